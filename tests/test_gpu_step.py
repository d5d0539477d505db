"""End-to-end parity of the training step (the native stepper, tfs_step_*) against the oracle
step (O1-O13), on one GPU: R = 1, and R = 2, 3, 4 vocabulary shards SIMULATED on the GPU
(tfs_comm in its one-process mode: the same phases and kernels as one process per GPU -- the
pull Gather through peer pointers, the id / gradient pushes into the owners' inboxes, the
owners' planned ScatterAdd -- with the barriers replaced by stream ordering).

Checked per step: sampled ids and num_tries bit-exact per replica; Part / route / Gather /
Stitch bit-exact (the gathered operand rows equal the oracle's Gather of E[x], W[y||s]); the
distinct ids per owner of the route plans; per-token loss and the table updates of every shard
element by element (tests/parity.py: |gpu - oracle| <= tol x the sum of |terms|, plus one
fp32 ulp of the new value per update); untouched rows bit-identical; graph replay over several
steps; determinism.
"""
import numpy as np
import pytest
import torch

import oracle
from oracle import step as ostep
import workloads
from parity import (TOL_BF16_ACC, TOL_BF16_EMU, TOL_F32, elem_err, ssm_allow, ssm_scales,
                    update_err)

pytestmark = pytest.mark.gpu

from paper_1605_08695_b200 import step as gstep  # noqa: E402
from paper_1605_08695_b200._lib import TFS_BF16, TFS_F32  # noqa: E402

DEV = "cuda"


def _cfg(w, R, dtype, lr=1.0, tokens=None, vocab=None, **kw):
    return gstep.StepConfig(vocab=vocab or w.vocab, dim=w.dim, tokens=tokens or
                            w.tokens_per_replica(R), num_sampled=w.num_sampled, num_shards=R,
                            lr=lr, seed=workloads.SAMPLER_SEED, operand_dtype=dtype, **kw)


def make_step(cfg, E, W, b):
    R = cfg.num_shards
    comm = gstep.Comm.simulated(cfg) if R > 1 else None
    st = gstep.Step(cfg, comm)
    for r in range(st.nlocal):
        st.load_tables(E[r::R], W[r::R], b[r::R], local=r)
    st.sync()
    return st


def _batches(w, R, step=0, tokens=None, vocab=None):
    xs, ys = zip(*[workloads.batch(w, R, r, step=step) for r in range(R)])
    xs, ys = list(xs), list(ys)
    if tokens is not None:
        xs, ys = [x[:tokens] for x in xs], [y[:tokens] for y in ys]
    if vocab is not None:
        xs, ys = [np.minimum(x, vocab - 1) for x in xs], [np.minimum(y, vocab - 1) for y in ys]
    return xs, ys


def _dev(arrs):
    return torch.from_numpy(np.concatenate(arrs)).to(DEV)


def _check_step(st, E, W, b, xs, ys, cfg, emu, tol, step, E2=None):
    """Run one step of `st` (counter = step) and compare with the oracle step over R shards."""
    R, B = cfg.num_shards, cfg.tokens
    ocfg = ostep.StepConfig(vocab=cfg.vocab, dim=cfg.dim, num_sampled=cfg.num_sampled,
                            num_shards=R, lr=cfg.lr, seed=cfg.seed, step=step, bf16=emu,
                            full_softmax=cfg.full_softmax, label_in=cfg.full_softmax and R > 1,
                            abs_bounds=True)
    E2, W2, b2, tr = ostep.step(E, W, b, xs, ys, ocfg)
    st.set_step(step)
    st.run(_dev(xs), _dev(ys))
    st.check("step")
    bf16_rows = cfg.operand_dtype == TFS_BF16
    for r in range(st.nlocal):
        t = tr[r]
        if not cfg.full_softmax:
            assert np.array_equal(st.tensor("qw", r)[B:].cpu().numpy(), t.sampled), r
            assert int(st.tensor("num_tries", r).item()) == t.num_tries
        if not (cfg.full_softmax and R > 1):
            # Part -> route -> owner Gather -> route back -> Stitch: exactly the lookup
            h = st.tensor("h", r)
            wr = st.tensor("w_rows", r)
            if bf16_rows:
                h, wr = (a.cpu().view(torch.int16).numpy().view(np.uint16) for a in (h, wr))
                assert np.array_equal(h, oracle.gather(E, xs[r], bf16=True))
                q = np.concatenate([ys[r], t.sampled])
                assert np.array_equal(wr, oracle.gather(W, q, bf16=True))
            else:
                assert np.array_equal(h.cpu().numpy(), E[xs[r]])
            assert np.array_equal(st.tensor("b_rows", r).cpu().numpy(),
                                  b[np.concatenate([ys[r], t.sampled])])
            loss = st.tensor("loss", r).cpu().numpy()
            e = elem_err(loss, t.ssm["loss"], t.ssm["abs_loss"])
            assert e <= tol, ("loss", r, e)
        if R > 1 and not cfg.full_softmax:  # distinct ids per owner of both route plans
            cnt = st.tensor("counts", r).cpu().numpy()
            q = np.concatenate([ys[r], t.sampled])
            for o in range(R):
                assert cnt[0, o] == np.unique(xs[r][xs[r] % R == o]).size
                assert cnt[1, o] == np.unique(q[q % R == o]).size
    # global loss = sum over ranks of the loss_sum shares
    got = sum(float(st.tensor("loss_sum", r).item()) for r in range(st.nlocal))
    want = sum(t.ssm["loss"].sum() for t in tr) / (R * B)
    scale = sum(t.ssm["abs_loss"].sum() for t in tr) / (R * B)
    assert abs(got - want) <= tol * scale, (got, want)
    aE, aW, ab = tr[0].abs_delta
    mE, mW, mb = tr[0].amb_delta
    for name, T0, To, A, M in (("E", E, E2, aE, mE), ("W", W, W2, aW, mW), ("b", b, b2, ab, mb)):
        for r in range(st.nlocal):
            g = st.tensor(name, r).cpu().numpy()
            t0, to, a, m = T0[r::R], To[r::R], A[r::R], M[r::R]
            touched = np.nonzero(np.any((a != 0).reshape(t0.shape[0], -1), axis=1))[0]
            untouched = np.setdiff1d(np.arange(t0.shape[0]), touched)
            assert np.array_equal(g[untouched], t0[untouched]), (name, r)
            e = update_err(g[touched], to[touched], a[touched], allow=m[touched])
            assert e <= tol, (name, r, e)
    return E2, W2, b2, tr


def gpu_tables(st, V):
    """The logical tables E, W, b assembled from every local rank's shard (row i of shard
    i mod R at local row i div R) -- the state the next step starts from."""
    R = st.R
    out = []
    for name in ("E", "W", "b"):
        parts = [st.tensor(name, r).cpu().numpy() for r in range(st.nlocal)]
        full = np.empty((V,) + parts[0].shape[1:], np.float32)
        for r in range(R):
            full[r::R] = parts[r]
        out.append(full)
    return out


# ------------------------------------------------------------------------------------- R = 1
@pytest.mark.parametrize("dtype,tol,emu", [(TFS_F32, TOL_F32, False), (TFS_BF16, TOL_BF16_ACC, False),
                                           (TFS_BF16, TOL_BF16_EMU, True)])
def test_step_config_T(dtype, tol, emu):
    w = workloads.WORKLOADS["T"]
    E, W, b = workloads.tables(w.vocab, w.dim)
    cfg = _cfg(w, 1, dtype)
    xs, ys = _batches(w, 1)
    _check_step(make_step(cfg, E, W, b), E, W, b, xs, ys, cfg, emu, tol, 0)


@pytest.mark.parametrize("dtype,tol,emu", [(TFS_F32, TOL_F32, False), (TFS_BF16, TOL_BF16_EMU, True)])
def test_step_config_L(dtype, tol, emu):
    w = workloads.WORKLOADS["L"]
    E, W, b = workloads.tables(w.vocab, w.dim)
    cfg = _cfg(w, 1, dtype)
    xs, ys = _batches(w, 1)
    _check_step(make_step(cfg, E, W, b), E, W, b, xs, ys, cfg, emu, tol, 3)


def test_step_config_F_full_softmax():
    """Config F: every one of the 40,000 classes is a candidate (the paper's full softmax,
    P:1159-1160) -- run at a reduced token count so the oracle finishes in seconds."""
    w = workloads.WORKLOADS["F"]
    E, W, b = workloads.tables(w.vocab, w.dim)
    cfg = _cfg(w, 1, TFS_BF16, tokens=64)
    xs, ys = _batches(w, 1, tokens=64)
    _check_step(make_step(cfg, E, W, b), E, W, b, xs, ys, cfg, True, TOL_BF16_EMU, 0)


def test_graph_replay_matches_eager_over_steps():
    """Capture once, replay three steps (the step counter advances inside the graph) ==
    three eager steps of a second stepper, bit for bit."""
    w = workloads.WORKLOADS["L"]
    E, W, b = workloads.tables(w.vocab, w.dim)
    cfg = _cfg(w, 1, TFS_BF16, lr=0.1)
    a, e = make_step(cfg, E, W, b), make_step(cfg, E, W, b)
    a.set_step(5)
    e.set_step(5)
    a.capture()
    for i in range(3):
        xs, ys = _batches(w, 1, step=i)
        la = a.run(_dev(xs), _dev(ys)).clone()
        le = e.run(_dev(xs), _dev(ys)).clone()
        torch.cuda.synchronize()
        assert torch.equal(la, le)
    for name in ("E", "W", "b"):
        assert torch.equal(a.tensor(name), e.tensor(name))
    assert int(a.tensor("step").item()) == 8


def test_step_host_buffers_match_device():
    """tfs_step_run with HOST x / y (copied inside the C call) and the loss read back to host
    == the device-input step."""
    w = workloads.WORKLOADS["T"]
    E, W, b = workloads.tables(w.vocab, w.dim)
    cfg = _cfg(w, 1, TFS_BF16)
    a, d = make_step(cfg, E, W, b), make_step(cfg, E, W, b)
    xs, ys = _batches(w, 1)
    xh = torch.from_numpy(xs[0]).pin_memory()
    yh = torch.from_numpy(ys[0]).pin_memory()
    lh = torch.zeros(1, dtype=torch.float32).pin_memory()
    a.run_host(xh, yh, lh)
    ld = d.run(_dev(xs), _dev(ys))
    torch.cuda.synchronize()
    assert lh.item() == ld.item()
    assert torch.equal(a.tensor("E"), d.tensor("E")) and torch.equal(a.tensor("W"), d.tensor("W"))


def test_step_deterministic():
    w = workloads.WORKLOADS["L"]
    E, W, b = workloads.tables(w.vocab, w.dim)
    cfg = _cfg(w, 1, TFS_BF16)
    xs, ys = _batches(w, 1)
    outs = []
    for _ in range(2):
        st = make_step(cfg, E, W, b)
        st.run(_dev(xs), _dev(ys))
        torch.cuda.synchronize()
        outs.append([st.tensor(n).clone() for n in ("E", "W", "b", "loss")])
    for a, bb in zip(*outs):
        assert torch.equal(a, bb)


@pytest.mark.slow
def test_step_config_X_full_outputs():
    """BASELINE's full size X (V = 800k, B = 2560, S = 8192; bf16 operands, the launch
    configuration bench.py times): the whole sampled-softmax output of the step -- loss, lse,
    dh, dW_true, db_true, dW_s, db_s of all 2560 tokens and 8192 classes -- against the
    bf16-emulating oracle element by element, and the E / W / b updates of every touched row."""
    w = workloads.WORKLOADS["X"]
    E, W, b = workloads.tables(w.vocab, w.dim)
    cfg = _cfg(w, 1, TFS_BF16)
    xs, ys = _batches(w, 1)
    x, y = xs[0], ys[0]
    B, S, c = x.size, w.num_sampled, 1.0 / x.size
    st = make_step(cfg, E, W, b)
    st.run(_dev(xs), _dev(ys))
    st.check("step X")
    s, T, les, ley = oracle.sample(w.vocab, S, True, cfg.seed, 0, 0, y)
    assert np.array_equal(st.tensor("qw")[B:].cpu().numpy(), s)
    assert int(st.tensor("num_tries").item()) == T
    o = oracle.sampled_softmax(E[x], y, W[y], b[y], ley.astype(np.float32).astype(np.float64), s,
                               W[s], b[s], les.astype(np.float32).astype(np.float64),
                               grad_scale=c, bf16=True)
    sc, al = ssm_scales(o, c), ssm_allow(o)
    dw, db = st.tensor("dw").cpu().numpy(), st.tensor("db").cpu().numpy()
    got = {"loss": st.tensor("loss").cpu().numpy(), "lse": st.tensor("lse").cpu().numpy(),
           "dh": st.tensor("dh").cpu().numpy(), "dw_true": dw[:B], "db_true": db[:B],
           "dw_s": dw[B:], "db_s": db[B:]}
    for k, v in got.items():
        e = elem_err(v, o[k], sc[k], al[k])
        assert e <= TOL_BF16_EMU, (k, e)
    # table updates of the touched rows (sub-tables indexed by the distinct ids)
    for name, T0, ids, grads, scale, amb in (
            ("E", E, x, o["dh"], o["abs_dh"], o["amb_dh"]),
            ("W", W, np.concatenate([y, s]), np.concatenate([o["dw_true"], o["dw_s"]]),
             np.concatenate([sc["dw_true"], o["abs_dw_s"]]),
             np.concatenate([np.zeros_like(o["dw_true"]), o["amb_dw_s"]])),
            ("b", b, np.concatenate([y, s]), np.concatenate([o["db_true"], o["db_s"]]),
             np.concatenate([sc["db_true"], o["abs_db_s"]]),
             np.concatenate([np.zeros_like(o["db_true"]), o["amb_db_s"]]))):
        u, inv = np.unique(ids, return_inverse=True)
        ref = oracle.scatter_add_sgd(T0[u], inv, grads, cfg.lr)
        _, a, _ = oracle.sort_reduce(inv, 1, scale)
        _, m, _ = oracle.sort_reduce(inv, 1, amb)
        g = st.tensor(name)[torch.from_numpy(u).to(DEV)].cpu().numpy()
        e = update_err(g, ref, cfg.lr * a, allow=cfg.lr * m)
        assert e <= TOL_BF16_EMU, (name, e)


@pytest.mark.slow
def test_step_config_Z_sampled_tokens():
    """Z (65,536 Zipf-1.1 tokens on one GPU, S = 8192): sampled ids exact; loss / lse / dh of
    64 tokens the oracle computes one by one (the dW_s columns would need the lse of all 65,536
    tokens, 275 GFLOP of fp64 -- the X test covers them at full size)."""
    w = workloads.WORKLOADS["Z"]
    E, W, b = workloads.tables(w.vocab, w.dim)
    cfg = _cfg(w, 1, TFS_BF16)
    xs, ys = _batches(w, 1)
    x, y = xs[0], ys[0]
    B, S = x.size, w.num_sampled
    st = make_step(cfg, E, W, b)
    st.run(_dev(xs), _dev(ys))
    st.check("step Z")
    s, T, les, ley = oracle.sample(w.vocab, S, True, cfg.seed, 0, 0, y)
    assert np.array_equal(st.tensor("qw")[B:].cpu().numpy(), s)
    tok = np.random.default_rng(0).permutation(B)[:64]
    o = oracle.sampled_softmax(E[x], y, W[y], b[y], ley.astype(np.float32).astype(np.float64), s,
                               W[s], b[s], les.astype(np.float32).astype(np.float64),
                               grad_scale=1.0 / B, bf16=True, tok_idx=tok, col_idx=np.zeros(0, np.int64))
    assert elem_err(st.tensor("loss").cpu().numpy()[tok], o["loss"], o["abs_loss"]) <= TOL_BF16_EMU
    assert elem_err(st.tensor("lse").cpu().numpy()[tok], o["lse"], o["abs_loss"]) <= TOL_BF16_EMU
    assert elem_err(st.tensor("dh").cpu().numpy()[tok], o["dh"], o["abs_dh"],
                    o["amb_dh"]) <= TOL_BF16_EMU


@pytest.mark.parametrize("kind", ["momentum", "adagrad"])
@pytest.mark.parametrize("R", [1, 2])
def test_step_sparse_optimizer(kind, R):
    """Sparse Momentum / Adagrad in the step, R = 1 (fp32 operands) and
    R = 2 simulated shards (bf16 operands; slot tables sharded like the tables): the oracle
    step's gradients at each state fed to the oracle's optimizer; two steps so the slots carry
    state.  Error scales propagate the gradients' term sums through the optimizer."""
    w = workloads.WORKLOADS["T"]
    dtype = TFS_F32 if R == 1 else TFS_BF16
    tol = TOL_F32 if R == 1 else TOL_BF16_EMU
    E, W, b = workloads.tables(w.vocab, w.dim)
    cfg = _cfg(w, R, dtype, lr=0.5, optimizer=kind)
    st = make_step(cfg, E, W, b)
    init = 0.0 if kind == "momentum" else cfg.adagrad_init
    tabs = {"E": E.copy(), "W": W.copy(), "b": b.copy()}
    slots = {k: np.full_like(v, init) for k, v in tabs.items()}
    sc = {k: 0.0 for k in ("E", "W", "b", "sE", "sW", "sb")}
    for step in range(2):
        xs, ys = _batches(w, R, step=step)
        ocfg = ostep.StepConfig(vocab=cfg.vocab, dim=cfg.dim, num_sampled=cfg.num_sampled,
                                num_shards=R, lr=1.0, seed=cfg.seed, step=step,
                                bf16=(dtype == TFS_BF16), abs_bounds=True)
        _, _, _, tr = ostep.step(tabs["E"], tabs["W"], tabs["b"], xs, ys, ocfg)
        gabs = tr[0].abs_delta                      # lr = 1: sum of |terms| per entry
        ids = {"E": np.concatenate(xs)}
        ids["W"] = ids["b"] = np.concatenate([np.concatenate([ys[r], tr[r].sampled])
                                              for r in range(R)])
        grads = {"E": np.concatenate([t.ssm["dh"] for t in tr]),
                 "W": np.concatenate([np.concatenate([t.ssm["dw_true"], t.ssm["dw_s"]]) for t in tr]),
                 "b": np.concatenate([np.concatenate([t.ssm["db_true"], t.ssm["db_s"]]) for t in tr])}
        for i, k in enumerate(("E", "W", "b")):
            tabs[k], slots[k] = oracle.scatter_opt(kind, tabs[k], slots[k], ids[k], grads[k],
                                                   cfg.lr, cfg.momentum)
            ga = gabs[i]
            if kind == "momentum":
                sc["s" + k] = cfg.momentum * sc["s" + k] + ga
                sc[k] = sc[k] + cfg.lr * sc["s" + k]
            else:
                a = np.maximum(slots[k].astype(np.float64), 1e-30)
                sc["s" + k] = sc["s" + k] + 2 * ga * ga
                sc[k] = sc[k] + cfg.lr * (ga / np.sqrt(a) + ga * sc["s" + k] / (2 * a ** 1.5))
        st.set_step(step)
        st.run(_dev(xs), _dev(ys))
        st.check("step")
    for k, T0 in (("E", E), ("W", W), ("b", b)):
        for r in range(st.nlocal):
            for got_t, ref, s0, key in ((st.tensor(k, r), tabs[k], T0, k),
                                        (st.tensor("slot_" + k, r), slots[k],
                                         np.full_like(T0, init), "s" + k)):
                g = got_t.cpu().numpy()
                rf, s0r, scale = ref[r::R], s0[r::R], np.broadcast_to(sc[key], T0.shape)[r::R]
                touched = np.nonzero(np.any((rf != s0r).reshape(rf.shape[0], -1), axis=1))[0]
                untouched = np.setdiff1d(np.arange(rf.shape[0]), touched)
                assert np.array_equal(g[untouched], s0r[untouched]), (key, r)
                e = update_err(g[touched], rf[touched], scale[touched], ulps=2)
                assert e <= tol, (key, r, e)


# ------------------------------------------------------------- R > 1 shards simulated on one GPU
@pytest.mark.parametrize("R", [2, 3, 4, 8])
@pytest.mark.parametrize("name,tol,emu", [("T", TOL_BF16_EMU, True), ("T", TOL_BF16_ACC, False),
                                          ("L", TOL_BF16_EMU, True)])
def test_sim_sharded_step_matches_oracle(R, name, tol, emu):
    """R vocabulary shards / replicas: ids mod R, the one-sided routes (pull Gather, id and
    gradient pushes into the owners' inboxes, merge-plan ScatterAdd on the owner), vs the
    oracle's synchronous step over R simulated shards (O3-O13)."""
    w = workloads.WORKLOADS[name]
    E, W, b = workloads.tables(w.vocab, w.dim)
    cfg = _cfg(w, R, TFS_BF16)
    xs, ys = _batches(w, R)
    _check_step(make_step(cfg, E, W, b), E, W, b, xs, ys, cfg, emu, tol, 2)


@pytest.mark.parametrize("R", [2, 4, 8])
def test_sim_sharded_steps_graph_replay(R):
    """Three steps of R simulated shards, captured once into a CUDA graph and replayed (inbox
    reuse across steps, the step counter inside the graph): each step against the oracle."""
    w = workloads.WORKLOADS["T"]
    E, W, b = workloads.tables(w.vocab, w.dim)
    cfg = _cfg(w, R, TFS_BF16)
    st = make_step(cfg, E, W, b)
    st.set_step(0)
    st.capture()
    for k in range(3):
        xs, ys = _batches(w, R, step=k)
        E, W, b = gpu_tables(st, w.vocab)        # identical inputs: the GPU's state (c.5)
        _check_step(st, E, W, b, xs, ys, cfg, True, TOL_BF16_EMU, k)


@pytest.mark.parametrize("R,vocab,tokens", [(2, 1000, 32), (3, 4003, 96), (4, 4003, 64),
                                            (8, 4003, 32)])
def test_sim_sharded_full_softmax(R, vocab, tokens):
    """The vocabulary-sharded full softmax (R-30): W, b stay on their shard, which
    scores all R*B tokens against its classes; ragged shards when R does not divide V; vs the
    oracle's label-in full-softmax step over the same global batch (bf16 emulation)."""
    w = workloads.Workload("Fs", vocab, 64, tokens, 0, R)
    E, W, b = workloads.tables(vocab, 64)
    cfg = _cfg(w, R, TFS_BF16)
    xs, ys = _batches(w, R)
    st = make_step(cfg, E, W, b)
    _check_step(st, E, W, b, xs, ys, cfg, True, TOL_BF16_EMU, 0)
    xs, ys = _batches(w, R, step=1)              # second step: updated W / its bf16 shadow
    E, W, b = gpu_tables(st, vocab)              # from the GPU's own state (identical inputs)
    _check_step(st, E, W, b, xs, ys, cfg, True, TOL_BF16_EMU, 1)


@pytest.mark.parametrize("R", [2, 3])
def test_sim_sharded_full_softmax_graph_replay(R):
    """The sharded full softmax captured once into a CUDA graph and replayed for three steps,
    each step against the oracle from the GPU's own state."""
    w = workloads.Workload("Fs", 1000, 64, 32, 0, R)
    E, W, b = workloads.tables(1000, 64)
    cfg = _cfg(w, R, TFS_BF16)
    st = make_step(cfg, E, W, b)
    st.set_step(0)
    st.capture()
    for k in range(3):
        xs, ys = _batches(w, R, step=k)
        E, W, b = gpu_tables(st, 1000)
        _check_step(st, E, W, b, xs, ys, cfg, True, TOL_BF16_EMU, k)


@pytest.mark.parametrize("R", [2, 4])
def test_sim_sharded_X_integer_paths(R):
    """BASELINE's X shape (V = 800k, B = 2560 and S = 8192 per replica) with R shards: the
    sampled ids / T of every replica, the distinct ids per owner, and the bits of every gathered
    operand row (bf16) and bias -- the integer and copy paths, checked in full."""
    w = workloads.WORKLOADS["X"]
    E, W, b = workloads.tables(w.vocab, w.dim)
    cfg = _cfg(w, R, TFS_BF16, lr=0.1)
    xs, ys = _batches(w, R)
    st = make_step(cfg, E, W, b)
    st.run(_dev(xs), _dev(ys))
    st.check("X step")
    B = cfg.tokens
    for r in range(R):
        s, T, _, _ = oracle.sample(w.vocab, w.num_sampled, True, cfg.seed, 0, r, ys[r])
        assert np.array_equal(st.tensor("qw", r)[B:].cpu().numpy(), s)
        assert int(st.tensor("num_tries", r).item()) == T
        q = np.concatenate([ys[r], s])
        h = st.tensor("h", r).cpu().view(torch.int16).numpy().view(np.uint16)
        wr = st.tensor("w_rows", r).cpu().view(torch.int16).numpy().view(np.uint16)
        assert np.array_equal(h, oracle.gather(E, xs[r], bf16=True))
        assert np.array_equal(wr, oracle.gather(W, q, bf16=True))
        assert np.array_equal(st.tensor("b_rows", r).cpu().numpy(), b[q])
        cnt = st.tensor("counts", r).cpu().numpy()
        for o in range(R):
            assert cnt[0, o] == np.unique(xs[r][xs[r] % R == o]).size
            assert cnt[1, o] == np.unique(q[q % R == o]).size
        assert np.all(np.isfinite(st.tensor("loss", r).cpu().numpy()))


def test_route_capacity_overflow_is_reported():
    """A configured slot capacity below a batch's distinct ids per owner is reported as
    TFS_ERR_CAPACITY (the default capacity is the worst case and cannot overflow)."""
    w = workloads.WORKLOADS["T"]
    E, W, b = workloads.tables(w.vocab, w.dim)
    cfg = _cfg(w, 2, TFS_BF16, cap_e=2)
    st = make_step(cfg, E, W, b)
    xs, ys = _batches(w, 2)
    st.run(_dev(xs), _dev(ys))
    torch.cuda.synchronize()
    assert any(st.error(r)[0] == 9 for r in range(2))


@pytest.mark.parametrize("R,full", [(1, False), (2, False), (3, False), (2, True)])
def test_step_with_delayed_side_stream(R, full, monkeypatch):
    """Race detector: TFS_DEBUG_SIDE_DELAY_US makes every side-stream phase start 3 ms late, so
    any work on the main stream that reads side-stream results without an event wait computes
    on stale data and fails the oracle comparison (round 2 found one this way: the W gradient
    push of the R > 1 step did not wait for the W route plan)."""
    monkeypatch.setenv("TFS_DEBUG_SIDE_DELAY_US", "3000")
    w = (workloads.Workload("Fs", 1000, 64, 32, 0, R) if full else workloads.WORKLOADS["T"])
    E, W, b = workloads.tables(w.vocab, w.dim)
    cfg = _cfg(w, R, TFS_BF16)
    st = make_step(cfg, E, W, b)
    for k in range(2):
        xs, ys = _batches(w, R, step=k)
        E, W, b = gpu_tables(st, w.vocab)
        _check_step(st, E, W, b, xs, ys, cfg, True, TOL_BF16_EMU, k)
