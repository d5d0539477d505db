"""Multi-GPU parity of the sharded step (R = 2 ranks over NCCL) against the oracle step with R
simulated shards: sampled ids bit-exact per replica, per-token loss, and each rank's updated
shard of E, W, b (normwise rel, R-19).  Needs >= 2 GPUs (gpurun --gpus 2); skipped otherwise."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def rel(g, o):
    return float(np.max(np.abs(g - o)) / max(np.max(np.abs(o)), 1e-300)) if o.size else 0.0


# A mid-size full-softmax case (the oracle's full softmax over F itself takes minutes).
EXTRA = {"Fm": dict(vocab=4000, dim=128, tokens=256),
         "Fo": dict(vocab=4003, dim=64, tokens=96)}   # V not a multiple of R (ragged shards)


def _workload(name):
    import workloads
    if name in EXTRA:
        return workloads.Workload(name, shards=2, num_sampled=0, **EXTRA[name])
    return workloads.WORKLOADS[name]


def _worker(rank, world, port, name, dtype, route, *rest):
    """Runs one rank; any exception is reported through the queue (so the parent fails fast
    with the traceback instead of waiting for a result that never comes)."""
    import traceback
    *flag, q = rest
    full = bool(flag and flag[0])
    try:
        _worker_body(rank, world, port, name, dtype, route, q, full)
    except BaseException:
        q.put((rank, {"error": traceback.format_exc()}))
        raise


def _worker_body(rank, world, port, name, dtype, route, q, full):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import oracle  # noqa: F401
    from oracle import step as ostep
    import workloads
    from paper_1605_08695_b200 import step as gstep
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        w = _workload(name)
        V, R = w.vocab, world
        E, W, b = workloads.tables(V, w.dim)
        xs, ys = zip(*[workloads.batch(w, R, r) for r in range(R)])
        cfg = gstep.StepConfig(vocab=V, dim=w.dim, tokens=xs[0].size, num_sampled=w.num_sampled,
                               lr=1.0, seed=workloads.SAMPLER_SEED, operand_dtype=dtype,
                               route=route, full_softmax=full)
        st = gstep.ShardedStep(cfg, torch.from_numpy(E[rank::R].copy()).to(dev),
                               torch.from_numpy(W[rank::R].copy()).to(dev),
                               torch.from_numpy(b[rank::R].copy()).to(dev), gstep.Router())
        st.run(torch.from_numpy(xs[rank]).to(dev), torch.from_numpy(ys[rank]).to(dev), 2)
        torch.cuda.synchronize()
        st.err.check("dist step")
        ocfg = ostep.StepConfig(vocab=V, dim=w.dim, num_sampled=w.num_sampled, num_shards=R,
                                lr=1.0, seed=workloads.SAMPLER_SEED, step=2, bf16=(dtype == 1),
                                full_softmax=full)
        E2, W2, b2, tr = ostep.step(E, W, b, list(xs), list(ys), ocfg)
        B = xs[0].size
        if full:  # the loss is formed where each label lives: compare the global sum
            want = sum(t.ssm["loss"].sum() for t in tr) / (R * B)
            res = {"sampled": True,
                   "loss": abs(float(st.ssm_out["loss_sum"].item()) - want) / abs(want)}
        else:
            res = {"sampled": np.array_equal(st.qw[B:].cpu().numpy(), tr[rank].sampled),
                   "loss": rel(st.ssm_out["loss"].cpu().numpy(), tr[rank].ssm["loss"])}
        for nm, T0, Tg, To in (("E", E, st.E, E2), ("W", W, st.W, W2), ("b", b, st.b, b2)):
            g = Tg.cpu().numpy()
            t0, to = T0[rank::R], To[rank::R]
            touched = np.nonzero(np.any((to != t0).reshape(t0.shape[0], -1), axis=1))[0]
            untouched = np.setdiff1d(np.arange(t0.shape[0]), touched)
            res[nm + "_untouched"] = bool(np.array_equal(g[untouched], t0[untouched]))
            res[nm] = rel(g[touched] - t0[touched], to[touched] - t0[touched])
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _run_ranks(args_of_rank):
    """Spawn one process per rank, collect (rank, result) pairs; a rank that raised fails the
    test with its traceback, and no rank is left running (a peer of a failed rank may be
    blocked in a device barrier)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, len(args_of_rank), port, *a, q))
             for r, a in enumerate(args_of_rank)]
    for p in procs:
        p.start()
    try:
        res = []
        for _ in procs:
            rank, r = q.get(timeout=600)
            assert "error" not in r, f"rank {rank}:\n{r['error']}"
            res.append((rank, r))
        for p in procs:
            p.join(timeout=120)
            assert p.exitcode == 0
        return res
    finally:
        for p in procs:
            if p.is_alive():
                p.kill()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("route", ["p2p", "nccl"])
@pytest.mark.parametrize("name,dtype,tol", [("T", 0, 1e-5), ("L", 1, 2e-3)])
def test_dist_step_matches_oracle(name, dtype, tol, route):
    res = _run_ranks([(name, dtype, route)] * 2)
    for rank, r in res:
        assert r["sampled"], rank
        assert r["loss"] <= tol, (rank, r)
        for nm in ("E", "W", "b"):
            assert r[nm + "_untouched"], (rank, nm)
            assert r[nm] <= tol, (rank, nm, r[nm])


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("name", ["T", "Fm"])
def test_dist_full_softmax_sharded_matches_oracle(name):
    """The vocabulary-sharded full softmax (W / b stay on their shard, which scores
    all R*B tokens) reaches the oracle's full-softmax step over the same global batch."""
    res = _run_ranks([(name, 1, "p2p", True)] * 2)
    for rank, r in res:
        assert r["loss"] <= 5e-3, (rank, r)
        for nm in ("E", "W", "b"):
            assert r[nm + "_untouched"], (rank, nm)
            assert r[nm] <= 5e-3, (rank, nm, r[nm])


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs 4 GPUs")
@pytest.mark.parametrize("name,dtype,route,full,tol", [
    ("T", 0, "p2p", False, 1e-5), ("T", 1, "nccl", False, 2e-3), ("Fo", 1, "p2p", True, 5e-3)])
def test_dist4_matches_oracle(name, dtype, route, full, tol):
    """R = 4 ranks (the bench's 4-GPU configuration): sampled step over both transports, and the
    sharded full softmax with V = 4003 (shards of 1001 / 1001 / 1001 / 1000 classes)."""
    res = _run_ranks([(name, dtype, route, full)] * 4)
    assert len(res) == 4
    for rank, r in res:
        assert r["sampled"], rank
        assert r["loss"] <= tol, (rank, r)
        for nm in ("E", "W", "b"):
            assert r[nm + "_untouched"], (rank, nm)
            assert r[nm] <= tol, (rank, nm, r[nm])
