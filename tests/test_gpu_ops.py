"""GPU parity of every libtfs entry point against the CPU oracle (run on a B200: -m gpu).

Integer outputs (partition, sampled ids, T, gathered / stitched bits) must be bit-exact.
Floating point uses the element-wise, cancellation-aware metric of tests/parity.py (reading
R-19): |g_i - o_i| <= tol * a_i for every element, a_i = the sum of the absolute values of the
terms forming o_i (returned by the oracle); tol = 1e-5 for fp32 operands, 2e-2 for bf16
operands against the fp64 unrounded oracle, 2e-3 against the oracle's bf16-emulating mode.
"""
import numpy as np
import pytest
import torch

import oracle
import workloads
from parity import (TOL_BF16_ACC, TOL_BF16_EMU, TOL_F32, elem_err, ssm_allow, ssm_scales,
                    update_err)

pytestmark = pytest.mark.gpu

from paper_1605_08695_b200 import ops  # noqa: E402
from paper_1605_08695_b200._lib import TFS_BF16, TFS_F32  # noqa: E402

DEV = "cuda"


def T(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(DEV)


# ------------------------------------------------------------------------------------- GEMM unit
@pytest.mark.parametrize("M,N,K,ks", [(128, 256, 64, 1), (256, 512, 512, 1), (300, 704, 192, 1),
                                      (2560, 512, 8192, 4), (40, 24, 64, 1), (1000, 256, 2560, 3)])
@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, False), (True, True)])
def test_tcgen05_gemm_matches_torch(M, N, K, ks, a_mn, b_mn):
    """C = A B^T with each operand read K-major ([rows, K]) or MN-major ([K, rows])."""
    g = torch.Generator().manual_seed(M * 7 + N)
    A = torch.randn(M, K, generator=g).to(torch.bfloat16)
    B = torch.randn(N, K, generator=g).to(torch.bfloat16)
    def place(X, mn):  # row stride padded to a multiple of 8 elements (16 bytes)
        X = X.T if mn else X
        r, c = X.shape
        buf = torch.zeros(r, (c + 7) // 8 * 8, dtype=torch.bfloat16, device=DEV)
        buf[:, :c] = X.to(DEV)
        return buf[:, :c]

    Ad, Bd = place(A, a_mn), place(B, b_mn)
    C = ops.debug_gemm_bf16(Ad, Bd, ks, a_mn=a_mn, b_mn=b_mn)
    got = C.cpu().double()
    ref = A.double() @ B.double().T
    err = (got - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err


# -------------------------------------------------------------------------------------- Partition
@pytest.mark.parametrize("n", [0, 1, 31, 4095, 4096, 4097, 10752, 70001])
@pytest.mark.parametrize("R", [1, 2, 3, 8])
def test_partition_bit_exact(n, R):
    V = 800_000
    rng = np.random.default_rng(n + R)
    ids = workloads.zipf_ids(rng, V, 1.0, n)
    local, pos, counts = ops.partition(T(ids), V, R)
    if n == 0:
        assert counts.cpu().tolist() == [0] * R
        return
    ol, op, oc = oracle.partition(ids, V, R)
    assert np.array_equal(local.cpu().numpy(), ol)
    assert np.array_equal(pos.cpu().numpy(), op)
    assert np.array_equal(counts.cpu().numpy(), oc)


def test_partition_explicit_mode_and_errors():
    ids = T(np.array([5, 9, 3, 7]))
    local, pos, counts = ops.partition(ids, 0, 2, assignments=T(np.array([1, 0, 1, 0], np.int32)))
    assert local.tolist() == [9, 7, 5, 3] and pos.tolist() == [1, 3, 0, 2]
    assert counts.tolist() == [2, 2]
    err = ops.ErrorSlot(DEV)
    bad = np.arange(9000) % 100
    bad[5000] = 100
    bad[7000] = -4
    ops.partition(T(bad), 100, 4, err=err)
    assert err.read() == (2, 5000)


# ----------------------------------------------------------------------------------------- Gather
@pytest.mark.parametrize("dim", [512, 64, 3, 1])
@pytest.mark.parametrize("bf16", [False, True])
def test_gather_bit_exact(dim, bf16):
    rng = np.random.default_rng(dim)
    table = rng.standard_normal((5000, dim)).astype(np.float32)
    ids = rng.integers(0, 5000, 3001)
    ids[:100] = 7  # duplicates
    out = ops.gather(T(table), T(ids), out_dtype=torch.bfloat16 if bf16 else torch.float32)
    ref = oracle.gather(table, ids, bf16=bf16)
    got = out.cpu().view(torch.int16).numpy().view(np.uint16) if bf16 else out.cpu().numpy()
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("dim", [512, 64, 3])
@pytest.mark.parametrize("bf16", [False, True])
def test_gather2_rows_and_companion_bit_exact(dim, bf16):
    """W rows and their bias in one pass == two oracle Gathers; padding ids leave both unwritten,
    a bad id is reported at its position."""
    rng = np.random.default_rng(dim + 1)
    table = rng.standard_normal((5000, dim)).astype(np.float32)
    bias = rng.standard_normal(5000).astype(np.float32)
    ids = rng.integers(0, 5000, 3001)
    ids[:100] = 7
    ids[200] = -1
    od = torch.bfloat16 if bf16 else torch.float32
    out = torch.full((ids.size, dim), 3.0, dtype=od, device=DEV)
    out2 = torch.full((ids.size,), 5.0, device=DEV)
    err = ops.ErrorSlot(DEV)
    ops.gather2(T(table), T(bias), T(ids), out, out2, err=err)
    assert err.read()[0] == 0
    keep = ids != -1
    ref = oracle.gather(table, ids[keep], bf16=bf16)
    got = out.cpu().view(torch.int16).numpy().view(np.uint16) if bf16 else out.cpu().numpy()
    assert np.array_equal(got[keep], ref)
    assert np.array_equal(out2.cpu().numpy()[keep], oracle.gather(bias.reshape(-1, 1), ids[keep])[:, 0])
    assert float(out2[200]) == 5.0 and float(out[200, 0].float()) == 3.0
    ids[2500] = 5000
    ops.gather2(T(table), T(bias), T(ids), out, out2, err=err)
    assert err.read() == (2, 2500)


@pytest.mark.parametrize("R", [1, 3, 4])
@pytest.mark.parametrize("bf16", [False, True])
def test_gather_peers2_simulated_shards(R, bf16):
    """The one-sided routed Gather (shard id % R, row id // R) through a pointer table, with the
    bias companion; R shards simulated on one GPU; == the oracle's Gather of the logical table."""
    rng = np.random.default_rng(R)
    V, d = 3001, 64
    W = rng.standard_normal((V, d)).astype(np.float32)
    b = rng.standard_normal(V).astype(np.float32)
    rows = -(-V // R)
    sh = [torch.zeros((rows, d), device=DEV) for _ in range(R)]
    sb = [torch.zeros(rows, device=DEV) for _ in range(R)]
    for r in range(R):
        n_r = W[r::R].shape[0]
        sh[r][:n_r] = T(W[r::R])
        sb[r][:n_r] = T(b[r::R])
    tab = torch.tensor([t.data_ptr() for t in sh], dtype=torch.int64, device=DEV)
    tab2 = torch.tensor([t.data_ptr() for t in sb], dtype=torch.int64, device=DEV)
    ids = workloads.zipf_ids(rng, V, 1.0, 2000)
    od = torch.bfloat16 if bf16 else torch.float32
    out = torch.empty((ids.size, d), dtype=od, device=DEV)
    out2 = torch.empty(ids.size, device=DEV)
    ops.gather_peers2(tab, tab2, rows, d, T(ids), V, R, out, out2)
    ref = oracle.gather(W, ids, bf16=bf16)
    got = out.cpu().view(torch.int16).numpy().view(np.uint16) if bf16 else out.cpu().numpy()
    assert np.array_equal(got, ref)
    assert np.array_equal(out2.cpu().numpy(), b[ids])


@pytest.mark.parametrize("R", [2, 3])
def test_gather_peers2_bf16_mirrors(R):
    """The pull from the owners' bf16 mirrors (bf16 RNE of the fp32 shards) == the pull of the
    fp32 shards rounded to bf16 == the oracle's bf16 Gather of the logical table, bit-exact."""
    rng = np.random.default_rng(10 + R)
    V, d = 3001, 64
    W = rng.standard_normal((V, d)).astype(np.float32)
    b = rng.standard_normal(V).astype(np.float32)
    rows = -(-V // R)
    sh = [torch.zeros((rows, d), device=DEV) for _ in range(R)]
    sb = [torch.zeros(rows, device=DEV) for _ in range(R)]
    for r in range(R):
        n_r = W[r::R].shape[0]
        sh[r][:n_r] = T(W[r::R])
        sb[r][:n_r] = T(b[r::R])
    mir = [t.to(torch.bfloat16) for t in sh]  # torch's RNE conversion: the mirrors' contents
    mtab = torch.tensor([t.data_ptr() for t in mir], dtype=torch.int64, device=DEV)
    tab2 = torch.tensor([t.data_ptr() for t in sb], dtype=torch.int64, device=DEV)
    ids = workloads.zipf_ids(rng, V, 1.0, 2000)
    ids[7] = -1
    out = torch.full((ids.size, d), 3.0, dtype=torch.bfloat16, device=DEV)
    out2 = torch.full((ids.size,), 5.0, device=DEV)
    ops.gather_peers2_bf16(mtab, tab2, rows, d, T(ids), V, R, out, out2)
    keep = ids != -1
    ref = oracle.gather(W, ids[keep], bf16=True)
    got = out.cpu().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got[keep], ref)
    assert np.array_equal(out2.cpu().numpy()[keep], b[ids[keep]])
    assert float(out[7, 0].float()) == 3.0 and float(out2[7]) == 5.0


def test_gather_out_of_range():
    err = ops.ErrorSlot(DEV)
    table = T(np.zeros((10, 8), np.float32))
    ids = np.arange(2000) % 10
    ids[1500] = 10
    ids[1700] = -1
    ops.gather(table, T(ids), err=err)
    assert err.read() == (2, 1500)


# ----------------------------------------------------------------------------------------- Stitch
@pytest.mark.parametrize("n,dim", [(1, 512), (777, 512), (4096, 64), (999, 3), (10000, 1)])
def test_stitch_bit_exact(n, dim):
    rng = np.random.default_rng(n)
    perm = rng.permutation(n)
    rows = rng.standard_normal((n, dim)).astype(np.float32)
    out = ops.stitch(T(perm), T(rows), err=ops.ErrorSlot(DEV))
    assert np.array_equal(out.cpu().numpy(), oracle.stitch(perm, rows))


def test_stitch_validation():
    rows = T(np.zeros((6, 4), np.float32))
    for pos, bad in (([0, 1, 1, 2, 3, 4], 2), ([0, 6, 1, 2, 3, 4], 1), ([5, 4, 3, -1, 1, 0], 3)):
        err = ops.ErrorSlot(DEV)
        ops.stitch(T(np.array(pos)), rows, err=err)
        assert err.read() == (3, bad)


# ---------------------------------------------------------------------------------------- Sampler
@pytest.mark.parametrize("V,S,unique", [(1000, 64, True), (40000, 512, True),
                                        (800000, 8192, True), (40000, 512, False),
                                        (1000, 999, True)])
def test_sampler_bit_exact(V, S, unique):
    rng = np.random.default_rng(V + S)
    labels = rng.integers(0, V, 300)
    smp = ops.Sampler(V, S, unique, DEV)
    for step, rep in ((0, 0), (5, 3)):
        s, les, ley, Tn = smp.sample(7, step, rep, T(labels))
        os_, oT, oles, oley = oracle.sample(V, S, unique, 7, step, rep, labels)
        assert np.array_equal(s.cpu().numpy(), os_)
        assert int(Tn.item()) == oT
        # log ec enters the logits as an additive correction: its error scale is that of a
        # logit, |log ec| + 1 (ec -> 1 gives log ec -> 0, where only the absolute error counts)
        assert elem_err(les.cpu().numpy(), oles, np.abs(oles) + 1.0) < 1e-6
        assert elem_err(ley.cpu().numpy(), oley, np.abs(oley) + 1.0) < 1e-6


def test_sampler_step_from_device_matches_host_step():
    V, S = 40000, 512
    labels = T(np.arange(100))
    smp = ops.Sampler(V, S, True, DEV)
    a = smp.sample(3, 11, 1, labels)[0].clone()
    b = smp.sample(3, 0, 1, labels, step_dev=torch.tensor([11], device=DEV))[0]
    assert torch.equal(a, b)


# --------------------------------------------------------------------------------- Sampled softmax
def _ssm_case(B, S, V, d, seed, hit_frac=0.2, logq=True, unique=True):
    rng = np.random.default_rng(seed)
    W = (rng.random((V, d), dtype=np.float32) - 0.5)
    bb = (rng.random(V, dtype=np.float32) - 0.5) * 0.2
    h = (rng.random((B, d), dtype=np.float32) - 0.5)
    labels = workloads.zipf_ids(rng, V, 1.0, B)
    s, Tn, les, ley = oracle.sample(V, S, unique, seed, 0, 0, labels)
    nh = int(B * hit_frac)
    labels[:nh] = rng.choice(s, nh)
    les = les.astype(np.float32)
    ley = oracle.sample(V, S, unique, seed, 0, 0, labels)[3].astype(np.float32)
    return dict(h=h, labels=labels, w_true=W[labels], b_true=bb[labels], le_t=ley, s=s,
                w_s=W[s], b_s=bb[s], le_s=les, V=V)


def _run_ssm(c, dtype, grad_scale, use_map=True, ws=None):
    """use_map: pass the vocabulary bound (candidate map in the workspace head) or 0."""
    out = ops.sampled_softmax(T(c["h"]), T(c["labels"]), T(c["w_true"]), T(c["b_true"]),
                              T(c["le_t"]), T(c["s"]), T(c["w_s"]), T(c["b_s"]), T(c["le_s"]),
                              grad_scale=grad_scale, operand_dtype=dtype,
                              vocab=c["V"] if use_map else 0, ws=ws)
    return {k: v.cpu().numpy() for k, v in out.items()}


def _oracle_ssm(c, grad_scale, bf16):
    return oracle.sampled_softmax(c["h"], c["labels"], c["w_true"], c["b_true"],
                                  c["le_t"].astype(np.float64), c["s"], c["w_s"], c["b_s"],
                                  c["le_s"].astype(np.float64), grad_scale=grad_scale, bf16=bf16)


KEYS = ("loss", "lse", "dh", "dw_true", "db_true", "dw_s", "db_s")


@pytest.mark.parametrize("B,S,d", [(32, 64, 64), (37, 100, 64), (256, 512, 512), (130, 300, 128)])
def test_ssm_fp32_parity(B, S, d):
    c = _ssm_case(B, S, 40000, d, seed=B + S)
    gs = 1.0 / B
    got = _run_ssm(c, TFS_F32, gs)
    ref = _oracle_ssm(c, gs, False)
    sc = ssm_scales(ref, gs)
    for k in KEYS:
        e = elem_err(got[k], ref[k], sc[k])
        assert e <= TOL_F32, (k, e)
    assert abs(got["loss_sum"][0] - gs * ref["loss"].sum()) <= TOL_F32 * gs * ref["abs_loss"].sum()


@pytest.mark.parametrize("use_map", [True, False])
@pytest.mark.parametrize("B,S,d", [(256, 512, 512), (130, 300, 128), (2560, 512, 512),
                                   (300, 1000, 64)])
def test_ssm_bf16_parity(B, S, d, use_map):
    c = _ssm_case(B, S, 40000, d, seed=3 * B + S)
    gs = 1.0 / B
    got = _run_ssm(c, TFS_BF16, gs, use_map)
    ref = _oracle_ssm(c, gs, False)       # accuracy: fp64, unrounded operands
    emu = _oracle_ssm(c, gs, True)        # rounding points: bf16-emulating oracle
    sr, se, ae = ssm_scales(ref, gs), ssm_scales(emu, gs), ssm_allow(emu)
    for k in KEYS:
        e1, e2 = elem_err(got[k], ref[k], sr[k]), elem_err(got[k], emu[k], se[k], ae[k])
        assert e1 <= TOL_BF16_ACC and e2 <= TOL_BF16_EMU, (k, e1, e2)


@pytest.mark.parametrize("use_map", [True, False])
@pytest.mark.parametrize("B,S,d,V", [(700, 2000, 128, 3000), (300, 4096, 64, 500)])
def test_ssm_bf16_duplicate_candidates(B, S, d, V, use_map):
    """Sampling with replacement from a small vocabulary: ids repeat among the candidates, so a
    label's columns span a range with other ids inside it (the epilogue's slow exclusion path)."""
    c = _ssm_case(B, S, V, d, seed=B + 7, hit_frac=0.6, unique=False)
    assert len(np.unique(c["s"])) < S
    gs = 1.0 / B
    got = _run_ssm(c, TFS_BF16, gs, use_map)
    emu = _oracle_ssm(c, gs, True)
    se, ae = ssm_scales(emu, gs), ssm_allow(emu)
    for k in KEYS:
        e = elem_err(got[k], emu[k], se[k], ae[k])
        assert e <= TOL_BF16_EMU, (k, e)


def test_ssm_candidate_map_left_zero():
    """The candidate map in the workspace head is zero again after every call, so one
    workspace serves calls with different candidate sets."""
    c1 = _ssm_case(256, 512, 3000, 64, seed=11, hit_frac=0.5)
    c2 = _ssm_case(256, 512, 3000, 64, seed=12, hit_frac=0.5)
    ws = ops.ssm_workspace(256, 512, 64, TFS_BF16, DEV, 3000)
    _run_ssm(c1, TFS_BF16, 0.01, ws=ws)
    torch.cuda.synchronize()
    assert int(ws[:3000 * 8].count_nonzero()) == 0
    got = _run_ssm(c2, TFS_BF16, 0.01, ws=ws)
    emu = _oracle_ssm(c2, 0.01, True)
    se, ae = ssm_scales(emu, 0.01), ssm_allow(emu)
    for k in KEYS:
        e = elem_err(got[k], emu[k], se[k], ae[k])
        assert e <= TOL_BF16_EMU, (k, e)


@pytest.mark.parametrize("V", [40000, 0])
def test_ssm_schedule_counters_left_zero_and_deterministic(V):
    """The logits / gradient GEMMs claim tiles dynamically through counters in the 256 bytes
    after the candidate map (include/tfs.h): they are zero again after every call, and repeated
    calls -- each with its own tile-to-CTA assignment -- give bit-identical outputs (X shape:
    five tiles per SM)."""
    B, S, d = 2560, 8192, 512
    c = _ssm_case(B, S, 40000, d, seed=5)
    ws = ops.ssm_workspace(B, S, d, TFS_BF16, DEV, V)
    head = (8 * V + 255) // 256 * 256
    outs = []
    for _ in range(3):
        o = ops.sampled_softmax(T(c["h"]), T(c["labels"]), T(c["w_true"]), T(c["b_true"]),
                                T(c["le_t"]), T(c["s"]), T(c["w_s"]), T(c["b_s"]), T(c["le_s"]),
                                grad_scale=1.0 / B, operand_dtype=TFS_BF16, vocab=V, ws=ws)
        torch.cuda.synchronize()
        assert int(ws[:head + 256].count_nonzero()) == 0
        outs.append({k: v.clone() for k, v in o.items()})
    for o in outs[1:]:
        for k in o:
            assert torch.equal(o[k], outs[0][k]), k


@pytest.mark.parametrize("B,S,d", [(2560, 8192, 512), (300, 1000, 64)])
def test_ssm_rows_ready_event(B, S, d):
    """tfs_ssm_args.rows_ready_event: a copy of dw_true / db_true / dw_s / db_s taken on another
    stream as soon as the event fires equals the call's final values (the event follows every
    write of them; dh's split-K reduction may still be running) -- outputs prefilled with NaN."""
    c = _ssm_case(B, S, 40000, d, seed=B + 7 * S)
    nan = lambda *sh: torch.full(sh, float("nan"), device=DEV)
    out = {"loss": nan(B), "lse": nan(B), "loss_sum": nan(1), "dh": nan(B, d), "dw_true": nan(B, d),
           "db_true": nan(B), "dw_s": nan(S, d), "db_s": nan(S)}
    ev = torch.cuda.Event()
    ev.record()  # (creates the event before the library records it)
    side = torch.cuda.Stream()
    torch.cuda.synchronize()
    ops.sampled_softmax(T(c["h"]), T(c["labels"]), T(c["w_true"]), T(c["b_true"]),
                        T(c["le_t"]), T(c["s"]), T(c["w_s"]), T(c["b_s"]), T(c["le_s"]),
                        grad_scale=1.0 / B, operand_dtype=TFS_BF16, vocab=c["V"], out=out,
                        rows_ready=ev)
    with torch.cuda.stream(side):
        side.wait_event(ev)
        snap = {k: out[k].clone() for k in ("dw_true", "db_true", "dw_s", "db_s")}
    torch.cuda.synchronize()
    for k, v in snap.items():
        assert torch.equal(v, out[k]), k
        assert not torch.isnan(v).any(), k


def test_ssm_deterministic():
    c = _ssm_case(512, 1024, 40000, 128, seed=1)
    a = _run_ssm(c, TFS_BF16, 0.01)
    b = _run_ssm(c, TFS_BF16, 0.01)
    for k in KEYS:
        assert np.array_equal(a[k], b[k]), k


# --------------------------------------------------------------------------- Sort-reduce / SGD
@pytest.mark.parametrize("n,R,dim", [(1, 1, 512), (2560, 1, 512), (10752, 8, 512), (5000, 3, 64),
                                     (70000, 2, 8)])
def test_sort_reduce_parity(n, R, dim):
    V = 800_000
    rng = np.random.default_rng(n)
    ids = workloads.zipf_ids(rng, V, 1.1, n)
    rows = rng.standard_normal((n, dim)).astype(np.float32)
    rows2 = rng.standard_normal(n).astype(np.float32)
    local, sums, sums2, counts, U = ops.sort_reduce(T(ids), V, R, T(rows), rows2=T(rows2))
    ol, osum, oc = oracle.sort_reduce(ids, R, rows.astype(np.float64))
    _, osum2, _ = oracle.sort_reduce(ids, R, rows2.astype(np.float64))
    _, asum, _ = oracle.sort_reduce(ids, R, np.abs(rows.astype(np.float64)))
    _, asum2, _ = oracle.sort_reduce(ids, R, np.abs(rows2.astype(np.float64)))
    u = int(U.item())
    assert u == ol.size
    assert np.array_equal(local[:u].cpu().numpy(), ol)
    assert np.array_equal(counts.cpu().numpy(), oc)
    assert elem_err(sums[:u].cpu().numpy(), osum, asum) <= TOL_F32
    assert elem_err(sums2[:u].cpu().numpy(), osum2, asum2) <= TOL_F32


def _update_scale(ids, g, lr):
    """lr x the sum of |gradient rows| of each distinct id (ascending ids, like np.unique)."""
    _, a, _ = oracle.sort_reduce(ids, 1, np.abs(np.asarray(g, np.float64)))
    return lr * a


@pytest.mark.parametrize("n,dim,zipf", [(2560, 512, 1.0), (10752, 64, 1.2), (65536, 16, 1.1),
                                        (100, 3, 1.0)])
def test_scatter_add_sgd_parity(n, dim, zipf):
    rows_t = 50_000
    rng = np.random.default_rng(n + dim)
    table = rng.standard_normal((rows_t, dim)).astype(np.float32)
    ids = workloads.zipf_ids(rng, rows_t, zipf, n)
    g = rng.standard_normal((n, dim)).astype(np.float32)
    t2 = rng.standard_normal(rows_t).astype(np.float32)
    g2 = rng.standard_normal(n).astype(np.float32)
    lr = 1.0
    dt, dt2 = T(table), T(t2)
    ops.scatter_add_sgd(dt, T(ids), T(g), lr, table2=dt2, grad2=T(g2))
    ref = oracle.scatter_add_sgd(table, ids, g.astype(np.float64), lr)
    ref2 = oracle.scatter_add_sgd(t2, ids, g2.astype(np.float64), lr)
    got = dt.cpu().numpy()
    touched = np.unique(ids)
    untouched = np.setdiff1d(np.arange(rows_t), touched)
    assert np.array_equal(got[untouched], table[untouched])
    sc = _update_scale(ids, g, lr)
    sc2 = _update_scale(ids, g2, lr)
    assert update_err(got[touched], ref[touched], sc) <= TOL_F32
    got2 = dt2.cpu().numpy()
    assert update_err(got2[touched], ref2[touched], sc2) <= TOL_F32


def test_scatter_add_sgd_errors_and_empty():
    table = T(np.zeros((10, 4), np.float32))
    ops.scatter_add_sgd(table, T(np.zeros(0, np.int64)), T(np.zeros((0, 4), np.float32)), 1.0)
    assert table.abs().sum().item() == 0
    err = ops.ErrorSlot(DEV)
    ids = np.array([1, 2, 10, 3, 11])
    ops.scatter_add_sgd(table, T(ids), T(np.ones((5, 4), np.float32)), 1.0, err=err)
    assert err.read() == (2, 2)
    assert table[1].tolist() == [-1.0] * 4 and table[3].tolist() == [-1.0] * 4


@pytest.mark.parametrize("dim", [512, 6])
def test_heavy_hitter_segments(dim):
    """One id repeated 15,000 times plus a Zipf tail: exercises the piece path (segments of more
    than 32 rows summed as 64-row pieces combined in piece order)."""
    rows_t, n = 3000, 20000
    rng = np.random.default_rng(dim)
    ids = workloads.zipf_ids(rng, rows_t, 1.2, n)
    ids[rng.permutation(n)[:15000]] = 5
    table = rng.standard_normal((rows_t, dim)).astype(np.float32)
    g = rng.standard_normal((n, dim)).astype(np.float32)
    dt = T(table)
    ops.scatter_add_sgd(dt, T(ids), T(g), 0.5)
    ref = oracle.scatter_add_sgd(table, ids, g.astype(np.float64), 0.5)
    touched = np.unique(ids)
    got = dt.cpu().numpy()
    assert update_err(got[touched], ref[touched], _update_scale(ids, g, 0.5)) <= TOL_F32
    local, sums, _, counts, U = ops.sort_reduce(T(ids), rows_t, 4, T(g))
    ol, osum, oc = oracle.sort_reduce(ids, 4, g.astype(np.float64))
    _, asum, _ = oracle.sort_reduce(ids, 4, np.abs(g.astype(np.float64)))
    u = int(U.item())
    assert np.array_equal(local[:u].cpu().numpy(), ol) and np.array_equal(counts.cpu().numpy(), oc)
    assert elem_err(sums[:u].cpu().numpy(), osum, asum) <= TOL_F32
    # determinism of the piece path
    dt2 = T(table)
    ops.scatter_add_sgd(dt2, T(ids), T(g), 0.5)
    assert torch.equal(dt.cpu(), dt2.cpu())


@pytest.mark.parametrize("n,dim,zipf", [(2560, 512, 1.0), (10752, 64, 1.2), (777, 6, 1.0)])
def test_planned_scatter_matches_unplanned(n, dim, zipf):
    """tfs_scatter_plan + tfs_scatter_add_sgd_planned == tfs_scatter_add_sgd, bit for bit, and
    one plan serves repeated applies with fresh gradients."""
    rng = np.random.default_rng(n + dim)
    V = 5000
    ids = workloads.zipf_ids(rng, V, zipf, n)
    g1 = rng.standard_normal((n, dim)).astype(np.float32)
    g2 = rng.standard_normal((n, dim)).astype(np.float32)
    gb = rng.standard_normal(n).astype(np.float32)
    t0 = rng.standard_normal((V, dim)).astype(np.float32)
    b0 = rng.standard_normal(V).astype(np.float32)
    a, ab = T(t0), T(b0)
    ops.scatter_add_sgd(a, T(ids), T(g1), 0.1, table2=ab, grad2=T(gb))
    ops.scatter_add_sgd(a, T(ids), T(g2), 0.1)
    b, bb = T(t0), T(b0)
    plan = ops.ScatterPlan(n, V, dim, DEV).build(T(ids))
    plan.apply(b, T(g1), 0.1, table2=bb, grad2=T(gb))
    plan.apply(b, T(g2), 0.1)
    assert torch.equal(a, b) and torch.equal(ab, bb)


@pytest.mark.parametrize("R,n,dim,cap", [(3, 700, 64, 400), (2, 2560, 512, 1500), (4, 999, 6, 300),
                                         (8, 600, 8, 7000)])  # last: merge beyond shared memory
def test_fixed_capacity_route_round_trip(R, n, dim, cap):
    """tfs_route_plan / tfs_gather_slots / tfs_route_unpack / tfs_route_reduce /
    tfs_scatter_*_slots with R requesters simulated on one GPU (the all-to-all is a tensor
    transpose of slot regions): the stitched rows equal table[ids] bit for bit, and the owner
    updates equal per-requester fixed-order sums added in requester order; the merge plan
    (sorted runs) equals the radix plan bit for bit."""
    rng = np.random.default_rng(R * n + dim)
    V, lr = 5000, 0.5
    table = rng.standard_normal((V, dim)).astype(np.float32)
    ids = [workloads.zipf_ids(rng, V, 1.1, n) for _ in range(R)]
    grads = [rng.standard_normal((n, dim)).astype(np.float32) for _ in range(R)]
    stride = cap + 5                     # regions wider than the slots
    rstride = (cap * dim + 8) // 4 * 4
    plans, send = [], torch.full((R, R, stride), -9, dtype=torch.int64, device=DEV)
    counts = torch.zeros((R, R), dtype=torch.int64, device=DEV)
    for r in range(R):
        plans.append(ops.RoutePlan(n, V, R, cap, dim, DEV).build(T(ids[r]), send[r], stride,
                                                                 counts=counts[r]))
    recv = send.transpose(0, 1).contiguous()               # recv[o][src] = send[src][o]
    for r in range(R):
        want = [len(np.unique(ids[r][ids[r] % R == o])) for o in range(R)]
        assert counts[r].tolist() == want
    rows = torch.zeros((R, R, rstride), dtype=torch.float32, device=DEV)
    for o in range(R):
        ops.gather_slots(T(np.ascontiguousarray(table[o::R])), recv[o], stride, R, cap, rows[o],
                         rstride)
    back = rows.transpose(0, 1).contiguous()               # back[r][o] = rows[o][r]
    for r in range(R):
        h = torch.empty((n, dim), dtype=torch.float32, device=DEV)
        plans[r].unpack(back[r], rstride, dim, h)
        assert np.array_equal(h.cpu().numpy(), table[ids[r]])
    gs = torch.zeros((R, R, rstride), dtype=torch.float32, device=DEV)
    for r in range(R):
        plans[r].reduce(T(grads[r]), dim, gs[r], rstride)
    gr = gs.transpose(0, 1).contiguous()
    for o in range(R):
        shard = table[o::R]
        res = []
        for sorted_runs in (True, False):
            t = T(np.ascontiguousarray(shard))
            p = ops.SlotScatterPlan(R, cap, shard.shape[0], dim, DEV)
            p.build(recv[o], stride, sorted_runs=sorted_runs)
            p.apply(t, gr[o], rstride, lr)
            res.append(t.cpu().numpy())
        assert np.array_equal(res[0], res[1])
        ref = shard.astype(np.float64)
        scale = np.zeros(shard.shape)
        for r in range(R):                                  # requester order
            acc = {}
            for i in range(n):
                if ids[r][i] % R == o:
                    acc.setdefault(ids[r][i] // R, []).append(grads[r][i].astype(np.float64))
            for loc, rows_ in acc.items():
                ref[loc] -= lr * np.sum(rows_, axis=0)
                scale[loc] += lr * np.sum(np.abs(rows_), axis=0)
        touched = np.unique(np.concatenate([ids[r][ids[r] % R == o] // R for r in range(R)]))
        assert update_err(res[0][touched], ref[touched].astype(np.float32),
                          scale[touched]) <= TOL_F32


def test_route_plan_capacity_overflow_is_reported():
    V, R, n = 1000, 2, 500
    ids = np.arange(n, dtype=np.int64) * 2            # every id owned by shard 0
    send = torch.empty((R, 100), dtype=torch.int64, device=DEV)
    err = ops.ErrorSlot(DEV)
    ops.RoutePlan(n, V, R, 100, 8, DEV).build(T(ids), send, 100, err=err)
    assert err.read() == (9, 0)


@pytest.mark.parametrize("B,S,d", [(2560, 512, 512), (300, 1000, 64)])
def test_ssm_bf16_operand_inputs_identical(B, S, d):
    """TFS_BF16_OPERANDS: h / w_true / w_s handed over already rounded (a bf16 Gather) give
    bit-identical outputs to the fp32 inputs rounded inside the call."""
    c = _ssm_case(B, S, 40000, d, seed=B + 2 * S)
    ref = _run_ssm(c, TFS_BF16, 1.0 / B)
    bf = lambda a: T(a).to(torch.bfloat16)
    out = ops.sampled_softmax(bf(c["h"]), T(c["labels"]), bf(c["w_true"]), T(c["b_true"]),
                              T(c["le_t"]), T(c["s"]), bf(c["w_s"]), T(c["b_s"]), T(c["le_s"]),
                              grad_scale=1.0 / B, operand_dtype=TFS_BF16, vocab=c["V"])
    for k in KEYS + ("loss_sum",):
        assert np.array_equal(out[k].cpu().numpy(), ref[k]), k


@pytest.mark.parametrize("kind", ["momentum", "adagrad"])
@pytest.mark.parametrize("n,dim,zipf", [(10752, 512, 1.0), (5000, 6, 1.2), (65536, 64, 1.1)])
def test_sparse_momentum_adagrad_match_oracle(kind, n, dim, zipf):
    """tfs_scatter_opt_planned against the oracle on Zipf ids with heavy
    duplicates, including the width-1 companion table with its own slot; two consecutive steps
    so the slots carry state; kind 'sgd' through the same entry equals the SGD apply bit for
    bit."""
    rng = np.random.default_rng(n + dim)
    V, lr, mu = 4000, 0.05, 0.9
    ids = workloads.zipf_ids(rng, V, zipf, n)
    t0 = rng.standard_normal((V, dim)).astype(np.float32)
    b0 = rng.standard_normal(V).astype(np.float32)
    s0 = (np.abs(rng.standard_normal((V, dim))) * 0.1).astype(np.float32)
    sb0 = (np.abs(rng.standard_normal(V)) * 0.1).astype(np.float32)
    gs = [rng.standard_normal((n, dim)).astype(np.float32) for _ in range(2)]
    gbs = [rng.standard_normal(n).astype(np.float32) for _ in range(2)]
    t, b, s, sb = T(t0), T(b0), T(s0), T(sb0)
    plan = ops.ScatterPlan(n, V, dim, DEV).build(T(ids))
    ro, rb, rs, rsb = t0, b0, s0, sb0
    # element-wise error scales propagated through the two steps from the gradient sums'
    # term scale ga = sum |g| per distinct id (momentum: m = mu m + g, T -= lr m; Adagrad:
    # a += g^2 -> 2 ga^2, T -= lr g / sqrt(a) -> lr (ga / sqrt(a) + ga S_a / (2 a^1.5)))
    touched = np.unique(ids)
    sc = {"T": 0.0, "S": 0.0, "b": 0.0, "sb": 0.0}
    for g, gb in zip(gs, gbs):
        plan.apply_opt(kind, t, T(g), lr, s, mu, table2=b, grad2=T(gb), slot2=sb)
        ro, rs = oracle.scatter_opt(kind, ro, rs, ids, g.astype(np.float64), lr, mu)
        rb, rsb = oracle.scatter_opt(kind, rb, rsb, ids, gb.astype(np.float64), lr, mu)
        for key, grad, slot_ref in (("T", g, rs), ("b", gb, rsb)):
            ga = _update_scale(ids, grad, 1.0)
            skey = "S" if key == "T" else "sb"
            if kind == "momentum":
                sc[skey] = mu * sc[skey] + ga
                sc[key] = sc[key] + lr * sc[skey]
            else:
                a = slot_ref[touched].astype(np.float64)
                sc[skey] = sc[skey] + 2 * ga * ga
                sc[key] = sc[key] + lr * (ga / np.sqrt(a) + ga * sc[skey] / (2 * a ** 1.5))
    for got, ref, init, key in ((t, ro, t0, "T"), (s, rs, s0, "S"), (b, rb, b0, "b"),
                                (sb, rsb, sb0, "sb")):
        gn = got.cpu().numpy()
        e = update_err(gn[touched], ref[touched], sc[key], ulps=2)
        assert e <= TOL_F32, (key, e)
        untouched = np.setdiff1d(np.arange(V), touched)
        assert np.array_equal(gn[untouched], init[untouched])
    a, c = T(t0), T(t0)
    plan.apply_opt("sgd", a, T(gs[0]), lr, None)
    plan.apply(c, T(gs[0]), lr)
    assert torch.equal(a, c)


@pytest.mark.parametrize("kind", ["sgd", "momentum", "adagrad"])
@pytest.mark.parametrize("n,zipf", [(10752, 1.0), (65536, 1.1)])
def test_sparse_update_keeps_bf16_mirror(kind, n, zipf):
    """tfs_sparse_opt.mirror: after the update every row of the bf16 mirror equals the RNE bf16
    of the updated fp32 row (whole segments and the heavy ids crossing windows alike), untouched
    rows keep their mirror bits, and the fp32 result is the one without a mirror."""
    V, dim = 50_000, 64
    rng = np.random.default_rng(n + len(kind))
    ids = workloads.zipf_ids(rng, V, zipf, n)
    t0 = rng.standard_normal((V, dim)).astype(np.float32)
    g = rng.standard_normal((n, dim)).astype(np.float32)
    plan = ops.ScatterPlan(n, V, dim, DEV).build(T(ids))
    slot = (torch.full((V, dim), 0.1, device=DEV) if kind != "sgd" else None)
    slot_c = slot.clone() if slot is not None else None
    t, c = T(t0), T(t0)
    mir = t.to(torch.bfloat16)
    plan.apply_opt(kind, t, T(g), 0.05, slot, 0.9, mirror=mir)
    plan.apply_opt(kind, c, T(g), 0.05, slot_c, 0.9)
    assert torch.equal(t, c)
    assert torch.equal(mir.view(torch.int16), t.to(torch.bfloat16).view(torch.int16))


# ------------------------------------------------------- vocabulary-sharded full softmax (halves)
def _full_softmax_oracle(h, labels, W, bb, c, bf16=False):
    """Full softmax via the oracle with all V classes as candidates and the label among them
    (flag LABEL_IN_CANDIDATES, reading R-30 -- pinned to the textbook dense softmax and its
    bf16 rounding point in test_oracle): per-class gradients directly."""
    V = W.shape[0]
    return oracle.sampled_softmax(h, labels, None, None, None, np.arange(V), W, bb, np.zeros(V),
                                  flags=oracle.LABEL_IN_CANDIDATES, grad_scale=c, bf16=bf16)


def _sharded_full_softmax(h, labels, W, bb, c, R):
    """R vocabulary shards (class v on shard v mod R) simulated on one GPU through the C ABI."""
    M, d = h.shape
    V = W.shape[0]
    th, ty = T(h), T(labels)
    shards = []
    for r in range(R):
        ids = np.arange(r, V, R)
        ws = ops.ssm_workspace(M, ids.size, d, TFS_BF16, DEV, V)
        args = (th, ty, T(ids), T(W[ids]), T(bb[ids]))
        st = ops.ssm_partial_stats(*args, vocab=V, ws=ws)
        shards.append((ids, ws, args, st))
    tab = lambda ts: torch.tensor([t.data_ptr() for t in ts], dtype=torch.int64, device=DEV)
    lse = torch.empty(M, device=DEV)
    ops.lse_combine_peers(tab([s[3] for s in shards]), R, M, lse)
    outs = [ops.ssm_backward_from_lse(*args, lse, grad_scale=c, ws=ws, vocab=V)
            for ids, ws, args, st in shards]
    dh = torch.empty(M, d, device=DEV)
    ops.reduce_peers(tab([o["dh"] for o in outs]), R, 0, M * d, dh)
    loss = torch.zeros(R, device=DEV)
    for r in range(R):
        ops.label_loss_sum(lse, outs[r]["z_label"], ty, R, r, c, loss[r:])
    dW = np.zeros_like(W, dtype=np.float64)
    db = np.zeros(V)
    for r, o in enumerate(outs):
        dW[shards[r][0]] = o["dw_s"].cpu().numpy()
        db[shards[r][0]] = o["db_s"].cpu().numpy()
    maps_zero = all(int(s[1][:8 * V].count_nonzero()) == 0 for s in shards)
    return lse.cpu().numpy(), dh.cpu().numpy(), dW, db, float(loss.sum()), maps_zero


@pytest.mark.parametrize("M,V,d,R", [(77, 500, 64, 1), (256, 1000, 64, 3), (300, 2000, 128, 2),
                                     (1024, 4000, 512, 4)])
def test_sharded_full_softmax_halves(M, V, d, R):
    """logits and gradients computed on each vocabulary shard, combined through
    (max, sum) pairs, equal the full softmax (loss, dh, dW, db)."""
    rng = np.random.default_rng(M + V + R)
    W = (rng.random((V, d), dtype=np.float32) - 0.5)
    bb = (rng.random(V, dtype=np.float32) - 0.5) * 0.2
    h = (rng.random((M, d), dtype=np.float32) - 0.5)
    labels = workloads.zipf_ids(rng, V, 1.0, M)
    c = 1.0 / M
    lse, dh, dW, db, loss_sum, maps_zero = _sharded_full_softmax(h, labels, W, bb, c, R)
    for o, tol in ((_full_softmax_oracle(h, labels, W, bb, c), TOL_BF16_ACC),
                   (_full_softmax_oracle(h, labels, W, bb, c, bf16=True), TOL_BF16_EMU)):
        assert elem_err(lse, o["lse"], o["abs_loss"]) <= tol
        for g, k in ((dh, "dh"), (dW, "dw_s"), (db, "db_s")):
            e = elem_err(g, o[k], o["abs_" + k], o["amb_" + k])
            assert e <= tol, (k, tol, e)
        want = c * o["loss"].sum()
        assert abs(loss_sum - want) <= tol * c * o["abs_loss"].sum()
    assert maps_zero
