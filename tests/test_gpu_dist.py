"""Multi-GPU parity of the sharded step (R = 2 or 4 processes, one per GPU, tfs_comm over CUDA
IPC / NVLink) against the oracle step with R shards: three captured-and-replayed steps, sampled
ids bit-exact per replica, the global loss, and each rank's updated shard of E, W, b element by
element (tests/parity.py).  Needs >= 2 GPUs (gpurun --gpus 2); skipped otherwise.  The same
phases are covered on one GPU by tests/test_gpu_step.py (ranks simulated)."""
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
    """One rank of a real multi-GPU run (one process per GPU, tfs_comm over CUDA IPC / NVLink):
    three steps captured once into a CUDA graph and replayed, each compared with the oracle's
    synchronous step over R shards (tests/parity.py metric)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import oracle  # noqa: F401
    from oracle import step as ostep
    import workloads
    from parity import update_err
    from paper_1605_08695_b200 import step as gstep
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        w = _workload(name)
        V, R = w.vocab, world
        E, W, b = workloads.tables(V, w.dim)
        B = w.tokens_per_replica(R)
        S = 0 if full else w.num_sampled      # full: the vocabulary-sharded full softmax
        cfg = gstep.StepConfig(vocab=V, dim=w.dim, tokens=B, num_sampled=S,
                               num_shards=R, lr=1.0, seed=workloads.SAMPLER_SEED,
                               operand_dtype=dtype)
        comm = gstep.Comm.distributed(cfg, timeout_ms=60000)
        st = gstep.Step(cfg, comm)
        st.load_tables(E[rank::R], W[rank::R], b[rank::R])
        st.sync()
        st.set_step(0)
        st.capture()
        res = {"sampled": True, "loss": 0.0}
        for k in range(3):
            xs, ys = zip(*[workloads.batch(w, R, r, step=k) for r in range(R)])
            ocfg = ostep.StepConfig(vocab=V, dim=w.dim, num_sampled=S or V, num_shards=R,
                                    lr=1.0, seed=workloads.SAMPLER_SEED, step=k,
                                    bf16=(dtype == 1), full_softmax=full, label_in=full,
                                    abs_bounds=True)
            E2, W2, b2, tr = ostep.step(E, W, b, list(xs), list(ys), ocfg)
            dist.barrier()
            st.run(torch.from_numpy(xs[rank]).to(dev), torch.from_numpy(ys[rank]).to(dev))
            st.check(f"dist step {k}")
            got = torch.tensor([float(st.tensor("loss_sum").item())], dtype=torch.float64,
                               device=dev)
            dist.all_reduce(got)
            want = sum(t.ssm["loss"].sum() for t in tr) / (R * B)
            scale = sum(t.ssm["abs_loss"].sum() for t in tr) / (R * B)
            res["loss"] = max(res["loss"], abs(float(got.item()) - want) / scale)
            if not full:
                res["sampled"] &= bool(np.array_equal(st.tensor("qw")[B:].cpu().numpy(),
                                                      tr[rank].sampled))
            aE, aW, ab = tr[0].abs_delta
            mE, mW, mb = tr[0].amb_delta
            nxt = []
            for nm, T0, To, A, Mb in (("E", E, E2, aE, mE), ("W", W, W2, aW, mW),
                                      ("b", b, b2, ab, mb)):
                g = st.tensor(nm).cpu().numpy()
                t0, to, a, m = T0[rank::R], To[rank::R], A[rank::R], Mb[rank::R]
                touched = np.nonzero(np.any((a != 0).reshape(t0.shape[0], -1), axis=1))[0]
                untouched = np.setdiff1d(np.arange(t0.shape[0]), touched)
                res[nm + "_untouched"] = res.get(nm + "_untouched", True) and bool(
                    np.array_equal(g[untouched], t0[untouched]))
                res[nm] = max(res.get(nm, 0.0), update_err(g[touched], to[touched], a[touched],
                                                           allow=m[touched]))
                # the next step starts from the GPUs' own state (identical inputs, c.5)
                parts = [None] * R
                dist.all_gather_object(parts, g)
                table = np.empty_like(T0)
                for r in range(R):
                    table[r::R] = parts[r]
                nxt.append(table)
            E, W, b = nxt
        q.put((rank, res))
        st.close()
        comm.close()
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
@pytest.mark.parametrize("name,tol", [("T", 2e-3), ("L", 2e-3)])
def test_dist_step_matches_oracle(name, tol):
    res = _run_ranks([(name, 1, "p2p")] * 2)
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
    all R*B tokens) reaches the oracle's label-in full-softmax step over the same global batch
    (bf16 emulation, R-30)."""
    res = _run_ranks([(name, 1, "p2p", True)] * 2)
    for rank, r in res:
        assert r["loss"] <= 2e-3, (rank, r)
        for nm in ("E", "W", "b"):
            assert r[nm + "_untouched"], (rank, nm)
            assert r[nm] <= 2e-3, (rank, nm, r[nm])


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs 4 GPUs")
@pytest.mark.parametrize("name,full", [("T", False), ("L", False), ("Fo", True)])
def test_dist4_matches_oracle(name, full):
    """R = 4 processes (the bench's 4-GPU configuration): the sampled step, and the sharded
    full softmax with V = 4003 (shards of 1001 / 1001 / 1001 / 1000 classes)."""
    res = _run_ranks([(name, 1, "p2p", full)] * 4)
    assert len(res) == 4
    for rank, r in res:
        assert r["sampled"], rank
        assert r["loss"] <= 2e-3, (rank, r)
        for nm in ("E", "W", "b"):
            assert r[nm + "_untouched"], (rank, nm)
            assert r[nm] <= 2e-3, (rank, nm, r[nm])
