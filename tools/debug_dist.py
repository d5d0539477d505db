"""Debug driver: the R-rank step (one process per GPU, torchrun) vs the oracle, step by step,
eager and graph-replayed, printing every table's element-wise error per step.

    torchrun --nproc-per-node 2 tools/debug_dist.py [T|L|Fm] [full]
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import oracle  # noqa: E402,F401
from oracle import step as ostep  # noqa: E402
import workloads  # noqa: E402
from parity import update_err  # noqa: E402
from paper_1605_08695_b200 import step as gstep  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "T"
    full = len(sys.argv) > 2 and sys.argv[2] == "full"
    rank, R = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    extra = {"Fm": dict(vocab=4000, dim=128, tokens=256)}
    w = (workloads.Workload(name, shards=R, num_sampled=0, **extra[name]) if name in extra
         else workloads.WORKLOADS[name])
    S = 0 if full else w.num_sampled
    V, B = w.vocab, w.tokens_per_replica(R)
    E, W, b = workloads.tables(V, w.dim)
    cfg = gstep.StepConfig(vocab=V, dim=w.dim, tokens=B, num_sampled=S, num_shards=R, lr=1.0,
                           seed=workloads.SAMPLER_SEED)
    comm = gstep.Comm.distributed(cfg, timeout_ms=20000)
    st = gstep.Step(cfg, comm)
    st.load_tables(E[rank::R], W[rank::R], b[rank::R])
    st.sync()
    for mode in ("eager", "graph"):
        st.set_step(0)
        if mode == "graph":
            st.capture()
        tabs = (E, W, b)
        for k in range(3):
            xs, ys = zip(*[workloads.batch(w, R, r, step=k) for r in range(R)])
            ocfg = ostep.StepConfig(vocab=V, dim=w.dim, num_sampled=S or V, num_shards=R, lr=1.0,
                                    seed=workloads.SAMPLER_SEED, step=k, bf16=True,
                                    full_softmax=full, label_in=full, abs_bounds=True)
            E2, W2, b2, tr = ostep.step(*tabs, list(xs), list(ys), ocfg)
            dist.barrier()
            st.run(torch.from_numpy(xs[rank]).to(dev), torch.from_numpy(ys[rank]).to(dev))
            torch.cuda.synchronize()
            errs = {"err": st.error(), "comm": comm.error()}
            got = torch.tensor([float(st.tensor("loss_sum").item())], dtype=torch.float64,
                               device=dev)
            dist.all_reduce(got)
            want = sum(t.ssm["loss"].sum() for t in tr) / (R * B)
            errs["loss"] = float(got.item()) - want
            nxt = []
            for nm, T0, To, A in zip("EWb", tabs, (E2, W2, b2), tr[0].abs_delta):
                g = st.tensor(nm).cpu().numpy()
                t0, to, a = T0[rank::R], To[rank::R], A[rank::R]
                touched = np.nonzero(np.any((a != 0).reshape(t0.shape[0], -1), axis=1))[0]
                unt = np.setdiff1d(np.arange(t0.shape[0]), touched)
                errs[nm] = (update_err(g[touched], to[touched], a[touched]),
                            bool(np.array_equal(g[unt], t0[unt])))
                parts = [None] * R
                dist.all_gather_object(parts, g)
                tab = np.empty_like(T0)
                for r in range(R):
                    tab[r::R] = parts[r]
                nxt.append(tab)
            tabs = tuple(nxt)
            print(f"rank {rank} {mode} step {k}: {errs}", flush=True)
        if mode == "graph":
            st.uncapture()
        st.load_tables(E[rank::R], W[rank::R], b[rank::R])
        st.sync()
        dist.barrier()
    st.close()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
