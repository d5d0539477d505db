"""Stress driver for the one-process-per-GPU step (torchrun): K eager steps then K graph replays
of workload W (default X), the error slots checked after every step; on an error, the inbox
contents are inspected (ids outside [-1, nloc)).

    torchrun --nproc-per-node 4 tools/stress_dist.py [X] [K]
"""
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads  # noqa: E402
from paper_1605_08695_b200 import step as gstep  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "X"
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    rank, R = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    w = workloads.WORKLOADS[name]
    B = w.tokens_per_replica(R)
    cfg = gstep.StepConfig(vocab=w.vocab, dim=w.dim, tokens=B, num_sampled=w.num_sampled,
                           num_shards=R, lr=0.1, seed=workloads.SAMPLER_SEED)
    comm = gstep.Comm.distributed(cfg, timeout_ms=20000)
    st = gstep.Step(cfg, comm)
    E, W, b = workloads.tables_device(w.vocab, w.dim, R, rank, dev)
    st.load_tables(E, W, b)
    st.sync()
    xs = [torch.from_numpy(workloads.batch(w, R, rank, step=i)[0]).to(dev) for i in range(16)]
    ys = [torch.from_numpy(workloads.batch(w, R, rank, step=i)[1]).to(dev) for i in range(16)]
    nloc = st.tensor("E").shape[0]
    for mode in ("eager", "graph"):
        if mode == "graph":
            st.capture()
        for i in range(K):
            st.run(xs[i % 16], ys[i % 16])
            torch.cuda.synchronize()
            code, idx = st.error()
            ccode, cidx = comm.error()
            bad = torch.tensor([code, ccode], device=dev)
            dist.all_reduce(bad, op=dist.ReduceOp.MAX)
            if code or ccode:
                heap = comm.heap()
                print(f"rank {rank} {mode} step {i}: err ({code}, {idx}) comm ({ccode}, {cidx})",
                      flush=True)
            if int(bad.max().item()):
                break
        if int(bad.max().item()):
            break
        if rank == 0:
            print(f"{mode}: {K} steps clean", flush=True)
    st.close()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
