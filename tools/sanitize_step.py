"""Small driver for compute-sanitizer (memcheck / racecheck / synccheck): the native step on
configs T and L (R = 1, bf16 and fp32 operands), T with R = 2 ranks simulated on one GPU, and
the sharded full softmax with R = 2 simulated ranks; each run eagerly, then once as a captured
CUDA graph.  Exits non-zero if any step reports a data error.

    compute-sanitizer --tool memcheck python tools/sanitize_step.py [T|L|all]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads  # noqa: E402
from paper_1605_08695_b200 import step as gstep  # noqa: E402
from paper_1605_08695_b200._lib import TFS_BF16, TFS_F32  # noqa: E402


def run(name, R=1, dtype=TFS_BF16, full=False, graph=True):
    w = workloads.WORKLOADS[name] if not full else workloads.Workload("Fs", 1000, 64, 32, 0, R)
    E, W, b = workloads.tables(w.vocab, w.dim)
    B = w.tokens_per_replica(R)
    cfg = gstep.StepConfig(vocab=w.vocab, dim=w.dim, tokens=B, num_sampled=w.num_sampled,
                           num_shards=R, lr=0.5, seed=workloads.SAMPLER_SEED,
                           operand_dtype=dtype)
    comm = gstep.Comm.simulated(cfg) if R > 1 else None
    st = gstep.Step(cfg, comm)
    for r in range(st.nlocal):
        st.load_tables(E[r::R], W[r::R], b[r::R], local=r)
    st.sync()
    xs, ys = zip(*[workloads.batch(w, R, r) for r in range(R)])
    import numpy as np
    x = torch.from_numpy(np.concatenate(xs)).cuda()
    y = torch.from_numpy(np.concatenate(ys)).cuda()
    st.run(x, y)
    if graph:
        st.capture()
        st.run(x, y)
    st.check(f"{name} R={R}")
    st.close()
    if comm is not None:
        comm.close()
    print(f"ok {name} R={R} dtype={dtype} full={full}", flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("T", "all"):
        run("T")
        run("T", dtype=TFS_F32, graph=False)
        run("T", R=2)
        run("T", R=2, full=True)
    if which in ("L", "all"):
        run("L", graph=False)
