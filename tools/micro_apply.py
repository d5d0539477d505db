"""Micro-benchmark of the planned ScatterAdd-SGD (plan build and apply) at the step's shapes.

    python tools/micro_apply.py            # (with TFS_ALLOW_VARIANT_LIB=1 TFS_LIB=... for A/B)

Per case: ids drawn like the workloads (Zipf over V = 800k, or the W-side mix of unique sampled
ids + Zipf labels), gradient rows fp32 [n x 512]; L2 flushed before every timed call; CUDA
events on the current stream; median of 30.  Prints plan / apply microseconds and the apply's
algorithmic bytes (gradient rows + table read-modify-write of the distinct rows) per second.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1605_08695_b200 import ops  # noqa: E402

V, D = 800_000, 512


def zipf(rng, s, n):
    r = np.arange(1, V + 1, dtype=np.float64)
    p = r ** -s
    p /= p.sum()
    return rng.choice(V, size=n, p=p).astype(np.int64)


def timed(fn, flush, reps=30):
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


def main():
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(1)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    table = torch.zeros((V, D), dtype=torch.float32, device=dev)
    cases = [
        ("E_X", zipf(rng, 1.0, 2560)),
        ("W_X", np.concatenate([zipf(rng, 1.0, 2560), rng.choice(V, 8192, replace=False)])),
        ("E_Z", zipf(rng, 1.1, 65536)),
        ("W_Z", np.concatenate([zipf(rng, 1.1, 65536), rng.choice(V, 8192, replace=False)])),
        ("uniq_40k", rng.choice(V, 40000, replace=False)),
    ]
    for name, ids_np in cases:
        n = ids_np.size
        ids = torch.from_numpy(ids_np).to(dev)
        grad = torch.randn((n, D), dtype=torch.float32, device=dev)
        plan = ops.ScatterPlan(n, V, D, dev)
        t_plan = timed(lambda: plan.build(ids), flush)
        plan.build(ids)
        t_apply = timed(lambda: plan.apply(table, grad, 1e-3), flush)
        u = np.unique(ids_np).size
        nbytes = n * D * 4 + 2 * u * D * 4
        print(f"{name:9s} n={n:6d} distinct={u:6d} plan {t_plan:7.1f} us  apply {t_apply:7.1f} us "
              f"{nbytes / t_apply / 1e3:7.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
