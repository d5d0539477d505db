"""Per-launch times of one sampled-softmax call at the X shape (B 2560, S 8192, d 512, bf16
operands as the step passes them, label ids and candidates in V = 800k), from the call's own
timing events (include/tfs.h): prep, logits GEMM, combine, gradient GEMM, column sums, grouped
dh / dW_s GEMM, finalize; median of 20 calls, L2 flushed before each.  For A/B of GEMM builds
(TFS_ALLOW_VARIANT_LIB=1 TFS_LIB=...).  Usage: python tools/time_ssm.py [B S]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1605_08695_b200 import ops  # noqa: E402
from paper_1605_08695_b200._lib import TFS_BF16  # noqa: E402

dev = "cuda"
B = int(sys.argv[1]) if len(sys.argv) > 1 else 2560
S = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
d, V = 512, 800000
g = torch.Generator(device=dev).manual_seed(0)
bf = lambda *s: ((torch.rand(*s, device=dev, generator=g) - 0.5)).to(torch.bfloat16)
h, wt, ws = bf(B, d), bf(B, d), bf(S, d)
bt = torch.rand(B, device=dev, generator=g) * 0.2 - 0.1
bs = torch.rand(S, device=dev, generator=g) * 0.2 - 0.1
lt = torch.zeros(B, device=dev) - 3
ls = torch.zeros(S, device=dev) - 3
labels = torch.randint(0, V, (B,), device=dev, generator=g)
sampled = torch.randperm(V, device=dev, generator=g)[:S]
wsb = ops.ssm_workspace(B, S, d, TFS_BF16, dev, V)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
out = None
names = ["prep", "logits_gemm", "combine", "grad", "colsum", "store_gemm", "finalize"]
rows = []
for it in range(25):
    flush.zero_()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
    for e in ev:
        e.record()  # create the events before handing them to the library
    torch.cuda.synchronize()
    out = ops.sampled_softmax(h, labels, wt, bt, lt, sampled, ws, bs, ls, grad_scale=1.0 / B,
                              vocab=V, out=out, ws=wsb, events=ev)
    torch.cuda.synchronize()
    if it >= 5:
        rows.append([ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(7)] +
                    [ev[0].elapsed_time(ev[7]) * 1e3])
med = np.median(np.array(rows), axis=0)
print(" ".join(f"{n}={v:.1f}" for n, v in zip(names + ["call"], med)))
