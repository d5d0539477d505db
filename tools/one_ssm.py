"""Profiling driver: N sampled-softmax calls (tfs_sampled_softmax_fwd_bwd, bf16 operands) at the
bench workload's shape (X: B = 2560 tokens, S = 8192 candidates, d = 512, V = 800k), seeded
synthetic inputs.  Used for the per-kernel ncu captures under profiles/ (see profiles/README)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1605_08695_b200 import ops
from paper_1605_08695_b200._lib import TFS_BF16
dev = "cuda"
B, S, d = 2560, 8192, 512
g = torch.Generator(device=dev).manual_seed(0)
h = torch.rand(B, d, device=dev, generator=g) - 0.5
wt = torch.rand(B, d, device=dev, generator=g) - 0.5
ws = torch.rand(S, d, device=dev, generator=g) - 0.5
bt = torch.rand(B, device=dev, generator=g) * 0.2 - 0.1
bs = torch.rand(S, device=dev, generator=g) * 0.2 - 0.1
lt = torch.zeros(B, device=dev) - 3
ls = torch.zeros(S, device=dev) - 3
labels = torch.randint(0, 800000, (B,), device=dev)
sampled = torch.randperm(800000, device=dev)[:S]
wsb = ops.ssm_workspace(B, S, d, TFS_BF16, dev, 800000)
out = None
for _ in range(int(os.environ.get("N", "3"))):
    out = ops.sampled_softmax(h, labels, wt, bt, lt, sampled, ws, bs, ls, grad_scale=1.0 / B, vocab=800000, out=out, ws=wsb)
torch.cuda.synchronize()
print("ok")
