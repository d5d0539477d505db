"""In-graph spans of the three tcgen05 GEMM launches of the X step (diagnostic build):

    python tools/build_variant.py variants/trace.so -DTFS_GEMM_TRACE
    TFS_ALLOW_VARIANT_LIB=1 TFS_LIB=$PWD/variants/trace.so python tools/gemm_spans_step.py [X]

Builds the R = 1 stepper as bench.py does, captures its CUDA graph, replays it (L2 flushed
before each replay, CUDA events around each replay) and, after each of the last few replays,
reads the per-CTA globaltimer stamps of the last STATS / GRAD / STORE launches
(`tfs_trace_gemm_spans`): when each GEMM's first CTA entered and its last CTA left, relative
to the STATS launch, next to the replay's event-timed step and two globaltimer marker kernels
launched on the replay's stream just before and after it (`tfs_trace_stamp`).  Shows whether the GEMMs run in
the graph as fast as alone (profiles/r2_gemm_spans_X.txt) and what lies between them."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import workloads
from paper_1605_08695_b200 import _lib
from paper_1605_08695_b200 import step as gstep
from paper_1605_08695_b200._lib import TFS_BF16

NAMES = ("STATS", "GRAD", "STORE")


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "X"
    w = workloads.WORKLOADS[wl]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    B, S, d = w.tokens_per_replica(1), w.num_sampled, w.dim
    cfg = gstep.StepConfig(vocab=w.vocab, dim=d, tokens=B, num_sampled=S, num_shards=1, lr=0.1,
                           seed=workloads.SAMPLER_SEED, operand_dtype=TFS_BF16)
    st = gstep.Step(cfg, None)
    E, W, b = workloads.tables_device(w.vocab, d, 1, 0, dev)
    st.load_tables(E, W, b)
    del E, W, b
    st.sync()
    xs, ys = [], []
    for i in range(4):
        x, y = workloads.batch(w, 1, 0, step=i)
        xs.append(torch.from_numpy(np.asarray(x)).to(dev))
        ys.append(torch.from_numpy(np.asarray(y)).to(dev))
    st.run(xs[0], ys[0])
    torch.cuda.synchronize()
    st.capture()
    L = _lib.lib()
    fn = L.tfs_trace_gemm_spans
    fn.argtypes = [ctypes.c_void_p]
    fn.restype = ctypes.c_int32
    stamp, stamps = L.tfs_trace_stamp, L.tfs_trace_stamps
    stamp.argtypes = [ctypes.c_int32, ctypes.c_void_p]
    stamps.argtypes = [ctypes.c_void_p]
    marks = np.zeros(8, dtype=np.uint64)
    cur = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    buf = np.zeros((3, 160, 3), dtype=np.uint64)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(12):
        flush.fill_(i & 0xFF)
        stamp(0, cur())
        ev0.record()
        st.run(xs[i % 4], ys[i % 4])
        ev1.record()
        stamp(1, cur())
        torch.cuda.synchronize()
        if i < 8:
            continue
        assert fn(buf.ctypes.data) == 0
        assert stamps(marks.ctypes.data) == 0
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        t0 = int(buf[0, :sms, 0].min())
        parts = [f"replay {i}: step {ev0.elapsed_time(ev1) * 1e3:.1f} us (events); markers"
                 f" {(int(marks[0]) - t0) / 1e3:.1f} / {(int(marks[1]) - t0) / 1e3:.1f}"]
        for m, name in enumerate(NAMES):
            n = sms  # grid = one CTA (or one CTA of a pair) per SM
            ent = buf[m, :n, 0].astype(np.int64)
            ext = buf[m, :n, 2].astype(np.int64)
            ok = ent > 0
            su = buf[m, :n, 1].astype(np.int64)
            parts.append(f"{name} {(ent[ok].min() - t0) / 1e3:.1f} -> {(ext[ok].max() - t0) / 1e3:.1f}"
                         f" ({(ext[ok].max() - ent[ok].min()) / 1e3:.1f} us; entry spread"
                         f" {(ent[ok].max() - ent[ok].min()) / 1e3:.1f}, setup done by"
                         f" {(su[ok].max() - ent[ok].min()) / 1e3:.1f}, first exit"
                         f" {(ext[ok].min() - ent[ok].min()) / 1e3:.1f})")
        print("\n  ".join(parts), flush=True)
    st.uncapture()
    st.close()


if __name__ == "__main__":
    main()
