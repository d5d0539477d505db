#!/usr/bin/env python
"""Benchmark: words/sec of the embed + sampled-softmax training step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload X] [--impl tfs|reference]

One JSON line on rank 0.  A "step" is one pass of the whole hot path of SURVEY §8(a) -- sample,
Part, route, Gather, route back, Stitch, sampled-softmax forward + backward, sort-reduce, route,
ScatterAdd-SGD -- over one synthetic batch of B tokens per GPU (weak scaling: B fixed per GPU).
Default workload X: V = 800,000, d = 512, B = 2,560 (128 x 20) per GPU, S = 8,192 per GPU,
Zipf(1.0) ids, bf16 tensor-core operands with fp32 accumulation and fp32 master tables.

The step is the native stepper of libtfs (tfs_step_*; one CUDA graph per step, one process per
GPU, tfs_comm over NVLink for R > 1).  Timing: W untimed warm-up steps; K timed steps, each
preceded by an L2 flush (a 256 MiB write, outside the timed interval); per-step CUDA events on
the launching stream; barrier + sync on both sides; max over ranks.  value = N*B*K / max-rank
time.  e2e: the same K steps through the C-ABI call tfs_step_run with HOST buffers: the H2D
copies of x, y from pinned memory and the D2H copy of the loss happen inside the call, every
step.  ``--impl reference`` times the CPU oracle (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "words/sec for embed+sampled-softmax step at 1/2/4/8 B200; HBM GB/s"
UNIT = "words/sec"
N_BATCHES = 16
FLUSH_BYTES = 256 << 20


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--workload", default="X", choices=sorted(workloads.WORKLOADS))
    p.add_argument("--impl", default="tfs", choices=["tfs", "reference"])
    p.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
    p.add_argument("--no-graph", action="store_true", help="eager launches instead of CUDA graph")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--phase-steps", type=int, default=20, help="instrumented eager steps")
    p.add_argument("--null-step", action="store_true",
                   help="SURVEY 8f #4 / P:1048-1055: step time of 32 random lookups per worker "
                        "from a 1 GB and a 16 GB embedding sharded over the GPUs")
    p.add_argument("--optimizer", default="sgd", choices=["sgd", "momentum", "adagrad"],
                   help="sparse optimizer of the ScatterAdd step (1 GPU; the paper uses SGD)")
    p.add_argument("--cap", type=int, default=0,
                   help="R > 1 route slots per owner (0 = the worst case, never overflows)")
    return p.parse_args()


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------------------------ clocks
class ClockSampler:
    """Polls NVML every 5 ms for SM clock and throttle reasons (start before, stop after)."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, torch_device):
        self.samples = []
        self.ok = False
        self.max_mhz = None
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            props = torch.cuda.get_device_properties(torch_device)
            h = None
            try:
                bus = "%08x:%02x:%02x.0" % (props.pci_domain_id, props.pci_bus_id,
                                           props.pci_device_id)
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(torch_device.index or 0)
            self.h = h
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # no NVML: report it, never fake numbers
            self.err = str(e)

    def _run(self):
        nv = self.nv
        while not self.stop:
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((time.time(), sm, r))
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        if not self.ok:
            return
        self.stop = False
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def finish(self, t0, t1):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "NVML unavailable"}
        self.stop = True
        self.t.join()
        win = [s for s in self.samples if t0 <= s[0] <= t1] or self.samples
        busy = [s for s in win if not (s[2] & 0x1)] or win
        reasons = set()
        for _, _, r in busy:
            for bit, name in self.REASONS.items():
                if r & bit and bit != 0x1:
                    reasons.add(name)
        return {"sm_mhz": statistics.median([s[1] for s in busy]) if busy else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                "samples": len(busy)}


# ---------------------------------------------------------------------------- oracle timing
def oracle_steps(w, n_steps, tokens, log=None):
    """The CPU oracle (oracle/step.py, single-threaded C++ + numpy glue) on a bounded sample:
    `tokens` of the B tokens of each batch, full V / S / d.  Returns (words, seconds)."""
    import oracle  # noqa: F401  (test infrastructure: bench's cpu_baseline / reference legs)
    from oracle import step as ostep
    E, W, b = workloads.tables(w.vocab, w.dim)
    cfg = ostep.StepConfig(vocab=w.vocab, dim=w.dim, num_sampled=w.num_sampled or w.vocab,
                           num_shards=1, lr=0.1, seed=workloads.SAMPLER_SEED,
                           full_softmax=(w.num_sampled == 0), inplace=True)
    words = 0
    secs = 0.0
    for i in range(n_steps):
        x, y = workloads.batch(w, 1, 0, step=i % N_BATCHES)
        cfg.step = i
        t = time.perf_counter()
        E, W, b, _ = ostep.step(E, W, b, [x[:tokens]], [y[:tokens]], cfg)
        secs += time.perf_counter() - t
        words += tokens
    return words, secs


def run_reference(args):
    """Reference arm: the oracle as it stands, on host cores, same metric/unit/config."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = workloads.WORKLOADS[args.workload]
    tokens = 16
    oracle_steps(w, args.warmup, tokens)
    words, secs = oracle_steps(w, args.steps, tokens)
    value = words / secs
    sample = (f"{tokens} of {w.tokens_per_replica(1)} tokens per step, V={w.vocab}, "
              f"d={w.dim}, S={w.num_sampled or w.vocab}; single-threaded oracle")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True,
            "scaling": "strong" if w.strong else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": args.workload, "vocab": w.vocab, "dim": w.dim,
                       "tokens_per_step": tokens, "num_sampled": w.num_sampled},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------- GPU timing
def graph_kernel_nodes(graph):
    """Number of kernel nodes in a captured CUDA graph (cuda-python), or None."""
    try:
        from cuda.bindings import runtime as rt
        g = graph.raw_cuda_graph()
        if isinstance(g, int):
            g = rt.cudaGraph_t(init_value=g)
        err, _, n = rt.cudaGraphGetNodes(g, 0)
        err, nodes, n = rt.cudaGraphGetNodes(g, n)
        k = 0
        for nd in nodes:
            err, t = rt.cudaGraphNodeGetType(nd)
            if t == rt.cudaGraphNodeType.cudaGraphNodeTypeKernel:
                k += 1
        return k
    except Exception:
        return None


def host_info():
    """Host cores and CPU model of the box the oracle baseline runs on."""
    model = None
    try:
        import subprocess
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "lscpu_model": model}


def so_info():
    import hashlib
    from paper_1605_08695_b200 import _lib
    with open(_lib.SO_PATH, "rb") as f:
        h = hashlib.sha256(f.read()).hexdigest()[:16]
    return {"path": os.path.relpath(_lib.SO_PATH, ROOT), "sha256_16": h,
            "product": _lib.SO_PATH == _lib.PRODUCT_SO}


def run_null_step(args, world, rank, dev):
    """The paper's sparse null step: "Each worker reads 32 randomly selected
    entries from a large embedding matrix containing 1 GB or 16 GB of data ... step times do
    not vary with the size of the embedding ... 5 to 20 ms".  Here: fp32 rows of 512, the
    matrix sharded by id mod R over the GPUs; one step = 32 fresh random ids per worker and
    their rows gathered (R = 1: tfs_gather; R > 1: tfs_gather_peers, one-sided NVLink pulls
    from the tfs_comm heaps behind a device barrier).  Reported: median step time."""
    import torch
    from paper_1605_08695_b200 import ops
    from paper_1605_08695_b200 import step as gstep
    from paper_1605_08695_b200 import _lib
    d, n_ids, steps = 512, 32, max(args.steps, 50)
    out = {}
    for gb in (1, 16):
        V = gb * (1 << 30) // (4 * d)
        rows = -(-V // world)
        comm = None
        if world > 1:
            import ctypes
            p = ctypes.c_void_p()
            L = _lib.lib()
            _lib.check(L.tfs_comm_create(world, rank, 1, dev.index, 65536 + 4 * rows * d, 60000,
                                         ctypes.byref(p)), "tfs_comm_create")
            h = ctypes.create_string_buffer(64)
            _lib.check(L.tfs_comm_export(p, h), "tfs_comm_export")
            _lib.check(L.tfs_comm_connect(p, gstep.exchange_handles(h.raw)), "tfs_comm_connect")
            comm = gstep.Comm(p, world, rank, 1, dev)
            shard = gstep.device_tensor(comm.heap() + 65536, (rows, d), torch.float32, dev)
            tab = comm.peer_bases() + 65536
        else:
            shard = torch.empty((rows, d), dtype=torch.float32, device=dev)
        shard.uniform_(-0.5, 0.5)
        gen = torch.Generator(device=dev).manual_seed(1234 + rank)
        ids = torch.empty(n_ids, dtype=torch.int64, device=dev)
        res = torch.empty((n_ids, d), dtype=torch.float32, device=dev)
        err = ops.ErrorSlot(dev)
        times = []
        for i in range(args.warmup + steps):
            ids.random_(0, V, generator=gen)
            torch.cuda.synchronize()
            if comm is not None:
                comm.barrier(0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if comm is not None:
                ops.gather_peers(tab, rows, d, ids, V, world, res, err=err)
                comm.barrier(1)
            else:
                ops.gather(shard, ids, out=res, err=err)
            e1.record()
            torch.cuda.synchronize()
            if i >= args.warmup:
                times.append(e0.elapsed_time(e1))
        err.check("null step")
        med = torch.tensor([float(np.median(times))], device=dev, dtype=torch.float64)
        if world > 1:
            import torch.distributed as dist
            dist.all_reduce(med, op=dist.ReduceOp.MAX)
            dist.barrier()
            comm.close()
        out[f"{gb}GB"] = {"median_ms": float(med.item()), "rows": V,
                          "p10_ms": float(np.percentile(times, 10)),
                          "p90_ms": float(np.percentile(times, 90))}
        del shard
        torch.cuda.empty_cache()
    if rank == 0:
        print(json.dumps({"metric": "sparse null step time (32 random embedding lookups per "
                                    "worker, P:1048-1055)", "unit": "ms", "n_gpus": world,
                          "higher_is_better": False, "steps": steps, "warmup": args.warmup,
                          "data": "synthetic", "config": {"workload": "null-step", "dim": d,
                          "lookups_per_worker": n_ids, "transport": "p2p" if world > 1
                          else "local"}, "paper_ms": [5, 20], "results": out}), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    from paper_1605_08695_b200 import _lib
    from paper_1605_08695_b200 import step as gstep
    from paper_1605_08695_b200._lib import TFS_BF16, TFS_F32

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if args.null_step:
        run_null_step(args, world, rank, dev)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    w = workloads.WORKLOADS[args.workload]
    R = world
    B = w.tokens_per_replica(R)
    S = w.num_sampled
    d = w.dim
    dtype = TFS_BF16 if args.dtype == "bf16" else TFS_F32
    cfg = gstep.StepConfig(vocab=w.vocab, dim=d, tokens=B, num_sampled=S, num_shards=R, lr=0.1,
                           seed=workloads.SAMPLER_SEED, operand_dtype=dtype,
                           optimizer=args.optimizer, cap_e=args.cap, cap_w=args.cap)
    comm = gstep.Comm.distributed(cfg, timeout_ms=60000) if R > 1 else None
    st = gstep.Step(cfg, comm)
    E, W, b = workloads.tables_device(w.vocab, d, R, rank, dev)
    st.load_tables(E, W, b)
    del E, W, b
    st.sync()
    # 16 distinct pre-generated batches per rank, resident in HBM and in pinned host memory.
    # x || y of a batch adjacent in one pinned buffer: the C call moves them in one H2D copy
    xs_h, ys_h = [], []
    for i in range(N_BATCHES):
        x, y = workloads.batch(w, R, rank, step=i)
        xy = torch.from_numpy(np.concatenate([x, y])).pin_memory()
        xs_h.append(xy[:B])
        ys_h.append(xy[B:])
    xs_d = [t.to(dev) for t in xs_h]
    ys_d = [t.to(dev) for t in ys_h]
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=dev)
    use_graph = not args.no_graph
    L = _lib.lib()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- one counted eager step: how many libtfs kernels a step launches
    barrier()
    c0 = L.tfs_debug_launch_count()
    st.run(xs_d[0], ys_d[0])
    torch.cuda.synchronize()
    launches_per_step = L.tfs_debug_launch_count() - c0
    st.check("bench step")
    kernel_nodes = None
    if use_graph:
        barrier()
        st.capture()
        kernel_nodes = st.graph_kernels()

    def one_step(i):
        return st.run(xs_d[i % N_BATCHES], ys_d[i % N_BATCHES])

    check_every = int(os.environ.get("TFS_BENCH_CHECK_EVERY", "0"))  # debugging aid (off)
    for i in range(args.warmup):
        one_step(i)
        if check_every and (i + 1) % check_every == 0:
            st.check(f"warmup step {i}")
    barrier()

    # ---- timed region: K steps, L2 flushed before each (outside the events)
    clocks = ClockSampler(dev)
    clocks.start()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier()
    t_wall0 = time.time()
    for i in range(args.steps):
        flush.zero_()
        starts[i].record()
        one_step(i)
        ends[i].record()
        if check_every and (i + 1) % check_every == 0:
            st.check(f"timed step {i}")
    barrier()
    t_wall1 = time.time()
    per_step = [s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)]
    local_ms = sum(per_step)
    clk = clocks.finish(t_wall0, t_wall1)
    if world > 1:
        tt = torch.tensor([local_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    else:
        total_ms = local_ms
    st.check("bench timed steps")
    words = R * B * args.steps
    value = words / (total_ms / 1e3)

    # ---- e2e: the C-ABI step call with HOST buffers (H2D of x, y and D2H of the loss inside)
    loss_host = torch.empty(args.steps, dtype=torch.float32).pin_memory()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        st.run_host(xs_h[i % N_BATCHES], ys_h[i % N_BATCHES], loss_host[i:i + 1])
    e1.record()
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    assert np.all(np.isfinite(loss_host.numpy()))
    e2e_value = words / (e2e_ms / 1e3)
    st.check("bench e2e steps")

    # ---- instrumented eager steps: per-phase (R = 1, serial) and per-GEMM device time
    if use_graph:
        st.uncapture()
    n_ph = max(1, min(args.phase_steps, args.steps))
    evs_all = []
    barrier()
    for i in range(n_ph):
        flush.zero_()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
        st.run(xs_d[i % N_BATCHES], ys_d[i % N_BATCHES], timing_events=evs)
        evs_all.append(evs)
    barrier()
    st.check("bench instrumented steps")

    def avg(i0, i1):
        return sum(e[i0].elapsed_time(e[i1]) for e in evs_all) / len(evs_all)

    phases = {}
    if R > 1 and S > 0:  # main-stream phase boundaries of the one-sided step (include/tfs.h)
        for name, (i0, i1) in (("barrier_B0", (0, 1)), ("commit", (1, 2)),
                               ("pull_W_and_wait_B1_side", (2, 3)), ("softmax_call", (9, 16)),
                               ("reduce_push_W", (16, 4)), ("barrier_B2", (4, 5)),
                               ("apply_W", (5, 6)), ("join_E_apply", (6, 7)),
                               ("total", (0, 7)),
                               ("side_phase1_from_B0", (1, 17)), ("side_B1_wait", (17, 18)),
                               ("side_owner_plans", (18, 19)), ("side_until_E_pushed", (19, 20)),
                               ("side_E_pushed_at", (0, 20)), ("main_W_pushed_at", (0, 4))):
            phases[name] = avg(i0, i1)
        allph = [None] * world  # every rank's phases (load balance across owners)
        dist.all_gather_object(allph, phases)
        phases = {"rank0": phases, "max_over_ranks": {k: max(p[k] for p in allph) for k in phases},
                  "per_rank_total": [p["total"] for p in allph],
                  "per_rank_barrier_B2": [p["barrier_B2"] for p in allph],
                  "per_rank_apply_W": [p["apply_W"] for p in allph]}
    if R == 1:
        for name, (i0, i1) in (("sample", (0, 1)), ("gather_E", (1, 2)), ("gather_W", (2, 3)),
                               ("sampled_softmax", (3, 4)), ("plan_E", (4, 5)),
                               ("plan_W", (5, 6)), ("apply_E", (6, 7)), ("apply_W", (7, 8))):
            phases[name] = avg(i0, i1)
    peaks, peak_src = load_peaks()
    # Sub-millisecond kernels timed inside eager steps at full clocks: the BURST peak.
    peak = peaks.get("bf16_tflops", 1675.0)
    hbm_peak = peaks.get("hbm_gbs", 6456.2)
    roofline = None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic_ssm.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.workload)
        except Exception:
            traffic = None
    S_eff = S if S > 0 else w.vocab  # candidates per replica (full softmax: all V classes)
    if S == 0 and R > 1:
        # per shard: M = R*B tokens x its V/R classes; STATS 2 M n d, GRAD + STORE 6 M n d flops
        M_, n_ = R * B, -(-w.vocab // R)
        kern = {"partial_stats": (avg(9, 10), 2.0 * M_ * n_ * d),
                "backward_from_lse": (avg(11, 12), 6.0 * M_ * n_ * d)}
        per = {k: {"ms": v, "tflops": f / (v / 1e3) / 1e12, "frac": f / (v / 1e3) / 1e12 / peak}
               for k, (v, f) in kern.items()}
        top = per["backward_from_lse"]
        roofline = {"kernel": "tfs_ssm_backward_from_lse (GRAD + column sums + grouped "
                              "dh / dW GEMM on this shard's classes)",
                    "bound": "tensor", "achieved": top["tflops"], "peak": peak,
                    "unit": "TFLOP/s", "frac": top["frac"], "traffic": None,
                    "peak_source": f"{peak_src} bf16 burst (sub-ms kernels at full clocks)",
                    "algorithmic": "6*M*n*d flops per call (M = R*B tokens, n = V/R classes); "
                                   "achieved = that / the call's CUDA-event duration",
                    "ms": top["ms"], "kernels": per}
        call_ms = None
    elif args.dtype == "f32":
        # the fp32 parity path: SIMT FFMA GEMMs (no tensor cores); peak = SMs x 128 FP32 lanes
        # x 2 flops x the max SM clock (B200_PROFILING.md unit counts), timed as the whole call
        call_ms = avg(9, 16)
        fp32_peak = 148 * 128 * 2 * 1.965e9 / 1e12
        t = call_ms / 1e3
        ach = 6.0 * B * S_eff * d / t / 1e12
        roofline = {"kernel": "tfs_sampled_softmax_fwd_bwd, fp32 path (SIMT FFMA GEMMs)",
                    "bound": "alu", "achieved": ach, "peak": fp32_peak, "unit": "TFLOP/s",
                    "frac": ach / fp32_peak, "traffic": None,
                    "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 x 1965 MHz",
                    "algorithmic": "6*B*S*d flops per call; achieved = that / the call's "
                                   "CUDA-event duration in instrumented eager steps",
                    "ms": call_ms,
                    "logits_gemm_ms": avg(9, 11)}
    else:
        zpass = int(_lib.lib().tfs_ssm_grad_from_logits()) == 1
        kern_ms = {"gemm_stats": avg(10, 11), "gemm_store": avg(14, 15)}
        flops = {"gemm_stats": 2.0 * B * S_eff * d, "gemm_store": 4.0 * B * S_eff * d}
        if not zpass:
            kern_ms["gemm_grad"] = avg(12, 13)
            flops["gemm_grad"] = 2.0 * B * S_eff * d
        call_ms = avg(9, 16)
        per = {k: {"ms": v, "tflops": flops[k] / (v / 1e3) / 1e12,
                   "frac": flops[k] / (v / 1e3) / 1e12 / peak} for k, v in kern_ms.items()}
        if zpass:
            # the elementwise gradient pass: reads the fp32 logits, writes bf16 G (+ slab sums)
            gp_ms = avg(12, 13)
            gp_bytes = B * S_eff * (4 + 2)
            per["grad_pass"] = {"ms": gp_ms, "GBps": gp_bytes / (gp_ms / 1e3) / 1e9,
                                "frac": gp_bytes / (gp_ms / 1e3) / 1e9 / hbm_peak,
                                "bound": "hbm", "bytes": gp_bytes}
        top = per["gemm_store"]
        roofline = {"kernel": "umma::gemm_kernel<STORE> (dh = G W_s and dW_s = G^T h, one "
                              "persistent tcgen05 launch)",
                    "bound": "tensor", "achieved": top["tflops"], "peak": peak,
                    "unit": "TFLOP/s", "frac": top["frac"],
                    "traffic": (traffic or {}).get("gemm_store"),
                    "peak_source": f"{peak_src} bf16 burst (sub-ms kernels at full clocks)",
                    "algorithmic": "4*B*S*d flops per launch (two GEMMs); achieved = that / the "
                                   "launch's CUDA-event duration in instrumented eager steps",
                    "ms": top["ms"], "kernels": per}
        t = call_ms / 1e3
        roofline["sampled_softmax_call"] = {
            "kernel": "tfs_sampled_softmax_fwd_bwd (whole call)", "bound": "tensor",
            "achieved": 6.0 * B * S_eff * d / t / 1e12, "peak": peak, "unit": "TFLOP/s",
            "frac": 6.0 * B * S_eff * d / t / 1e12 / peak,
            "traffic": (traffic or {}).get("ssm_total"),
            "algorithmic": "6*B*S*d flops per call (3 GEMMs; the logits recompute is overhead)",
            "ms": call_ms}
    hbm = None
    if R == 1 and S > 0:
        # Algorithmic bytes per call, each call timed alone by CUDA
        # events on its stream in the serial instrumented steps.
        #  Gather: the ids, the DISTINCT rows read once (repeats are L2 hits), every requested
        #    row written (bf16 operand rows in bf16 mode; the bias in fp32).
        #  ScatterAdd-SGD apply: every gradient row read once (fp32), each distinct row of the
        #    table read and written (W with its bias).
        #  Plan: ids read, sorted keys / permutation / segments written -- latency-bound (us).
        qw = st.tensor("qw")
        x_last = st.tensor("x")
        u_e = int(torch.unique(x_last).numel())
        u_w = int(torch.unique(qw).numel())
        n_e, n_w = B, B + S
        row_in = 4 * d
        row_out = (2 if args.dtype == "bf16" else 4) * d
        calls = {
            "gather_E": 8 * n_e + u_e * row_in + n_e * row_out,
            "gather_W": 8 * n_w + u_w * (row_in + 4) + n_w * (row_out + 4),
            "apply_E": n_e * row_in + 2 * u_e * row_in,
            "apply_W": n_w * (row_in + 4) + 2 * u_w * (row_in + 4),
        }
        per = {}
        for k, nbytes in calls.items():
            t_ = phases[k] / 1e3
            per[k] = {"bytes": nbytes, "us": phases[k] * 1e3, "GBps": nbytes / t_ / 1e9,
                      "frac": nbytes / t_ / 1e9 / hbm_peak}
        g_bytes = calls["gather_E"] + calls["gather_W"]
        s_bytes = calls["apply_E"] + calls["apply_W"]
        t_g = (phases["gather_E"] + phases["gather_W"]) / 1e3
        t_s = (phases["apply_E"] + phases["apply_W"]) / 1e3
        hbm = {"gather_GBps": g_bytes / t_g / 1e9, "gather_frac": g_bytes / t_g / 1e9 / hbm_peak,
               "scatter_GBps": s_bytes / t_s / 1e9,
               "scatter_frac": s_bytes / t_s / 1e9 / hbm_peak,
               "scatter_plan_us": {"E": phases["plan_E"] * 1e3, "W": phases["plan_W"] * 1e3},
               "calls": per, "distinct_rows": [u_e, u_w], "peak": hbm_peak, "unit": "GB/s",
               "note": "per-call CUDA-event times of serial instrumented eager steps (L2 "
                       "flushed before each step); bytes = algorithmic (DESIGN.md §6)"}
        roofline["scatter"] = {"kernel": "ScatterAdd-SGD apply (seg_window + crossing "
                                         "segments), E and W calls",
                               "bound": "hbm", "achieved": hbm["scatter_GBps"],
                               "peak": hbm_peak, "unit": "GB/s", "frac": hbm["scatter_frac"],
                               "traffic": None, "algorithmic": "per distinct row: read its "
                               "gradient rows + read and write the table row"}
        roofline["gather"] = {"kernel": "Gather (gather_vec4, bf16 out), E and W calls",
                              "bound": "hbm", "achieved": hbm["gather_GBps"], "peak": hbm_peak,
                              "unit": "GB/s", "frac": hbm["gather_frac"], "traffic": None}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        tokens = 128
        words_o, secs_o = oracle_steps(w, 3, tokens)
        hi = host_info()
        rate = words_o / secs_o
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle",
               "nproc": hi["nproc"], "lscpu_model": hi["lscpu_model"],
               "ideal_all_cores_extrapolation": rate * (hi["nproc"] or 1),
               "sample": f"3 oracle steps of {tokens} of the {B} tokens of a batch (full "
                         f"V={w.vocab}, S={S or w.vocab}, d={d}); single-threaded C++ oracle "
                         f"+ numpy glue on 1 of {hi['nproc']} cores; {secs_o:.1f} s; the "
                         f"all-cores figure is an extrapolation (x nproc), not a measurement"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if w.strong else "weak",  # Z: a fixed global batch
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": args.workload, "vocab": w.vocab, "dim": d,
                       "tokens_per_gpu": B, "global_batch": R * B, "num_sampled": S,
                       "zipf_s": w.zipf_s,
                       "softmax": ("sampled" if S > 0 else "full" if R == 1 else
                                   "full, vocabulary-sharded: each GPU scores all R*B tokens "
                                   "against its V/R classes (P:706-714)"),
                       "parallelism": f"vocab-sharded x{R} (ids mod R), "
                       f"data-parallel x{R}", "l2": "flushed before every timed step "
                       "(256 MiB write outside the timed interval)",
                       "cuda_graph": use_graph, "batches": N_BATCHES,
                       "optimizer": args.optimizer, "runtime": "native tfs_step (C ABI)",
                       "route_slots": ({"transport": "one-sided NVLink (tfs_comm IPC heaps)",
                                        "cap": args.cap or "worst case (B, B+S)"}
                                       if R > 1 else None)},
            "clocks": clk,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 2 * B * 8,
                    "d2h_bytes_per_step": 4, "api": "tfs_step_run with host x / y / loss"},
            "gpu_launches": launches_per_step * args.steps,
            "gpu_launches_per_step": launches_per_step,
            "graph_kernel_nodes": kernel_nodes,
            "roofline": roofline,
            "hbm": hbm,
            "phases_ms": phases,
            "per_step_ms_p10_p50_p90": [float(np.percentile(per_step, q)) for q in (10, 50, 90)],
            "cpu_baseline": cpu,
            "library": so_info(),
        }
        print(json.dumps(line), flush=True)
    st.close()
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()
        comm.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
