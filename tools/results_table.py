"""BASELINE.md §6 rows from bench JSON lines (profiles/r2_final_*.json): words/s (with the
per-step p10-p90 range), step time, gather / scatter GB/s (R = 1 calls), the logits GEMM's
TFLOP/s, and the oracle baseline.  Prints markdown rows.

    python tools/results_table.py profiles/r2_final_bench_*.json
"""
import json
import sys


def row(path):
    d = json.loads(open(path).read().strip().splitlines()[-1])
    c = d["config"]
    B = c["tokens_per_gpu"] * d["n_gpus"]
    p10, p50, p90 = d.get("per_step_ms_p10_p50_p90", [None] * 3)
    wps = lambda ms: B / (ms / 1e3) / 1e6 if ms else None
    rng = f"{wps(p90):.2f}-{wps(p10):.2f}M" if p10 else "-"
    h = d.get("hbm") or {}
    g = f"{h['gather_GBps']:.0f} ({h['gather_frac']:.2f})" if h else "-"
    s = f"{h['scatter_GBps']:.0f} ({h['scatter_frac']:.2f})" if h else "-"
    k = (d.get("roofline") or {}).get("kernels", {})
    st = k.get("gemm_stats") or k.get("partial_stats")
    gemm = f"{st['tflops']:.0f} ({st['frac']:.2f})" if st else "-"
    cpu = d.get("cpu_baseline")
    cpu_s = f"{cpu['value']:.0f} (1 of {cpu.get('nproc')} cores)" if cpu else "-"
    opt = c.get("optimizer", "sgd")
    tag = (" f32" if d.get("dtype") == "f32" else "") + (f" {opt}" if opt != "sgd" else "")
    return (f"| {c['workload']}{tag} | {d['n_gpus']} | "
            f"{d['value'] / 1e6:.2f}M ({rng}) | {d['ms_per_step'] * 1e3:.1f} | {g} | {s} | {gemm} | "
            f"{cpu_s} | {d['e2e']['value'] / 1e6:.2f}M |")


if __name__ == "__main__":
    print("| Config | GPUs | Words/sec (p90-p10 step range) | Step us | Gather GB/s (frac of 6456) | "
          "Scatter GB/s (frac) | Logits GEMM TF/s (frac of 1675) | Oracle words/s | e2e words/s |")
    print("|---|---|---|---|---|---|---|---|---|")
    for p in sys.argv[1:]:
        try:
            print(row(p))
        except Exception as e:  # a line that is not a bench line
            print(f"<!-- {p}: {e} -->")
