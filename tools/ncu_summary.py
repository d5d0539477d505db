"""Key metrics of every kernel in an ncu report (ncu -i REP --page details --csv), one block per
launch: duration, DRAM / L2 / SM throughput, tensor pipe, issue slots, occupancy, registers.

    python tools/ncu_summary.py gpurun_out/prof_final/x_full.ncu-rep > profiles/r2_ncu_full_X.txt
"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Issue Slots Busy", "Eligible Warps Per Scheduler",
        "Achieved Occupancy", "Registers Per Thread", "Grid Size", "Block Size", "L2 Hit Rate",
        "Executed Instructions"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "lts__throughput.avg.pct_of_peak_sustained_elapsed"]


def main():
    rep = sys.argv[1]
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(det)))
    h = r[0]
    ki, mi, vi, ui, ii = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value",
                                                "Metric Unit", "ID"))
    out = {}
    for x in r[1:]:
        e = out.setdefault(x[ii], {"name": x[ki].split("(")[0]})
        if x[mi] in WANT and x[mi] not in e:
            e[x[mi]] = f"{x[vi]} {x[ui]}".strip()
    rr = list(csv.reader(io.StringIO(raw)))
    rh, units = rr[0], rr[1]
    for n, row in enumerate(rr[2:]):
        e = out.get(str(n))
        if e is None:
            continue
        for m in RAW:
            if m in rh:
                j = rh.index(m)
                e[m] = f"{row[j]} {units[j]}".strip()
    print(f"# ncu --set full summary of {rep}")
    for k in sorted(out, key=int):
        e = out[k]
        print(f"== {k} {e.pop('name')}")
        for m, v in e.items():
            print(f"   {m}: {v}")


if __name__ == "__main__":
    main()
