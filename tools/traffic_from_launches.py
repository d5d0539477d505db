"""Per-launch DRAM traffic of the sampled-softmax call from an ncu launch list (the
`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum` CSV of a bench
run; the last complete call is used) -> profiles/traffic_ssm.json[workload]: bytes per launch of
each GEMM and of the whole call (bench.py reports them as roofline.traffic).

    python tools/traffic_from_launches.py profiles/r2_launches_X.csv X
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SSM = ("prep_kernel", "gemm_kernel<0", "bf16_combine", "gemm_kernel<1", "g_colsum", "db_colpart",
       "gemm_kernel<2", "split_finalize")


def main():
    path, workload = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(path)))
    hdr, data = None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            e = data.setdefault(int(d["ID"]), {"name": d["Kernel Name"]})
            e[d["Metric Name"]] = float(d["Metric Value"]) * (1e9 if d["Metric Unit"] == "Gbyte"
                                                              else 1e6 if d["Metric Unit"] == "Mbyte"
                                                              else 1e3 if d["Metric Unit"] == "Kbyte"
                                                              else 1.0)
    ids = sorted(data)
    # the last COMPLETE call: from a prep_kernel to the split_finalize after its STORE GEMM
    starts = [i for i in ids if "prep_kernel" in data[i]["name"]]
    def complete(s0):
        seen = False
        for i in ids:
            if i <= s0:
                continue
            n = data[i]["name"]
            if "prep_kernel" in n:
                return False
            if "gemm_kernel<2" in n:
                return True
        return False
    start = next(s0 for s0 in reversed(starts) if complete(s0))
    out, total = {}, 0.0
    for i in ids:
        if i < start:
            continue
        n = data[i]["name"]
        if not any(k in n for k in SSM):
            if "gemm_store" in out:
                break
            continue
        b = data[i].get("dram__bytes_read.sum", 0) + data[i].get("dram__bytes_write.sum", 0)
        key = {"gemm_kernel<0": "gemm_stats", "gemm_kernel<1": "gemm_grad",
               "gemm_kernel<2": "gemm_store"}.get(next((k for k in SSM if k in n), ""), None)
        if key and key not in out:
            out[key] = b
        total += b
    # stop at the first non-softmax kernel after the STORE GEMM (its finalize passes included)
    out["ssm_total"] = total
    out["source"] = os.path.relpath(path, ROOT)
    dst = os.path.join(ROOT, "profiles", "traffic_ssm.json")
    allw = json.load(open(dst)) if os.path.exists(dst) else {}
    allw[workload] = out
    json.dump(allw, open(dst, "w"), indent=1)
    print(workload, out)


if __name__ == "__main__":
    main()
