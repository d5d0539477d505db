"""Role timeline of CTA 0 of each tcgen05 GEMM launch (diagnostic build):

    python tools/build_variant.py variants/trace.so -DTFS_GEMM_TRACE
    TFS_ALLOW_VARIANT_LIB=1 TFS_LIB=$PWD/variants/trace.so TFS_TRACE_DUMP=1 N=3 \\
        python tools/one_ssm.py 2> trace.log
    python tools/gemm_timeline.py trace.log

Prints, per launch kind (0 logits, 1 gradient, 2 grouped dh / dW_s), microseconds after the
CTA's setup: producer stage-ready times, MMA tile start / stage-data arrival / tile issued,
epilogue tile ready / done (slots in umma.cuh, 'role timeline')."""
import sys

CLK_GHZ = 1.965
ROWS = [("producer stage ready", 16, 128), ("MMA tile start", 128, 144),
        ("MMA stage data", 160, 288), ("MMA tile issued", 144, 160),
        ("epilogue tile ready", 288, 304), ("epilogue tile done", 304, 320)]


def main():
    lines = [l for l in open(sys.argv[1]) if l.startswith("TRACE")]
    seen = {}
    for l in lines:  # the last launch of each kind
        head, rest = l.split(":", 1)
        seen[head.split()[1]] = (head, rest)
    for mode in sorted(seen):
        head, rest = seen[mode]
        d = {int(a): int(b) / (CLK_GHZ * 1e3) for a, b in (x.split(":") for x in rest.split())}
        print(head)
        for name, a, b in ROWS:
            v = [d[k] for k in sorted(d) if a <= k < b]
            print(f"  {name:22s}", " ".join(f"{x:.2f}" for x in v))


if __name__ == "__main__":
    main()
