"""Build an experiment variant of libtfs.so with extra -D switches, for A/B timing only.

    python tools/build_variant.py OUT.so -DTFS_KSUB=1
    TFS_ALLOW_VARIANT_LIB=1 TFS_LIB=$PWD/OUT.so python tools/one_ssm.py      # run against it

Tuning switches of the product source (every variant computes correct results): TFS_KSUB_* set
k-blocks per pipeline stage (TFS_KSUB_SOFTMAX, TFS_KSUB_STORE), TFS_STORE_CTA=1 builds the
grouped STORE GEMM with single CTAs instead of CTA pairs,
TFS_SEG_CHUNK / TFS_SEG_MINB tune the sparse apply.  (Round 1's wrong-result role-isolation
switches were removed from the product source; their numbers stay in profiles/r1_summary.md.)
bench.py records the path and hash of the library it loaded.
"""
import glob
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1605_08695_b200", "csrc")


def main():
    out, flags = sys.argv[1], sys.argv[2:]
    arch = ["-gencode", "arch=compute_100a,code=sm_100a"]
    with tempfile.TemporaryDirectory() as tmp:
        objs = []
        for src in sorted(glob.glob(os.path.join(CSRC, "*.cu"))):
            obj = os.path.join(tmp, os.path.basename(src) + ".o")
            subprocess.check_call(["nvcc", *arch, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler",
                                   "-fPIC", "-I", os.path.join(ROOT, "include"), *flags, "-c",
                                   src, "-o", obj])
            objs.append(obj)
        subprocess.check_call(["nvcc", *arch, "-shared", "-cudart=static", "-o", out, *objs])
    print("built", out)


if __name__ == "__main__":
    main()
