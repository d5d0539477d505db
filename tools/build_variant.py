"""Build an experiment variant of libtfs.so with extra -D switches, for A/B timing only.

    python tools/build_variant.py OUT.so -DTFS_EXP_NO_TMA -DTFS_EXP_NO_MMA   # barrier skeleton
    TFS_LIB=$PWD/OUT.so python tools/one_ssm.py                              # run against it

Switches (paper_1605_08695_b200/csrc): TFS_EXP_NO_TMA / TFS_EXP_NO_MMA / TFS_EXP_NO_EPI isolate
the three roles of the tcgen05 GEMM (results are wrong; timing only), TFS_EXP_NO_HITS and
TFS_EXP_CB_GLOBAL vary its epilogue, TFS_KSUB sets k-blocks per pipeline stage, TFS_UMMA_CTAS=2
builds the CTA-pair GEMM, TFS_SEG_CHUNK / TFS_SEG_MINB tune the sparse apply.  The numbers these
produced are in profiles/r1_summary.md.
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
