"""Build an alternate libaegis variant for A/B timing (dev tool; runs here, no GPU).

    python tools/ab_build.py <name> [-DFLAG=V ...]   ->  paper_2604_03425_b200/libaegis_<name>.so

Select it on the GPU with AEGIS_LIB=paper_2604_03425_b200/libaegis_<name>.so
(paper_2604_03425_b200/_lib.py).  Same sources and flags as csrc/Makefile plus
the extra defines.
"""
import concurrent.futures
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2604_03425_b200", "csrc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]


def main():
    name, extra = sys.argv[1], sys.argv[2:]
    out = os.path.join(CSRC, "build_" + name)
    os.makedirs(out, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))

    def comp(src):
        obj = os.path.join(out, os.path.basename(src)[:-3] + ".o")
        subprocess.run(["nvcc"] + FLAGS + extra + ["-c", src, "-o", obj], check=True)
        return obj

    with concurrent.futures.ThreadPoolExecutor(8) as ex:
        objs = list(ex.map(comp, srcs))
    lib = os.path.join(ROOT, "paper_2604_03425_b200", f"libaegis_{name}.so")
    subprocess.run(["nvcc"] + ARCH + ["-shared", "-o", lib] + objs + ["-lcudart"], check=True)
    print("built", lib)


if __name__ == "__main__":
    main()
