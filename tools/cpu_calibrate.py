"""Check the CPU arm's extrapolation model (bench.cpu_baseline) against a full
oracle run of BASELINE config 1 (FFN 768->3072->768, T = 128, N = 2^16) on the
host cores.  Dev tool; CPU only (runs on the GPU box's host for its core count).

    python tools/cpu_calibrate.py [--out profiles/r01_cpu_calibration.txt]
"""
import argparse
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import bench  # noqa: E402
from oracle_py import Oracle  # noqa: E402
from paper_2604_03425_b200 import plan_graph  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    threads = os.cpu_count() or 1
    args = argparse.Namespace(tokens=128)
    model = bench.cpu_baseline(args, kind=1)
    g = plan_graph(log_n=16, tokens=128, layers=1, kind=1)
    o = Oracle(16, threads=threads)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "ffn.heops")
        g.dump(path)
        t0 = time.time()
        o.run_graph(path)
        full = time.time() - t0
    txt = (f"# CPU arm calibration, config 1 (FFN T=128, N=2^16), {threads} host threads\n"
           f"full oracle run      : {full:9.1f} s (includes key/table setup)\n"
           f"bench extrapolation  : {model['value']:9.1f} s\n"
           f"ratio model / full   : {model['value'] / full:9.3f}\n"
           f"model sample         : {model['sample']}\n")
    print(txt)
    if a.out:
        open(a.out, "w").write(txt)


if __name__ == "__main__":
    main()
