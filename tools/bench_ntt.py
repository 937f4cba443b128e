"""NTT / INTT throughput at N = 2^16 for each butterfly implementation (dev tool; GPU).

    python tools/bench_ntt.py [--shapes 48x17,12x35,1x8]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2604_03425_b200 import Context, _lib  # noqa: E402


def timed(c, fn, reps=10):
    st = torch.cuda.ExternalStream(c.stream)
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="48x17,12x35,4x8")
    ap.add_argument("--impls", default="2,1,0")
    a = ap.parse_args()
    c = Context(log_n=16)
    lib = _lib.load()
    names = {0: "int-v1", 1: "f64-v2", 2: "f64-v1"}
    for sh in a.shapes.split(","):
        lanes, level = map(int, sh.split("x"))
        b = c.bundle(lanes, 1, level)
        b.fill_input(1)
        limbs = lanes * level
        for impl in map(int, a.impls.split(",")):
            lib.aegis_ntt_impl(impl)
            tf = timed(c, lambda: c.ntt(b))
            ti = timed(c, lambda: c.ntt(b, inverse=True))
            alg = 16 * 65536 * limbs
            print(f"{names[impl]:7s} {limbs:4d} limbs: fwd {tf * 1e6 / limbs:7.1f} ns/limb ({alg / tf / 1e6:7.1f} GB/s)"
                  f"  inv {ti * 1e6 / limbs:7.1f} ns/limb ({alg / ti / 1e6:7.1f} GB/s)", flush=True)
        b.free()
    lib.aegis_ntt_impl(1)


if __name__ == "__main__":
    main()
