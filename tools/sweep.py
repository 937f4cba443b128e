"""BASELINE config 5: NTT / INTT and key-switch throughput vs limb count at
N = 2^16 and 2^17 on one B200 (dev tool; GPU).

    python tools/sweep.py [--out profiles/r01_sweep.txt]

NTT: `lanes` x L limbs per call, GB/s = 2 * 8N * limbs / t (algorithmic).
KS : one Relin (hybrid key switch, dnum = ceil(L/4)) of `lanes` lanes at level L,
     microseconds per lane.  Contexts use a 60-prime chain so L runs to 60.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2604_03425_b200 import Context  # noqa: E402


def timed(c, fn, reps=3):
    st = torch.cuda.ExternalStream(c.stream)
    fn()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        e1.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--levels", default="8,16,24,35,48,60")
    a = ap.parse_args()
    lines = ["# NTT / key-switch sweep (BASELINE config 5), one B200; min of 3 timed calls",
             f"{'N':>7s} {'L':>3s} {'lanes':>5s} {'NTT fwd GB/s':>13s} {'ns/limb':>8s} {'INTT GB/s':>10s} "
             f"{'KS us/lane':>11s}"]
    for log_n in (16, 17):
        n = 1 << log_n
        c = Context(log_n=log_n, chain_length=60, bootstrap_level=14)
        c.keys_generate([0])
        for L in map(int, a.levels.split(",")):
            lanes = 16 if log_n == 16 else 8
            b = c.bundle(lanes, 1, L)
            b.fill_input(1)
            tf = timed(c, lambda: c.ntt(b))
            ti = timed(c, lambda: c.ntt(b, inverse=True))
            alg = 2 * 8 * n * lanes * L
            b.free()
            x = c.bundle(lanes, 2, L)
            x.fill_input(2)
            p3 = c.bundle(lanes, 3, L)
            c.cmult(p3, x, x, L)  # valid 3-component product for the Relin
            tk = timed(c, lambda: c.relin(p3, L))
            p3.free()
            x.free()
            ln = (f"{n:7d} {L:3d} {lanes:5d} {alg / tf / 1e6:13.1f} {tf * 1e6 / (lanes * L):8.1f} "
                  f"{alg / ti / 1e6:10.1f} {tk * 1e3 / lanes:11.1f}")
            print(ln, flush=True)
            lines.append(ln)
        c.close()
    if a.out:
        open(a.out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
