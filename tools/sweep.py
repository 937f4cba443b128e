"""BASELINE config 5: NTT / INTT and key-switch throughput vs limb count at
N = 2^16 and 2^17 on one B200 (dev tool; GPU).

    python tools/sweep.py [--out profiles/r02_sweep.txt] [--lanes 16]

NTT: `lanes` x L limbs per call, GB/s = 2 * 8N * limbs / t (algorithmic).
KS : one Relin (hybrid key switch, dnum = ceil(L/4)) of `lanes` lanes at level L,
     microseconds per lane.  Contexts use a 60-prime chain so L runs to 60.
"""
import argparse
import json
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
    ap.add_argument("--lanes", type=int, default=16)
    a = ap.parse_args()
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6550.0) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6550.0
    fp64 = json.load(open(os.path.join(ROOT, "profiles", "r02_pipe_peaks.json")))["dfma_tfma_s"] * 1e12
    lines = ["# NTT / key-switch sweep (BASELINE config 5), one B200; min of 3 timed calls",
             f"# HBM peak {hbm:.0f} GB/s (MEASURED_PEAKS.json); FP64 peak {fp64 / 1e12:.2f} T DFMA-class ops/s "
             "(profiles/r02_pipe_peaks.json, at the 1965 MHz max clock)",
             "# NTT frac = algorithmic GB/s / HBM; NTT fp64 = 8 ops per butterfly x N/2 log N butterflies / t / peak",
             "# KS bytes = SURVEY 8(d): (B (3 l + 2 l) + 2 d (l + 4)) 8N per Relin batch of B lanes;",
             "# KS fp64 floor = limb transforms (INTT l + ModUp d (l+4) - l + ModDown INTT 8 + NTT 2 l) x FP64 ops / peak",
             f"{'N':>7s} {'L':>3s} {'lanes':>5s} {'NTT fwd GB/s':>13s} {'frac':>5s} {'fp64':>5s} {'ns/limb':>8s} "
             f"{'INTT GB/s':>10s} {'KS us/lane':>11s} {'KS GB/s':>8s} {'frac':>5s} {'KS fp64':>7s}"]
    for log_n in (16, 17):
        n = 1 << log_n
        c = Context(log_n=log_n, chain_length=60, bootstrap_level=14)
        c.keys_generate([0])
        for L in map(int, a.levels.split(",")):
            lanes = a.lanes if log_n == 16 else max(1, a.lanes // 2)
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
            d = -(-L // 4)
            ks_bytes = (lanes * (3 * L + 2 * L) + 2 * d * (L + 4)) * 8 * n
            ops_per_limb = 8 * (n // 2) * log_n
            ntt_fp64 = ops_per_limb * lanes * L / (tf / 1e3) / fp64
            n_ntt = L + (d * (L + 4) - L) + 8 + 2 * L
            ks_fp64 = n_ntt * ops_per_limb * lanes / (tk / 1e3) / fp64
            ks_gbs = ks_bytes / (tk / 1e3) / 1e9
            ln = (f"{n:7d} {L:3d} {lanes:5d} {alg / tf / 1e6:13.1f} {alg / tf / 1e6 / hbm:5.2f} {ntt_fp64:5.2f} "
                  f"{tf * 1e6 / (lanes * L):8.1f} {alg / ti / 1e6:10.1f} {tk * 1e3 / lanes:11.1f} {ks_gbs:8.1f} "
                  f"{ks_gbs / hbm:5.2f} {ks_fp64:7.2f}")
            print(ln, flush=True)
            lines.append(ln)
        c.close()
    if a.out:
        open(a.out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
