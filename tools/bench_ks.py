"""Per-HE-op device time on a batch of lanes at N = 2^16 (dev tool; GPU).

    python tools/bench_ks.py [--lanes 64] [--level 25] [--reps 3]

Under `ncu --metrics gpu__time_duration.sum` the same script gives the
kernel-level split of each operator.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2604_03425_b200 import Context  # noqa: E402


def timed(c, fn, reps):
    st = torch.cuda.ExternalStream(c.stream)
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
    ap.add_argument("--lanes", type=int, default=64)
    ap.add_argument("--level", type=int, default=25)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    c = Context(log_n=16)
    c.keys_generate([0, 1001])
    L, n = a.level, a.lanes
    x = c.bundle(n, 2, L)
    x.fill_input(1)
    y = c.bundle(n, 2, L)
    y.fill_input(2)
    p3 = c.bundle(n, 3, L)
    out = c.bundle(n, 2, L)
    limb = 8 << 16
    res = {}
    res["cmult"] = timed(c, lambda: c.cmult(p3, x, y, L), a.reps)
    res["relin"] = timed(c, lambda: c.relin(p3, L), a.reps)
    res["rot"] = timed(c, lambda: c.rot(out, x, 1, L), a.reps)
    res["rescale"] = timed(c, lambda: c.rescale(out, x, L), a.reps)
    res["cadd"] = timed(c, lambda: c.cadd(out, x, y, L), a.reps)
    res["ntt_fwd"] = timed(c, lambda: c.ntt(x), a.reps)
    for k, v in res.items():
        print(f"{k:8s} {n} lanes @ l={L}: {v:8.3f} ms  {v * 1e3 / n:8.1f} us/lane", flush=True)
    print(f"(cmult alg bytes/lane {7 * L * limb / 1e6:.0f} MB -> {7 * L * limb * n / res['cmult'] / 1e6:.0f} GB/s)")


if __name__ == "__main__":
    main()
