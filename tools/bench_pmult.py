"""Device time of one bundled PCMM step (pmult_acc) at the T=2048 layer's
shapes, N = 2^16.  Dev tool; GPU.

    python tools/bench_pmult.py [--shapes qkv,ffn1,ffn2,small]

qkv : 4 token groups x 12 input cts -> 36 outputs in 3 sub-tensors, level 35
ffn1: 4 x 12 -> 48 outputs (4 sub-tensors of 12), level 17
ffn2: 4 x 48 -> 12 outputs, level 17
small: T = 512 (1 token group) qkv at level 35
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2604_03425_b200 import Context  # noqa: E402

SHAPES = {  # tg, c_in, c_out, chunk_period, level
    "qkv": (4, 12, 36, 48, 35),
    "ffn1": (4, 12, 48, 48, 17),
    "ffn2": (4, 48, 12, 0, 17),
    "small": (1, 12, 36, 0, 35),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="qkv,ffn1,ffn2,small")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    c = Context(log_n=16)
    st = torch.cuda.ExternalStream(c.stream)
    for name in a.shapes.split(","):
        tg, c_in, c_out, chunk, level = SHAPES[name]
        x = c.bundle(tg * c_in, 2, level)
        x.fill_input(1)
        acc = c.bundle(tg * c_out, 2, level)
        acc.fill_input(2)
        fn = lambda: c.pmult_acc(acc, x, 77, c_in * c_out, level, chunk_period=chunk)  # noqa: E731
        fn()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn()
            e1.record(st)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        macs = tg * c_in * c_out * 2 * level * 65536
        print(f"{name:6s} tg={tg} {c_in}x{c_out} L={level}: {min(ts):8.3f} ms  "
              f"{macs / min(ts) / 1e6:8.1f} G modmul/s  (all {[round(t, 3) for t in ts]})", flush=True)
        x.free()
        acc.free()


if __name__ == "__main__":
    main()
