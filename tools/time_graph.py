"""Quick timing of graph execution and NTT throughput on one GPU (dev tool)."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_03425_b200 import Context  # noqa: E402


def timed(c, fn, reps=3):
    st = torch.cuda.ExternalStream(c.stream)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return ts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=128)
    ap.add_argument("--kind", type=int, default=1)
    ap.add_argument("--layers", type=int, default=1)
    ap.add_argument("--ntt", action="store_true")
    ap.add_argument("--max-ops", type=int, default=-1)
    a = ap.parse_args()
    c = Context(log_n=16)
    if a.ntt:
        for lanes, level in ((48, 17), (12, 35)):
            b = c.bundle(lanes, 1, level)
            b.fill_input(1)
            ts = timed(c, lambda: c.ntt(b), 5)
            limbs = lanes * level
            t = min(ts) / 1e3
            print(f"NTT fwd {limbs} limbs: {min(ts):.3f} ms  {16 * 65536 * limbs / t / 1e9:.1f} GB/s algorithmic "
                  f"({t / limbs * 1e9:.0f} ns/limb)")
            ts = timed(c, lambda: c.ntt(b, inverse=True), 5)
            t = min(ts) / 1e3
            print(f"NTT inv {limbs} limbs: {min(ts):.3f} ms  {16 * 65536 * limbs / t / 1e9:.1f} GB/s")
            b.free()
    g = c.graph(kind=a.kind, tokens=a.tokens, layers=a.layers)
    c.keys_generate(g.key_ids())
    c.sync()
    t0 = time.time()
    ts = timed(c, lambda: g.run(max_ops=a.max_ops), 2)
    print(f"graph kind={a.kind} T={a.tokens} layers={a.layers}: {ts} ms  wall {time.time() - t0:.1f}s "
          f"peak {g.peak_bytes() / 2**30:.1f} GiB  launches {c.launch_count()}")


if __name__ == "__main__":
    main()
