"""Device time of representative HE-op groups of the T=2048 layer, run through
the graph executor (hoisting and liveness as in the real layer).  Dev tool; GPU.

    python tools/bench_ops.py [--lanes 256] [--rots 8] [--which rot,relin,softrot]

rot     : one source bundle at level 17 rotated by `rots` offsets (hoisted
          ModUp, as att_out's 63 rotations of the score tensor)
relin   : CMult + Relin at level 25 (softmax squaring)
softrot : a single non-hoisted rotation at level 30 (softmax rot-add ladder)
"""
import argparse
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2604_03425_b200 import Context  # noqa: E402


def op(i, kind, out, lanes, level, ins, rot=0, acc=0):
    s = f"O {i} {kind} {rot} {out} 0 {lanes} {acc} 0 -1 0 {level} 0 0 {len(ins)}"
    for b in ins:
        s += f" {b} 0 {lanes}"
    return s


def graph(which, lanes, rots):
    L = ["# heops v1 bench", "inputs 0"]
    if which in ("rot", "rot34"):
        lvl = 17 if which == "rot" else 34
        L.append(f"B 0 {lanes} {lvl} 2 0 0 0 0 src")
        for r in range(rots):
            L.append(f"B {r + 1} {lanes} {lvl} 2 2 0 0 0 rot{r}")
        for r in range(rots):
            L.append(op(r, 5, r + 1, lanes, lvl, [0], rot=r + 1))
    elif which == "relin":
        lvl = 25
        L += [f"B 0 {lanes} {lvl} 2 0 0 0 0 src", f"B 1 {lanes} {lvl} 2 1 0 0 0 sq"]
        L += [op(0, 4, 1, lanes, lvl, [0, 0]), op(1, 6, 1, lanes, lvl, [1])]
    elif which == "caddw":  # score accumulation: 48 product lanes added (wrapped) into 1,536
        lvl = 33
        L[1] = "inputs 0 1"
        L += [f"B 0 {lanes} {lvl} 2 0 0 0 0 acc", f"B 1 {max(1, lanes // 32)} {lvl} 2 0 0 0 0 prod"]
        L.append(f"O 0 2 0 0 0 {lanes} 1 0 -1 0 {lvl} 0 0 1 1 0 {max(1, lanes // 32)}")
    elif which == "softrot":
        lvl = 30
        L += [f"B 0 {lanes} {lvl} 2 0 0 0 0 src", f"B 1 {lanes} {lvl} 2 2 0 0 0 rot"]
        L.append(op(0, 5, 1, lanes, lvl, [0], rot=4))
    return "\n".join(L) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lanes", type=int, default=256)
    ap.add_argument("--rots", type=int, default=8)
    ap.add_argument("--which", default="rot,relin,softrot")
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    c = Context(log_n=16)
    st = torch.cuda.ExternalStream(c.stream)
    with tempfile.TemporaryDirectory() as d:
        for w in a.which.split(","):
            p = os.path.join(d, w + ".heops")
            open(p, "w").write(graph(w, a.lanes, a.rots))
            g = c.load_graph(p)
            c.keys_generate(g.key_ids())
            g.run()
            g.run()
            ts = []
            hs = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                h0 = time.perf_counter()
                g.run()
                hs.append(round((time.perf_counter() - h0) * 1e3, 1))
                e1.record(st)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            if os.environ.get("AEGIS_DEBUG"):
                print("  host ms per run (enqueue):", hs)
            ms = min(ts)
            units = a.lanes * (a.rots if w.startswith("rot") else 1)
            print(f"{w:8s} {a.lanes} lanes: {ms:9.3f} ms/run  {ms * 1e3 / units:8.1f} us per lane-op "
                  f"(min of {a.reps}; all {[round(t, 1) for t in ts]})", flush=True)


if __name__ == "__main__":
    main()
