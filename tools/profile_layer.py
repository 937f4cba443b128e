"""Per-op device-time breakdown of one encrypted layer (dev tool; GPU).

    python tools/profile_layer.py [--tokens 2048] [--out profiles/r01_layer_T2048_ops.txt]
"""
import argparse
import collections
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_03425_b200 import Context  # noqa: E402

KINDS = ["encode", "padd", "cadd", "pmult", "cmult", "rot", "relin", "rescale", "boot"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=2048)
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-hoist", action="store_true")
    ap.add_argument("--dce", action="store_true", help="dead-lane elimination variant")
    a = ap.parse_args()
    c = Context(log_n=16)
    g = c.graph(kind=0, tokens=a.tokens)
    c.keys_generate(g.key_ids())
    if a.no_hoist:
        g.set_hoisting(False)
    if a.dce:
        g.set_dce(True)
    g.run()  # warm
    g.set_profiling(True)
    g.run()
    t = g.op_times()
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "g.heops")
        g.dump(p)
        bundles, ops = {}, []
        for ln in open(p):
            f = ln.split()
            if f and f[0] == "B":
                bundles[int(f[1])] = f[9]
            elif f and f[0] == "O":
                ops.append((KINDS[int(f[2])], bundles[int(f[4])].rsplit(".", 1)[0], int(f[6]), int(f[11])))
    by = collections.defaultdict(lambda: [0, 0.0])
    node = collections.defaultdict(float)
    kind = collections.defaultdict(float)
    for (k, n, lanes, lvl), ms in zip(ops, t):
        key = (n.split(".")[1] if "." in n else n, k)
        by[key][0] += 1
        by[key][1] += ms
        node[key[0]] += ms
        kind[k] += ms
    tot = float(t.sum())
    lines = [f"# per-op device time, T={a.tokens}, N=2^16, hoisting={'off' if a.no_hoist else 'on'}: "
             f"total {tot / 1e3:.2f} s over {len(t)} HE ops"]
    lines.append("## by layer node")
    for k, v in sorted(node.items(), key=lambda x: -x[1]):
        lines.append(f"  {k:18s} {v / 1e3:8.3f} s  {100 * v / tot:5.1f}%")
    lines.append("## by op kind")
    for k, v in sorted(kind.items(), key=lambda x: -x[1]):
        lines.append(f"  {k:18s} {v / 1e3:8.3f} s  {100 * v / tot:5.1f}%")
    lines.append("## by (node, kind)")
    for k, v in sorted(by.items(), key=lambda x: -x[1][1])[:25]:
        lines.append(f"  {k[0]:18s} {k[1]:8s} n={v[0]:4d} {v[1] / 1e3:8.3f} s  avg {v[1] / v[0]:8.2f} ms")
    txt = "\n".join(lines)
    print(txt)
    if a.out:
        open(a.out, "w").write(txt + "\n")


if __name__ == "__main__":
    main()
