"""Run one encrypted layer with the kernel probe on (GPU; driven under ncu by
tools/round_measure*.sh).  Prints the probe totals of the probed kernel as one
JSON line so an ncu capture of the same run can be divided by the same
algorithmic bytes (profiles/r02_cfwd_a_*).

    python tools/ncu_top.py [--tokens 2048] [--kind 0] [--kernel cfwd_a] [--max-ops -1]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=2048)
    ap.add_argument("--kind", type=int, default=0)
    ap.add_argument("--kernel", default="cfwd_a")
    ap.add_argument("--max-ops", type=int, default=-1)
    a = ap.parse_args()
    from paper_2604_03425_b200 import Context
    c = Context(log_n=16)
    g = c.graph(kind=a.kind, tokens=a.tokens)
    c.keys_generate(g.key_ids())
    c.sync()
    c.probe_start(a.kernel)
    g.run(max_ops=a.max_ops)
    c.sync()
    n, ms, b = c.probe_read()
    print(json.dumps({"kernel": a.kernel, "tokens": a.tokens, "launches": n, "probe_ms": ms, "alg_bytes": b,
                      "alg_bytes_per_launch": b / max(n, 1)}), flush=True)


if __name__ == "__main__":
    main()
