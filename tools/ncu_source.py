"""Stall samples per SASS opcode / hottest instructions from an ncu report (dev tool; no GPU).

    python tools/ncu_source.py <report.ncu-rep> <kernel regex> [launch_skip]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    skip = sys.argv[3] if len(sys.argv) > 3 else "0"
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--launch-skip", skip,
                          "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    data = rows[2:]
    si, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    val = lambda r: int(r[si]) if r[si].strip().isdigit() else 0  # noqa: E731
    tot = sum(val(r) for r in data) or 1
    agg, cnt = collections.Counter(), collections.Counter()
    for r in data:
        t = r[src].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
        agg[op.split(".")[0]] += val(r)
        cnt[op.split(".")[0]] += 1
    print(f"{rows[0][1]}: {tot} stall samples")
    for k, v in agg.most_common(16):
        print(f"  {k:10s} {v:7d} {100 * v / tot:5.1f}%  ({cnt[k]} instrs)")
    print("hottest:")
    for r in sorted(data, key=lambda r: -val(r))[:20]:
        print(f"  {val(r):6d}  {r[src][:90]}")


if __name__ == "__main__":
    main()
