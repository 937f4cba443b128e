"""Per-kernel device-time split of an ncu launch-list CSV (dev tool; no GPU).

    python tools/kernel_split.py <launches.csv> [runs]

Launches are grouped by kernel name (templates kept); `runs` divides the totals
(e.g. the number of graph runs the captured script made).
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    runs = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    H = rows[h]
    ki, mi, vi, ui = H.index("Kernel Name"), H.index("Metric Name"), H.index("Metric Value"), H.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        k = r[ki].split("(")[0].replace("void ", "").split("::")[-1]
        v = float(r[vi].replace(",", "")) * {"usecond": 1e3, "msecond": 1e6}.get(r[ui], 1.0)
        agg[k].append(v)
    tot = sum(sum(v) for v in agg.values())
    print(f"total {tot / 1e6 / runs:.2f} ms per run ({runs:g} runs)")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"  {k:28s} {len(v) / runs:7.1f}/run {sum(v) / 1e6 / runs:9.2f} ms/run {100 * sum(v) / tot:5.1f}%"
              f"  avg {sum(v) / len(v) / 1e3:8.1f} us")


if __name__ == "__main__":
    main()
