"""Summarise ncu outputs into text files for profiles/ (run here, no GPU).

    python tools/summarize_ncu.py launches <launches.csv> <out.txt>
    python tools/summarize_ncu.py full <report.ncu-rep> <out.txt>
"""
import collections
import csv
import io
import re
import subprocess
import sys


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").split("::")[-1]
        v = float(r[vi].replace(",", ""))
        v *= {"usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list ({path}); gpu__time_duration.sum, --clock-control none, serialised\n")
        f.write(f"# total kernel time {tot / 1e6:.2f} ms over {sum(v[0] for v in agg.values())} launches\n")
        f.write(f"{'kernel':60s} {'launches':>9s} {'total_ms':>10s} {'share':>7s} {'avg_us':>9s}\n")
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"{k[:60]:60s} {v[0]:9d} {v[1] / 1e6:10.2f} {100 * v[1] / tot:6.1f}% {v[1] / v[0] / 1e3:9.1f}\n")



METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "sm__inst_executed_pipe_fp64.sum.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.sum.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.sum.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
]


def full(path, out):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary of {path}\n")
        for r in rows[2:]:
            f.write(f"\n## {r[h.index('Kernel Name')][:110]}\n")
            for m in METRICS:
                if m in h:
                    i = h.index(m)
                    f.write(f"  {m:80s} {r[i]} {units[i]}\n")



if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
