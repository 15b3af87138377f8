"""Summarise ncu reports (.ncu-rep from `ncu --set full`) and launch lists (--metrics
gpu__time_duration.sum CSV) into small tracked files under profiles/.

  python tools/ncu_summary.py rep  <file.ncu-rep> [...]   → one JSON object per kernel launch
  python tools/ncu_summary.py list <launches.csv>         → per-kernel totals and shares
"""
import collections
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")][:120]}
        for m in METRICS:
            if m in h:
                i = h.index(m)
                d[m] = f"{r[i]} {units[i]}".strip()
        res.append(d)
    return res


def launch_list(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(t for _, t in agg.values())
    return {"total_us": tot, "launches": sum(n for n, _ in agg.values()),
            "kernels": [{"kernel": k, "launches": n, "us": round(t, 1), "share": round(t / tot, 4)}
                        for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])]}


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "rep":
        for p in sys.argv[2:]:
            for d in rep(p):
                print(json.dumps(d))
    else:
        print(json.dumps(launch_list(sys.argv[2]), indent=1))
