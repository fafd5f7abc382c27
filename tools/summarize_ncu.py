"""Summaries of ncu outputs for profiles/ (run here, no GPU needed).

  python tools/summarize_ncu.py launches <launches.csv> [steps]   -> markdown table of per-kernel device time
  python tools/summarize_ncu.py full <report.ncu-rep>            -> key metrics per captured kernel
  python tools/summarize_ncu.py lines <report.ncu-rep> <kernel regex> [n]  -> top CUDA lines by stall samples
"""

from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys


def launches(path: str, steps: int = 1) -> str:
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[d["Metric Unit"]]
        name = d["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values())
    out = [f"{len(data)} launches, {tot:.1f} us device time over {steps} step(s) "
           f"({tot / steps:.1f} us/step, serialised, cold cache)", "",
           "| kernel | launches | us | us/step | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {v[0]} | {v[1]:.1f} | {v[1] / steps:.1f} | {100 * v[1] / tot:.1f}% |")
    return "\n".join(out)


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio"]


def full(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {m: hdr.index(m) for m in METRICS if m in hdr}
    out = ["| kernel | " + " | ".join(f"{m} ({units[i]})" for m, i in idx.items()) + " |",
           "|" + "---|" * (len(idx) + 1)]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        out.append(f"| `{name}` | " + " | ".join(r[i] for i in idx.values()) + " |")
    return "\n".join(out)


def lines(path: str, kernel: str, n: int = 15) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass,cuda",
                          "--kernel-name", f"regex:{kernel}", "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    agg = collections.defaultdict(lambda: [0, ""])
    hdr, last = None, ""
    for r in rows:
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        try:
            samples = int(r[4] or 0)
        except ValueError:
            continue
        key = r[0] or last  # SASS rows after the first of a CUDA line carry no line number
        last = key
        agg[key][0] += samples
        if not agg[key][1]:
            agg[key][1] = r[1].strip()
    tot = sum(v[0] for v in agg.values()) or 1
    out = [f"{kernel}: {tot} stall samples", "", "| line | samples | share | source |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:n]:
        out.append(f"| {k} | {v[0]} | {100 * v[0] / tot:.1f}% | `{v[1][:90]}` |")
    return "\n".join(out)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    if kind == "launches":
        print(launches(path, int(sys.argv[3]) if len(sys.argv) > 3 else 1))
    elif kind == "lines":
        print(lines(path, sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 15))
    else:
        print(full(path))
