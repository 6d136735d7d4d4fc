#!/usr/bin/env python
"""Summarise ncu outputs for profiles/<round>/SUMMARY.md.

    python scripts/summarize_ncu.py launches.csv [full.ncu-rep] > SUMMARY.md

* launches.csv: `ncu --metrics gpu__time_duration.sum --csv` launch list. Per
  kernel name: launches, total and mean device time, share of all librlhead
  launches (cold-cache and serialised under ncu: compare shares).
* full.ncu-rep: `ncu --set full` capture; key counters per captured launch.
"""
import collections
import csv
import subprocess
import sys

OURS = ("k_tc_gemm", "k_merge", "k_gather", "k_flags", "k_compact", "k_scan", "k_validate", "k_dz",
        "k_grpo", "k_stats_reduce", "k_zero_inactive", "k_simt")


def short(name):
    return name.replace("void ", "").replace("rlh::", "").split("(")[0]


def launches(path):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    hdr = rows[0]
    i_name, i_val = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        n = short(r[i_name])
        if not n.startswith(OURS):
            continue
        v = float(r[i_val].replace(",", "")) / 1e6  # ns -> ms
        c, t = agg.get(n, (0, 0.0))
        agg[n] = (c + 1, t + v)
    tot = sum(t for _, t in agg.values())
    print("| kernel | launches | total ms | mean ms | share |")
    print("|---|---|---|---|---|")
    for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{n}` | {c} | {t:.2f} | {t / c:.3f} | {100 * t / tot:.1f}% |")
    print()


KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    print("| kernel | " + " | ".join(k for k in KEYS) + " |")
    print("|---" * (len(KEYS) + 1) + "|")
    for r in rows[2:]:
        vals = [f"{r[idx[k]]} {units[idx[k]]}" if k in idx else "n/a" for k in KEYS]
        print(f"| `{short(r[idx['Kernel Name']])}` | " + " | ".join(vals) + " |")
    print()


if __name__ == "__main__":
    launches(sys.argv[1])
    if len(sys.argv) > 2:
        full(sys.argv[2])
