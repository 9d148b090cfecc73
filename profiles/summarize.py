#!/usr/bin/env python
"""Summarise ncu captures into the text files kept under profiles/.

  python profiles/summarize.py launches <launches.csv>      # per-kernel share of device time
  python profiles/summarize.py full <report.ncu-rep>        # key metrics + top stall lines per kernel
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__waves_per_multiprocessor", "launch__occupancy_limit_shared_mem",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]


def launches(path):
    tot = defaultdict(float)
    cnt = defaultdict(int)
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    hdr = rows[0]
    ik, im, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", ""))
        if r[iu] in ("nsecond", "ns"):
            v /= 1e3
        elif r[iu] in ("msecond", "ms"):
            v *= 1e3
        name = r[ik].split("(")[0]
        tot[name] += v
        cnt[name] += 1
    all_us = sum(tot.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>7s}")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k[:60]:60s} {cnt[k]:8d} {tot[k]:12.1f} {tot[k] / cnt[k]:10.2f} {tot[k] / all_us * 100:6.1f}%")


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print("=" * 100)
        print(r[hdr.index("Kernel Name")])
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:70s} {r[i]:>16s} {units[i]}")
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    blocks = src.split('"Kernel Name"')
    for b in blocks[1:]:
        lines = b.splitlines()
        name = lines[0].split(",")[1] if lines else "?"
        rr = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
        if not rr:
            continue
        h = rr[0]
        try:
            iS, iW = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
        except ValueError:
            continue
        data = [x for x in rr[1:] if len(x) > iW]
        tot = sum(float(x[iW] or 0) for x in data) or 1.0
        print("-" * 100)
        print("top stall-sampled SASS lines:", name)
        for x in sorted(data, key=lambda x: -float(x[iW] or 0))[:12]:
            print(f"  {float(x[iW] or 0) / tot * 100:5.1f}%  {x[iS][:100]}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
