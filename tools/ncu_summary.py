"""Summaries of ncu output for profiles/ (tuning aid).

    python tools/ncu_summary.py launches LAUNCHES.csv      # per-kernel share table
    python tools/ncu_summary.py full REPORT.ncu-rep        # key raw metrics per launch
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_read.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__t_sector_hit_rate.pct"]


def short(name):
    name = re.sub(r"\(.*\)$", "", name)
    name = re.sub(r"svdsc::|\(anonymous namespace\)::|<unnamed>::|unnamed>::|void ", "", name)
    return name.replace("(int)", "").strip()


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[h + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        k = short(r[ki])
        v = float(r[vi].replace(",", ""))
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
        us = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
        tot[k] += us
        cnt[k] += 1
    T = sum(tot.values())
    print(f"{'kernel':34s} {'launches':>9s} {'total ms':>10s} {'share':>6s} {'avg us':>9s}")
    for k in sorted(tot, key=lambda q: -tot[q]):
        print(f"{k[:34]:34s} {cnt[k]:9d} {tot[k] / 1e3:10.3f} {100 * tot[k] / T:5.1f}% {tot[k] / cnt[k]:9.2f}")
    print(f"{'TOTAL':34s} {sum(cnt.values()):9d} {T / 1e3:10.3f}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print(short(r[hdr.index("Kernel Name")]))
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"    {k:60s} {r[i]:>16s} {units[i]}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
