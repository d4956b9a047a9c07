"""Sum an ncu --csv launch list (gpu__time_duration.sum) per kernel name.

    python tools/launch_sum.py gpurun_out/launches.csv [--top 30]
"""
import collections
import csv
import re
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[1:]:
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3)
        name = re.sub(r"\(.*", "", r[ki])[:70]
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{name:70s} {c:6d} {t:11.1f} us {t / c:9.2f} us/launch {100 * t / tot:5.1f}%")
    print(f"total {tot:.1f} us")


if __name__ == "__main__":
    main()
