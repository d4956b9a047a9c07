"""Summarize an ncu --metrics gpu__time_duration.sum --csv launch list: per
kernel count, total, share and average (cold-cache, serialised launches)."""
import collections
import csv
import re
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hi = [i for i, r in enumerate(rows) if r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[hi + 1:]:
        name = r[ki]
        m = re.search(r"(k_[A-Za-z0-9_]+)", name)
        name = m.group(1) if m else name[:40]
        if "<" in r[ki]:
            tm = re.search(r"k_[A-Za-z0-9_]+<([^>]*)>", r[ki])
            if tm:
                name += "<" + tm.group(1) + ">"
        tot[name] += float(r[vi].replace(",", "")) * scale[r[ui]]
        cnt[name] += 1
    S = sum(tot.values())
    print(f"{'kernel':34s} {'launches':>8s} {'total ms':>10s} {'share':>6s} {'avg us':>9s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:34s} {cnt[k]:8d} {v / 1e3:10.3f} {100 * v / S:5.1f}% {v / cnt[k]:9.2f}")
    print(f"{'TOTAL':34s} {sum(cnt.values()):8d} {S / 1e3:10.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
