"""Top SASS lines by warp-stall samples from `ncu -i rep --page source --csv`
(SASS view), with the dominant stall reasons per line."""
import csv
import sys


def main(path, top=30):
    rows = [r for r in csv.reader(open(path)) if r]
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
    h = rows[hi]
    si = h.index("Source")
    ai = h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
    data = []
    for r in rows[hi + 1:]:
        if r[0] == "Kernel Name":
            break  # next kernel's section
        if len(r) < len(h):
            continue
        v = float(r[ai] or 0)
        reasons = sorted(((float(r[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:3]
        data.append((v, r[si].strip(), reasons))
    tot = sum(d[0] for d in data) or 1
    for v, src, reasons in sorted(data, key=lambda d: -d[0])[:top]:
        rs = " ".join(f"{n}:{100 * x / tot:.1f}" for x, n in reasons if x)
        print(f"{100 * v / tot:5.1f}%  {src[:70]:70s} {rs}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
