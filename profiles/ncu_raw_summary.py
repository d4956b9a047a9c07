"""Key raw metrics per captured kernel from `ncu -i rep --page raw --csv`."""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]


def main(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    for r in rows[2:]:
        name = r[ki].split("(")[0].replace("unnamed>::", "")[:48]
        print(name)
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"    {k:58s} {r[i]:>14s} {units[i]}")


if __name__ == "__main__":
    main(sys.argv[1])
