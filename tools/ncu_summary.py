"""Summarise an .ncu-rep (raw page) into a markdown table for profiles/."""
import csv
import subprocess
import sys

WANT = [("Kernel Name", "kernel"), ("gpu__time_duration.sum", "time"),
        ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%pk"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%pk"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ_%"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
        ("launch__block_size", "block")]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    cols = [(h.index(k), lab) for k, lab in WANT if k in h]
    print("| " + " | ".join(f"{lab} ({units[i]})" if units[i] else lab for i, lab in cols) + " |")
    print("|" + "---|" * len(cols))
    for r in rows[2:]:
        cells = []
        for i, lab in cols:
            v = r[i]
            if lab == "kernel":
                v = v.split("(")[0].replace("void ", "")[:60]
            cells.append(v)
        print("| " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
