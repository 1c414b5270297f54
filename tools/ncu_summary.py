"""Summarise `ncu --set full` reports: one line of key metrics per profiled launch.

  python tools/ncu_summary.py gpurun_out/prof_*.ncu-rep > profiles/<round>_ncu_summary.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "dur"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "inst"),
    ("lts__t_sector_hit_rate.pct", "l2hit%"),
]


def main():
    for rep in sys.argv[1:]:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        if len(rows) < 3:
            print(rep, ": no data")
            continue
        h, units = rows[0], rows[1]
        for r in rows[2:]:
            name = r[h.index("Kernel Name")].split("(")[0]
            parts = [rep.split("/")[-1], name[:60]]
            for k, short in KEYS:
                if k in h:
                    i = h.index(k)
                    parts.append(f"{short}={r[i]}{units[i] if units[i] not in ('', '%') else ''}")
            print("  ".join(parts))


if __name__ == "__main__":
    main()
