"""Markdown summary of `ncu --page raw --csv` exports: per captured launch,
duration, DRAM bytes, DRAM throughput, FP64-pipe and issue utilisation.
Usage: python tools/ncu_summary.py name=export.csv ..."""
import csv
import sys

COLS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]

print("| capture | kernel | " + " | ".join(c[1] for c in COLS) + " |")
print("|---|---|" + "---|" * len(COLS))
for arg in sys.argv[1:]:
    name, path = arg.split("=", 1)
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        kern = r[hdr.index("Kernel Name")][:40] if "Kernel Name" in hdr else "?"
        vals = []
        for key, _ in COLS:
            if key in hdr:
                i = hdr.index(key)
                vals.append(f"{r[i]} {units[i]}".strip())
            else:
                vals.append("-")
        print(f"| {name} | `{kern}` | " + " | ".join(vals) + " |")
