"""Print the per-launch device times of an ncu --csv launch list."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hi]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for r in rows[hi + 1:hi + 1 + n]:
    print(f"{r[vi]:>10s} {r[ui]:5s} {r[ki][:80]}")
