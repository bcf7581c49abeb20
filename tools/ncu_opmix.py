"""Executed-instruction mix of one kernel by SASS opcode (ncu source page).

usage: python tools/ncu_opmix.py <report.ncu-rep> <kernel-regex> [N]
"""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
# the page repeats the whole listing per matching launch record: keep the first
kn = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
if len(kn) > 1:
    rows = rows[:kn[1]]
hi = [i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r][0]
hdr = rows[hi]
src, ie = hdr.index("Source"), hdr.index("Instructions Executed")
mix = collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= ie:
        continue
    s = r[src].strip()
    if not s:
        continue
    toks = s.split()
    op = toks[0]
    if op.startswith("@"):
        op = toks[1] if len(toks) > 1 else op
    op = op.split(".")[0]
    try:
        mix[op] += int(float(r[ie] or 0))
    except ValueError:
        pass
tot = sum(mix.values()) or 1
print(f"total warp instructions {tot}")
for op, n in mix.most_common(top):
    print(f"{op:10s} {n:12d} {n / tot:6.1%}")
