"""Top CUDA source lines of one kernel by warp-stall samples (ncu source page,
cuda,sass view: rows with a line number carry the per-line aggregates).

usage: python tools/ncu_hot.py <report.ncu-rep> <kernel-regex> [N]
"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
       f"regex:{kern}"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
# the page repeats the whole listing per matching launch record: keep the first
kn = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
if len(kn) > 1:
    rows = rows[:kn[1]]
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
hdr = rows[hi]
si = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ri = [hdr.index(h) for h in reasons]
recs = []
for r in rows[hi + 1:]:
    if len(r) <= max(ri) or not r[0] or r[0] == "Line No":
        continue
    try:
        tot = float(r[si] or 0)
    except ValueError:
        continue
    if tot <= 0:
        continue
    rs = sorted(((float(r[i] or 0), reasons[k]) for k, i in enumerate(ri)), reverse=True)[:3]
    recs.append((tot, r[0], r[1].strip()[:80], r[ie], rs))
allt = sum(t for t, *_ in recs) or 1
for tot, line, s, ins, rs in sorted(recs, reverse=True)[:top]:
    why = " ".join(f"{n.replace('stall_', '')}={v / tot:.0%}" for v, n in rs if v)
    print(f"{tot / allt:6.1%} L{line:>5} i={ins:>9} {s:80s} {why}")
