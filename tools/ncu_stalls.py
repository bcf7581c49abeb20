"""Per-segment (between BAR.SYNCs) stall-reason totals from an ncu source page."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else None)
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kern:
    cmd += ["-k", f"regex:{kern}"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
# the page repeats the whole listing per matching launch record: keep the first
kn = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
if len(kn) > 1:
    rows = rows[:kn[1]]
hi = [i for i, r in enumerate(rows) if "Address" in r and "Source" in r][0]
hdr = rows[hi]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ri = [hdr.index(h) for h in reasons]
src = hdr.index("Source")
ie = hdr.index("Instructions Executed")
seg, acc, inst = 0, {}, {}
for r in rows[hi + 1:]:
    if len(r) <= max(ri):
        continue
    a = acc.setdefault(seg, [0] * len(ri))
    for k, i in enumerate(ri):
        try:
            a[k] += int(r[i] or 0)
        except ValueError:
            pass
    try:
        inst[seg] = inst.get(seg, 0) + int(r[ie] or 0)
    except ValueError:
        pass
    if "BAR.SYNC" in r[src]:
        seg += 1
tot = sum(sum(v) for v in acc.values())
for sg, a in acc.items():
    s = sum(a)
    top = sorted(zip(reasons, a), key=lambda t: -t[1])[:5]
    print(f"seg {sg}: {100 * s / tot:5.1f}%  insts {inst.get(sg, 0):>10d}  " +
          "  ".join(f"{n[6:]}={100 * v / max(s, 1):.0f}%" for n, v in top))
