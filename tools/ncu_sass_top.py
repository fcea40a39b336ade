"""Summarise an ncu report's SASS source page: top instructions by stall samples / executions."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows[:10]) if "Source" in r)
h = rows[hi]
S, E, SMP = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[hi + 1:] if len(r) > SMP]
tot_s = sum(float(r[SMP] or 0) for r in data)
tot_e = sum(float(r[E] or 0) for r in data)
print(f"total samples {tot_s:.0f}, total warp-instructions {tot_e:.3g}")
op = Counter()
ops = Counter()
for r in data:
    mn = r[S].split()[0] if r[S].split() else "?"
    if mn.startswith("@"):
        mn = r[S].split()[1]
    op[mn.split(".")[0]] += float(r[E] or 0)
    ops[mn.split(".")[0]] += float(r[SMP] or 0)
print("by opcode (exec share, stall share):")
for k, v in op.most_common(18):
    print(f"  {k:10s} {v / tot_e:6.3f} {ops[k] / tot_s:6.3f}")
print("top stall instructions:")
for r in sorted(data, key=lambda r: -float(r[SMP] or 0))[:n]:
    print(f"  {r[0]:>6s} {float(r[SMP] or 0) / tot_s:6.3f} {r[S][:90]}")
