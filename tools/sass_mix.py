"""Instruction mix of an ncu source-page SASS export (tools/prof.sh *_sass.csv): executed warp instructions
and stall samples per opcode, and the hottest instructions."""
import csv
import sys
from collections import Counter

fn = sys.argv[1]
rows = list(csv.reader(open(fn)))
h = rows[1]
iS, iE, iSm = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
ex, sm = Counter(), Counter()
hot = []
tot_e = tot_s = 0
for r in rows[2:]:
    if len(r) <= iSm:
        continue
    src = r[iS].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    e = float(r[iE] or 0)
    s = float(r[iSm] or 0)
    ex[op] += e
    sm[op] += s
    tot_e += e
    tot_s += s
    hot.append((s, e, r[0], src))
print(f"total warp instructions {tot_e:.3g}, stall samples {tot_s:.0f}")
for op, e in ex.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"  {op:10s} {100 * e / tot_e:5.1f} % inst   {100 * sm[op] / max(tot_s, 1):5.1f} % samples")
print("hottest:")
for s, e, a, src in sorted(hot, reverse=True)[:30]:
    print(f"  {a:>6s} {100 * s / max(tot_s, 1):5.2f} % {e:12.0f}  {src[:90]}")
