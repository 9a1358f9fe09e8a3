"""Aggregate an ncu source page (--page source --csv --print-source sass) by
opcode: executed warp-instructions and stall samples per opcode class."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ex, st = Counter(), Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= iE:
        continue
    src = r[iS].strip()
    if not src:
        continue
    op = src.split()[0]
    if op.startswith("@"):
        op = src.split()[1]
    key = op if op.startswith(("VI", "LD", "ST")) else op.split(".")[0]
    n = float(r[iE] or 0)
    ex[key] += n
    st[key] += float(r[iW] or 0)
    tot += n
print(f"total warp-instructions {tot:.4g}")
for k, v in ex.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{k:22s} {v:12.4g} {100 * v / tot:6.2f}%  stall-samples {st[k]:.0f}")
