"""Summarise an ncu source page (SASS) export: top stall instructions and
per-region sample totals.  usage: ncu_src.py page.csv [ntop]"""
import csv
import sys

r = list(csv.reader(open(sys.argv[1])))
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = r[1]
rows = r[2:]
si = h.index("Warp Stall Sampling (All Samples)")
src = h.index("Source")
ex = h.index("Instructions Executed")
tot = sum(int(x[si] or 0) for x in rows)
print("total samples", tot, "instructions", len(rows))
top = sorted(range(len(rows)), key=lambda i: -int(rows[i][si] or 0))[:ntop]
for i in sorted(top):
    print(f"{i:5d} {rows[i][si]:>6} {rows[i][ex]:>9}  {rows[i][src][:90]}")
marks = [i for i, x in enumerate(rows) if "BAR.SYNC" in x[src] or "EXIT" in x[src] or "CCTL.IVALL" in x[src]]
print("barrier/exit/cctl at", marks)
