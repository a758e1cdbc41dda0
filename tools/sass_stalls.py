#!/usr/bin/env python3
"""Summarise an `ncu --page source --csv --print-source sass` export: stall
samples per opcode and the hottest instructions (with their neighbours)."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr, data = rows[i0], rows[i0 + 1:]
ci = {h: i for i, h in enumerate(hdr)}
S = ci["Warp Stall Sampling (All Samples)"]
tot = sum(int(r[S]) for r in data)
by_op = Counter()
for r in data:
    op = r[1].split()[0] if r[1].split() else "?"
    if op.startswith("@"):
        op = r[1].split()[1]
    by_op[op.split(".")[0]] += int(r[S])
print("total samples", tot)
for op, v in by_op.most_common(15):
    print(f"  {op:10s} {100 * v / tot:5.1f}%")
top = sorted(range(len(data)), key=lambda i: -int(data[i][S]))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for i in sorted(top):
    print(f"{i:5d} {100 * int(data[i][S]) / tot:5.2f}%  {data[i][1].strip()[:90]}")
# stall reasons of the hottest instructions
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print("\nreason totals:", ", ".join(f"{h[6:]} {100 * sum(int(r[ci[h]]) for r in data) / tot:.1f}%" for h in reasons
                                  if sum(int(r[ci[h]]) for r in data) > 0.01 * tot))
for i in sorted(top)[:]:
    rs = sorted(((int(data[i][ci[h]]), h[6:]) for h in reasons), reverse=True)[:3]
    if int(data[i][S]) > 0.01 * tot:
        print(f"{i:5d} {data[i][1].strip()[:50]:50s} " + " ".join(f"{n}:{v}" for v, n in rs if v))
# executed-instruction mix
X = ci["Instructions Executed"]
tx = sum(int(r[X] or 0) for r in data)
mix = Counter()
for r in data:
    t = r[1].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    mix[op.split(".")[0]] += int(r[X] or 0)
print("\nexecuted warp instructions", tx, "; mix:", ", ".join(f"{o} {100 * v / tx:.1f}%" for o, v in mix.most_common(18)))
