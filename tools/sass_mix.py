"""Aggregate an `ncu --page source --print-source sass --csv` dump by opcode:
executed warp instructions and stall samples per opcode (profiling helper)."""
import csv, sys, collections

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ie, ss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
cnt, st = collections.Counter(), collections.Counter()
tot = tots = 0
for r in rows[2:]:
    if len(r) < len(h):
        continue
    op = r[1].strip().split()[0] if r[1].strip() else "?"
    if op.startswith("@"):
        op = r[1].strip().split()[1]
    n = int(r[ie] or 0); s = int(r[ss] or 0)
    cnt[op] += n; st[op] += s; tot += n; tots += s
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print(f"total warp instr {tot}, stall samples {tots}")
for op, n in cnt.most_common(top):
    print(f"{op:14s} {n:12d} {100*n/tot:6.2f}%  stalls {100*st[op]/max(tots,1):6.2f}%")
