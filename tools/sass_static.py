"""Static SASS opcode mix of selected kernels in libgs_b200.so (cuobjdump -sass;
no GPU needed).  Usage: python tools/sass_static.py [regex ...] > profiles/...md
Counts instructions per opcode in each matching kernel's SASS: evidence of the
FP64 tensor-core (DMMA), TMA / bulk-copy (UBLKCP, UTMALDG) and mbarrier
(SYNCS) instructions the kernels issue."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1607_04091_b200", "libgs_b200.so")


def main():
    pats = [re.compile(p) for p in (sys.argv[1:] or ["k2f_interp_mma", "k2f_spread_mma", "k_ndft_fwd", "k_ndft_adj"])]
    txt = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    kern, counts = None, collections.OrderedDict()
    for line in txt.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            kern = m.group(1)
            dem = subprocess.run(["c++filt", kern], capture_output=True, text=True).stdout.strip()
            kern = dem if any(p.search(dem) for p in pats) else None
            if kern:
                counts[kern] = collections.Counter()
            continue
        if kern is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m:
            counts[kern][m.group(2).split(".")[0]] += 1
    print("# Static SASS opcode mix (cuobjdump -sass of libgs_b200.so)\n")
    for k, c in counts.items():
        tot = sum(c.values())
        print(f"## `{k}`\n\n{tot} SASS instructions. Top opcodes:\n")
        print("| opcode | count | share |\n|---|---|---|")
        for op, n in c.most_common(18):
            print(f"| {op} | {n} | {100.0 * n / tot:.1f}% |")
        keys = ["DMMA", "DFMA", "DMUL", "DADD", "UBLKCP", "UTMALDG", "UBLKPF", "SYNCS", "LDGSTS", "LDS", "LDG"]
        print("\nKey opcodes: " + ", ".join(f"{o} {c.get(o, 0)}" for o in keys) + "\n")


if __name__ == "__main__":
    main()
