#!/usr/bin/env python3
"""Copy the reference's only stored golden vectors for this path -- the
60-digit edge-function moments of tests/family_fixtures.hpp -- into
tests/golden/edge_moments.json (data only).  moments[r*p + j] is the r-th
moment of edge function j; r = 0 equals phihat_edge(0) = boundary_fourier_at_zero
(fourier.cpp:60-72), r = 1 gives its derivative: d/dxi phihat(0) = -2 pi i m1."""
import json
import re
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/proj/tests/family_fixtures.hpp"
out = sys.argv[2] if len(sys.argv) > 2 else "tests/golden/edge_moments.json"
t = open(src).read()
data = {}
for m in re.finditer(r"constexpr double k(Left|Right)MomentsP(\d)\[\] = \{(.*?)\};", t, re.S):
    vals = [float(v) for v in re.findall(r"[-+]?[0-9.]+(?:[eE][-+]?[0-9]+)?", m.group(3))]
    data.setdefault(m.group(2), {})[m.group(1).lower()] = [v.hex() for v in vals]
json.dump(data, open(out, "w"), indent=1, sort_keys=True)
print("wrote", out)
