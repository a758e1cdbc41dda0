#!/usr/bin/env python3
"""CTA timeline of the fast-path interpolation (debug build with -DF_TIMELINE)
or spreading (-DF_TIMELINE=2) kernel: tools/build_variant.sh tl -DF_TIMELINE, then
GS_B200_LIB=ablibs/tl.so python tools/timeline.py).  Per chunk: SM clock at
entry, staging complete, compute complete; prints phase lengths and, per SM,
how much of the kernel span had 0 / 1 / 2+ CTAs in their compute phase."""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1607_04091_b200 as gs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--problems", type=int, default=8)
ap.add_argument("--workload", default="c5", help="c5 | c4 | c3 (2D NFFT configs)")
a = ap.parse_args()
gen = bench.ProductGen()
inp = [bench.problem_inputs(a.workload, b, gen) for b in range(min(a.problems, bench.problem_count(a.workload)))]
sets = [gs.SamplingSet(2, x[3]) for x in inp]
mu = np.concatenate([x[4] for x in inp]) if inp[0][4] is not None else None
op = gs.freq2wave(sets, inp[0][1], inp[0][2], bandwidth=max(x[5] for x in inp), weights=mu)
L = gs.load_library()
y = torch.randn(op.rows() * op.batch, dtype=torch.complex128, device="cuda")
sess = gs.CglsSession(op, y)
sess.step(2)
torch.cuda.synchronize()
L.gs_debug_timeline_clear()
sess.step(1)  # the interpolation launch of this iteration is recorded
torch.cuda.synchronize()
sess.close()
rows = 1 << 16
buf = np.zeros((rows, 5), dtype=np.uint64)
assert L.gs_debug_timeline(buf.ctypes.data_as(C.c_void_p), C.c_int64(rows)) == 0
buf = buf[buf[:, 0] != 0].astype(np.int64)
t0, t1, t2, sm = buf[:, 0], buf[:, 1], buf[:, 2], buf[:, 3]
print(f"chunks {len(buf)}; cycles per CTA: staging median {np.median(t1 - t0):.0f} (p90 {np.percentile(t1 - t0, 90):.0f}),"
      f" compute median {np.median(t2 - t1):.0f} (p90 {np.percentile(t2 - t1, 90):.0f})"
      + (f", fold+write median {np.median(buf[:, 4] - t2):.0f}" if buf[:, 4].any() else ""))
occ = np.zeros(4)
spans = []
for s in np.unique(sm):
    m = sm == s
    a0, a1, a2 = t0[m], t1[m], t2[m]
    lo, hi = a0.min(), max(a2.max(), buf[m, 4].max())
    spans.append(hi - lo)
    ev = sorted([(x, 1) for x in a1] + [(x, -1) for x in a2])
    cur, last = 0, lo
    for x, d in ev:
        occ[min(cur, 3)] += x - last
        cur += d
        last = x
    occ[0] += hi - last
    # CTAs resident: entries vs exits
print(f"SM span median {np.median(spans):.0f} cycles; time with 0/1/2/3+ CTAs computing: "
      + " ".join(f"{100 * v / occ.sum():.1f}%" for v in occ))
print(f"sum over chunks: staging {np.sum(t1 - t0) / occ.sum():.2f}x span, compute {np.sum(t2 - t1) / occ.sum():.2f}x span")
