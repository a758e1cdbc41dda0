#!/usr/bin/env python3
"""Small driver for ncu: build a workload's operator (bench.py inputs) for a
few problems, run `reps` T / T* pairs on resident device tensors, exit."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1607_04091_b200 as gs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c5")
ap.add_argument("--problems", type=int, default=4)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--cgls", action="store_true", help="run CGLS iterations (sorted-order session path)")
a = ap.parse_args()
gen = bench.ProductGen()
inp = [bench.problem_inputs(a.workload, b, gen) for b in range(a.problems)]
dim, p, J = inp[0][:3]
sets = [gs.SamplingSet(dim, x[3]) for x in inp]
mu = np.concatenate([x[4] for x in inp]) if inp[0][4] is not None else None
op = gs.freq2wave(sets, p, J, bandwidth=max(x[5] for x in inp), weights=mu)
x = torch.randn(op.cols() * op.batch, dtype=torch.complex128, device="cuda")
y = torch.randn(op.rows() * op.batch, dtype=torch.complex128, device="cuda")
if a.cgls:
    sess = gs.CglsSession(op, y)
    sess.step(a.reps)
    sess.close()
else:
    for _ in range(a.reps):
        gs.apply_forward(op, x)
        gs.apply_adjoint(op, y)
torch.cuda.synchronize()
print("route", op.route, "ok")
