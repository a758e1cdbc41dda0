#!/usr/bin/env python3
"""Fixed cost of one public-API solve (H2D of the data, preamble, D2H of the
solution) vs its per-iteration cost: times gs_solve_least_squares from pinned
host buffers at a few iteration counts on the C5 workload."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1607_04091_b200 as gs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--problems", type=int, default=64)
a = ap.parse_args()
gen = bench.ProductGen()
inp = [bench.problem_inputs("c5", b, gen) for b in range(a.problems)]
sets = [gs.SamplingSet(2, x[3]) for x in inp]
mu = np.concatenate([x[4] for x in inp])
op = gs.freq2wave(sets, 4, 8, bandwidth=max(x[5] for x in inp), weights=mu)
b = torch.randn(op.rows() * op.batch, dtype=torch.complex128).pin_memory()
x = torch.empty(op.cols() * op.batch, dtype=torch.complex128).pin_memory()
bench.gs_solve_host(op, b, x, 2)
for iters in (1, 2, 11, 41):
    t = time.perf_counter()
    for _ in range(3):
        bench.gs_solve_host(op, b, x, iters)
    t = (time.perf_counter() - t) / 3
    print(f"iters {iters:3d}: {t * 1e3:8.2f} ms per call")
