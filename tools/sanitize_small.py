"""Small solves through every route (uniform 1D, 1D NFFT, tensor, 2D NFFT): a
debug driver for bounds / assert builds of the kernels: python tools/sanitize_small.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (input generators only)
import paper_1607_04091_b200 as gs  # noqa: E402

rng = np.random.default_rng(0)


def rc(n):
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)


cases = [
    ("uniform haar", 1, 1, 6, oracle.gen_grid(128, 1.0), 64.0, None),
    ("uniform db2", 1, 2, 6, oracle.gen_grid(160, 0.5), None, None),
    ("nfft1d db4", 1, 4, 6, oracle.gen_jitter(200, 0.5, 0.2, 3, 1), None, "w"),
    ("tensor db2", 2, 2, 4, oracle.gen_grid(32, 1.0, 2), 16.0, None),
    ("nfft2d db4", 2, 4, 5, oracle.gen_jitter(48, 0.5, 0.2, 4, 2), None, "w"),
    # spiral: uneven bands -> the balanced band schedule of the DMMA kernels, multi-chunk tiles
    ("nfft2d db4 spiral", 2, 4, 5, oracle.gen_spiral(6, 1024.0, 15.0), 16.0, None),
    ("nfft2d db2 spiral", 2, 2, 5, oracle.gen_spiral(6, 1024.0, 15.0), 16.0, None),
]
for name, dim, p, J, c, bw, w in cases:
    K = bw if bw is not None else float(np.max(np.abs(c))) + 1e-9
    mu = oracle.voronoi(dim, c, K) if w else None
    op = gs.freq2wave(gs.SamplingSet(dim, c), p, J, bandwidth=K, weights=mu)
    y = gs.apply_forward(op, rc(op.cols()))
    z = gs.apply_adjoint(op, rc(op.rows()))
    x, st = gs.solve_least_squares(op, y + 1e-3 * rc(op.rows()), max_iterations=4, tolerance=1e-300)
    print(name, op.route, "balanced" if getattr(op, "balanced_schedule", False) else "static", st.iterations,
          float(np.linalg.norm(x)), float(np.linalg.norm(z)))
print("sanitize ok")
