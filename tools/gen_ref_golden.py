"""Golden vectors produced by the REFERENCE ITSELF (tests/golden/ref_*.npz).

oracle/_ref/libgs_ref.so is the unmodified reference library (its sources
compiled where they lie with Eigen / FFTW stand-ins: oracle/Makefile,
oracle/ref_driver.cpp); oracle.ref binds it.  For each BASELINE config this
script runs, on the config's seeded inputs (bench.py problem_inputs /
coeffs_and_noise -- the same generators the GPU tests use, SHA-256 asserted):

  gs::freq2wave (unweighted)   b = T x_true + noise         (the data vector)
  gs::freq2wave (weighted)     y = T_w x_true,  z = T_w^* b (one apply each)
  gs::solve_least_squares      x_K after the config's K iterations, tol 1e-300

and stores a sample of each vector (head + strided entries; the vectors run to
2^20 entries), its 2-norm, the residual history and the input hashes.  Where
the oracle's fixture of the same config exists (tests/golden/cgls_*.npz, made
by tools/gen_cgls_fixtures.py) the agreement of the two iterates is printed
and stored (`oracle_vs_ref_x`): that is the oracle pinned against the
reference at config size.

Usage: python tools/gen_ref_golden.py c1 c2 c3 c4 c5:0 c5:85 ...   (one process per spec is fine)
Timing on one core: c1/c2 seconds, c3 ~4 min, c5:b ~6 min, c4 ~35 min.
"""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import oracle  # noqa: E402
from oracle import ref  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sample_idx(n, count=2048):
    head = np.arange(min(64, n))
    stride = np.linspace(0, n - 1, min(count, n)).astype(np.int64)
    return np.unique(np.concatenate([head, stride]))


def main(spec):
    workload, _, b = spec.partition(":")
    b = int(b or 0)
    iters = bench.CONFIG_ITERS[workload]
    assert ref.available(), "oracle/_ref/libgs_ref.so missing (needs /root/reference)"
    t0 = time.time()
    dim, p, J, c, mu, bw, sig = bench.problem_inputs(workload, b, bench.ProductGen())
    op_u = ref.Op(dim, p, J, c, bandwidth=bw)
    x_true, noise = bench.coeffs_and_noise(b, op_u.cols, op_u.rows, sig)
    data = op_u.forward(x_true) + noise
    del op_u
    op = ref.Op(dim, p, J, c, weights=mu, bandwidth=bw)
    t1 = time.time()
    y = op.forward(x_true)
    z = op.adjoint(data)
    t2 = time.time()
    x, st = op.solve(data, max_iterations=iters, tolerance=1e-300)
    t3 = time.time()
    assert st["iterations"] == iters
    im, ic = sample_idx(data.size), sample_idx(x.size)
    out = dict(workload=workload, problem=b, iters=iters, backend=ref.backend(),
               coords_sha=sha(c), weights_sha=sha(mu) if mu is not None else "",
               uniform_fast=bool(op.uniform_fast),
               m_idx=im, c_idx=ic,
               b_val=data[im], b_norm=np.linalg.norm(data),
               y_val=y[im], y_norm=np.linalg.norm(y),
               z_val=z[ic], z_norm=np.linalg.norm(z),
               x_val=x[ic], x_norm=np.linalg.norm(x),
               history=np.asarray(st["history"]))
    name = f"ref_{workload}" + (f"_b{b}" if workload == "c5" else "") + ".npz"
    fx = os.path.join(OUT, f"cgls_{workload}" + (f"_b{b}" if workload == "c5" else "") + ".npz")
    msg = ""
    if os.path.exists(fx):
        f = np.load(fx)
        e = oracle.rel_error(f["x"], x)
        eb = np.max(np.abs(f["b_val"] - data[f["b_idx"]])) / np.linalg.norm(data) * np.sqrt(data.size)
        out.update(oracle_vs_ref_x=e, oracle_vs_ref_b=eb, oracle_sens=float(f["sens"]))
        msg = f"; oracle fixture vs reference: iterate {e:.3e} (oracle sensitivity {float(f['sens']):.2e}), b sample {eb:.1e}"
    np.savez(os.path.join(OUT, name), **out)
    print(f"{spec}: construction {t1 - t0:.0f} s, applies {t2 - t1:.1f} s, {iters} iterations {t3 - t2:.0f} s"
          f"{msg} -> {name}", flush=True)


if __name__ == "__main__":
    for s in sys.argv[1:]:
        main(s)
