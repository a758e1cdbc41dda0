"""The B200 path against the REFERENCE ITSELF.

Two anchors, both independent of the oracle restatement:

* committed golden vectors the unmodified reference produced on the BASELINE
  configs' seeded inputs (tests/golden/ref_*.npz, tools/gen_ref_golden.py):
  the data vector b = T x_true + noise, one T_w x and one T_w^* b, and the
  CGLS iterate after the config's own iteration count -- all five configs,
  full size;
* the reference library oracle/_ref/libgs_ref.so run live beside the GPU on
  seeded mid-size problems (it travels with the snapshot; skipped if absent).

Bars (north star): T x and T* y <= 1e-10 relative; CGLS iterate <= 1e-8, or
-- on configs whose CG amplifies roundoff beyond that (C4, C5 b=85; DESIGN.md
"Parity") -- within the documented sensitivity, printed as a deviation."""
import hashlib
import os

import numpy as np
import pytest

from oracle import ref, rel_error

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
TOL_APPLY = 1e-10
TOL_CGLS = 1e-8


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def golden(name):
    path = os.path.join(GOLD, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated")
    f = np.load(path, allow_pickle=False)
    return {k: f[k] for k in f.files}


def sample_err(v, val, norm):
    """max entry error relative to the vector's rms entry (||v|| / sqrt(n))."""
    return float(np.max(np.abs(v - val)) / float(norm) * np.sqrt(v.size if v.size else 1))


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5_b0", "c5_b85", "c5_b170", "c5_b255"])
def test_gpu_matches_reference_golden(name):
    import bench
    import paper_1607_04091_b200 as gs
    fx = golden(f"ref_{name}.npz")
    workload, b = str(fx["workload"]), int(fx["problem"])
    dim, p, J, c, mu, bw, sig = bench.problem_inputs(workload, b, bench.ProductGen())
    assert sha(c) == str(fx["coords_sha"])
    if mu is not None:
        assert sha(mu) == str(fx["weights_sha"])
    op_u = gs.freq2wave(gs.SamplingSet(dim, c), p, J, bandwidth=bw)
    x_true, noise = bench.coeffs_and_noise(b, op_u.cols(), op_u.rows(), sig)
    data = gs.apply_forward(op_u, x_true) + noise
    del op_u
    op = gs.freq2wave(gs.SamplingSet(dim, c), p, J, bandwidth=bw, weights=mu)
    im, ic = fx["m_idx"], fx["c_idx"]
    M, Nc = data.size, op.cols()
    eb = float(np.max(np.abs(data[im] - fx["b_val"])) / float(fx["b_norm"]) * np.sqrt(M))
    ey = float(np.max(np.abs(gs.apply_forward(op, x_true)[im] - fx["y_val"])) / float(fx["y_norm"]) * np.sqrt(M))
    ez = float(np.max(np.abs(gs.apply_adjoint(op, data)[ic] - fx["z_val"])) / float(fx["z_norm"]) * np.sqrt(Nc))
    K = int(fx["iters"])
    x, st = gs.solve_least_squares(op, data, max_iterations=K, tolerance=1e-300)
    assert st.iterations == K
    ex = float(np.linalg.norm(x[ic] - fx["x_val"]) / np.linalg.norm(fx["x_val"]))
    h = np.asarray(st.history)
    big = fx["history"] > 1e-6  # residuals well above their own roundoff
    eh = float(np.max(np.abs(h[big] - fx["history"][big]) / fx["history"][big]))
    sens = float(fx["oracle_sens"]) if "oracle_sens" in fx else 0.0
    print(f"{name} ({op.route}) vs the reference itself: b {eb:.1e}, T x {ey:.1e}, T* y {ez:.1e}; "
          f"CGLS iterate after {K} iterations {ex:.3e} (1e-15-data sensitivity {sens:.1e}); residual history (entries > 1e-6) {eh:.1e}")
    assert max(eb, ey, ez) <= TOL_APPLY
    if ex > TOL_CGLS:
        ops = os.path.join(GOLD, f"cgls_{workload}_opsens.npz")
        sens_op = float(np.load(ops)["sens_op"]) if os.path.exists(ops) else 0.0
        print(f"DEVIATION {name}: CGLS iterate {ex:.3e} > 1e-8 vs the reference; CG amplifies roundoff here "
              f"(1e-15 data perturbation moves the iterate {sens:.2e}, 1-ulp row weights {sens_op:.2e})")
        assert max(sens, sens_op) > TOL_CGLS / 20 and (ex <= 20 * sens or ex <= 100 * sens_op), (ex, sens, sens_op)


LIVE = [  # dim, p, J, M per axis, eps, pattern, weights
    (1, 1, 9, 1024, 1.0, "grid", False), (1, 4, 10, 4096, 0.5, "jitter", True), (1, 8, 8, 1000, 0.5, "jitter", True),
    (2, 1, 5, 64, 0.5, "jitter", False), (2, 2, 6, 128, 1.0, "grid", False), (2, 4, 6, 128, 0.5, "jitter", True),
    (2, 3, 6, 100, 0.5, "jitter", True),
]


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref/libgs_ref.so absent")
@pytest.mark.parametrize("dim,p,J,M,eps,kind,weighted", LIVE)
def test_gpu_matches_reference_live(dim, p, J, M, eps, kind, weighted):
    import paper_1607_04091_b200 as gs
    from paper_1607_04091_b200 import inputs
    pts = ref.gen_grid(M, eps, dim) if kind == "grid" else ref.gen_jitter(M, eps, 0.2, 23, dim)
    K = M * eps / 2 + 1
    mu = inputs.voronoi_weights(dim, pts, K) if weighted else None
    r = ref.Op(dim, p, J, pts, weights=mu, bandwidth=K)
    g = gs.freq2wave(gs.SamplingSet(dim, pts), p, J, bandwidth=K, weights=mu)
    assert (g.rows(), g.cols()) == (r.rows, r.cols)
    rng = np.random.default_rng(3)
    x = rng.standard_normal(r.cols) + 1j * rng.standard_normal(r.cols)
    y = rng.standard_normal(r.rows) + 1j * rng.standard_normal(r.rows)
    ef = rel_error(gs.apply_forward(g, x), r.forward(x))
    ea = rel_error(gs.apply_adjoint(g, y), r.adjoint(y))
    data = r.forward(x)
    xg, sg = gs.solve_least_squares(g, data, max_iterations=30, tolerance=1e-300)
    xr, sr = r.solve(data, max_iterations=30, tolerance=1e-300)
    ec = rel_error(xg, xr)
    print(f"live reference, dim {dim} p {p} J {J} M {M} {kind} ({g.route}): T x {ef:.1e}, T* y {ea:.1e}, "
          f"CGLS(30) {ec:.1e}")
    assert ef <= TOL_APPLY and ea <= TOL_APPLY
    assert sg.iterations == sr["iterations"] == 30
    assert ec <= TOL_CGLS
