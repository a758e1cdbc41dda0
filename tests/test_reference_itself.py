"""The reference ITSELF as the parity anchor.

oracle/_ref/libgs_ref.so is the unmodified reference library -- its own
sources compiled where they lie under /root/reference/proj/src against an
Eigen subset (tests/cpp/shim/Eigen/Dense) and an FFTW stand-in
(oracle/refshim), recipe in oracle/Makefile.  These tests

* run the reference's OWN unit-test files against that library (the stand-ins
  carry the reference through its suites),
* compare the oracle restatement (oracle/gs_oracle.cpp) with it function by
  function on seeded inputs, and
* check the oracle against the committed golden vectors the reference produced
  at the BASELINE configs' sizes (tests/golden/ref_*.npz, made by
  tools/gen_ref_golden.py) -- these run wherever the fixtures are, with or
  without the library.

CPU only.  The library exists where it was built (the container that has
/root/reference) and wherever the snapshot travels."""
import os
import subprocess

import numpy as np
import pytest

import oracle
from oracle import ref, rel_error

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_ref")
GOLD = os.path.join(ROOT, "tests", "golden")
SUITES = ["test_nufft", "test_freq2wave", "test_solver", "test_fourier", "test_scaling", "test_patterns",
          "test_weights", "test_dyadic"]
# One case of the reference's suites asserts BIT equality of (sqrt(mu) * rx) * ry with
# sqrt(mu) * (rx * ry) (test_freq2wave.cpp:211 on the 2D densify of freq2wave.cpp:443).  The two
# association orders round differently (about 1 entry in 5 agrees on x86-64 / GCC), so the
# reference fails that one check on its own arithmetic here; everything else must pass.
KNOWN = {"test_freq2wave": "row weights scale the rows by sqrt(mu) exactly"}

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref/libgs_ref.so absent (built where /root/reference is)")


def suite_binary(name):
    path = os.path.join(BIN, "self_" + name)
    if not os.path.exists(path):
        if ref.buildable():
            subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp"), "refself"])
        else:
            pytest.skip("reference test sources absent and suites not prebuilt")
    return path


@needs_ref
@pytest.mark.parametrize("name", SUITES)
def test_reference_passes_its_own_suite(name):
    out = subprocess.run([suite_binary(name)], capture_output=True, text=True, timeout=900)
    fails = [l[len("[FAIL] "):] for l in out.stdout.splitlines() if l.startswith("[FAIL]")]
    summary = [l for l in out.stdout.splitlines() if l.startswith("test cases:")]
    print(f"reference itself, {name}: {summary[-1] if summary else out.stdout[-300:]}")
    allowed = [KNOWN[name]] if name in KNOWN else []
    assert [f for f in fails if f not in allowed] == [], out.stdout[-3000:]
    assert summary, out.stdout[-1000:]


CASES = [  # dim, p, J, M per axis, eps, pattern
    (1, 1, 6, 128, 1.0, "grid"), (1, 2, 6, 160, 0.5, "jitter"), (1, 4, 7, 512, 0.5, "jitter"),
    (1, 8, 6, 200, 0.5, "jitter"), (2, 1, 4, 32, 0.5, "jitter"), (2, 2, 4, 32, 1.0, "grid"),
    (2, 3, 5, 64, 0.5, "jitter"), (2, 4, 5, 64, 0.5, "jitter"),
]


@needs_ref
@pytest.mark.parametrize("dim,p,J,M,eps,kind", CASES)
def test_oracle_matches_reference(dim, p, J, M, eps, kind):
    """Factors bit for bit; T x, T* y, densify, CGLS iterate to roundoff."""
    pts = oracle.gen_grid(M, eps, dim) if kind == "grid" else oracle.gen_jitter(M, eps, 0.2, 7, dim)
    ptr = ref.gen_grid(M, eps, dim) if kind == "grid" else ref.gen_jitter(M, eps, 0.2, 7, dim)
    assert np.array_equal(pts, ptr)
    K = M * eps / 2 + 1
    mu = None
    if kind == "jitter":
        mu = oracle.voronoi(dim, pts, K)
        assert np.max(np.abs(mu - ref.voronoi(dim, pts, K))) <= 1e-13 * np.max(mu)
    a = oracle.Op(dim, p, J, pts, weights=mu, bandwidth=K)
    b = ref.Op(dim, p, J, pts, weights=mu, bandwidth=K)
    assert (a.rows, a.cols, a.uniform_fast) == (b.rows, b.cols, b.uniform_fast)
    for ax in range(dim):
        for fa, fb in zip(a.factors(ax), b.factors(ax)):
            assert (fa is None) == (fb is None)
            if fa is not None:
                assert np.array_equal(fa, fb)
    rng = np.random.default_rng(5)
    x = rng.standard_normal(a.cols) + 1j * rng.standard_normal(a.cols)
    y = rng.standard_normal(a.rows) + 1j * rng.standard_normal(a.rows)
    ef, ea = rel_error(a.forward(x), b.forward(x)), rel_error(a.adjoint(y), b.adjoint(y))
    data = b.forward(x)
    xa, sa = a.solve(data, max_iterations=25, tolerance=1e-300)
    xb, sb = b.solve(data, max_iterations=25, tolerance=1e-300)
    ec = rel_error(xa, xb)
    print(f"dim {dim} p {p} J {J} M {M} {kind}: T x {ef:.1e}, T* y {ea:.1e}, CGLS(25) {ec:.1e}")
    assert ef <= 1e-13 and ea <= 1e-13
    assert sa["iterations"] == sb["iterations"] == 25
    assert ec <= 1e-10
    if a.rows * a.cols <= 1 << 20:
        assert np.max(np.abs(a.densify() - b.densify())) <= 1e-15


@needs_ref
def test_oracle_matches_reference_transforms():
    rng = np.random.default_rng(11)
    for dim, N in [(1, (64, 0)), (2, (16, 12))]:
        M = 150
        pts = rng.uniform(-0.5, 0.5, M * dim)
        n = N[0] * (N[1] if dim == 2 else 1)
        g = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        y = rng.standard_normal(M) + 1j * rng.standard_normal(M)
        assert rel_error(oracle.ndft(dim, N, pts, g), ref.ndft(dim, N, pts, g)) <= 1e-14
        assert rel_error(oracle.ndft(dim, N, pts, y, adjoint=True), ref.ndft(dim, N, pts, y, adjoint=True)) <= 1e-14
        for sigma, w in [(2.0, 6), (1.5, 4), (1.25, 8)]:
            fa, na = oracle.nfft(dim, N, pts, g, sigma=sigma, w=w)
            fb, nb = ref.nfft(dim, N, pts, g, sigma=sigma, w=w)
            assert na[:dim] == nb[:dim]
            # sigma = 1.25 with 17 taps on a 20-point grid: the deconvolution amplifies the FFTs' roundoff
            tol = 1e-13 if sigma >= 1.5 else 1e-11
            assert rel_error(fa, fb) <= tol
            assert rel_error(oracle.nfft(dim, N, pts, y, adjoint=True, sigma=sigma, w=w)[0],
                             ref.nfft(dim, N, pts, y, adjoint=True, sigma=sigma, w=w)[0]) <= tol
    x = rng.standard_normal(48) + 1j * rng.standard_normal(48)
    for M, eps, N in [(96, 0.5, 48), (64, 1.0, 48), (200, 0.25, 48)]:
        assert rel_error(oracle.uniform_fft(x, M, eps, N), ref.uniform_fft(x, M, eps, N)) <= 1e-13
        yy = rng.standard_normal(M) + 1j * rng.standard_normal(M)
        assert rel_error(oracle.uniform_adjoint_fft(yy, eps, N), ref.uniform_adjoint_fft(yy, eps, N)) <= 1e-13
    for p in range(1, 9):
        assert np.array_equal(oracle.family_taps(p), ref.family_taps(p))
        for xi in (0.0, 0.37, -2.6, 11.25):
            assert abs(oracle.fourier_scaling(p, xi) - ref.fourier_scaling(p, xi)) <= 1e-16
        if p >= 2:
            for left in (True, False):
                assert np.array_equal(oracle.boundary_at_zero(p, left), ref.boundary_at_zero(p, left)) or \
                    rel_error(oracle.boundary_at_zero(p, left), ref.boundary_at_zero(p, left)) <= 1e-13
                for xi in (0.0, 0.41, -3.3):
                    assert rel_error(oracle.fourier_boundary(p, left, xi), ref.fourier_boundary(p, left, xi)) <= 1e-13
                Ua, Va = oracle.boundary_UV(p, left)
                Ub, Vb = ref.boundary_UV(p, left)
                assert np.array_equal(Ua, Ub) and np.array_equal(Va, Vb)


@needs_ref
def test_oracle_matches_reference_dyadic():
    for p in (1, 2, 4):
        ta, tb = oracle.scaling_dyadic(p, 5), ref.scaling_dyadic(p, 5)
        assert ta.support_begin == tb.support_begin and np.max(np.abs(ta.values - tb.values)) <= 1e-13
        if p >= 2:
            for la, lb in zip(oracle.boundary_dyadic(p, True, 4), ref.boundary_dyadic(p, True, 4)):
                assert np.max(np.abs(la.values - lb.values)) <= 1e-12
        rng = np.random.default_rng(p)
        c1 = rng.standard_normal(32)
        assert np.max(np.abs(oracle.weval(1, p, 5, 7, c1) - ref.weval(1, p, 5, 7, c1))) <= 1e-12
        c2 = rng.standard_normal(16 * 16)
        assert np.max(np.abs(oracle.weval(2, p, 4, 6, c2) - ref.weval(2, p, 4, 6, c2))) <= 1e-12


# ---------------------------------------------------------------- committed reference goldens
def golden(name):
    path = os.path.join(GOLD, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated")
    f = np.load(path, allow_pickle=False)
    return {k: f[k] for k in f.files}


@pytest.mark.parametrize("workload", ["c1", "c2"])
def test_oracle_reproduces_reference_golden_small(workload):
    """C1 / C2 at full size: the oracle against what the reference produced."""
    import bench
    fx = golden(f"ref_{workload}.npz")
    dim, p, J, c, mu, bw, sig = bench.problem_inputs(workload, 0, oracle)
    assert bench_sha(c) == str(fx["coords_sha"])
    op_u = oracle.Op(dim, p, J, c, bandwidth=bw)
    x_true, noise = bench.coeffs_and_noise(0, op_u.cols, op_u.rows, sig)
    data = op_u.forward(x_true) + noise
    op = oracle.Op(dim, p, J, c, weights=mu, bandwidth=bw)
    assert op.uniform_fast == bool(fx["uniform_fast"])
    im, ic = fx["m_idx"], fx["c_idx"]
    scale = lambda v, n: np.max(np.abs(v)) / float(n) * np.sqrt(len(v))  # noqa: E731
    eb = scale(data[im] - fx["b_val"], fx["b_norm"])
    ey = scale(op.forward(x_true)[im] - fx["y_val"], fx["y_norm"])
    ez = scale(op.adjoint(data)[ic] - fx["z_val"], fx["z_norm"])
    x, st = op.solve(data, max_iterations=int(fx["iters"]), tolerance=1e-300)
    ex = np.linalg.norm(x[ic] - fx["x_val"]) / np.linalg.norm(fx["x_val"])
    print(f"{workload}: oracle vs reference golden: b {eb:.1e}, T x {ey:.1e}, T* y {ez:.1e}, CGLS iterate {ex:.1e}")
    assert max(eb, ey, ez) <= 1e-12
    assert ex <= 1e-8


def bench_sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["c3", "c4", "c5_b0", "c5_b85", "c5_b170", "c5_b255"])
def test_oracle_fixture_agrees_with_reference_golden(name):
    """Config-size CGLS: the oracle iterate fixture (cgls_*.npz) against the
    sample of the REFERENCE's iterate (ref_*.npz) for the same seeded inputs."""
    rf = golden(f"ref_{name}.npz")
    of = golden(f"cgls_{name}.npz")
    assert str(rf["coords_sha"]) == str(of["coords_sha"]) and str(rf["weights_sha"]) == str(of["weights_sha"])
    ic = rf["c_idx"]
    e = np.linalg.norm(of["x"][ic] - rf["x_val"]) / np.linalg.norm(rf["x_val"])
    common, io, ir = np.intersect1d(of["b_idx"], rf["m_idx"], return_indices=True)
    eb = float(np.max(np.abs(of["b_val"][io] - rf["b_val"][ir])) / float(rf["b_norm"]) * np.sqrt(float(rf["m_idx"][-1] + 1)))
    assert common.size >= 64 and eb <= 1e-12
    sens = float(of["sens"])
    print(f"{name}: oracle fixture vs reference iterate {e:.3e} after {int(rf['iters'])} iterations "
          f"(oracle's own 1e-15-data sensitivity {sens:.2e}); b = T x_true + noise on {common.size} shared entries {eb:.1e}")
    # same algorithm, different FFT butterflies: roundoff-level differences amplified by CG
    assert e <= max(1e-8, 50 * sens)
