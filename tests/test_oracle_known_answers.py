"""Pins the CPU oracle (oracle/gs_oracle.cpp) against every known-answer relation
the reference's own tests hold for the T / T* / CGLS path, plus the reference's
stored golden vectors (60-digit edge moments, tests/family_fixtures.hpp).

Each test cites the reference test it restates (paths relative to
/root/reference/proj).  CPU only: runs in the no-GPU suite.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import OracleError, rel_error

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rc(n, rng):
    return rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)


def pts1(m, rng):
    return rng.uniform(-0.5, 0.4999, m)


# ---------------------------------------------------------------- scaling
def test_haar_and_db2_taps():  # test_scaling.cpp:13-38
    assert list(oracle.family_taps(1)) == [0.5, 0.5]
    s3 = math.sqrt(3.0)
    want = [(1 + s3) / 8, (3 + s3) / 8, (3 - s3) / 8, (1 - s3) / 8]
    assert np.max(np.abs(oracle.family_taps(2) - want)) < 1e-15
    t = oracle.family_taps(2)
    ks = np.arange(-1, 3)
    sign = np.where(ks % 2 == 0, 1.0, -1.0)
    assert abs(np.sum(sign * t)) < 1e-15 and abs(np.sum(sign * ks * t)) < 1e-15


def test_every_family_sums_to_one():  # test_scaling.cpp:40-48
    for p in range(1, 9):
        t = oracle.family_taps(p)
        assert t.size == 2 * p and abs(t.sum() - 1.0) < 1e-12


def test_boundary_staircase_support():  # test_scaling.cpp:56-74
    for p in range(2, 9):
        for left in (True, False):
            U, V = oracle.boundary_UV(p, left)
            for k in range(p):
                for c in range(2 * p - 1):
                    if c > 2 * k:
                        assert V[k, c] == 0.0
                assert V[k, 2 * k] != 0.0


# ---------------------------------------------------------------- fourier
def test_haar_closed_form():  # test_fourier.cpp:24-30
    assert oracle.fourier_scaling(1, 0.0) == 1.0
    assert abs(oracle.fourier_scaling(1, 0.5) - (-2j / math.pi)) < 1e-15
    assert abs(oracle.fourier_scaling(1, 1.0)) < 1e-15


def test_normalization_and_conjugate_symmetry():  # test_fourier.cpp:32-45
    rng = np.random.default_rng(11)
    for p in range(1, 9):
        assert abs(oracle.fourier_scaling(p, 0.0) - 1.0) < 1e-12
        for xi in rng.uniform(-20, 20, 25):
            a = oracle.fourier_scaling(p, xi)
            b = oracle.fourier_scaling(p, -xi)
            assert abs(b - np.conj(a)) < 1e-12


def test_product_truncation():  # test_fourier.cpp:47-56
    for p in (2, 5, 8):
        for xi in (0.3, 7.7, -31.4, 64.0, -64.0):
            assert abs(oracle.fourier_scaling(p, xi, 40) - oracle.fourier_scaling(p, xi, 50)) < 1e-10


def test_boundary_fixed_point_residual():  # test_fourier.cpp:86-101
    for p in range(2, 9):
        for left in (True, False):
            v = oracle.boundary_at_zero(p, left)
            U, V = oracle.boundary_UV(p, left)
            res = v - U @ v - V @ np.ones(2 * p - 1)
            assert np.linalg.norm(res) < 1e-12
    with pytest.raises(OracleError) as e:
        oracle.boundary_at_zero(1, True)
    assert e.value.code == 5


def test_boundary_recursion_stationary_and_converged():  # test_fourier.cpp:103-112
    fixed = oracle.boundary_at_zero(2, True)
    assert np.linalg.norm(fixed - oracle.fourier_boundary(2, True, 0.0, 17)) < 1e-13
    d30 = oracle.fourier_boundary(2, True, 0.3, 30)
    d40 = oracle.fourier_boundary(2, True, 0.3, 40)
    assert np.max(np.abs(d30 - d40)) < 1e-10


def _moments():
    raw = json.load(open(os.path.join(GOLDEN, "edge_moments.json")))
    return {int(p): {s: np.array([float.fromhex(v) for v in vals]) for s, vals in d.items()}
            for p, d in raw.items()}


def test_edge_transforms_at_zero_match_golden_moments():
    """family_fixtures.hpp (60-digit golden data): phihat_edge(0) = 0th moment."""
    for p, d in _moments().items():
        for side in ("left", "right"):
            v0 = oracle.boundary_at_zero(p, side == "left")
            assert np.max(np.abs(v0 - d[side][:p])) < 1e-14, (p, side)
            # the full recursion at xi = 0 reproduces it as well
            assert np.max(np.abs(oracle.fourier_boundary(p, side == "left", 0.0) - d[side][:p])) < 1e-13


def test_edge_transform_slopes_match_golden_first_moments():
    """d/dxi phihat_edge(0) = -2 pi i * (first moment), central difference."""
    h = 1e-5
    for p, d in _moments().items():
        if p > 6:
            continue
        for side in ("left", "right"):
            lt = side == "left"
            slope = (oracle.fourier_boundary(p, lt, h) - oracle.fourier_boundary(p, lt, -h)) / (2 * h)
            want = -2j * math.pi * d[side][p:2 * p]
            assert np.max(np.abs(slope - want)) < 1e-6 * (1 + np.max(np.abs(want))), (p, side)


# ---------------------------------------------------------------- nufft
def _ndft_np(N, pts, x):  # tests/oracles.hpp:25-34, opposite loop nesting
    k = np.arange(-N // 2, N // 2)
    return np.exp(-2j * np.pi * np.outer(pts, k)) @ x


def test_direct_ndft_and_pairing():  # test_nufft.cpp:15-60
    rng = np.random.default_rng(21)
    p = pts1(7, rng)
    imp = np.zeros(8, complex)
    imp[4] = 1
    assert np.max(np.abs(oracle.ndft(1, (8,), p, imp) - 1)) < 1e-14
    x = rc(8, rng)
    assert rel_error(oracle.ndft(1, (8,), p, x), _ndft_np(8, p, x)) < 1e-12
    p2 = rng.uniform(-0.5, 0.4999, 18)
    x2 = rc(24, rng)
    k0 = np.arange(-2, 2)
    k1 = np.arange(-3, 3)
    want = np.array([np.sum(x2.reshape(4, 6) * np.exp(-2j * np.pi * (np.add.outer(k0 * p2[2 * m], k1 * p2[2 * m + 1]))))
                     for m in range(9)])
    assert rel_error(oracle.ndft(2, (4, 6), p2, x2), want) < 1e-12
    with pytest.raises(OracleError):
        oracle.ndft(1, (8,), np.array([0.5]), x)
    y = rc(7, rng)
    lhs = np.vdot(y, oracle.ndft(1, (8,), p, x))
    rhs = np.vdot(oracle.ndft(1, (8,), p, y, adjoint=True), x)
    assert abs(lhs - rhs) / (np.linalg.norm(x) * np.linalg.norm(y)) < 1e-12


def test_plan_preconditions():  # test_nufft.cpp:62-74
    rng = np.random.default_rng(23)
    p = pts1(5, rng)
    _, nov = oracle.nfft(1, (16,), p, None)
    assert nov[0] == 32
    for args in [((16,), np.array([0.5]), 2.0, 6), ((15,), p, 2.0, 6), ((16,), p, 1.1, 6), ((16,), p, 2.0, 1)]:
        with pytest.raises(OracleError) as e:
            oracle.nfft(1, args[0], args[1], None, sigma=args[2], w=args[3])
        assert e.value.code == 5


def test_fast_tracks_direct_and_pairs():  # test_nufft.cpp:76-107, 174-185
    rng = np.random.default_rng(24)
    p = pts1(100, rng)
    imp = np.zeros(64, complex)
    imp[32] = 1
    assert np.max(np.abs(oracle.nfft(1, (64,), p, imp)[0] - 1)) < 1e-7
    x = rc(64, rng)
    y = rc(100, rng)
    fast = oracle.nfft(1, (64,), p, x)[0]
    assert rel_error(fast, oracle.ndft(1, (64,), p, x)) < 1e-7
    fadj = oracle.nfft(1, (64,), p, y, adjoint=True)[0]
    assert rel_error(fadj, oracle.ndft(1, (64,), p, y, adjoint=True)) < 1e-7
    assert abs(np.vdot(y, fast) - np.vdot(fadj, x)) / (np.linalg.norm(x) * np.linalg.norm(y)) < 1e-12
    p2 = rng.uniform(-0.5, 0.4999, 20)
    x2 = rc(64, rng)
    y2 = rc(10, rng)
    assert rel_error(oracle.nfft(2, (8, 8), p2, x2)[0], oracle.ndft(2, (8, 8), p2, x2)) < 1e-7
    assert rel_error(oracle.nfft(2, (8, 8), p2, y2, adjoint=True)[0],
                     oracle.ndft(2, (8, 8), p2, y2, adjoint=True)) < 1e-7
    for n, m in ((64, 1000), (256, 4096)):
        pp = pts1(m, rng)
        xx = rc(n, rng)
        assert rel_error(oracle.nfft(1, (n,), pp, xx)[0], oracle.ndft(1, (n,), pp, xx)) < 1e-7


def test_fast_linearity():  # test_nufft.cpp:109-122
    rng = np.random.default_rng(25)
    p = pts1(40, rng)
    a, b = rc(32, rng), rc(32, rng)
    al, be = 0.3 - 1.1j, -0.8 + 0.2j
    fa, fb, fc = (oracle.nfft(1, (32,), p, v)[0] for v in (a, b, al * a + be * b))
    assert np.max(np.abs(fc - al * fa - be * fb)) < 1e-12


def test_uniform_reduction_equals_direct():  # test_nufft.cpp:124-172
    rng = np.random.default_rng(26)
    assert np.all(oracle.uniform_fft(np.zeros(8), 16, 0.5, 8) == 0)
    x = rc(8, rng)
    pts = (np.arange(1, 17) - 9) / 16.0
    assert rel_error(oracle.uniform_fft(x, 16, 0.5, 8), oracle.ndft(1, (8,), pts, x)) < 1e-12
    x4 = rc(4, rng)
    p4 = (np.arange(1, 9) - 5) / 8.0
    want4 = np.exp(-2j * np.pi * np.outer(p4, np.arange(-2, 2))) @ x4
    assert rel_error(oracle.uniform_fft(x4, 8, 1.0, 8), want4) < 1e-12
    for args in ((x, 16, 0.3, 8), (x, 4, 0.5, 8)):
        with pytest.raises(OracleError):
            oracle.uniform_fft(*args)
    N, M, eps = 16, 40, 0.25
    pts = eps / N * (np.arange(1, M + 1) - 1.0 - M / 2.0)
    y = rc(M, rng)
    assert rel_error(oracle.uniform_adjoint_fft(y, eps, N), oracle.ndft(1, (16,), pts, y, adjoint=True)) < 1e-12


# ---------------------------------------------------------------- freq2wave
def _pairing(op, rng):
    x, y = rc(op.cols, rng), rc(op.rows, rng)
    return abs(np.vdot(y, op.forward(x)) - np.vdot(op.adjoint(y), x)) / (np.linalg.norm(x) * np.linalg.norm(y))


def test_haar_uniform_diagonal():  # test_freq2wave.cpp:41-53
    g = oracle.gen_grid(16, 0.5)
    op = oracle.Op(1, 1, 3, g)
    assert op.rows == 16 and op.cols == 8 and op.uniform_fast
    D, L, R = op.factors(0)
    assert L is None
    for m in range(16):
        assert abs(D[m] - 2 ** -1.5 * oracle.fourier_scaling(1, g[m] / 8)) < 1e-15


def test_densify_rows_match_formulas():  # test_freq2wave.cpp:55-101
    op = oracle.Op(1, 1, 2, np.array([0.0]))
    d = op.densify()
    assert d.shape == (1, 4) and np.max(np.abs(d - 0.5)) < 1e-15
    op = oracle.Op(1, 2, 3, np.array([1.7]))
    row = op.densify()[0]
    z = 1.7 / 8
    amp = 2 ** -1.5
    vl = oracle.fourier_boundary(2, True, z)
    vr = oracle.fourier_boundary(2, False, z)
    pl, pr = amp * np.exp(1j * np.pi * 1.7), amp * np.exp(-1j * np.pi * 1.7)
    assert abs(row[0] - pl * vl[0]) < 1e-13 and abs(row[1] - pl * vl[1]) < 1e-13
    assert abs(row[6] - pr * vr[1]) < 1e-13 and abs(row[7] - pr * vr[0]) < 1e-13
    for c in range(2, 6):
        want = amp * np.exp(-2j * np.pi * (c - 4) * z) * oracle.fourier_scaling(2, z)
        assert abs(row[c] - want) < 1e-13
    row2 = oracle.Op(2, 2, 3, np.array([1.7, -0.9])).densify()[0]
    rx = oracle.Op(1, 2, 3, np.array([1.7])).densify()[0]
    ry = oracle.Op(1, 2, 3, np.array([-0.9])).densify()[0]
    assert np.max(np.abs(row2 - np.outer(ry, rx).ravel())) < 1e-10


def test_construction_preconditions():  # test_freq2wave.cpp:103-120
    with pytest.raises(OracleError) as e:
        oracle.Op(1, 2, 1, oracle.gen_grid(8, 0.1))
    assert e.value.code == 5
    with pytest.raises(OracleError):
        oracle.Op(1, 1, 3, np.array([0.0, 4.0]))
    oracle.Op(1, 1, 3, np.array([0.0, -4.0]))
    with pytest.raises(OracleError):
        oracle.Op(1, 1, 3, np.array([0.0, 3.0]), bandwidth=2.0)


def test_1d_dense_section():  # test_freq2wave.cpp:122-153
    rng = np.random.default_rng(31)
    op = oracle.Op(1, 1, 3, oracle.gen_grid(16, 0.5))
    d = op.densify()
    assert np.all(op.forward(np.zeros(op.cols)) == 0) and np.all(op.adjoint(np.zeros(op.rows)) == 0)
    x, y = rc(op.cols, rng), rc(op.rows, rng)
    assert rel_error(op.forward(x), d @ x) < 1e-10
    assert rel_error(op.adjoint(y), d.conj().T @ y) < 1e-10
    op = oracle.Op(1, 4, 4, oracle.gen_jitter(64, 0.225, 0.05, 77))
    assert not op.uniform_fast
    x = rc(op.cols, rng)
    assert rel_error(op.forward(x), op.densify() @ x) < 1e-6


def test_2d_dense_section_and_haar():  # test_freq2wave.cpp:155-182
    rng = np.random.default_rng(33)
    for p, m in ((2, 20), (1, 18)):
        op = oracle.Op(2, p, 3, rng.uniform(-3.9, 3.9, 2 * m))
        d = op.densify()
        x, y = rc(op.cols, rng), rc(op.rows, rng)
        assert rel_error(op.forward(x), d @ x) < 1e-6
        assert rel_error(op.adjoint(y), d.conj().T @ y) < 1e-6


def test_pairing_1d_2d():  # test_freq2wave.cpp:184-194
    rng = np.random.default_rng(34)
    op1 = oracle.Op(1, 3, 4, rng.uniform(-7.9, 7.9, 60))
    op2 = oracle.Op(2, 2, 3, rng.uniform(-3.9, 3.9, 100))
    for _ in range(5):
        assert _pairing(op1, rng) < 1e-7 and _pairing(op2, rng) < 1e-7


def test_row_weights_exact():  # test_freq2wave.cpp:196-220
    rng = np.random.default_rng(35)
    for dim in (1, 2):
        c = rng.uniform(-3.9, 3.9, 12 * dim)
        w = rng.uniform(0.1, 2.0, 12)
        plain = oracle.Op(dim, 2, 3, c)
        wtd = oracle.Op(dim, 2, 3, c, weights=w)
        dp, dw = plain.densify(), wtd.densify()
        for m in range(12):
            # 1D rows are bit-identical; 2D rows (w*rx)*ry vs w*(rx*ry) differ by one rounding
            if dim == 1:
                assert np.all(dw[m] == math.sqrt(w[m]) * dp[m])
            else:
                assert np.max(np.abs(dw[m] - math.sqrt(w[m]) * dp[m])) <= 4e-16 * np.max(np.abs(dw[m]))
        x = rc(plain.cols, rng)
        assert np.max(np.abs(wtd.forward(x) - np.sqrt(w) * plain.forward(x))) < 1e-12


def test_uniform_vs_generic_and_periodized():  # test_freq2wave.cpp:222-253
    rng = np.random.default_rng(36)
    g = oracle.gen_grid(32, 0.25)
    fast = oracle.Op(1, 1, 4, g)
    gen = oracle.Op(1, 1, 4, g, allow_uniform=False)
    assert fast.uniform_fast and not gen.uniform_fast
    x, y = rc(16, rng), rc(32, rng)
    assert rel_error(fast.forward(x), gen.forward(x)) < 1e-7
    assert rel_error(fast.adjoint(y), gen.adjoint(y)) < 1e-7
    g = oracle.gen_grid(128, 0.5)
    with pytest.raises(OracleError):
        oracle.Op(1, 1, 4, g)
    op = oracle.Op(1, 1, 4, g, bandwidth=64.0)
    x = rc(op.cols, rng)
    d = op.densify()
    assert rel_error(op.forward(x), d @ x) < 1e-10
    gen = oracle.Op(1, 1, 4, g, bandwidth=64.0, allow_uniform=False)
    assert rel_error(gen.forward(x), d @ x) < 1e-6


def test_linearity_and_shape_errors():  # test_freq2wave.cpp:255-294
    rng = np.random.default_rng(38)
    op = oracle.Op(2, 3, 3, rng.uniform(-3.9, 3.9, 30))
    al, be = 0.6 - 0.4j, -1.2 + 0.9j
    a, b = rc(op.cols, rng), rc(op.cols, rng)
    assert np.max(np.abs(op.forward(al * a + be * b) - al * op.forward(a) - be * op.forward(b))) < 1e-12
    u, v = rc(op.rows, rng), rc(op.rows, rng)
    assert np.max(np.abs(op.adjoint(al * u + be * v) - al * op.adjoint(u) - be * op.adjoint(v))) < 1e-12
    op = oracle.Op(1, 1, 3, oracle.gen_grid(16, 0.5))
    with pytest.raises(OracleError) as e:
        op.densify(64)
    assert e.value.code == 5
    for f in (op.forward, op.adjoint):
        with pytest.raises(OracleError) as e:
            f(np.zeros(7, complex))
        assert e.value.code == 4


# ---------------------------------------------------------------- solver
def test_in_span_recovery():  # test_solver.cpp:19-33
    rng = np.random.default_rng(51)
    op = oracle.Op(1, 4, 5, oracle.gen_grid(128, 0.25))
    truth = rc(op.cols, rng)
    x, st = op.solve(op.forward(truth))
    assert st["converged"] and st["iterations"] <= 50
    assert np.linalg.norm(x - truth) / np.linalg.norm(truth) < 1e-6
    assert st["history"].size == st["iterations"] + 1


def test_lsq_residual_monotone():  # test_solver.cpp:35-54
    rng = np.random.default_rng(57)
    op = oracle.Op(1, 2, 4, oracle.gen_grid(32, 0.5))
    data = rc(op.rows, rng)
    prev = None
    for cap in range(1, 13):
        x, _ = op.solve(data, max_iterations=cap, tolerance=1e-300)
        lsq = np.linalg.norm(data - op.forward(x))
        if prev is not None:
            assert lsq <= prev * (1 + 1e-12)
        prev = lsq


def test_zero_data_and_dense_oracle():  # test_solver.cpp:56-82
    op = oracle.Op(1, 1, 3, oracle.gen_grid(16, 0.5))
    x, st = op.solve(np.zeros(16))
    assert st["converged"] and st["iterations"] == 0 and np.all(x == 0)
    rng = np.random.default_rng(52)
    data = rc(16, rng)
    x, st = op.solve(data)
    assert st["converged"]
    d = op.densify()
    expect = np.linalg.solve(d.conj().T @ d, d.conj().T @ data)
    assert np.linalg.norm(x - expect) / np.linalg.norm(expect) < 1e-8


def test_row_permutation_invariance():  # test_solver.cpp:84-114
    rng = np.random.default_rng(53)
    pts = oracle.gen_jitter(48, 0.3, 0.07, 99)
    data = oracle.Op(1, 2, 4, pts).forward(rc(16, rng)) + (1e-3 - 1e-3j)
    perm = rng.permutation(48)
    a = oracle.Op(1, 2, 4, pts).solve(data)[0]
    b = oracle.Op(1, 2, 4, pts[perm]).solve(data[perm])[0]
    assert np.linalg.norm(a - b) / np.linalg.norm(a) < 1e-10


def test_weighted_solve():  # test_solver.cpp:116-129
    rng = np.random.default_rng(54)
    pts = oracle.gen_jitter(40, 0.4, 0.09, 7)
    mu = oracle.voronoi(1, pts, 8.0)
    op = oracle.Op(1, 2, 4, pts, weights=mu)
    truth = rc(op.cols, rng)
    raw = oracle.Op(1, 2, 4, pts).forward(truth)
    x, st = op.solve(raw)
    assert st["converged"] and np.linalg.norm(x - truth) / np.linalg.norm(truth) < 1e-6


def test_nonconvergence_initial_guess_validation():  # test_solver.cpp:131-188
    rng = np.random.default_rng(55)
    op = oracle.Op(1, 2, 4, oracle.gen_grid(64, 0.25))
    x, st = op.solve(rc(64, rng), max_iterations=1)
    assert not st["converged"] and st["iterations"] == 1 and st["history"].size == 2
    op = oracle.Op(1, 1, 4, oracle.gen_grid(32, 0.5))
    truth = rc(op.cols, rng)
    x, st = op.solve(op.forward(truth), x0=truth)
    assert st["converged"] and st["iterations"] == 0 and np.all(x == truth)
    op = oracle.Op(1, 1, 3, oracle.gen_grid(16, 0.5))
    with pytest.raises(OracleError) as e:
        op.solve(np.zeros(15))
    assert e.value.code == 4
    with pytest.raises(OracleError) as e:
        op.solve(np.ones(16), tolerance=0.0)
    assert e.value.code == 5


# ---------------------------------------------------------------- patterns / weights
def test_patterns():  # test_patterns.cpp:14-80
    g = oracle.gen_grid(128, 0.5)
    assert g[0] == -32.0 and g[127] == 31.5
    t = oracle.gen_grid(4, 0.5, 2)
    assert t[0] == -1.0 and t[1] == -1.0 and t[3] == -0.5
    assert np.all(oracle.gen_jitter(64, 0.5, 0.0, 123) == oracle.gen_grid(64, 0.5))
    assert np.all(oracle.gen_jitter(64, 0.5, 0.1, 42) == oracle.gen_jitter(64, 0.5, 0.1, 42))
    big = oracle.gen_jitter(5463, 0.5, 0.125, 7)
    assert np.all(np.diff(big) > 0)
    plane = oracle.gen_jitter(9, 0.5, 0.1, 3, 2)
    assert np.max(np.abs(plane - oracle.gen_grid(9, 0.5, 2))) <= 0.1
    s = oracle.gen_spiral(1, 4.0, 2.0).reshape(-1, 2)
    assert np.max(np.abs(s[0])) < 1e-15 and abs(s[1, 1] - 0.5) < 1e-14 and abs(s[2, 0] + 1.0) < 1e-14
    big = oracle.gen_spiral(27, 27681.0 / 27.0, 16.0).reshape(-1, 2)
    assert big.shape[0] == 27681 and np.max(np.hypot(big[:, 0], big[:, 1])) <= 16 + 1e-12
    with pytest.raises(OracleError):
        oracle.gen_jitter(8, 0.5, 0.25, 1)


def test_voronoi_small():  # test_weights.cpp (1D exact cells, 2D total area)
    mu = oracle.voronoi(1, np.array([-1.0, 0.0, 2.0]), 3.0)
    assert np.allclose(mu, [2.5, 1.5, 2.0])
    pts = oracle.gen_jitter(6, 0.5, 0.1, 5, 2)
    mu = oracle.voronoi(2, pts, 1.6)
    assert abs(mu.sum() - 3.2 * 3.2) < 1e-12
