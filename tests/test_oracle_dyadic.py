"""Pins the oracle's restatement of dyadic.cpp (the dyadic
cascades and weval) to every known answer the reference's own tests hold for
it: test_dyadic.cpp (haar indicator, partition of unity, unit integral,
boundary dilation equations, weval constants / shifted tables / validation /
linearity / 2D separability, polynomial reproduction from the 60-digit edge
moments) and acceptance.cpp criteria 7-8 (including the cross-check of the hot
path's boundary Fourier transforms against quadrature of the dyadic tables)."""
import json
import math
import os

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def binom(n, k):
    acc = 1.0
    for i in range(k):
        acc = acc * (n - i) / (i + 1)
    return acc


def scaling_moments(p, count):  # test_dyadic.cpp:26-40
    taps = oracle.family_taps(p)
    mu = [1.0]
    for r in range(1, count):
        acc = 0.0
        for j in range(r):
            ps = sum(taps[k + p - 1] * float(k) ** (r - j) for k in range(-p + 1, p + 1))
            acc += binom(r, j) * ps * mu[j]
        mu.append(acc / (2.0 ** r - 1.0))
    return mu


def pou_error(t, p):  # test_dyadic.cpp:42-53
    n = 1 << t.resolution
    worst = 0.0
    for i in range(n):
        s = sum(t.value_at(i - (k << t.resolution)) for k in range(-p, p + 1))
        worst = max(worst, abs(s - 1.0))
    return worst


def test_haar_table_is_the_indicator():
    t = oracle.scaling_dyadic(1, 3)
    assert t.values.size == 9 and np.all(t.values[:8] == 1.0) and t.values[8] == 0.0


def test_db2_partition_of_unity_and_unit_integral():
    t = oracle.scaling_dyadic(2, 8)
    assert pou_error(t, 2) < 1e-8
    assert abs(np.sum(t.values) * 2.0 ** -8 - 1.0) < 1e-6


@pytest.mark.parametrize("p", range(2, 9))
def test_partition_of_unity_db2_to_db8(p):
    assert pou_error(oracle.scaling_dyadic(p, 10), p) < 1e-6


def dilation_residual(p, left, R):
    """boundary tables against their dilation equations (test_dyadic.cpp:84-113)"""
    U, V = oracle.boundary_UV(p, left)  # H / sqrt2, h / sqrt2 (scaling.cpp:71-72)
    H, h = U * math.sqrt(2.0), V * math.sqrt(2.0)
    interior = oracle.scaling_dyadic(p, R)
    tabs = oracle.boundary_dyadic(p, left, R)
    worst = 0.0
    for k in range(p):
        t = tabs[k]
        for i in range(0, t.values.size, 2):
            nx = (t.support_begin << R) + i
            rhs = sum(H[k, l] * tabs[l].value_at(2 * nx) for l in range(p))
            for m in range(p, p + 2 * k + 1):
                arg = 2 * nx - (m << R) if left else 2 * nx + ((m + 1) << R)
                rhs += h[k, m - p] * interior.value_at(arg)
            worst = max(worst, abs(t.values[i] / math.sqrt(2.0) - rhs))
    return worst


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("left", [True, False])
def test_boundary_tables_satisfy_dilation_equations(p, left):
    assert dilation_residual(p, left, 6) < 1e-10


def test_boundary_tables_reject_haar():
    with pytest.raises(oracle.OracleError):
        oracle.boundary_dyadic(1, True, 6)


def test_weval_constant_haar_is_one():
    J, R = 4, 8
    ev = oracle.weval(1, 1, J, R, np.full(1 << J, 2.0 ** (-0.5 * J)))
    assert ev.size == (1 << R) + 1
    assert np.allclose(ev[:-1], 1.0, rtol=1e-14, atol=0) and ev[-1] == 0.0


def test_weval_unit_interior_coefficient_is_the_shifted_table():
    J, R, col = 5, 10, 13
    c = np.zeros(1 << J)
    c[col] = 1.0
    ev = oracle.weval(1, 2, J, R, c)
    t = oracle.scaling_dyadic(2, R - J)
    amp = 2.0 ** (0.5 * J)
    want = np.array([amp * t.value_at(i - (col << (R - J))) for i in range(ev.size)])
    assert np.max(np.abs(ev - want)) < 1e-12


def test_weval_validation_and_zero():
    c = np.zeros(32)
    for args, code in [((5, 4, c), 5), ((4, 8, c), 4), ((1, 4, np.zeros(2)), 5)]:
        with pytest.raises(oracle.OracleError) as e:
            oracle.weval(1, 2, *args)
        assert e.value.code == code
    assert np.all(oracle.weval(1, 2, 5, 8, c) == 0.0)


def test_weval_is_linear():
    J, R = 4, 7
    rng = np.random.default_rng(5)
    a, b = rng.uniform(-1, 1, 1 << J), rng.uniform(-1, 1, 1 << J)
    ea, eb, ec = (oracle.weval(1, 3, J, R, v) for v in (a, b, 0.7 * a - 1.3 * b))
    assert np.max(np.abs(ec - 0.7 * ea + 1.3 * eb)) < 1e-12


def test_weval_2d_constant_haar_and_separability():
    J, R = 3, 6
    n, g = 1 << J, (1 << R) + 1
    e = oracle.weval(2, 1, J, R, np.full(n * n, 2.0 ** -J)).reshape(g, g)
    assert np.allclose(e[:-1, :-1], 1.0, rtol=1e-13, atol=0)
    rng = np.random.default_rng(9)
    ax, by = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    outer = np.outer(by, ax).ravel()  # outer[j n + i] = ax[i] by[j]
    e2 = oracle.weval(2, 2, J, R, outer).reshape(g, g)
    ex, ey = oracle.weval(1, 2, J, R, ax), oracle.weval(1, 2, J, R, by)
    assert np.max(np.abs(e2 - np.outer(ey, ex))) < 1e-12
    assert np.all(oracle.weval(2, 2, J, R, np.zeros(n * n)) == 0.0)


@pytest.mark.parametrize("p", [2, 4, 6, 8])
def test_edge_corrected_basis_reproduces_polynomials(p):
    """test_dyadic.cpp:215-266 with the 60-digit edge moments (tests/golden)."""
    fx = json.load(open(os.path.join(ROOT, "tests", "golden", "edge_moments.json")))[str(p)]
    left = [float.fromhex(v) for v in fx["left"]]
    right = [float.fromhex(v) for v in fx["right"]]
    J = 4
    R, n, half = J + 3, 1 << J, 2.0 ** (J - 1)
    mu = scaling_moments(p, p)
    for r in range(p):
        amp = 2.0 ** (-0.5 * J) * 2.0 ** (-J * r)
        c = np.zeros(n)
        for col in range(n):
            acc = 0.0
            if col < p:
                acc = sum(binom(r, s) * (-half) ** (r - s) * left[s * p + col] for s in range(r + 1))
            elif col >= n - p:
                j = n - 1 - col
                acc = sum(binom(r, s) * half ** (r - s) * right[s * p + j] for s in range(r + 1))
            else:
                for s in range(r + 1):
                    mom = sum(binom(s, j) * mu[j] * float(col) ** (s - j) for j in range(s + 1))
                    acc += binom(r, s) * (-half) ** (r - s) * mom
            c[col] = amp * acc
        ev = oracle.weval(1, p, J, R, c)
        x = np.arange(ev.size) * 2.0 ** -R - 0.5
        assert np.max(np.abs(ev - x ** r)) < 1e-8


def fourier_quadrature(t, xi):  # tests/oracles.hpp:52-61
    h = 2.0 ** -t.resolution
    w = np.ones(t.values.size)
    w[0] = w[-1] = 0.5
    x = t.support_begin + h * np.arange(t.values.size)
    return np.sum(w * t.values * np.exp(-2j * np.pi * xi * x)) * h


@pytest.mark.parametrize("p", [2, 4, 8])
def test_boundary_fourier_matches_quadrature_of_dyadic_tables(p):
    """acceptance.cpp criterion 8: the hot path's edge transforms
    (fourier_boundary) against trapezoid quadrature of the R = 14 tables."""
    worst = 0.0
    for left in (True, False):
        tabs = oracle.boundary_dyadic(p, left, 14)
        for xi in (-8.0, -2.3, 0.4, 1.7, 8.0):
            v = oracle.fourier_boundary(p, left, xi)
            for k in range(p):
                worst = max(worst, abs(v[k] - fourier_quadrature(tabs[k], xi)))
    assert worst < 1e-6
