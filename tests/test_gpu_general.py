"""Option generality of the operator (VERDICT r1 item 6 / ADVICE): values the
fused config kernels do not take run through the general routes
(csrc/general_route.cuh: device NfftPlan + general-length FFT, composed as
freq2wave.cpp:215-387) and match the oracle -- the reference algorithm at
the same options -- at the T.x bar (1e-10) and the CGLS bar (1e-8).

  * sigma = 1.25 / 1.5 (non-power-of-two oversampled grids), 1D and 2D
  * kernel half-width w = 8 (17 taps; the fused kernels stop at 15)
  * J = 12 non-uniform 1D (n_ov = 8192 > 4096)
  * uniform 1D with DFT lengths 6144 (non-power-of-two) and 16384 (> 8192)
"""
import math

import numpy as np
import pytest

import oracle
from oracle import rel_error

pytestmark = pytest.mark.gpu


def gs():
    import paper_1607_04091_b200 as m
    return m


def rc(n, rng):
    return (rng.standard_normal(n) + 1j * rng.standard_normal(n)) / math.sqrt(2)


def check(dim, p, J, coords, iters=20, weights=None, bandwidth=None, **opt):
    g = gs()
    rng = np.random.default_rng(len(coords) + p)
    ref = oracle.Op(dim, p, J, coords, weights=weights, bandwidth=bandwidth, **opt)
    op = g.freq2wave(g.SamplingSet(dim, coords), p, J, weights=weights, bandwidth=bandwidth, **opt)
    x, y = rc(ref.cols, rng), rc(ref.rows, rng)
    ef = rel_error(g.apply_forward(op, x), ref.forward(x))
    ea = rel_error(g.apply_adjoint(op, y), ref.adjoint(y))
    b = ref.forward(rc(ref.cols, rng)) + 1e-3 * rc(ref.rows, rng)
    xr, _ = ref.solve(b, max_iterations=iters, tolerance=1e-300)
    xg, sg = g.solve_least_squares(op, b, max_iterations=iters, tolerance=1e-300)
    ec = rel_error(xg, xr)
    print(f"general dim={dim} p={p} J={J} M={ref.rows} {opt}: route {op.route} n_over {op.n_over} "
          f"fwd {ef:.2e} adj {ea:.2e} cgls({iters}) {ec:.2e}")
    assert ef <= 1e-10 and ea <= 1e-10 and ec <= 1e-8 and sg.iterations == iters
    D, L, R = ref.factors(0)
    Dg, Lg, Rg = op.factors(0)
    assert np.max(np.abs(Dg - D)) <= 1e-13 * np.max(np.abs(D))
    return op


@pytest.mark.parametrize("sigma,w", [(1.25, 6), (1.5, 6), (2.0, 8), (1.5, 4)])
def test_1d_nfft_options(sigma, w):
    c = oracle.gen_jitter(1000, 0.25, 0.05, 11)
    K = float(np.max(np.abs(c)))
    mu = oracle.voronoi(1, c, K)
    op = check(1, 4, 7, c, weights=mu, bandwidth=K, sigma=sigma, w=w)
    assert op.route == "nfft_1d"


def test_1d_nfft_large_scale():
    """J = 12 non-uniform (n_ov 8192, four-step FFT): ADVICE r1 (jitter1d --scale 2)."""
    c = oracle.gen_jitter(9000, 0.5, 0.2, 3)
    K = float(np.max(np.abs(c)))
    op = check(1, 3, 12, c, bandwidth=K, iters=10)
    assert op.n_over == 8192


@pytest.mark.parametrize("sigma,w,p", [(1.5, 6, 4), (1.25, 6, 2), (2.0, 8, 3), (1.25, 5, 1)])
def test_2d_nfft_options(sigma, w, p):
    rng = np.random.default_rng(5)
    c = rng.uniform(-15.9, 15.9, 2 * 700)
    check(2, p, 5, c, sigma=sigma, w=w)


@pytest.mark.parametrize("J,M,p", [(11, 5000, 2), (13, 16384, 1)])
def test_1d_uniform_any_length(J, M, p):
    """Uniform grids whose DFT length q N / eps is 6144 (non-power-of-two) or
    16384 (> 8192): the reference's uniform_fast route at any length."""
    n = 1 << J
    c = oracle.gen_grid(M, 1.0)
    op = check(1, p, J, c, bandwidth=float(M) / 2, iters=10)
    assert op.route == "uniform_1d" and op.uniform_fast
