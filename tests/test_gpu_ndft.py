"""GPU direct NDFT (a14: ndft_forward / ndft_adjoint, nufft.cpp:74-132) through
the C-ABI, against the oracle's restatement of the reference loops.

Mirrors the reference's tests/test_nufft.cpp:15-60 (impulse, zero, the
double-loop oracle at 1e-12, the pairing identity, the range check) and adds
config-size cases (C2's 1024 modes x 4096 points; a 2D 64x64 grid) plus the
exact-NDFT operator route (GS_ROUTE_NDFT_1D) on C2 against the oracle's
KB-NFFT operator (bar 1e-10: the KB aliasing error is ~1e-11)."""
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
    return rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)


def pts(m, rng, dim=1):
    return rng.uniform(-0.5, 0.4999, m * dim)


def test_direct_forward_impulse_zero_and_oracle():  # test_nufft.cpp:15-42
    rng = np.random.default_rng(21)
    p = pts(7, rng)
    imp = np.zeros(8, complex)
    imp[4] = 1.0
    assert np.max(np.abs(gs().ndft_forward(1, [8], p, imp) - 1.0)) < 1e-14
    assert np.all(gs().ndft_forward(1, [8], p, np.zeros(8, complex)) == 0)
    x = rc(8, rng)
    assert rel_error(gs().ndft_forward(1, [8], p, x), oracle.ndft(1, [8, 0], p, x)) < 1e-12
    p2 = pts(9, rng, 2)
    x2 = rc(24, rng)
    assert rel_error(gs().ndft_forward(2, [4, 6], p2, x2), oracle.ndft(2, [4, 6], p2, x2)) < 1e-12
    with pytest.raises(gs().DomainError):
        gs().ndft_forward(1, [8], np.array([0.5]), x)
    with pytest.raises(gs().ShapeError):
        gs().ndft_forward(1, [8], p, rc(7, rng))


def test_direct_adjoint_trivial_and_pairing():  # test_nufft.cpp:44-60
    g = gs()
    z = g.ndft_adjoint(1, [8], np.array([0.0]), np.array([1.0 + 0j]))
    assert np.max(np.abs(z - 1.0)) < 1e-14
    rng = np.random.default_rng(22)
    p = pts(11, rng)
    assert np.all(g.ndft_adjoint(1, [8], p, np.zeros(11, complex)) == 0)
    x, y = rc(8, rng), rc(11, rng)
    lhs = np.vdot(y, g.ndft_forward(1, [8], p, x))
    rhs = np.vdot(g.ndft_adjoint(1, [8], p, y), x)
    assert abs(lhs - rhs) / (np.linalg.norm(x) * np.linalg.norm(y)) < 1e-12


@pytest.mark.parametrize("dim,N,M", [(1, [1024], 4096), (1, [1000], 3001), (2, [64, 64], 5000), (2, [30, 18], 777)])
def test_direct_config_sizes_vs_oracle(dim, N, M):
    """C2 shape (1024 modes, 4096 points), a non-multiple-of-16 length and 2D grids."""
    rng = np.random.default_rng(23 + M)
    p = pts(M, rng, dim)
    nm = N[0] * (N[1] if dim == 2 else 1)
    NN = N if dim == 2 else [N[0], 0]
    x, y = rc(nm, rng), rc(M, rng)
    ef = rel_error(gs().ndft_forward(dim, N, p, x), oracle.ndft(dim, NN, p, x))
    ea = rel_error(gs().ndft_adjoint(dim, N, p, y), oracle.ndft(dim, NN, p, y, adjoint=True))
    print(f"ndft dim={dim} N={N} M={M}: forward {ef:.2e} adjoint {ea:.2e}")
    assert ef < 1e-12 and ea < 1e-12


def test_direct_odd_length_semantics():
    """k = -N/2 .. N/2-1 with C++ integer division (nufft.cpp:81): odd lengths
    leave their last index out exactly as the reference loop does."""
    rng = np.random.default_rng(29)
    p = pts(50, rng)
    x, y = rc(7, rng), rc(50, rng)
    assert rel_error(gs().ndft_forward(1, [7], p, x), oracle.ndft(1, [7, 0], p, x)) < 1e-12
    z = gs().ndft_adjoint(1, [7], p, y)
    zr = oracle.ndft(1, [7, 0], p, y, adjoint=True)
    assert rel_error(z, zr) < 1e-12 and z[-1] == 0


def test_direct_device_tensors():
    import torch
    g = gs()
    rng = np.random.default_rng(31)
    p = pts(300, rng)
    x = rc(64, rng)
    yd = g.ndft_forward(1, [64], torch.from_numpy(p).cuda(), torch.from_numpy(x).cuda())
    assert rel_error(yd.cpu().numpy(), oracle.ndft(1, [64, 0], p, x)) < 1e-12


def test_exact_ndft_route_c2():
    """C2 on the exact NDFT route: T / T* against the oracle's KB operator
    (<= 1e-10; the difference is the KB error) and CGLS after the config's 100
    iterations (<= 1e-8)."""
    g = gs()
    rng = np.random.default_rng(20160613)
    c = oracle.gen_jitter(4096, 0.5, 0.2, 20160613)
    K = float(np.max(np.abs(c)))
    mu = oracle.voronoi(1, c, K)
    ref = oracle.Op(1, 4, 10, c, weights=mu, bandwidth=K)
    op = g.freq2wave(g.SamplingSet(1, c), "db4", 10, bandwidth=K, weights=mu, exact_ndft=True)
    assert op.route == "ndft_1d" and not op.uniform_fast
    x = rc(1024, rng)
    y = rc(4096, rng)
    ef = rel_error(g.apply_forward(op, x), ref.forward(x))
    ea = rel_error(g.apply_adjoint(op, y), ref.adjoint(y))
    # exact vs exact: the route's T against a dense NDFT section through the oracle's factors
    D, L, R = ref.factors(0)
    zeta = np.array([oracle.wrap_half_open(v / 1024.0) for v in c])
    xt = x.copy()
    xt[:4] = 0
    xt[-4:] = 0
    core = oracle.ndft(1, [1024, 0], zeta, xt)
    exact = D * core + L @ x[:4] + R @ x[-4:]
    ee = rel_error(g.apply_forward(op, x), exact)
    print(f"ndft route C2: vs KB oracle fwd {ef:.2e} adj {ea:.2e}; vs exact section {ee:.2e}")
    assert ef <= 1e-10 and ea <= 1e-10 and ee <= 1e-12
    raw = oracle.Op(1, 4, 10, c, bandwidth=K).forward(rc(1024, rng)) + 1e-3 * rc(4096, rng)
    xr, _ = ref.solve(raw, max_iterations=100, tolerance=1e-300)
    xg, sg = g.solve_least_squares(op, raw, max_iterations=100, tolerance=1e-300)
    e = rel_error(xg, xr)
    print(f"ndft route C2 CGLS(100) vs KB oracle: {e:.2e}")
    assert sg.iterations == 100 and e <= 1e-8
