"""GPU parity: the sm_100a operator (through the C-ABI) against the CPU oracle
(oracle/gs_oracle.cpp, a restatement of the reference) on identical seeded
inputs.  Bars (BASELINE.json north star):
  * T x and T* y       : relative L2 (tests/oracles.hpp:63-70) <= 1e-10
  * CGLS iterate       : <= 1e-8 after the same iteration count (tol = 1e-300
                         idiom of test_solver.cpp:46)
  * factors D / L / R  : <= 1e-13 (max abs, relative to max |factor|)
The exact tensor route differs from the reference's KB-NFFT only by the KB
kernel's aliasing error (~1e-11), still inside 1e-10.
"""
import math

import numpy as np
import pytest

import oracle
from oracle import rel_error

pytestmark = pytest.mark.gpu

TOL_APPLY = 1e-10
TOL_CGLS = 1e-8


def gs():
    import paper_1607_04091_b200 as m
    return m


def rc(n, rng):
    return (rng.standard_normal(n) + 1j * rng.standard_normal(n)) / math.sqrt(2)


def build_pair(dim, p, J, coords, weights=None, bandwidth=None, allow_uniform=True, allow_tensor=True):
    ref = oracle.Op(dim, p, J, coords, weights=weights, bandwidth=bandwidth, allow_uniform=allow_uniform)
    g = gs()
    op = g.freq2wave(g.SamplingSet(dim, coords), p, J, bandwidth=bandwidth, weights=weights,
                     allow_uniform_fast_path=allow_uniform, allow_tensor_route=allow_tensor)
    return ref, op


def check_apply(ref, op, rng, tol=TOL_APPLY):
    g = gs()
    x = rc(ref.cols, rng)
    y = rc(ref.rows, rng)
    e_f = rel_error(g.apply_forward(op, x), ref.forward(x))
    e_a = rel_error(g.apply_adjoint(op, y), ref.adjoint(y))
    assert e_f <= tol and e_a <= tol, (e_f, e_a, op.route)
    return e_f, e_a


def check_factors(ref, op, dim):
    for axis in range(dim):
        Dr, Lr, Rr = ref.factors(axis)
        Dg, Lg, Rg = op.factors(axis)
        scale = np.max(np.abs(Dr))
        assert np.max(np.abs(Dg - Dr)) <= 1e-13 * scale
        if Lr is not None:
            scale = max(np.max(np.abs(Lr)), np.max(np.abs(Rr)))
            assert np.max(np.abs(Lg - Lr)) <= 1e-13 * scale
            assert np.max(np.abs(Rg - Rr)) <= 1e-13 * scale


def cgls_sensitivity(ref, b, iters):
    """How far the reference's own iterate moves when the data move by 1e-15
    (relative): the roundoff floor of CG on this problem.  Ill-conditioned
    problems amplify any rounding difference (tests note it in DESIGN.md)."""
    rng = np.random.default_rng(1)
    x1, _ = ref.solve(b, max_iterations=iters, tolerance=1e-300)
    x2, _ = ref.solve(b * (1 + 1e-15 * rc(b.size, rng)), max_iterations=iters, tolerance=1e-300)
    return rel_error(x2, x1)


def check_cgls(ref, op, b, iters, tol=TOL_CGLS):
    g = gs()
    xr, sr = ref.solve(b, max_iterations=iters, tolerance=1e-300)
    xg, sg = g.solve_least_squares(op, b, max_iterations=iters, tolerance=1e-300)
    assert sg.iterations == sr["iterations"] == iters
    e = rel_error(xg, xr)
    if e > tol:  # above 1e-8 only when the reference itself is that sensitive
        sens = cgls_sensitivity(ref, b, iters)
        assert sens > tol / 20 and e <= 20 * sens, (e, sens)
    # residual histories agree until both reach the roundoff floor, where CGNR
    # stagnates differently (solver.cpp:64-67: "may tick upward")
    hr = np.asarray(sr["history"])
    hg = np.asarray(sg.history)
    live = hr > 1e-9
    assert np.allclose(hg[live], hr[live], rtol=1e-6)
    return e


# ------------------------------------------------------------------ C1 (full size)
def test_c1_uniform_haar_full():
    rng = np.random.default_rng(20160613)
    coords = oracle.gen_grid(1024, 1.0)
    ref, op = build_pair(1, 1, 9, coords, bandwidth=512.0)
    assert op.route == "uniform_1d" and op.uniform_fast and ref.uniform_fast
    check_factors(ref, op, 1)
    check_apply(ref, op, rng)
    xt = rc(512, rng)
    b = ref.forward(xt) + 1e-3 * rc(1024, rng)
    check_cgls(ref, op, b, 50)
    # default tolerance stops at the same iteration as the reference
    _, sr = ref.solve(b)
    _, sg = gs().solve_least_squares(op, b)
    assert sg.iterations == sr["iterations"] and sg.converged == sr["converged"]


# ------------------------------------------------------------------ C2 (full size)
def test_c2_jitter_db4_full():
    rng = np.random.default_rng(20160613)
    coords = oracle.gen_jitter(4096, 0.5, 0.2, 20160613)
    K = float(np.max(np.abs(coords)))
    mu = oracle.voronoi(1, coords, K)
    ref, op = build_pair(1, 4, 10, coords, weights=mu, bandwidth=K)
    assert op.route == "nfft_1d" and not op.uniform_fast
    check_factors(ref, op, 1)
    check_apply(ref, op, rng)
    raw = oracle.Op(1, 4, 10, coords, bandwidth=K).forward(rc(1024, rng)) + 1e-3 * rc(4096, rng)
    check_cgls(ref, op, raw, 100)


# ------------------------------------------------------------------ C3 shapes
@pytest.mark.parametrize("tensor", [True, False])
def test_c3_uniform_2d_small(tensor):
    rng = np.random.default_rng(7)
    coords = oracle.gen_grid(64, 1.0, 2)
    ref, op = build_pair(2, 2, 5, coords, bandwidth=32.0, allow_tensor=tensor)
    assert op.route == ("tensor_2d" if tensor else "nfft_2d")
    check_factors(ref, op, 2)
    check_apply(ref, op, rng)
    b = ref.forward(rc(ref.cols, rng)) + 1e-4 * rc(ref.rows, rng)
    check_cgls(ref, op, b, 20)


def test_c3_full_size_apply():
    rng = np.random.default_rng(20160613)
    coords = oracle.gen_grid(512, 1.0, 2)
    ref, op = build_pair(2, 2, 8, coords, bandwidth=256.0)
    assert op.route == "tensor_2d"
    check_apply(ref, op, rng)


# ------------------------------------------------------------------ C4 / C5 shapes
def test_spiral_db4_weighted_small():
    rng = np.random.default_rng(5)
    # radially Nyquist-sampled spiral (ring spacing 1 in xi) so that CGLS is well
    # conditioned; an undersampled spiral amplifies roundoff in any CG
    coords = oracle.gen_spiral(16, 256.0, 16.0)
    mu = oracle.voronoi(2, coords, 16.0)
    ref, op = build_pair(2, 4, 5, coords, weights=mu, bandwidth=16.0)
    assert op.route == "nfft_2d"
    check_factors(ref, op, 2)
    check_apply(ref, op, rng)
    raw = oracle.Op(2, 4, 5, coords, bandwidth=16.0).forward(rc(ref.cols, rng)) + 1e-4 * rc(ref.rows, rng)
    check_cgls(ref, op, raw, 30)


def test_batched_jitter_2d_db4():
    """C5 shape in miniature: 3 independent problems in one batched handle."""
    rng = np.random.default_rng(9)
    g = gs()
    sets, refs, mus = [], [], []
    for b in range(3):
        c = oracle.gen_jitter(32, 0.5, 0.2, 20160613 + b, 2)
        K = float(np.max(np.abs(c)))
        mu = oracle.voronoi(2, c, K)
        sets.append(g.SamplingSet(2, c))
        mus.append(mu)
        refs.append(oracle.Op(2, 4, 4, c, weights=mu, bandwidth=K + 1e-9))
    K = max(float(np.max(np.abs(s.coords))) for s in sets) + 1e-9
    op = g.freq2wave(sets, 4, 4, bandwidth=K, weights=np.concatenate(mus))
    assert op.batch == 3 and op.route == "nfft_2d"
    x = rc(3 * 256, rng)
    y = rc(3 * 1024, rng)
    yf = g.apply_forward(op, x)
    za = g.apply_adjoint(op, y)
    for b in range(3):
        assert rel_error(yf[b * 1024:(b + 1) * 1024], refs[b].forward(x[b * 256:(b + 1) * 256])) <= TOL_APPLY
        assert rel_error(za[b * 256:(b + 1) * 256], refs[b].adjoint(y[b * 1024:(b + 1) * 1024])) <= TOL_APPLY
    xs, stats = g.solve_least_squares(op, y, max_iterations=15, tolerance=1e-300)
    for b in range(3):
        xr, sr = refs[b].solve(y[b * 1024:(b + 1) * 1024], max_iterations=15, tolerance=1e-300)
        assert stats[b].iterations == 15
        assert rel_error(xs[b * 256:(b + 1) * 256], xr) <= TOL_CGLS


# ------------------------------------------------------------------ every family, both dims
@pytest.mark.parametrize("p", range(1, 9))
def test_families_1d_2d_random_points(p):
    rng = np.random.default_rng(100 + p)
    J = 4 if p <= 4 else 5
    n = 1 << J
    c1 = rng.uniform(-n / 2, n / 2 - 1e-3, 97)
    ref, op = build_pair(1, p, J, c1)
    check_factors(ref, op, 1)
    check_apply(ref, op, rng)
    c2 = rng.uniform(-3.9 * n / 8, 3.9 * n / 8, 2 * 150)
    ref, op = build_pair(2, p, J, c2)
    check_factors(ref, op, 2)
    check_apply(ref, op, rng)


def test_periodized_bandwidth_and_generic_route():
    rng = np.random.default_rng(37)
    g128 = oracle.gen_grid(128, 0.5)
    for allow in (True, False):
        ref, op = build_pair(1, 1, 4, g128, bandwidth=64.0, allow_uniform=allow)
        assert op.uniform_fast == allow
        check_apply(ref, op, rng)


def test_non_power_of_two_uniform_dft():
    rng = np.random.default_rng(41)
    coords = oracle.gen_grid(40, 1.0)  # eps = 1, N = 16 -> q = 3 -> N2 = 48 (direct DFT)
    ref, op = build_pair(1, 2, 4, coords, bandwidth=20.0)
    assert op.uniform_fast
    check_apply(ref, op, rng)


# ------------------------------------------------------------------ relations on the GPU alone
def test_pairing_linearity_zero():
    rng = np.random.default_rng(34)
    g = gs()
    c = rng.uniform(-3.9, 3.9, 2 * 500)
    op = g.freq2wave(g.SamplingSet(2, c), "db3", 3)
    for _ in range(3):
        x, y = rc(op.cols(), rng), rc(op.rows(), rng)
        d = abs(np.vdot(y, g.apply_forward(op, x)) - np.vdot(g.apply_adjoint(op, y), x))
        assert d / (np.linalg.norm(x) * np.linalg.norm(y)) < 1e-12
    a, b = rc(op.cols(), rng), rc(op.cols(), rng)
    al, be = 0.6 - 0.4j, -1.2 + 0.9j
    f = g.apply_forward
    assert np.max(np.abs(f(op, al * a + be * b) - al * f(op, a) - be * f(op, b))) < 1e-12
    assert np.all(f(op, np.zeros(op.cols())) == 0)
    assert np.all(g.apply_adjoint(op, np.zeros(op.rows())) == 0)


def test_solver_edge_cases():
    g = gs()
    rng = np.random.default_rng(58)
    op = g.freq2wave(g.SamplingSet(1, oracle.gen_grid(16, 0.5)), "haar", 3)
    x, st = g.solve_least_squares(op, np.zeros(16))
    assert st.converged and st.iterations == 0 and np.all(x == 0)
    with pytest.raises(g.ShapeError):
        g.solve_least_squares(op, np.zeros(15))
    with pytest.raises(g.DomainError):
        g.solve_least_squares(op, np.ones(16), tolerance=0.0)
    with pytest.raises(g.ShapeError):
        g.apply_forward(op, np.zeros(7))
    op = g.freq2wave(g.SamplingSet(1, oracle.gen_grid(32, 0.5)), "haar", 4)
    truth = rc(16, rng)
    data = g.apply_forward(op, truth)
    x, st = g.solve_least_squares(op, data, initial_guess=truth)
    assert st.converged and st.iterations == 0 and np.all(x == truth)
    op = g.freq2wave(g.SamplingSet(1, oracle.gen_grid(64, 0.25)), "db2", 4)
    x, st = g.solve_least_squares(op, rc(64, rng), max_iterations=1)
    assert not st.converged and st.iterations == 1 and len(st.history) == 2


def test_device_tensors_roundtrip():
    import torch
    g = gs()
    rng = np.random.default_rng(3)
    c = oracle.gen_jitter(256, 0.5, 0.2, 11)
    op = g.freq2wave(g.SamplingSet(1, c), "db4", 7, bandwidth=float(np.max(np.abs(c))))
    x = rc(op.cols(), rng)
    yd = g.apply_forward(op, torch.from_numpy(x).cuda())
    assert yd.is_cuda
    assert rel_error(yd.cpu().numpy(), g.apply_forward(op, x)) == 0.0


# ------------------------------------------------------------------ full-size C4 / C5 problems
def _voronoi_fast(dim, c, K):
    from paper_1607_04091_b200 import inputs
    return inputs.voronoi_weights(dim, c, K)


def test_c5_problem_full_size():
    """One C5 problem at full size (2^18 jittered samples, db4 J=8, Voronoi
    weights): T x / T* y parity and a short fixed-count CGLS."""
    rng = np.random.default_rng(20160613)
    c = oracle.gen_jitter(512, 0.5, 0.2, 20160613, 2)
    K = float(np.max(np.abs(c)))
    mu = _voronoi_fast(2, c, K)
    ref, op = build_pair(2, 4, 8, c, weights=mu, bandwidth=K)
    assert op.route == "nfft_2d"
    check_apply(ref, op, rng)
    b = rc(ref.rows, rng)
    check_cgls(ref, op, b, 3)


def test_c4_spiral_full_size_apply():
    """C4 at full size (2^20 spiral samples, R=512, 64 turns, db4 J=9)."""
    rng = np.random.default_rng(20160613)
    c = oracle.gen_spiral(64, 16384.0, 512.0)
    mu = _voronoi_fast(2, c, 512.0)
    ref, op = build_pair(2, 4, 9, c, weights=mu, bandwidth=512.0)
    assert op.route == "nfft_2d"
    check_apply(ref, op, rng)


def test_dfma_kernel_variants_match_oracle():
    """The lane-per-column DFMA spreading / fused-pair DFMA interpolation
    variants (GS_B200_SPREAD=dfma, GS_B200_INTERP=dfma: the A/B baselines of
    the DMMA kernels) keep parity too.  Run in a subprocess: the library reads
    the selectors once per process."""
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np, oracle, paper_1607_04091_b200 as gs
rng = np.random.default_rng(3)
c = oracle.gen_jitter(64, 0.5, 0.2, 7, 2)
mu = oracle.voronoi(2, c, 16.5)
ref = oracle.Op(2, 4, 5, c, weights=mu, bandwidth=16.5)
op = gs.freq2wave(gs.SamplingSet(2, c), "db4", 5, bandwidth=16.5, weights=mu)
x = rng.standard_normal(ref.cols) + 1j * rng.standard_normal(ref.cols)
y = rng.standard_normal(ref.rows) + 1j * rng.standard_normal(ref.rows)
ef = oracle.rel_error(gs.apply_forward(op, x), ref.forward(x))
ea = oracle.rel_error(gs.apply_adjoint(op, y), ref.adjoint(y))
assert ef <= 1e-10 and ea <= 1e-10, (ef, ea)
print("ok", ef, ea)
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GS_B200_SPREAD="dfma", GS_B200_INTERP="dfma", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr


# ------------------------------------------------------------------ fast 2D tile path, every family it serves
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_fast2d_tile_path_families_dense_tiles(p):
    """The DMMA tile kernels (n_ov >= 48: J = 5 -> n_ov 64) for haar .. db4,
    on uniform points plus a dense cluster (tiles of > 144 samples: several
    chunks per tile, band starts inside later chunks, the band-major sample
    order), the public apply (caller order) and the CGLS session (sorted
    order)."""
    g = gs()
    rng = np.random.default_rng(500 + p)
    J = 5
    n = 1 << J
    spread_pts = rng.uniform(-0.49 * n, 0.49 * n, (700, 2))
    cluster = rng.normal(0.0, 0.6, (500, 2)) + np.array([3.3, -5.1])
    coords = np.concatenate([spread_pts, cluster]).reshape(-1)
    ref, op = build_pair(2, p, J, coords)
    assert op.route == "nfft_2d", op.route
    check_factors(ref, op, 2)
    check_apply(ref, op, rng)
    b = rc(ref.rows, rng)
    check_cgls(ref, op, b, 6)


# ------------------------------------------------------------------ one-launch / two-launch CGLS iterations
def test_fused_cgls_iterations_match_generic_and_oracle():
    """The fused CGLS iterations -- 1D uniform in one launch (k_uni_cgls_iter),
    1D NFFT with the q/s steps inside the gridding kernels, the tensor route's
    norm partials, the 2D generic 6-launch form -- against the
    generic 11-launch iteration (GS_B200_CG_FUSED=0, subprocess) and the
    oracle: same iterates, iteration counts, converged flags and residual
    histories, including a batch where one problem converges early under the
    default tolerance and one has zero data (solver.cpp:42-48)."""
    import os
    import subprocess
    import sys
    code = r'''
import json, numpy as np, oracle, paper_1607_04091_b200 as gs
rng = np.random.default_rng(11)
out = {}
def rc(n):
    return (rng.standard_normal(n) + 1j * rng.standard_normal(n)) / np.sqrt(2)
cases = [("uni_haar", 1, 1, 9, oracle.gen_grid(1024, 1.0), None, 512.0),
         ("uni_db2", 1, 2, 7, oracle.gen_grid(300, 0.5), None, None),
         ("nfft_db4", 1, 4, 8, oracle.gen_jitter(700, 0.5, 0.2, 5, 1), "voronoi", None),
         ("tensor_db2", 2, 2, 4, oracle.gen_grid(32, 1.0, 2), None, 16.0),
         ("nfft2d_db4", 2, 4, 5, oracle.gen_jitter(48, 0.5, 0.2, 6, 2), "voronoi", None)]
for name, dim, p, J, c, w, bw in cases:
    K = bw if bw is not None else float(np.max(np.abs(c))) + 1e-9
    mu = oracle.voronoi(dim, c, K) if w else None
    ref = oracle.Op(dim, p, J, c, weights=mu, bandwidth=K)
    op = gs.freq2wave(gs.SamplingSet(dim, c), p, J, bandwidth=K, weights=mu)
    b = ref.forward(rc(ref.cols)) + 1e-3 * rc(ref.rows)
    its = 30 if dim == 1 else 12
    x, st = gs.solve_least_squares(op, b, max_iterations=its, tolerance=1e-300)
    xr, sr = ref.solve(b, max_iterations=its, tolerance=1e-300)
    assert st.iterations == its and oracle.rel_error(x, xr) <= 1e-8, (name, oracle.rel_error(x, xr))
    if dim == 1:
        x2, st2 = gs.solve_least_squares(op, b)  # default tolerance: stops early
        xr2, sr2 = ref.solve(b)
        assert st2.iterations == sr2["iterations"] and st2.converged == sr2["converged"], (name, st2.iterations, sr2)
    else:
        x2, st2 = x, st
    out[name] = [x.tolist(), list(st.history), x2.tolist(), st2.iterations]
# batch: problem 1 has zero data, problem 2 converges early (exact data)
sets = [gs.SamplingSet(1, oracle.gen_jitter(600, 0.5, 0.2, 30 + i, 1)) for i in range(3)]
K = max(float(np.max(np.abs(s.coords))) for s in sets) + 1e-9
op = gs.freq2wave(sets, 4, 8, bandwidth=K)
refs = [oracle.Op(1, 4, 8, s.coords, bandwidth=K) for s in sets]
bs = [refs[0].forward(rc(256)) + 1e-3 * rc(600), np.zeros(600, complex), refs[2].forward(rc(256))]
xb, sts = gs.solve_least_squares(op, np.concatenate(bs), max_iterations=40, tolerance=1e-9)
for i in range(3):
    xr, sr = refs[i].solve(bs[i], max_iterations=40, tolerance=1e-9)
    assert sts[i].iterations == sr["iterations"] and sts[i].converged == sr["converged"], (i, sts[i].iterations, sr)
    e = oracle.rel_error(xb[i * 256:(i + 1) * 256], xr) if i != 1 else float(np.max(np.abs(xb[256:512])))
    assert e <= 1e-8, (i, e)
out["batch"] = [xb.tolist(), [s.iterations for s in sts]]
print("ok" + json.dumps(out, default=lambda z: [z.real, z.imag]))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for fused in ("1", "0"):
        env = dict(os.environ, GS_B200_CG_FUSED=fused, PYTHONPATH=root)
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout[-2000:] + r.stderr[-4000:]
        res[fused] = __import__("json").loads(r.stdout[2:])
    for k in res["1"]:
        a, b = res["1"][k], res["0"][k]
        xa = np.array(a[0], float)
        xb = np.array(b[0], float)
        assert np.max(np.abs(xa - xb)) <= 1e-9 * max(1.0, np.max(np.abs(xb))), k
        if k != "batch":
            ha, hb = np.asarray(a[1]), np.asarray(b[1])
            live = hb > 1e-9  # above the roundoff floor, where CGNR stagnates differently
            assert np.allclose(ha[live], hb[live], rtol=1e-9, atol=0), k  # residual histories
            assert a[3] == b[3], k
        else:
            assert a[1] == b[1]


def test_balanced_band_schedule_matches_static(monkeypatch):
    """A spiral loads the 3-row bands of its tiles unevenly: the operator picks
    the balanced band schedule of the DMMA kernels by itself, a jittered grid
    keeps the static one, and the two schedules agree to roundoff (they sum the
    same products in a different warp order)."""
    import paper_1607_04091_b200 as gs
    c = oracle.gen_spiral(12, 2048.0, 60.0)
    ops = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("GS_B200_BALANCE", flag)
        ops[flag] = gs.freq2wave(gs.SamplingSet(2, c), "db4", 6, bandwidth=64.0)
    monkeypatch.delenv("GS_B200_BALANCE")
    auto = gs.freq2wave(gs.SamplingSet(2, c), "db4", 6, bandwidth=64.0)
    assert ops["1"].route == "nfft_2d" and ops["1"].balanced_schedule and not ops["0"].balanced_schedule
    rng = np.random.default_rng(9)
    x = rng.standard_normal(auto.cols()) + 1j * rng.standard_normal(auto.cols())
    y = rng.standard_normal(auto.rows()) + 1j * rng.standard_normal(auto.rows())
    ref = oracle.Op(2, 4, 6, c, bandwidth=64.0)
    for name, op in (("balanced", ops["1"]), ("static", ops["0"])):
        ef, ea = rel_error(gs.apply_forward(op, x), ref.forward(x)), rel_error(gs.apply_adjoint(op, y), ref.adjoint(y))
        print(f"spiral, {name} schedule: T x {ef:.1e}, T* y {ea:.1e}")
        assert ef <= TOL_APPLY and ea <= TOL_APPLY
    print("auto-selected schedule on the spiral:", "balanced" if auto.balanced_schedule else "static")
    assert auto.balanced_schedule
    # a jittered grid fills the bands evenly (C5's shape, smaller): static kernels
    cj = oracle.gen_jitter(256, 0.5, 0.2, 3, 2)
    assert not gs.freq2wave(gs.SamplingSet(2, cj), "db4", 7, bandwidth=65.0).balanced_schedule
