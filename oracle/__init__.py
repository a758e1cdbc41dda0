"""ctypes front-end of the CPU oracle (oracle/gs_oracle.cpp).

TEST INFRASTRUCTURE ONLY.  Importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs -- never from the product
package ``paper_1607_04091_b200`` (which fails loudly without its CUDA library).

Every call restates the reference C++ path cited in gs_oracle.cpp; complex
vectors are numpy complex128 (layout-identical to std::complex<double>).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libgs_oracle.so")
_lib = None

_dp = C.POINTER(C.c_double)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build():
    subprocess.check_call(["make", "-s", "-C", _HERE])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        L.orc_wrap_half_open.restype = C.c_double
        L.orc_wrap_half_open.argtypes = [C.c_double]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _chk(rc):
    if rc != 0:
        raise OracleError(rc, lib().orc_last_error().decode())


def _c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Op:
    """Freq2WaveOp restated (freq2wave.cpp:86-193)."""

    def __init__(self, dim, p, J, coords, weights=None, bandwidth=None, sigma=2.0, w=6,
                 depth=30, terms=48, allow_uniform=True):
        coords = _f64(coords).ravel()
        self.dim = dim
        M = coords.size // dim
        wts = None if weights is None else _f64(weights)
        h = C.c_void_p()
        bw = 0.0 if bandwidth is None else float(bandwidth)
        _chk(lib().orc_op_create(C.c_int(dim), C.c_int(p), C.c_int(J), C.c_longlong(M), _p(coords),
                                 _p(wts), C.c_int(bandwidth is not None), C.c_double(bw),
                                 C.c_double(sigma), C.c_int(w), C.c_int(depth), C.c_int(terms),
                                 C.c_int(1 if allow_uniform else 0), C.byref(h)))
        self._h = h
        rows, cols, uf, eps = C.c_longlong(), C.c_longlong(), C.c_int(), C.c_double()
        lib().orc_op_info(h, C.byref(rows), C.byref(cols), C.byref(uf), C.byref(eps))
        self.rows, self.cols = rows.value, cols.value
        self.uniform_fast = bool(uf.value)
        self.uniform_epsilon = eps.value
        self.p = p
        self.J = J

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_op_destroy(self._h)
            self._h = None

    def forward(self, x):
        x = _c128(x)
        y = np.empty(self.rows, np.complex128)
        _chk(lib().orc_forward_n(self._h, _p(x.view(np.float64)), C.c_longlong(x.size), _p(y.view(np.float64))))
        return y

    def adjoint(self, y):
        y = _c128(y)
        z = np.empty(self.cols, np.complex128)
        _chk(lib().orc_adjoint_n(self._h, _p(y.view(np.float64)), C.c_longlong(y.size), _p(z.view(np.float64))))
        return z

    def factors(self, axis=0):
        D = np.empty(self.rows, np.complex128)
        L = R = None
        if self.p >= 2:
            L = np.empty(self.rows * self.p, np.complex128)
            R = np.empty(self.rows * self.p, np.complex128)
        lib().orc_factors(self._h, C.c_int(axis), _p(D.view(np.float64)),
                          _p(L.view(np.float64)) if L is not None else None,
                          _p(R.view(np.float64)) if R is not None else None)
        if L is not None:  # Eigen col-major M x p
            L = L.reshape(self.p, self.rows).T.copy()
            R = R.reshape(self.p, self.rows).T.copy()
        return D, L, R

    def densify(self, cap=1 << 24):
        out = np.empty((self.rows, self.cols), np.complex128)
        _chk(lib().orc_densify(self._h, C.c_longlong(cap), _p(out.view(np.float64))))
        return out

    def solve(self, b, x0=None, max_iterations=0, tolerance=1e-10):
        b = _c128(b)
        x = np.empty(self.cols, np.complex128)
        it, res, conv, hl = C.c_int(), C.c_double(), C.c_int(), C.c_int()
        mi = max_iterations if max_iterations > 0 else 2 * self.cols
        hist = np.empty(mi + 2, np.float64)
        x0a = None if x0 is None else _c128(x0)
        _chk(lib().orc_solve(self._h, _p(b.view(np.float64)), C.c_longlong(b.size), _p(x0a.view(np.float64)) if x0a is not None else None,
                             C.c_int(max_iterations), C.c_double(tolerance), _p(x.view(np.float64)),
                             C.byref(it), C.byref(res), C.byref(conv), _p(hist), C.byref(hl)))
        return x, dict(iterations=it.value, residual=res.value, converged=bool(conv.value),
                       history=hist[:hl.value].copy())


def fourier_scaling(p, xi, terms=48):
    out = np.empty(2)
    _chk(lib().orc_fourier_scaling(C.c_int(p), C.c_double(xi), C.c_int(terms), _p(out)))
    return complex(out[0], out[1])


def fourier_boundary(p, left, xi, depth=30, terms=48):
    out = np.empty(p, np.complex128)
    _chk(lib().orc_fourier_boundary(C.c_int(p), C.c_int(1 if left else 0), C.c_double(xi), C.c_int(depth),
                                    C.c_int(terms), _p(out.view(np.float64))))
    return out


def boundary_at_zero(p, left):
    out = np.empty(p, np.complex128)
    _chk(lib().orc_boundary_at_zero(C.c_int(p), C.c_int(1 if left else 0), _p(out.view(np.float64))))
    return out


def boundary_UV(p, left):
    U = np.empty((p, p))
    V = np.empty((p, 2 * p - 1))
    _chk(lib().orc_boundary_UV(C.c_int(p), C.c_int(1 if left else 0), _p(U), _p(V)))
    return U, V


def family_taps(p):
    out = np.empty(2 * p)
    _chk(lib().orc_family_taps(C.c_int(p), _p(out)))
    return out


def ndft(dim, N, pts, data, adjoint=False):
    pts = _f64(pts).ravel()
    M = pts.size // dim
    data = _c128(data)
    N0, N1 = (N[0], N[1] if dim == 2 else 0)
    out = np.empty(M if not adjoint else N0 * (N1 if dim == 2 else 1), np.complex128)
    _chk(lib().orc_ndft(C.c_int(int(adjoint)), C.c_int(dim), C.c_int(N0), C.c_int(N1), C.c_longlong(M), _p(pts),
                        _p(data.view(np.float64)), _p(out.view(np.float64))))
    return out


def nfft(dim, N, pts, data, adjoint=False, sigma=2.0, w=6):
    pts = _f64(pts).ravel()
    M = pts.size // dim
    N0, N1 = (N[0], N[1] if dim == 2 else 0)
    nov = (C.c_int * 2)()
    out = np.empty(M if not adjoint else N0 * (N1 if dim == 2 else 1), np.complex128)
    d = None if data is None else _c128(data)
    _chk(lib().orc_nfft(C.c_int(int(adjoint)), C.c_int(dim), C.c_int(N0), C.c_int(N1), C.c_longlong(M), _p(pts),
                        C.c_double(sigma), C.c_int(w), _p(d.view(np.float64)) if d is not None else None,
                        _p(out.view(np.float64)), nov))
    return out, (nov[0], nov[1])


def kb_weights(pts, n_over, N, sigma=2.0, w=6):
    pts = _f64(pts)
    M = pts.size
    base = np.empty(M, np.int64)
    wts = np.empty((M, 2 * w + 1))
    dec = np.empty(N)
    _chk(lib().orc_kb_weights(C.c_int(1), C.c_longlong(M), _p(pts), C.c_int(n_over), C.c_double(sigma), C.c_int(w),
                              base.ctypes.data_as(C.POINTER(C.c_longlong)), _p(wts), _p(dec), C.c_int(N)))
    return base, wts, dec


def uniform_fft(x, M, eps, N):
    x = _c128(x)
    out = np.empty(M, np.complex128)
    _chk(lib().orc_uniform(C.c_int(0), _p(x.view(np.float64)), C.c_longlong(x.size), C.c_longlong(M),
                           C.c_double(eps), C.c_longlong(N), _p(out.view(np.float64))))
    return out


def uniform_adjoint_fft(y, eps, N):
    y = _c128(y)
    out = np.empty(N, np.complex128)
    _chk(lib().orc_uniform(C.c_int(1), _p(y.view(np.float64)), C.c_longlong(y.size), C.c_longlong(y.size),
                           C.c_double(eps), C.c_longlong(N), _p(out.view(np.float64))))
    return out


def gen_grid(M, eps, dim=1):
    out = np.empty(M * (M * 2 if dim == 2 else 1))
    _chk(lib().orc_gen_grid(C.c_longlong(M), C.c_double(eps), C.c_int(dim), _p(out)))
    return out


def gen_jitter(M, eps, eta, seed, dim=1):
    out = np.empty(M * (M * 2 if dim == 2 else 1))
    _chk(lib().orc_gen_jitter(C.c_longlong(M), C.c_double(eps), C.c_double(eta), C.c_ulonglong(seed),
                              C.c_int(dim), _p(out)))
    return out


def gen_spiral(turns, ppt, K):
    count = int(round(turns * ppt))
    out = np.empty(2 * count)
    _chk(lib().orc_gen_spiral(C.c_int(turns), C.c_double(ppt), C.c_double(K), _p(out)))
    return out


def voronoi(dim, coords, K):
    coords = _f64(coords).ravel()
    M = coords.size // dim
    mu = np.empty(M)
    _chk(lib().orc_voronoi(C.c_int(dim), C.c_longlong(M), _p(coords), C.c_double(K), _p(mu)))
    return mu


def voronoi_fast(dim, coords, K, threads=0):
    """Bucketed exact Voronoi (same cells as voronoi(), roundoff-level areas) for
    point sets beyond the reference's O(M^2) loop; harness only."""
    c = _f64(coords).ravel()
    mu = np.empty(c.size // dim)
    n = threads or (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1))
    _chk(lib().orc_voronoi_fast(C.c_int(dim), C.c_longlong(mu.size), _p(c), C.c_double(K), _p(mu), C.c_int(n)))
    return mu


class FTable:
    """dyadic.hpp FunctionTable: samples at support_begin + i / 2^R."""

    def __init__(self, R, support_begin, values):
        self.resolution, self.support_begin, self.values = R, support_begin, values

    def value_at(self, numerator):
        idx = numerator - (self.support_begin << self.resolution)
        return float(self.values[idx]) if 0 <= idx < self.values.size else 0.0


def _table(call):
    n, sb = C.c_longlong(0), C.c_longlong(0)
    _chk(call(None, C.byref(n), C.byref(sb)))
    out = np.empty(n.value)
    _chk(call(_p(out), C.byref(n), C.byref(sb)))
    return out, sb.value


def scaling_dyadic(p, R):
    v, sb = _table(lambda o, n, s: lib().orc_scaling_dyadic(C.c_int(p), C.c_int(R), o, n, s))
    return FTable(R, sb, v)


def boundary_dyadic(p, left, R):
    out = []
    for k in range(p):
        v, sb = _table(lambda o, n, s, k=k: lib().orc_boundary_dyadic(C.c_int(p), C.c_int(int(left)), C.c_int(R),
                                                                      C.c_int(k), o, n, s))
        out.append(FTable(R, sb, v))
    return out


def weval(dim, p, J, R, coeffs):
    coeffs = _f64(coeffs).ravel()
    g = (1 << R) + 1
    out = np.empty(g if dim == 1 else g * g)
    _chk(lib().orc_weval(C.c_int(dim), C.c_int(p), C.c_int(J), C.c_int(R), _p(coeffs), C.c_longlong(coeffs.size),
                         _p(out)))
    return out


def wrap_half_open(z):
    return lib().orc_wrap_half_open(float(z))


def rel_error(got, want):
    """tests/oracles.hpp:63-70 -- the parity metric."""
    got = np.asarray(got)
    want = np.asarray(want)
    num = float(np.sum(np.abs(got - want) ** 2))
    den = float(np.sum(np.abs(want) ** 2))
    return math.sqrt(num) if den == 0.0 else math.sqrt(num / den)
