"""B200-native generalized sampling: the T / T* / CGLS hot path.

Python mirror of the reference C++ operator API (namespace ``gs``,
/root/reference/proj/include/gs/{freq2wave,solver,error}.hpp) over the C-ABI
in ``include/gs_b200.h`` (``libgs_b200.so``, sm_100a).  Same names, argument
meaning and error classes:

    op = freq2wave(SamplingSet(dim, coords), "db4", J, bandwidth=K, weights=mu)
    y  = apply_forward(op, x)        # freq2wave.hpp:61
    z  = apply_adjoint(op, y)        # freq2wave.hpp:64
    x, stats = solve_least_squares(op, b, SolveOptions(...))   # solver.hpp:29-31

Vectors are numpy complex128 arrays (host) or torch complex128 CUDA tensors
(device; no copies).  There is no CPU fallback: without the CUDA library or a
GPU every call raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = [
    "Error", "UsageError", "FileFormatError", "ShapeError", "DomainError", "NumericalError", "CudaError",
    "SamplingSet", "Freq2WaveOptions", "Freq2WaveOp", "SolveOptions", "SolveStats",
    "freq2wave", "apply_forward", "apply_adjoint", "solve_least_squares", "CglsSession",
    "ndft_forward", "ndft_adjoint", "NfftPlan", "plan_nfft", "nfft_forward", "nfft_adjoint",
    "uniform_ndft_fft", "uniform_ndft_adjoint_fft", "family_p", "ROUTES", "lib_path", "load_library",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.environ.get("GS_B200_LIB") or os.path.join(_HERE, "libgs_b200.so")  # env: A/B builds only
_lib = None


def lib_path():
    return _LIB


# ------------------------------------------------------------------ errors (error.hpp:9-41)
class Error(RuntimeError):
    exit_code = 1

    def __init__(self, msg):
        super().__init__(msg)


class UsageError(Error):
    exit_code = 2


class FileFormatError(Error):
    exit_code = 3


class ShapeError(Error):
    exit_code = 4


class DomainError(Error):
    exit_code = 5


class NumericalError(Error):
    exit_code = 6


class CudaError(Error):
    exit_code = 7


_ERRS = {2: UsageError, 3: FileFormatError, 4: ShapeError, 5: DomainError, 6: NumericalError, 7: CudaError}
ROUTES = {1: "uniform_1d", 2: "nfft_1d", 3: "nfft_2d", 4: "tensor_2d", 5: "ndft_1d"}


class _Desc(C.Structure):
    _fields_ = [("dim", C.c_int), ("family_p", C.c_int), ("J", C.c_int), ("M", C.c_int64), ("batch", C.c_int),
                ("coords", C.POINTER(C.c_double)), ("weights", C.POINTER(C.c_double)), ("bandwidth", C.c_double),
                ("sigma", C.c_double), ("w", C.c_int), ("boundary_depth", C.c_int), ("product_terms", C.c_int),
                ("allow_uniform_fast_path", C.c_int), ("allow_tensor_route", C.c_int), ("device", C.c_int),
                ("exact_ndft", C.c_int)]


class _Info(C.Structure):
    _fields_ = [("dim", C.c_int), ("family_p", C.c_int), ("J", C.c_int), ("batch", C.c_int), ("route", C.c_int),
                ("rows", C.c_int64), ("cols", C.c_int64), ("uniform_fast", C.c_int), ("uniform_epsilon", C.c_double),
                ("weighted", C.c_int), ("n_over", C.c_int), ("device_bytes", C.c_int64)]


class _Stats(C.Structure):
    _fields_ = [("iterations", C.c_int), ("residual", C.c_double), ("converged", C.c_int)]


def load_library():
    """Load libgs_b200.so (built by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB):
        raise CudaError(f"CUDA library {_LIB} not built (run __graft_entry__.build()); no CPU fallback exists")
    L = C.CDLL(_LIB)
    L.gs_last_error.restype = C.c_char_p
    vp = C.c_void_p
    dp = C.POINTER(C.c_double)
    L.gs_op_create.argtypes = [C.POINTER(_Desc), C.POINTER(vp)]
    L.gs_op_destroy.argtypes = [vp]
    L.gs_op_info.argtypes = [vp, C.POINTER(_Info)]
    L.gs_apply_forward.argtypes = [vp, vp, C.c_int64, vp, vp]
    L.gs_apply_adjoint.argtypes = [vp, vp, C.c_int64, vp, vp]
    L.gs_solve_least_squares.argtypes = [vp, vp, C.c_int64, vp, C.c_int, C.c_double, vp, C.POINTER(_Stats), dp, vp]
    L.gs_cgls_begin.argtypes = [vp, vp, C.c_int64, vp, C.c_double, C.c_int, vp, C.POINTER(vp)]
    L.gs_cgls_step.argtypes = [vp, C.c_int, vp]
    L.gs_cgls_active.argtypes = [vp, vp, C.POINTER(C.c_int)]
    L.gs_cgls_finish.argtypes = [vp, vp, C.POINTER(_Stats), dp, vp]
    L.gs_cgls_destroy.argtypes = [vp]
    L.gs_op_export_factors.argtypes = [vp, C.c_int, C.c_int, dp, dp, dp]
    L.gs_nfft_plan_create.argtypes = [C.c_int, C.POINTER(C.c_int), vp, C.c_int64, C.c_double, C.c_int, C.c_int,
                                      C.POINTER(vp)]
    L.gs_nfft_plan_forward.argtypes = [vp, vp, C.c_int64, vp, vp]
    L.gs_nfft_plan_adjoint.argtypes = [vp, vp, C.c_int64, vp, vp]
    L.gs_nfft_plan_info.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                    C.POINTER(C.c_int)]
    L.gs_nfft_plan_destroy.argtypes = [vp]
    L.gs_uniform_ndft_fft.argtypes = [vp, C.c_int64, C.c_int64, C.c_double, C.c_int64, vp, vp]
    L.gs_uniform_ndft_adjoint_fft.argtypes = [vp, C.c_int64, C.c_double, C.c_int64, vp, vp]
    L.gs_ndft_forward.argtypes = [C.c_int, C.POINTER(C.c_int), vp, C.c_int64, vp, C.c_int64, vp, vp]
    L.gs_ndft_adjoint.argtypes = [C.c_int, C.POINTER(C.c_int), vp, C.c_int64, vp, C.c_int64, vp, vp]
    _lib = L
    return L


def _check(rc):
    if rc != 0:
        msg = load_library().gs_last_error().decode()
        raise _ERRS.get(rc, Error)(msg)


def _check_inputs(rc):
    if rc != 0:
        L = load_library()
        L.gs_inputs_last_error.restype = C.c_char_p
        raise _ERRS.get(rc, Error)(L.gs_inputs_last_error().decode())


# ------------------------------------------------------------------ value types
_FAMILIES = {"haar": 1, "db1": 1, **{f"db{p}": p for p in range(2, 9)}}


def family_p(family) -> int:
    """family_from_string (scaling.cpp:16-22): haar / db1..db8 -> p."""
    if isinstance(family, int):
        if 1 <= family <= 8:
            return family
        raise DomainError("unsupported family")
    if family not in _FAMILIES:
        raise DomainError(f"unsupported family: {family}")
    return _FAMILIES[family]


@dataclass
class SamplingSet:
    """nufft.hpp:16-23 -- point-major coordinates (x[, y])."""
    dim: int
    coords: np.ndarray

    def __post_init__(self):
        self.coords = np.ascontiguousarray(self.coords, dtype=np.float64).ravel()

    def size(self):
        return self.coords.size // self.dim


@dataclass
class Freq2WaveOptions:
    """freq2wave.hpp:12-24."""
    bandwidth: Optional[float] = None
    weights: Optional[np.ndarray] = None
    sigma: float = 2.0
    w: int = 6
    boundary_depth: int = 30
    product_terms: int = 48
    allow_uniform_fast_path: bool = True
    allow_tensor_route: bool = False  # opt-in: exact tensor route for uniform 2D grids
    exact_ndft: bool = False  # 1D: direct NDFT core instead of the KB NFFT (GS_ROUTE_NDFT_1D)


@dataclass
class SolveOptions:
    """solver.hpp:10-14."""
    max_iterations: int = 0
    tolerance: float = 1e-10
    initial_guess: Optional[np.ndarray] = None


@dataclass
class SolveStats:
    """solver.hpp:16-22."""
    iterations: int = 0
    residual: float = 0.0
    history: list = field(default_factory=list)
    converged: bool = False


def _is_torch(a):
    return type(a).__module__.startswith("torch")


def _ptr_len(a, complex_expected=True):
    """(pointer, complex length, keepalive) of a numpy array or torch tensor."""
    if _is_torch(a):
        import torch
        if a.dtype != torch.complex128:
            raise ShapeError("expected a complex128 tensor")
        if not a.is_contiguous():
            a = a.contiguous()
        return a.data_ptr(), a.numel(), a
    arr = np.ascontiguousarray(a, dtype=np.complex128)
    return arr.ctypes.data, arr.size, arr


def _stream_ptr(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return getattr(stream, "cuda_stream", None)


class Freq2WaveOp:
    """Handle to the device-resident operator (Freq2WaveOp, freq2wave.hpp:32-55)."""

    def __init__(self, handle, keep):
        self._h = handle
        self._keep = keep
        info = _Info()
        _check(load_library().gs_op_info(handle, C.byref(info)))
        self.dim = info.dim
        self.p = info.family_p
        self.J = info.J
        self.n = 1 << info.J
        self.batch = info.batch
        self.route = ROUTES.get(info.route, "?")
        self._rows = info.rows
        self._cols = info.cols
        self.uniform_fast = bool(info.uniform_fast)
        self.uniform_epsilon = info.uniform_epsilon
        self._weighted = bool(info.weighted)
        self.n_over = info.n_over
        self.device_bytes = info.device_bytes
        # 2D gridding kernels on the balanced band schedule (uneven patterns, e.g. spirals)
        self.balanced_schedule = bool(load_library().gs_op_balanced_schedule(handle))

    def rows(self):
        return self._rows

    def cols(self):
        return self._cols

    def weighted(self):
        return self._weighted

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            load_library().gs_op_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def factors(self, axis=0, problem=0):
        """(D, L, R) of one axis in the reference layout (Dx/Lx/Rx, freq2wave.hpp:42-43)."""
        M = self._rows
        D = np.empty(M, np.complex128)
        L = R = None
        dp = C.POINTER(C.c_double)
        if self.p >= 2:
            L = np.empty(M * self.p, np.complex128)
            R = np.empty(M * self.p, np.complex128)
        _check(load_library().gs_op_export_factors(
            self._h, problem, axis, D.ctypes.data_as(dp),
            L.ctypes.data_as(dp) if L is not None else None, R.ctypes.data_as(dp) if R is not None else None))
        if L is not None:
            L = L.reshape(self.p, M).T.copy()
            R = R.reshape(self.p, M).T.copy()
        return D, L, R


def freq2wave(samples, family, J, options: Optional[Freq2WaveOptions] = None, *, batch=1, device=0, **kw):
    """gs::freq2wave (freq2wave.cpp:86-193), built on the device.

    ``samples`` is a SamplingSet (or a list of them for a batch of independent
    equal-shape problems); keyword arguments override Freq2WaveOptions fields.
    """
    opt = options or Freq2WaveOptions()
    for k, v in kw.items():
        setattr(opt, k, v)
    sets = samples if isinstance(samples, (list, tuple)) else [samples]
    dim = sets[0].dim
    M = sets[0].size()
    for s in sets:
        if s.dim != dim or s.size() != M:
            raise ShapeError("batched sampling sets must share dim and size")
    coords = np.ascontiguousarray(np.concatenate([s.coords for s in sets]), dtype=np.float64)
    weights = None
    if opt.weights is not None:
        weights = np.ascontiguousarray(np.asarray(opt.weights, dtype=np.float64).ravel())
        if weights.size != M * len(sets):
            raise ShapeError("weight count does not match sample count")
    dp = C.POINTER(C.c_double)
    d = _Desc()
    d.dim = dim
    d.family_p = family_p(family)
    d.J = int(J)
    d.M = M
    d.batch = len(sets)
    d.coords = coords.ctypes.data_as(dp)
    d.weights = weights.ctypes.data_as(dp) if weights is not None else None
    d.bandwidth = float("nan") if opt.bandwidth is None else float(opt.bandwidth)
    d.sigma = opt.sigma
    d.w = opt.w
    d.boundary_depth = opt.boundary_depth
    d.product_terms = opt.product_terms
    d.allow_uniform_fast_path = int(bool(opt.allow_uniform_fast_path))
    d.allow_tensor_route = int(bool(opt.allow_tensor_route))
    d.exact_ndft = int(bool(opt.exact_ndft))
    d.device = device
    h = C.c_void_p()
    _check(load_library().gs_op_create(C.byref(d), C.byref(h)))
    return Freq2WaveOp(h, None)


def _out_like(inp, n):
    if _is_torch(inp):
        import torch
        return torch.empty(n, dtype=torch.complex128, device=inp.device)
    return np.empty(n, np.complex128)


def apply_forward(op: Freq2WaveOp, coeffs, stream=None):
    """y = T x  (freq2wave.cpp:215-303)."""
    p, n, keep = _ptr_len(coeffs)
    out = _out_like(keep, op.rows() * op.batch)
    q = out.data_ptr() if _is_torch(out) else out.ctypes.data
    _check(load_library().gs_apply_forward(op.handle, p, n, q, _stream_ptr(stream)))
    return out


def apply_adjoint(op: Freq2WaveOp, samples, stream=None):
    """z = T* y  (freq2wave.cpp:305-387)."""
    p, n, keep = _ptr_len(samples)
    out = _out_like(keep, op.cols() * op.batch)
    q = out.data_ptr() if _is_torch(out) else out.ctypes.data
    _check(load_library().gs_apply_adjoint(op.handle, p, n, q, _stream_ptr(stream)))
    return out


def _ndft(adjoint, dim, N, points, data, stream=None):
    pts = points if _is_torch(points) else np.ascontiguousarray(points, dtype=np.float64).ravel()
    pp = pts.data_ptr() if _is_torch(pts) else pts.ctypes.data
    M = (pts.numel() if _is_torch(pts) else pts.size) // dim
    Nv = (C.c_int * 2)(int(N[0]), int(N[1]) if dim == 2 else 0)
    q, n, keep = _ptr_len(data)
    out = _out_like(keep, M if not adjoint else int(N[0]) * (int(N[1]) if dim == 2 else 1))
    o = out.data_ptr() if _is_torch(out) else out.ctypes.data
    fn = load_library().gs_ndft_adjoint if adjoint else load_library().gs_ndft_forward
    _check(fn(int(dim), Nv, pp, M, q, n, o, _stream_ptr(stream)))
    return out


def ndft_forward(dim, N, points, grid, stream=None):
    """gs::ndft_forward (nufft.cpp:74-101): y_m = sum_k x_k exp(-2 pi i k.xi_m), on the device."""
    return _ndft(False, dim, N, points, grid, stream)


def ndft_adjoint(dim, N, points, samples, stream=None):
    """gs::ndft_adjoint (nufft.cpp:103-132): z_k = sum_m y_m exp(+2 pi i k.xi_m), on the device."""
    return _ndft(True, dim, N, points, samples, stream)


class NfftPlan:
    """gs::NfftPlan (nufft.hpp:36-62): Kaiser-Bessel window-gridding NDFT pair on
    the device; ``points`` scaled to [-1/2, 1/2), point-major."""

    def __init__(self, dim, N, points, sigma=2.0, w=6, device=0):
        pts = np.ascontiguousarray(points, dtype=np.float64).ravel()
        Nv = (C.c_int * 2)(int(N[0]), int(N[1]) if dim == 2 and len(N) > 1 else 0)
        h = C.c_void_p()
        _check(load_library().gs_nfft_plan_create(int(dim), Nv, pts.ctypes.data, pts.size // max(1, int(dim)),
                                                  float(sigma), int(w), int(device), C.byref(h)))
        self._h = h
        d, m, g, nov = C.c_int(), C.c_int64(), C.c_int64(), (C.c_int * 2)()
        _check(load_library().gs_nfft_plan_info(h, C.byref(d), C.byref(m), C.byref(g), nov))
        self._dim, self._m, self._g, self._nov = d.value, m.value, g.value, (nov[0], nov[1])

    def dim(self):
        return self._dim

    def points_count(self):
        return self._m

    def grid_size(self):
        return self._g

    def oversampled_length(self, axis):
        return self._nov[axis]

    def forward(self, grid, stream=None):
        q, n, keep = _ptr_len(grid)
        out = _out_like(keep, self._m)
        o = out.data_ptr() if _is_torch(out) else out.ctypes.data
        _check(load_library().gs_nfft_plan_forward(self._h, q, n, o, _stream_ptr(stream)))
        return out

    def adjoint(self, samples, stream=None):
        q, n, keep = _ptr_len(samples)
        out = _out_like(keep, self._g)
        o = out.data_ptr() if _is_torch(out) else out.ctypes.data
        _check(load_library().gs_nfft_plan_adjoint(self._h, q, n, o, _stream_ptr(stream)))
        return out

    def close(self):
        if getattr(self, "_h", None):
            load_library().gs_nfft_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def plan_nfft(dim, N, points, sigma=2.0, w=6, device=0):
    """gs::plan_nfft (nufft.cpp:367-370)."""
    return NfftPlan(dim, N, points, sigma, w, device)


def nfft_forward(plan, grid, stream=None):
    return plan.forward(grid, stream)


def nfft_adjoint(plan, samples, stream=None):
    return plan.adjoint(samples, stream)


def uniform_ndft_fft(x, M, epsilon, N, stream=None):
    """gs::uniform_ndft_fft (nufft.cpp:402-429) on the device, any DFT length."""
    q, n, keep = _ptr_len(x)
    out = _out_like(keep, int(M))
    o = out.data_ptr() if _is_torch(out) else out.ctypes.data
    _check(load_library().gs_uniform_ndft_fft(q, n, int(M), float(epsilon), int(N), o, _stream_ptr(stream)))
    return out


def uniform_ndft_adjoint_fft(samples, epsilon, N, stream=None):
    """gs::uniform_ndft_adjoint_fft (nufft.cpp:431-459) on the device."""
    q, n, keep = _ptr_len(samples)
    out = _out_like(keep, int(N))
    o = out.data_ptr() if _is_torch(out) else out.ctypes.data
    _check(load_library().gs_uniform_ndft_adjoint_fft(q, n, float(epsilon), int(N), o, _stream_ptr(stream)))
    return out


def solve_least_squares(op: Freq2WaveOp, samples, options: Optional[SolveOptions] = None, stream=None, **kw):
    """CGNR resident on the GPU (solver.cpp:19-91).  Returns (x, SolveStats) or,
    for a batched operator, (x[batch*cols], [SolveStats]*batch)."""
    opt = options or SolveOptions()
    for k, v in kw.items():
        setattr(opt, k, v)
    if not (opt.tolerance > 0):
        raise DomainError("tolerance must be positive")
    p, n, keep = _ptr_len(samples)
    x0p = None
    keep0 = None
    if opt.initial_guess is not None:
        x0p, n0, keep0 = _ptr_len(opt.initial_guess)
        if n0 != op.cols() * op.batch:
            raise ShapeError("initial guess length mismatch")
    B = op.batch
    max_iter = opt.max_iterations if opt.max_iterations > 0 else 2 * op.cols()
    x = np.empty(op.cols() * B, np.complex128)
    stats = (_Stats * B)()
    hist = np.zeros(B * (max_iter + 1), np.float64)
    _check(load_library().gs_solve_least_squares(
        op.handle, p, n, x0p, int(opt.max_iterations), float(opt.tolerance), x.ctypes.data, stats,
        hist.ctypes.data_as(C.POINTER(C.c_double)), _stream_ptr(stream)))
    out = []
    for b in range(B):
        st = stats[b]
        hl = st.iterations + 1
        out.append(SolveStats(st.iterations, st.residual, list(hist[b * (max_iter + 1): b * (max_iter + 1) + hl]),
                              bool(st.converged)))
    return (x, out[0]) if B == 1 else (x, out)


class CglsSession:
    """Split CGLS (preamble / n iterations / result) for benchmarking and
    warm restarts: begin() runs solver.cpp:28-68, step(k) runs k iterations of
    solver.cpp:70-88 with no host synchronisation."""

    def __init__(self, op: Freq2WaveOp, samples, tolerance=1e-300, history_capacity=2, initial_guess=None,
                 stream=None):
        self.op = op
        p, n, self._keep = _ptr_len(samples)
        x0p = None
        if initial_guess is not None:
            x0p, _, self._keep0 = _ptr_len(initial_guess)
        self._cap = max(2, history_capacity)
        h = C.c_void_p()
        _check(load_library().gs_cgls_begin(op.handle, p, n, x0p, float(tolerance), self._cap, _stream_ptr(stream),
                                            C.byref(h)))
        self._h = h

    def step(self, iterations, stream=None):
        _check(load_library().gs_cgls_step(self._h, int(iterations), _stream_ptr(stream)))

    def active(self, stream=None):
        a = C.c_int()
        _check(load_library().gs_cgls_active(self._h, _stream_ptr(stream), C.byref(a)))
        return bool(a.value)

    def result(self, out=None, stream=None):
        B = self.op.batch
        x = out if out is not None else np.empty(self.op.cols() * B, np.complex128)
        q = x.data_ptr() if _is_torch(x) else x.ctypes.data
        stats = (_Stats * B)()
        _check(load_library().gs_cgls_finish(self._h, q, stats, None, _stream_ptr(stream)))
        return x, [SolveStats(s.iterations, s.residual, [], bool(s.converged)) for s in stats]

    def close(self):
        if getattr(self, "_h", None):
            load_library().gs_cgls_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
