"""Dyadic-grid evaluation on the GPU (dyadic.hpp; front-end row SURVEY 8(f)4):
scaling-function and edge-function tables by the dilation-equation cascade,
and weval_1d / weval_2d of a reconstruction on the closed grid over
[-1/2, 1/2].  Same names and semantics as the reference; every refinement
level and contraction runs in csrc/kernels_dyadic.cuh."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _check, _is_torch, _stream_ptr, family_p, load_library

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)


def _lib():
    L = load_library()
    if not getattr(L, "_dyadic_typed", False):
        vp = C.c_void_p
        L.gs_scaling_dyadic.argtypes = [C.c_int, C.c_int, _dp, _i64p, _i64p, vp]
        L.gs_boundary_dyadic.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp, _i64p, _i64p, vp]
        L.gs_weval.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int64, vp, vp]
        L._dyadic_typed = True
    return L


class FunctionTable:
    """dyadic.hpp:13-25: values[i] = phi(support_begin + i / 2^resolution)."""

    def __init__(self, family, resolution, support_begin, values):
        self.family, self.resolution, self.support_begin, self.values = family, resolution, support_begin, values

    def value_at(self, numerator: int) -> float:
        idx = numerator - (self.support_begin << self.resolution)
        return float(self.values[idx]) if 0 <= idx < self.values.size else 0.0


class ReconstructionEvaluation:
    """dyadic.hpp:40-48: 2^R + 1 points per axis; 2D values row-major, row = y."""

    def __init__(self, resolution, dim, values):
        self.resolution, self.dim, self.values = resolution, dim, values

    def points_per_axis(self) -> int:
        return (1 << self.resolution) + 1


def evaluate_scaling_dyadic(family, R, stream=None) -> FunctionTable:
    p = family_p(family)
    n, sb = C.c_int64(0), C.c_int64(0)
    L = _lib()
    _check(L.gs_scaling_dyadic(p, int(R), None, C.byref(n), C.byref(sb), _stream_ptr(stream)))
    out = np.empty(n.value)
    _check(L.gs_scaling_dyadic(p, int(R), out.ctypes.data_as(_dp), C.byref(n), C.byref(sb), _stream_ptr(stream)))
    return FunctionTable(family, int(R), sb.value, out)


def evaluate_boundary_dyadic(family, side, R, stream=None) -> list:
    """side: "left" / "right" (gs::Side).  Returns the p edge-function tables."""
    p = family_p(family)
    left = 1 if side in ("left", 0, True) else 0
    L = _lib()
    tabs = []
    for k in range(max(p, 1)):
        n, sb = C.c_int64(0), C.c_int64(0)
        _check(L.gs_boundary_dyadic(p, left, int(R), k, None, C.byref(n), C.byref(sb), _stream_ptr(stream)))
        out = np.empty(n.value)
        _check(L.gs_boundary_dyadic(p, left, int(R), k, out.ctypes.data_as(_dp), C.byref(n), C.byref(sb),
                                    _stream_ptr(stream)))
        tabs.append(FunctionTable(family, int(R), sb.value, out))
    return tabs


def _weval(dim, coeffs, family, J, R, stream):
    p = family_p(family)
    g = (1 << int(R)) + 1 if R >= 0 else 1
    if _is_torch(coeffs):
        import torch
        c = coeffs.contiguous().to(torch.float64)
        out = torch.empty(g if dim == 1 else g * g, dtype=torch.float64, device=c.device)
        cp, op, n = c.data_ptr(), out.data_ptr(), c.numel()
    else:
        c = np.ascontiguousarray(coeffs, dtype=np.float64).ravel()
        ok = 0 <= R <= (28 if dim == 1 else 15)  # larger R: the library raises DomainError
        out = np.empty((g if dim == 1 else g * g) if ok else 1)
        cp, op, n = c.ctypes.data, out.ctypes.data, c.size
    _check(_lib().gs_weval(dim, p, int(J), int(R), cp, n, op, _stream_ptr(stream)))
    return ReconstructionEvaluation(int(R), dim, out)


def weval_1d(coeffs, family, J, R, stream=None) -> ReconstructionEvaluation:
    """sum_n w_n phi^int_{J,k(n)} on the closed grid at resolution R >= J (dyadic.hpp:50-54)."""
    return _weval(1, coeffs, family, J, R, stream)


def weval_2d(coeffs, family, J, R, stream=None) -> ReconstructionEvaluation:
    """Tensor-product evaluation, coefficients x-fastest (dyadic.hpp:56-60)."""
    return _weval(2, coeffs, family, J, R, stream)
