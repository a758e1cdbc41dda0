"""Benchmark input harness: the reference's sampling patterns
(patterns.cpp, bit-identical generators) and exact O(M log M) Voronoi density
weights (weights.cpp semantics), implemented in csrc/host_inputs.cpp."""
import ctypes as C

import numpy as np

from . import _check_inputs, load_library

_dp = C.POINTER(C.c_double)


def _lib():
    L = load_library()
    if not getattr(L, "_inputs_typed", False):
        L.gs_inputs_last_error.restype = C.c_char_p
        L.gs_gen_grid.argtypes = [C.c_int64, C.c_double, C.c_int, _dp]
        L.gs_gen_jitter.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_uint64, C.c_int, _dp]
        L.gs_gen_spiral.argtypes = [C.c_int, C.c_double, C.c_double, _dp]
        L.gs_voronoi_weights.argtypes = [C.c_int, C.c_int64, _dp, C.c_double, _dp, C.c_int]
        L._inputs_typed = True
    return L


def gen_grid(M, eps, dim=1):
    out = np.empty(M * (2 * M if dim == 2 else 1))
    _check_inputs(_lib().gs_gen_grid(M, eps, dim, out.ctypes.data_as(_dp)))
    return out


def gen_jitter(M, eps, eta, seed, dim=1):
    out = np.empty(M * (2 * M if dim == 2 else 1))
    _check_inputs(_lib().gs_gen_jitter(M, eps, eta, seed, dim, out.ctypes.data_as(_dp)))
    return out


def gen_spiral(turns, points_per_turn, K):
    out = np.empty(2 * int(round(turns * points_per_turn)))
    _check_inputs(_lib().gs_gen_spiral(turns, points_per_turn, K, out.ctypes.data_as(_dp)))
    return out


def voronoi_weights(dim, coords, K, threads=0):
    coords = np.ascontiguousarray(coords, dtype=np.float64).ravel()
    M = coords.size // dim
    mu = np.empty(M)
    _check_inputs(_lib().gs_voronoi_weights(dim, M, coords.ctypes.data_as(_dp), float(K), mu.ctypes.data_as(_dp),
                                            int(threads)))
    return mu
