"""Benchmark input harness: the reference's sampling patterns
(patterns.cpp, bit-identical generators), exact O(M log M) Voronoi density
weights and the density report (weights.cpp semantics), the bench harness's
seeded coefficients (bench.cpp:30-36) and the truncated-cosine test signal
(signals.cpp), implemented in csrc/host_inputs.cpp."""
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
        L.gs_density.argtypes = [C.c_int, C.c_int64, _dp, C.c_double, _dp, C.c_int]
        L.gs_seeded_coefficients.argtypes = [C.c_int64, C.c_uint64, _dp]
        L.gs_truncated_cosine.argtypes = [C.c_int64, _dp, _dp]
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


def voronoi_weights(dim, coords, K, threads=0, device=None):
    """voronoi_weights (weights.cpp:94-133): host (multi-threaded) by default;
    device=<ordinal> runs the 2D cells on that GPU (gs_voronoi_weights_gpu,
    bit-identical to the host's)."""
    coords = np.ascontiguousarray(coords, dtype=np.float64).ravel()
    M = coords.size // dim
    mu = np.empty(M)
    if device is not None:
        from . import _check
        L = _lib()
        L.gs_voronoi_weights_gpu.argtypes = [C.c_int, C.c_int64, _dp, C.c_double, _dp, C.c_int, C.c_void_p]
        _check(L.gs_voronoi_weights_gpu(dim, M, coords.ctypes.data_as(_dp), float(K), mu.ctypes.data_as(_dp),
                                        int(device), None))
        return mu
    _check_inputs(_lib().gs_voronoi_weights(dim, M, coords.ctypes.data_as(_dp), float(K), mu.ctypes.data_as(_dp),
                                            int(threads)))
    return mu


class DensityReport:
    """weights.hpp DensityReport: delta_raw, delta_scaled = delta_raw / 2 and
    the quarter bound delta_scaled / (2K) < 1/4 (weights.cpp:172-176)."""

    def __init__(self, delta_raw, K):
        self.delta_raw = float(delta_raw)
        self.delta_scaled = self.delta_raw / 2.0
        self.satisfies_quarter_bound = (self.delta_scaled / (2.0 * K)) < 0.25


def density(dim, coords, K, threads=0):
    coords = np.ascontiguousarray(coords, dtype=np.float64).ravel()
    d = C.c_double(0.0)
    _check_inputs(_lib().gs_density(dim, coords.size // dim, coords.ctypes.data_as(_dp), float(K), C.byref(d),
                                    int(threads)))
    return DensityReport(d.value, K)


def seeded_coefficients(n, seed):
    out = np.empty(2 * n)
    _check_inputs(_lib().gs_seeded_coefficients(int(n), int(seed), out.ctypes.data_as(_dp)))
    return out.view(np.complex128)


def truncated_cosine_transform(xi):
    xi = np.ascontiguousarray(xi, dtype=np.float64).ravel()
    out = np.empty(2 * xi.size)
    _check_inputs(_lib().gs_truncated_cosine(xi.size, xi.ctypes.data_as(_dp), out.ctypes.data_as(_dp)))
    return out.view(np.complex128)
