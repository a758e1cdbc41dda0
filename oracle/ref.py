"""The reference itself, behind the oracle's ctypes front-end.

TEST INFRASTRUCTURE ONLY (same import rule as ``oracle``).

``oracle/_ref/libgs_ref.so`` is the UNMODIFIED reference library: its sources
compiled where they lie under /root/reference/proj/src by ``make -C oracle
ref`` against an Eigen subset and an FFTW stand-in (oracle/Makefile,
oracle/ref_driver.cpp).  It exports the symbols of libgs_oracle.so, so this
module is the oracle's own binding executed a second time against that
library: ``oracle.ref.Op``, ``oracle.ref.nfft`` ... call the reference where
``oracle.Op``, ``oracle.nfft`` ... call the restatement.

The library can only be built where /root/reference exists (the build
container); it is git-ignored and travels to the GPU box with the snapshot.
``available()`` says whether it is present.
"""
from __future__ import annotations

import importlib.util
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libgs_ref.so")
REFERENCE_ROOT = "/root/reference/proj"


def buildable():
    return os.path.exists(os.path.join(REFERENCE_ROOT, "src", "freq2wave.cpp"))


def build():
    """(Re)build oracle/_ref/libgs_ref.so when the reference sources are present."""
    if buildable():
        subprocess.check_call(["make", "-s", "-C", _HERE, "ref"])


def available():
    if not os.path.exists(LIB_PATH) and buildable():
        build()
    return os.path.exists(LIB_PATH)


def _bind():
    spec = importlib.util.spec_from_file_location("oracle._ref_binding", os.path.join(_HERE, "__init__.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod._LIB_PATH = LIB_PATH
    mod.build = build
    return mod


_b = _bind()

Op = _b.Op
OracleError = _b.OracleError
fourier_scaling = _b.fourier_scaling
fourier_boundary = _b.fourier_boundary
boundary_at_zero = _b.boundary_at_zero
boundary_UV = _b.boundary_UV
family_taps = _b.family_taps
ndft = _b.ndft
nfft = _b.nfft
uniform_fft = _b.uniform_fft
uniform_adjoint_fft = _b.uniform_adjoint_fft
gen_grid = _b.gen_grid
gen_jitter = _b.gen_jitter
gen_spiral = _b.gen_spiral
voronoi = _b.voronoi
scaling_dyadic = _b.scaling_dyadic
boundary_dyadic = _b.boundary_dyadic
weval = _b.weval
lib = _b.lib


def backend():
    import ctypes as C
    f = lib().orc_backend
    f.restype = C.c_char_p
    return f().decode()
