"""CPU-side checks of the drop-in boundary: the sm_100a C-ABI library loads
without a GPU, exports every entry point include/gs_b200.h declares, reports
its build arch, and applies the reference's construction-time validation
(freq2wave.cpp:93-140 error classes) before touching the device."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gs_b200.h")


def _lib():
    import paper_1607_04091_b200 as gs
    return gs, gs.load_library()


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|long long|const char\*)\s+(gs_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    gs, L = _lib()
    names = declared_functions()
    assert len(names) >= 12
    for name in names:
        assert hasattr(L, name), name
    assert L.gs_build_arch() == 100


def test_sass_is_sm_100a():
    import subprocess
    gs, _ = _lib()
    out = subprocess.run(["cuobjdump", "--list-elf", gs.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("kw,cls", [
    (dict(dim=3), "DomainError"),
    (dict(J=30), "DomainError"),
    (dict(J=1, family="db2"), "DomainError"),          # 2^J < 2p
    (dict(coords=[0.0, 4.0]), "DomainError"),         # + 2^{J-1} outside [-1/2, 1/2)
    (dict(coords=[0.0, float("nan")]), "DomainError"),
    (dict(bandwidth=2.0, coords=[0.0, 3.0]), "DomainError"),
    (dict(weights=[1.0, -1.0]), "DomainError"),
    (dict(weights=[1.0]), "ShapeError"),
    (dict(J=3, family="db2", boundary_depth=0), "DomainError"),   # fourier.cpp:87
    (dict(J=3, family="db2", product_terms=0), "DomainError"),    # fourier.cpp:36
])
def test_construction_validation_matches_reference(kw, cls):
    gs, _ = _lib()
    dim = kw.pop("dim", 1)
    J = kw.pop("J", 3)
    fam = kw.pop("family", "haar")
    coords = kw.pop("coords", [0.0, -4.0])
    with pytest.raises(getattr(gs, cls)):
        gs.freq2wave(gs.SamplingSet(dim, np.array(coords)), fam, J, **kw)


def test_unknown_family():
    gs, _ = _lib()
    with pytest.raises(gs.DomainError):
        gs.family_p("db9")
    assert gs.family_p("db4") == 4 and gs.family_p("haar") == 1


def test_no_gpu_fails_loudly():
    """Without a CUDA device, valid construction raises CudaError (no CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    gs, _ = _lib()
    with pytest.raises(gs.CudaError):
        gs.freq2wave(gs.SamplingSet(1, np.array([0.0, -4.0])), "haar", 3)


def test_haar_ignores_depth_and_terms():
    """haar evaluates neither the product nor the recursion (fourier.cpp:35),
    so depth / terms <= 0 pass validation and only the missing GPU fails."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    gs, _ = _lib()
    with pytest.raises(gs.CudaError):
        gs.freq2wave(gs.SamplingSet(1, np.array([0.0, -4.0])), "haar", 3, boundary_depth=0, product_terms=0)


@pytest.mark.parametrize("args", [
    (1, [16], [0.5], 2.0, 6), (1, [15], [0.1], 2.0, 6), (1, [16], [0.1], 1.1, 6), (1, [16], [0.1], 2.0, 1),
    (3, [16], [0.1], 2.0, 6)])
def test_nfft_plan_validation_matches_reference(args):
    """NfftPlan ctor checks (nufft.cpp:181-188) raise before the device is touched."""
    gs, _ = _lib()
    dim, N, p, sigma, w = args
    with pytest.raises(gs.DomainError):
        gs.plan_nfft(dim, N, np.array(p), sigma, w)


def test_uniform_reduction_validation():
    """uniform_setup (nufft.cpp:389-400): 1/epsilon integer, M >= N, x length <= N."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    gs, _ = _lib()
    x = np.ones(8, complex)
    for args in ((x, 16, 0.3, 8), (x, 4, 0.5, 8), (np.ones(9, complex), 16, 0.5, 8)):
        with pytest.raises(gs.DomainError):
            gs.uniform_ndft_fft(*args)
