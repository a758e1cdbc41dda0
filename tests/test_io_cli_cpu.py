"""CPU checks of the front-end rows: the reference's file
formats (io.cpp:104-323) byte for byte, their error classes, the `gs` CLI
commands that need no GPU (gen, weights), the density report
(weights.cpp:135-176) against a brute-force supremum, and the bench harness's
random streams pinned to an independent MT19937-64 implementation."""
import itertools
import json
import math
import os
import struct

import numpy as np
import pytest

import paper_1607_04091_b200 as gs
from paper_1607_04091_b200 import cli, inputs
from paper_1607_04091_b200 import io as gsio


# ------------------------------------------------------------------ MT19937-64 (C++ [rand.eng.mers])
class MT64:
    """Independent restatement of std::mt19937_64, used to pin the C++ streams."""
    W, N, M, R = 64, 312, 156, 31
    A = 0xB5026F5AA96619E9
    U, D, S, B, T, C, L = 29, 0x5555555555555555, 17, 0x71D67FFFEDA60000, 37, 0xFFF7EEE000000000, 43
    F = 6364136223846793005
    MASK = (1 << 64) - 1

    def __init__(self, seed=5489):
        self.mt = [0] * self.N
        self.mt[0] = seed & self.MASK
        for i in range(1, self.N):
            self.mt[i] = (self.F * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & self.MASK
        self.idx = self.N

    def __call__(self):
        if self.idx >= self.N:
            lo, hi = (1 << self.R) - 1, self.MASK ^ ((1 << self.R) - 1)
            for i in range(self.N):
                y = (self.mt[i] & hi) | (self.mt[(i + 1) % self.N] & lo)
                self.mt[i] = self.mt[(i + self.M) % self.N] ^ (y >> 1) ^ (self.A if y & 1 else 0)
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> self.U) & self.D
        y ^= (y << self.S) & self.B
        y ^= (y << self.T) & self.C
        y ^= y >> self.L
        return y & self.MASK

    def uniform(self, a, b):
        # libstdc++ generate_canonical<double, 53> over a 64-bit engine: one draw / 2^64
        u = float(self()) / 18446744073709551616.0
        if u >= 1.0:
            u = math.nextafter(1.0, 0.0)
        return (b - a) * u + a


def test_mt64_restatement_matches_the_standard_known_answer():
    g = MT64()
    for _ in range(9999):
        g()
    assert g() == 9981545732273789042  # [rand.predef]: 10000th output of default mt19937_64


def test_seeded_coefficients_match_bench_cpp_stream():
    seed = 20160613
    x = inputs.seeded_coefficients(64, seed)
    g = MT64(seed ^ 0x9E3779B97F4A7C15)
    ref = []
    for _ in range(64):
        re = g.uniform(-1.0, 1.0)
        im = g.uniform(-1.0, 1.0)
        ref.append(complex(re, im))
    assert np.array_equal(x, np.array(ref))


def test_jitter_pattern_matches_patterns_cpp_stream():
    M, eps, eta, seed = 37, 0.5, 0.2, 7
    pts = inputs.gen_jitter(M, eps, eta, seed, 1)
    g = MT64(seed)
    ref = sorted(eps * (m - M / 2.0) + g.uniform(-eta, eta) for m in range(M))
    assert np.array_equal(pts, np.array(ref))
    pts2 = inputs.gen_jitter(8, eps, eta, seed, 2)  # 2D: x-major grid, then one shift per coordinate
    g = MT64(seed)
    axis = [eps * (m - 4.0) for m in range(8)]
    grid = [c for x in axis for y in axis for c in (x, y)]
    assert np.array_equal(pts2, np.array([c + g.uniform(-eta, eta) for c in grid]))


# ------------------------------------------------------------------ density report
def brute_density_2d(pts, K):
    """sup over [-K,K]^2 of the nearest-sample distance: the maximum over every
    candidate Voronoi vertex (circumcentres, bisector/edge crossings, corners)."""
    cand = [(-K, -K), (K, -K), (K, K), (-K, K)]
    for a, b, c in itertools.combinations(pts, 3):
        d = 2 * (a[0] * (b[1] - c[1]) + b[0] * (c[1] - a[1]) + c[0] * (a[1] - b[1]))
        if abs(d) < 1e-14:
            continue
        ux = ((a @ a) * (b[1] - c[1]) + (b @ b) * (c[1] - a[1]) + (c @ c) * (a[1] - b[1])) / d
        uy = ((a @ a) * (c[0] - b[0]) + (b @ b) * (a[0] - c[0]) + (c @ c) * (b[0] - a[0])) / d
        cand.append((ux, uy))
    for a, b in itertools.combinations(pts, 2):
        mid, nrm = (a + b) / 2, b - a
        for fixed, axis in ((-K, 0), (K, 0), (-K, 1), (K, 1)):
            o = 1 - axis
            if abs(nrm[o]) < 1e-14:
                continue
            t = mid[o] + (nrm[axis] * (mid[axis] - fixed)) / nrm[o]
            p = [0.0, 0.0]
            p[axis], p[o] = fixed, t
            cand.append(tuple(p))
    best = 0.0
    for q in cand:
        if abs(q[0]) <= K + 1e-12 and abs(q[1]) <= K + 1e-12:
            best = max(best, np.min(np.hypot(pts[:, 0] - q[0], pts[:, 1] - q[1])))
    return best


def test_density_known_answers():
    assert inputs.density(1, np.array([-0.5, 0.5]), 1.0).delta_raw == 0.5
    r = inputs.density(1, np.array([-0.9, 0.1, 0.2]), 1.0)  # gaps: ends 0.1 / 0.8, half gaps 0.5 / 0.05
    assert r.delta_raw == pytest.approx(0.8) and r.delta_scaled == pytest.approx(0.4)
    assert r.satisfies_quarter_bound  # 0.4 / (2 K) = 0.2 < 1/4
    assert not inputs.density(1, np.array([0.9]), 1.0).satisfies_quarter_bound  # 1.9 / 2 / 2 >= 1/4
    quad = np.array([-0.5, -0.5, 0.5, -0.5, -0.5, 0.5, 0.5, 0.5])
    assert inputs.density(2, quad, 1.0).delta_raw == pytest.approx(math.sqrt(0.5), rel=1e-15)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_density_2d_matches_brute_force_supremum(seed):
    rng = np.random.default_rng(seed)
    pts = rng.uniform(-1, 1, size=(14, 2))
    d = inputs.density(2, pts.ravel(), 1.0).delta_raw
    assert d == pytest.approx(brute_density_2d(pts, 1.0), rel=1e-12)


def test_truncated_cosine_transform_closed_form():
    xi = np.array([0.0, 1.0, -1.0, 0.3, 2.5, -7.25])

    def g(a):
        return 0.5 if a == 0 else (complex(math.cos(math.pi * a), math.sin(math.pi * a)) - 1) / complex(0, 2 * math.pi * a)

    ref = np.array([0.5 * (g(v - 1) + g(v + 1)) for v in xi])
    assert np.allclose(inputs.truncated_cosine_transform(xi), ref, rtol=0, atol=1e-15)
    assert inputs.truncated_cosine_transform(np.array([1.0]))[0] == pytest.approx(0.25)


# ------------------------------------------------------------------ file formats
def test_frequency_file_binary_layout_and_round_trip(tmp_path):
    s = gs.SamplingSet(2, np.array([0.25, -1.5, 3.0, 1e-300]))
    p = tmp_path / "f.bin"
    gsio.write_frequency_file(p, s, "binary")
    raw = p.read_bytes()
    assert raw[:4] == b"GSFQ" and struct.unpack("<IIQ", raw[4:20]) == (1, 2, 2) and len(raw) == 20 + 32
    assert np.frombuffer(raw[20:], "<f8").tolist() == [0.25, -1.5, 3.0, 1e-300]
    back = gsio.read_frequency_file(p)
    assert back.dim == 2 and np.array_equal(back.coords, s.coords)
    q = tmp_path / "f.csv"
    gsio.write_frequency_file(q, s, "csv")
    assert q.read_text().splitlines()[:2] == ["xi_x,xi_y", "0.25,-1.5"]
    assert np.array_equal(gsio.read_frequency_file(q).coords, s.coords)  # %.17g round-trips exactly


def test_sample_and_coefficient_and_weight_files_round_trip(tmp_path):
    z = np.array([1 + 2j, -0.1 + 1e-17j, np.pi - 1j / 3])
    for fmt in ("csv", "binary"):
        p = tmp_path / f"s.{fmt}"
        gsio.write_sample_file(p, z, fmt)
        assert np.array_equal(gsio.read_sample_file(p), z)
    raw = (tmp_path / "s.binary").read_bytes()
    assert raw[:4] == b"GSSM" and struct.unpack("<IIQ", raw[4:20]) == (1, 1, 3)
    vals = np.arange(16) * (1 - 0.5j)
    cf = gsio.CoefficientFile(2, "db2", 2, vals)
    p = tmp_path / "c.gscf"
    gsio.write_coefficient_file(p, cf)
    raw = p.read_bytes()
    assert raw[:4] == b"GSCF" and struct.unpack("<IIBI", raw[4:17]) == (1, 2, 2, 2) and len(raw) == 17 + 256
    back = gsio.read_coefficient_file(p)
    assert (back.dim, back.family, back.J) == (2, "db2", 2) and np.array_equal(back.values, vals)
    gsio.write_coefficient_file(p, gsio.CoefficientFile(1, "haar", 3, np.ones(8)))
    assert p.read_bytes()[12] == 0 and gsio.read_coefficient_file(p).family == "haar"
    mu = np.array([0.5, 1.25, 1e-9])
    gsio.write_weight_file(tmp_path / "w.csv", mu)
    assert (tmp_path / "w.csv").read_text().startswith("mu\n")
    assert np.array_equal(gsio.read_weight_file(tmp_path / "w.csv"), mu)


@pytest.mark.parametrize("content,reader,msg", [
    (b"", "freq", "missing header"),
    (b"xi_q\n1\n", "freq", "bad frequency file header"),
    (b"xi_x\n", "freq", "has no points"),
    (b"xi_x,xi_y\n1,2\n3\n", "freq", "wrong column count at line 3"),
    (b"xi_x\n1.5x\n", "freq", "cannot parse number"),
    (b"GSFQ" + struct.pack("<I", 2), "freq", "unsupported frequency file version"),
    (b"GSFQ" + struct.pack("<II", 1, 3), "freq", "dim must be 1 or 2"),
    (b"GSFQ" + struct.pack("<IIQ", 1, 1, 4) + b"\0" * 8, "freq", "truncated file reading coordinates"),
    (b"re,im\n1\n", "samp", "wrong column count"),
    (b"GSSM" + struct.pack("<IIQ", 1, 1, 2) + b"\0" * 16, "samp", "truncated"),
    (b"XXXX", "coef", "bad magic"),
    (b"GSCF" + struct.pack("<IIBI", 1, 1, 9, 2), "coef", "unknown family tag 9"),
    (b"GSCF" + struct.pack("<IIBI", 1, 2, 4, 14), "coef", "scale out of range"),
    (b"GSCF" + struct.pack("<IIB", 1, 1, 4), "coef", "truncated file reading J"),
    (b"m\n1\n", "wts", "bad weight file header"),
])
def test_malformed_files_raise_file_format_error(tmp_path, content, reader, msg):
    p = tmp_path / "bad"
    p.write_bytes(content)
    fn = {"freq": gsio.read_frequency_file, "samp": gsio.read_sample_file, "coef": gsio.read_coefficient_file,
          "wts": gsio.read_weight_file}[reader]
    with pytest.raises(gs.FileFormatError, match=msg):
        fn(p)
    assert gs.FileFormatError.exit_code == 3


# ------------------------------------------------------------------ CLI without a GPU
def test_cli_gen_and_weights(tmp_path, capsys):
    f = str(tmp_path / "pts.bin")
    assert cli.main(["gen", "jitter", "--M", "64", "--epsilon", "0.5", "--eta", "0.2", "--seed", "5",
                     "-o", f, "--format", "bin", "--truncated-cosine-samples", str(tmp_path / "y.bin")]) == 0
    assert "wrote 64 points to" in capsys.readouterr().out
    s = gsio.read_frequency_file(f)
    assert np.array_equal(s.coords, inputs.gen_jitter(64, 0.5, 0.2, 5, 1))
    y = gsio.read_sample_file(tmp_path / "y.bin")
    assert np.array_equal(y, inputs.truncated_cosine_transform(s.coords))
    w = str(tmp_path / "w.csv")
    assert cli.main(["weights", f, "--bandwidth", "16.5", "-o", w]) == 0
    out = capsys.readouterr().out.splitlines()
    rep = inputs.density(1, s.coords, 16.5)
    assert out[0] == "delta_raw %.12g" % rep.delta_raw and out[2].startswith("quarter_bound")
    assert np.array_equal(gsio.read_weight_file(w), inputs.voronoi_weights(1, s.coords, 16.5))
    # spiral: 2D, points-per-turn derived from --M
    assert cli.main(["gen", "spiral", "--M", "300", "--turns", "3", "--bandwidth", "8", "-o",
                     str(tmp_path / "sp.csv")]) == 0
    assert gsio.read_frequency_file(tmp_path / "sp.csv").size() == 300


def test_cli_usage_and_error_exit_codes(tmp_path, capsys):
    assert cli.main([]) == 2
    assert cli.main(["gen", "blob", "-o", str(tmp_path / "x")]) == 2           # UsageError
    assert cli.main(["gen", "grid", "--M", "4", "-o", str(tmp_path / "x"), "--format", "xml"]) == 2
    assert cli.main(["weights", str(tmp_path / "missing"), "--bandwidth", "1"]) == 3  # FileFormatError
    gsio.write_frequency_file(tmp_path / "f.csv", gs.SamplingSet(1, np.array([0.0, 1.0, 2.0])))
    gsio.write_sample_file(tmp_path / "y.csv", np.ones(2))
    assert cli.main(["reconstruct", str(tmp_path / "f.csv"), str(tmp_path / "y.csv"), "--family", "haar",
                     "--scale-J", "2", "-o", str(tmp_path / "c")]) == 4           # count mismatch: ShapeError
    assert cli.main(["reconstruct", str(tmp_path / "f.csv"), str(tmp_path / "y.csv"), "--family", "haar",
                     "--scale-J", "2", "--weighted", "--unweighted", "-o", str(tmp_path / "c")]) == 2
    assert cli.main(["evaluate", str(tmp_path / "missing"), "--resolution", "3", "-o", "e"]) == 3
    assert cli.main(["bench", "nosuch"]) == 5
    capsys.readouterr()


def test_bench_registry_scaling_follows_bench_cpp():
    s, J = cli.bench_sampling_set(cli.REGISTRY[0], 0.25, 1)   # uniform1d: M 8192 -> 2048, J 12 -> 10
    assert J == 10 and s.size() == 2048
    assert s.coords[1] - s.coords[0] == pytest.approx(0.5 * (8192 / 2048) * 0.25)
    s, J = cli.bench_sampling_set(cli.REGISTRY[4], 1.0, 1)    # spiral: 27 turns, 27681 points
    assert J == 5 and s.size() == 27681
    with pytest.raises(gs.DomainError):
        cli.bench_sampling_set(cli.REGISTRY[0], 0.0, 1)
