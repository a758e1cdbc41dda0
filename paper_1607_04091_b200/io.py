"""File formats of the reference front end (io.hpp / io.cpp:104-323), so the
GPU operator reads and writes the same files `gs gen / weights / reconstruct`
exchange:

* frequency files: CSV header ``xi_x`` or ``xi_x,xi_y``, or binary ``GSFQ``
  (u32 version = 1, u32 dim, u64 count, little-endian f64 point-major);
* sample files: CSV header ``re,im``, or binary ``GSSM`` (same header layout,
  interleaved re/im f64);
* coefficient files: binary ``GSCF`` (u32 version, u32 dim, u8 family tag:
  0 = haar, p for dbp, u32 J, interleaved complex values);
* weight files: CSV header ``mu``.

Numbers are written with ``%.17g`` (io.cpp:62-66).  Malformed files raise
:class:`FileFormatError` (exit code 3) with the reference's messages.
"""
from __future__ import annotations

import struct

import numpy as np

from . import FileFormatError, SamplingSet, ShapeError, family_p


def _fmt(v: float) -> str:
    return "%.17g" % v


def _parse(token: str, context: str) -> float:
    # strtod semantics of io.cpp:68-76: the whole token must be a number
    t = token
    try:
        if t != t.rstrip() or not t.strip() or "_" in t:  # strtod: leading blanks only, no digit separators
            raise ValueError
        return float(t)
    except ValueError:
        raise FileFormatError(f"cannot parse number '{token}' in {context}") from None


def _read_text(path) -> bytes:
    try:
        with open(path, "rb") as f:
            raw = f.read()
    except OSError:
        raise FileFormatError(f"cannot open for reading: {path}") from None
    return raw


def _lines(raw: bytes):
    for line in raw.decode("utf-8", errors="replace").split("\n"):
        yield line[:-1] if line.endswith("\r") else line


class _Reader:
    def __init__(self, raw: bytes, pos: int = 4):
        self.raw, self.pos = raw, pos

    def take(self, fmt: str, what: str):
        n = struct.calcsize(fmt)
        if self.pos + n > len(self.raw):
            raise FileFormatError(f"truncated file reading {what}")
        v = struct.unpack_from(fmt, self.raw, self.pos)
        self.pos += n
        return v[0] if len(v) == 1 else v

    def doubles(self, count: int, what: str) -> np.ndarray:
        n = 8 * count
        if self.pos + n > len(self.raw):
            raise FileFormatError(f"truncated file reading {what}")
        v = np.frombuffer(self.raw, dtype="<f8", count=count, offset=self.pos).astype(np.float64)
        self.pos += n
        return v


def _open_out(path, binary: bool):
    try:
        return open(path, "wb") if binary else open(path, "w", newline="\n")
    except OSError:
        raise FileFormatError(f"cannot open for writing: {path}") from None


# ------------------------------------------------------------------ frequency files (io.cpp:104-165)
def write_frequency_file(path, samples: SamplingSet, fmt: str = "csv") -> None:
    coords = np.ascontiguousarray(samples.coords, dtype=np.float64)
    dim = samples.dim
    if fmt == "csv":
        with _open_out(path, False) as out:
            out.write("xi_x\n" if dim == 1 else "xi_x,xi_y\n")
            pts = coords.reshape(-1, dim)
            for row in pts:
                out.write(",".join(_fmt(v) for v in row) + "\n")
        return
    with _open_out(path, True) as out:
        out.write(b"GSFQ" + struct.pack("<IIQ", 1, dim, coords.size // dim))
        out.write(coords.astype("<f8").tobytes())


def read_frequency_file(path) -> SamplingSet:
    raw = _read_text(path)
    if raw[:4] == b"GSFQ":
        r = _Reader(raw)
        if r.take("<I", "version") != 1:
            raise FileFormatError("unsupported frequency file version")
        dim = r.take("<I", "dim")
        if dim not in (1, 2):
            raise FileFormatError("frequency file dim must be 1 or 2")
        count = r.take("<Q", "count")
        return SamplingSet(dim, r.doubles(count * dim, "coordinates"))
    lines = _lines(raw)
    header = next(lines, None)
    if header is None or (header == "" and raw == b""):
        raise FileFormatError("missing header")
    if header == "xi_x":
        dim = 1
    elif header == "xi_x,xi_y":
        dim = 2
    else:
        raise FileFormatError(f"bad frequency file header: {header}")
    vals = []
    for lineno, line in enumerate(lines, start=2):
        if not line:
            continue
        fields = line.split(",")
        if len(fields) != dim:
            raise FileFormatError(f"wrong column count at line {lineno}")
        vals.extend(_parse(f, "frequency file") for f in fields)
    if not vals:
        raise FileFormatError("frequency file has no points")
    return SamplingSet(dim, np.array(vals, dtype=np.float64))


# ------------------------------------------------------------------ sample files (io.cpp:167-225)
def write_sample_file(path, samples, fmt: str = "csv") -> None:
    z = np.ascontiguousarray(samples, dtype=np.complex128).ravel()
    if fmt == "csv":
        with _open_out(path, False) as out:
            out.write("re,im\n")
            for v in z:
                out.write(f"{_fmt(v.real)},{_fmt(v.imag)}\n")
        return
    with _open_out(path, True) as out:
        out.write(b"GSSM" + struct.pack("<IIQ", 1, 1, z.size))
        out.write(z.view(np.float64).astype("<f8").tobytes())


def read_sample_file(path) -> np.ndarray:
    raw = _read_text(path)
    if raw[:4] == b"GSSM":
        r = _Reader(raw)
        if r.take("<I", "version") != 1:
            raise FileFormatError("unsupported sample file version")
        r.take("<I", "dim")
        count = r.take("<Q", "count")
        return r.doubles(2 * count, "samples").view(np.complex128).copy()
    lines = _lines(raw)
    header = next(lines, None)
    if header is None or (header == "" and raw == b""):
        raise FileFormatError("missing header")
    if header != "re,im":
        raise FileFormatError(f"bad sample file header: {header}")
    vals = []
    for lineno, line in enumerate(lines, start=2):
        if not line:
            continue
        fields = line.split(",")
        if len(fields) != 2:
            raise FileFormatError(f"wrong column count at line {lineno}")
        vals.append(complex(_parse(fields[0], "sample file"), _parse(fields[1], "sample file")))
    if not vals:
        raise FileFormatError("sample file has no values")
    return np.array(vals, dtype=np.complex128)


# ------------------------------------------------------------------ coefficient files (io.cpp:227-275)
class CoefficientFile:
    """io.hpp CoefficientFile: dim, family name, J, values (2^(dim J) complex)."""

    def __init__(self, dim=1, family="haar", J=0, values=None):
        self.dim, self.family, self.J = int(dim), family, int(J)
        self.values = np.zeros(0, np.complex128) if values is None else np.asarray(values, np.complex128)


def _family_tag(family) -> int:
    p = family_p(family)
    return 0 if p == 1 else p


def write_coefficient_file(path, cf: CoefficientFile) -> None:
    z = np.ascontiguousarray(cf.values, dtype=np.complex128).ravel()
    with _open_out(path, True) as out:
        out.write(b"GSCF" + struct.pack("<IIBI", 1, cf.dim, _family_tag(cf.family), cf.J))
        out.write(z.view(np.float64).astype("<f8").tobytes())


def read_coefficient_file(path) -> CoefficientFile:
    raw = _read_text(path)
    if raw[:4] != b"GSCF":
        raise FileFormatError("not a coefficient file (bad magic)")
    r = _Reader(raw)
    if r.take("<I", "version") != 1:
        raise FileFormatError("unsupported coefficient file version")
    dim = r.take("<I", "dim")
    if dim not in (1, 2):
        raise FileFormatError("coefficient file dim must be 1 or 2")
    tag = r.take("<B", "family tag")
    if tag == 0:
        family = "haar"
    elif 2 <= tag <= 8:
        family = f"db{tag}"
    else:
        raise FileFormatError(f"unknown family tag {tag}")
    J = r.take("<I", "J")
    if J < 0 or dim * J > 26:
        raise FileFormatError("coefficient file scale out of range")
    count = 1 << (dim * J)
    return CoefficientFile(dim, family, J, r.doubles(2 * count, "coefficients").view(np.complex128).copy())


# ------------------------------------------------------------------ evaluations (io.cpp:277-297)
def write_evaluation_csv(path, ev) -> None:
    """1D: header x,value; x = i / 2^R - 1/2."""
    if ev.dim != 1:
        raise ShapeError("CSV evaluation output is 1D only")
    vals = np.asarray(ev.values, dtype=np.float64).ravel()
    with _open_out(path, False) as out:
        out.write("x,value\n")
        for i, v in enumerate(vals[: ev.points_per_axis()]):
            out.write(f"{_fmt(i * 2.0 ** -ev.resolution - 0.5)},{_fmt(v)}\n")


def write_evaluation_pgm(path, ev) -> None:
    """2D: binary 16-bit big-endian PGM, value range in the comment line."""
    if ev.dim != 2:
        raise ShapeError("PGM evaluation output is 2D only")
    vals = np.asarray(ev.values, dtype=np.float64).ravel()
    g = ev.points_per_axis()
    lo, hi = float(vals.min()), float(vals.max())
    scale = 65535.0 / (hi - lo) if hi > lo else 0.0
    t = (vals - lo) * scale  # std::lround: half away from zero
    words = (np.sign(t) * np.floor(np.abs(t) + 0.5)).astype(np.int64).astype(">u2")
    with _open_out(path, True) as out:
        out.write(f"P5\n# min {_fmt(lo)} max {_fmt(hi)}\n{g} {g}\n65535\n".encode())
        out.write(words.tobytes())


# ------------------------------------------------------------------ weight files (io.cpp:299-321)
def write_weight_file(path, mu) -> None:
    with _open_out(path, False) as out:
        out.write("mu\n")
        for v in np.asarray(mu, dtype=np.float64).ravel():
            out.write(_fmt(v) + "\n")


def read_weight_file(path) -> np.ndarray:
    raw = _read_text(path)
    lines = _lines(raw)
    header = next(lines, None)
    if header is None or (header == "" and raw == b""):
        raise FileFormatError("missing header")
    if header != "mu":
        raise FileFormatError(f"bad weight file header: {header}")
    return np.array([_parse(line, "weight file") for line in lines if line], dtype=np.float64)


def require_same_count(samples: SamplingSet, data) -> None:
    """gs_main.cpp:115-117"""
    if np.asarray(data).size != samples.size():
        raise ShapeError("frequency and sample files disagree on the point count")
