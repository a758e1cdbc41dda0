"""GPU dyadic evaluation against the oracle's restatement of
dyadic.cpp (pinned by tests/test_oracle_dyadic.py): refinement tables of the
interior and edge functions, weval_1d / weval_2d, validation error classes,
device-tensor inputs and the `gs evaluate` CSV / PGM outputs.  Floating-point
bar: max |GPU - oracle| <= 1e-13 x max |oracle| (the cascade and the
contractions are the same sums in a different order)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
TOL = 1e-13


def close(got, want, tol=TOL):
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape
    scale = max(1.0, float(np.max(np.abs(want)))) if want.size else 1.0
    err = float(np.max(np.abs(got - want))) if want.size else 0.0
    assert err <= tol * scale, err


@pytest.mark.parametrize("p", range(1, 9))
def test_scaling_tables_match_oracle(p):
    from paper_1607_04091_b200 import dyadic
    t = dyadic.evaluate_scaling_dyadic(p, 9)
    r = oracle.scaling_dyadic(p, 9)
    assert t.support_begin == r.support_begin
    close(t.values, r.values)


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("side", ["left", "right"])
def test_boundary_tables_match_oracle(p, side):
    from paper_1607_04091_b200 import dyadic
    tabs = dyadic.evaluate_boundary_dyadic(p, side, 7)
    ref = oracle.boundary_dyadic(p, side == "left", 7)
    for t, r in zip(tabs, ref):
        assert t.support_begin == r.support_begin
        close(t.values, r.values)


@pytest.mark.parametrize("p,J,R", [(1, 4, 8), (2, 5, 10), (3, 4, 7), (4, 6, 9), (8, 5, 8)])
def test_weval_1d_matches_oracle(p, J, R):
    from paper_1607_04091_b200 import dyadic
    rng = np.random.default_rng(p * 100 + J)
    c = rng.uniform(-1, 1, 1 << J)
    c[3] = 0.0  # zero weights are skipped (dyadic.cpp:193)
    ev = dyadic.weval_1d(c, p, J, R)
    assert ev.values.size == (1 << R) + 1 and ev.points_per_axis() == (1 << R) + 1
    close(ev.values, oracle.weval(1, p, J, R, c))


@pytest.mark.parametrize("p,J,R", [(1, 3, 6), (2, 4, 7), (4, 4, 8), (4, 6, 9)])
def test_weval_2d_matches_oracle(p, J, R):
    from paper_1607_04091_b200 import dyadic
    rng = np.random.default_rng(p * 7 + J)
    n = 1 << J
    c = rng.uniform(-1, 1, n * n)
    ev = dyadic.weval_2d(c, p, J, R)
    close(ev.values, oracle.weval(2, p, J, R, c))


def test_weval_device_tensors_and_validation():
    import torch
    import paper_1607_04091_b200 as gs
    from paper_1607_04091_b200 import dyadic
    c = torch.linspace(-1, 1, 64, dtype=torch.float64, device="cuda")
    ev = dyadic.weval_1d(c, "db4", 6, 9)
    assert ev.values.is_cuda
    close(ev.values.cpu().numpy(), oracle.weval(1, 4, 6, 9, c.cpu().numpy()))
    with pytest.raises(gs.DomainError):
        dyadic.weval_1d(np.zeros(32), "db2", 5, 4)     # R < J
    with pytest.raises(gs.ShapeError):
        dyadic.weval_1d(np.zeros(32), "db2", 4, 8)     # wrong length
    with pytest.raises(gs.DomainError):
        dyadic.weval_1d(np.zeros(2), "db2", 1, 4)      # 2^J < 2p
    with pytest.raises(gs.DomainError):
        dyadic.evaluate_boundary_dyadic("haar", "left", 4)
    assert np.all(dyadic.weval_2d(np.zeros(256), "db2", 4, 6).values == 0.0)


def test_cli_evaluate_csv_and_pgm(tmp_path, capsys):
    from paper_1607_04091_b200 import cli
    from paper_1607_04091_b200 import io as gsio
    rng = np.random.default_rng(3)
    c1 = rng.uniform(-1, 1, 32) + 1j * rng.uniform(-1, 1, 32)
    gsio.write_coefficient_file(tmp_path / "c1", gsio.CoefficientFile(1, "db2", 5, c1))
    assert cli.main(["evaluate", str(tmp_path / "c1"), "--resolution", "8", "-o", str(tmp_path / "e.csv")]) == 0
    rows = (tmp_path / "e.csv").read_text().splitlines()
    assert rows[0] == "x,value" and len(rows) == 1 + 257 and rows[1].startswith("-0.5,")
    vals = np.array([float(r.split(",")[1]) for r in rows[1:]])
    close(vals, oracle.weval(1, 2, 5, 8, c1.real))
    c2 = rng.uniform(-1, 1, 256).astype(np.complex128)
    gsio.write_coefficient_file(tmp_path / "c2", gsio.CoefficientFile(2, "db4", 4, c2))
    assert cli.main(["evaluate", str(tmp_path / "c2"), "--resolution", "6", "-o", str(tmp_path / "e.pgm")]) == 0
    raw = (tmp_path / "e.pgm").read_bytes()
    head, _, rest = raw.partition(b"\n65535\n")
    lines = head.split(b"\n")
    assert lines[0] == b"P5" and lines[1].startswith(b"# min ") and lines[2] == b"65 65"
    words = np.frombuffer(rest, ">u2")
    ref = oracle.weval(2, 4, 4, 6, c2.real)
    want = np.floor((ref - ref.min()) * (65535.0 / (ref.max() - ref.min())) + 0.5)
    assert words.size == 65 * 65 and np.max(np.abs(words - want)) <= 1
    capsys.readouterr()
