"""GPU checks of the command-line front end: `gs reconstruct`
writes the coefficient file + stats sidecar of gs_main.cpp:108-171 with the
GPU solve, whose iterate matches the oracle's solve on the same files; `gs
bench` runs a registry problem (bench.cpp) and appends the reference's CSV
record."""
import json

import numpy as np
import pytest

import oracle
from oracle import rel_error

pytestmark = pytest.mark.gpu


def test_cli_reconstruct_matches_oracle_solve(tmp_path, capsys):
    import paper_1607_04091_b200 as gs
    from paper_1607_04091_b200 import cli, inputs
    from paper_1607_04091_b200 import io as gsio
    f, y, c = str(tmp_path / "f.bin"), str(tmp_path / "y.bin"), str(tmp_path / "c.gscf")
    assert cli.main(["gen", "jitter", "--M", "512", "--epsilon", "0.5", "--eta", "0.2", "--seed", "11",
                     "-o", f, "--format", "bin", "--truncated-cosine-samples", y]) == 0
    capsys.readouterr()
    s = gsio.read_frequency_file(f)
    K = float(np.max(np.abs(s.coords))) + 0.25
    rc = cli.main(["reconstruct", f, y, "--family", "db2", "--scale-J", "6", "--bandwidth", repr(K),
                   "--max-iter", "25", "--tol", "1e-300", "-o", c])
    assert rc == 6  # tol 1e-300 never converges: exit code of a non-converged solve (gs_main.cpp:170)
    out = capsys.readouterr().out
    assert out.startswith("iterations 25 residual") and out.strip().endswith("(not converged)")
    cf = gsio.read_coefficient_file(c)
    assert (cf.dim, cf.family, cf.J, cf.values.size) == (1, "db2", 6, 64)
    side = json.load(open(c + ".stats.json"))
    assert side["iterations"] == 25 and side["weighted"] is True and side["converged"] is False
    # oracle on the same files: weighted (auto: bandwidth given, non-uniform points)
    mu = inputs.voronoi_weights(1, s.coords, K)
    ref = oracle.Op(1, 2, 6, s.coords, weights=mu, bandwidth=K)
    xr, sr = ref.solve(gsio.read_sample_file(y), max_iterations=25, tolerance=1e-300)
    assert sr["iterations"] == 25
    assert rel_error(cf.values, xr) <= 1e-8


def test_cli_reconstruct_converges_on_uniform_haar(tmp_path, capsys):
    from paper_1607_04091_b200 import cli
    from paper_1607_04091_b200 import io as gsio
    f, y, c = str(tmp_path / "f.csv"), str(tmp_path / "y.csv"), str(tmp_path / "c.gscf")
    assert cli.main(["gen", "grid", "--M", "1024", "--epsilon", "1", "-o", f,
                     "--truncated-cosine-samples", y]) == 0
    assert cli.main(["reconstruct", f, y, "--family", "haar", "--scale-J", "9", "--bandwidth", "512",
                     "-o", c]) == 0  # uniform grid -> unweighted, exact uniform route, converges (C1 recipe)
    side = json.load(open(c + ".stats.json"))
    assert side["converged"] is True and side["weighted"] is False and side["iterations"] <= 10
    assert gsio.read_coefficient_file(c).values.size == 512
    capsys.readouterr()


def test_cli_bench_appends_reference_csv_record(tmp_path, capsys):
    from paper_1607_04091_b200 import cli
    rep = str(tmp_path / "bench.csv")
    assert cli.main(["bench", "jitter1d", "--scale", "0.25", "--repeats", "1", "--report", rep]) == 0
    line = capsys.readouterr().out.strip()
    assert line.startswith("jitter1d ") and " init " in line and " s/iter " in line
    rows = open(rep).read().splitlines()
    assert rows[0] == "problem,rows,cols,init_seconds,solve_seconds,iterations,seconds_per_iteration"
    fields = rows[1].split(",")
    assert fields[0] == "jitter1d" and int(fields[1]) == round(5463 * 0.25) and int(fields[2]) == 512
    assert int(fields[5]) > 0
