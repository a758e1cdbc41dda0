"""Command-line front end over the GPU operator: the `gs`
subcommands of tools/gs_main.cpp with the same options, files, printed lines,
sidecar JSON and exit codes, routed through this package's C-ABI
(``python -m paper_1607_04091_b200 <command> ...``).

    gen          sampling pattern -> frequency file       (gs_main.cpp:44-66)
    weights      Voronoi weights + density report          (gs_main.cpp:74-84)
    reconstruct  least-squares reconstruction on the GPU   (gs_main.cpp:108-171)
    evaluate     coefficients on a dyadic grid (GPU)       (gs_main.cpp:179-198)
    bench        registry benchmark problem on the GPU     (gs_main.cpp:205-213,
                                                            bench.cpp:40-150)
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

from . import (DomainError, Error, Freq2WaveOptions, SamplingSet, ShapeError, SolveOptions, UsageError,
               apply_forward, family_p, freq2wave, solve_least_squares)
from . import inputs
from . import io as gsio


def _format(name: str) -> str:
    if name == "csv":
        return "csv"
    if name in ("bin", "binary"):
        return "binary"
    raise UsageError(f"unknown format: {name}")


# ------------------------------------------------------------------ gen
def cmd_gen(a) -> int:
    if a.kind == "grid":
        s = SamplingSet(a.dim, inputs.gen_grid(a.M, a.epsilon, a.dim))
    elif a.kind == "jitter":
        s = SamplingSet(a.dim, inputs.gen_jitter(a.M, a.epsilon, a.eta, a.seed, a.dim))
    elif a.kind == "spiral":
        ppt = a.points_per_turn
        if ppt <= 0 and a.M > 0:
            ppt = a.M / a.turns
        s = SamplingSet(2, inputs.gen_spiral(a.turns, ppt, a.bandwidth))
    else:
        raise UsageError(f"unknown pattern kind: {a.kind}")
    fmt = _format(a.format)
    gsio.write_frequency_file(a.output, s, fmt)
    if a.truncated_cosine_samples:
        if s.dim != 1:
            raise ShapeError("truncated cosine samples are 1D only")
        gsio.write_sample_file(a.truncated_cosine_samples, inputs.truncated_cosine_transform(s.coords), fmt)
    print(f"wrote {s.size()} points to {a.output}")
    return 0


# ------------------------------------------------------------------ weights
def cmd_weights(a) -> int:
    s = gsio.read_frequency_file(a.freq_file)
    mu = inputs.voronoi_weights(s.dim, s.coords, a.bandwidth)
    rep = inputs.density(s.dim, s.coords, a.bandwidth)
    if a.output:
        gsio.write_weight_file(a.output, mu)
    print("delta_raw %.12g" % rep.delta_raw)
    print("delta_scaled %.12g" % rep.delta_scaled)
    print("quarter_bound %s" % ("satisfied" if rep.satisfies_quarter_bound else "violated"))
    return 0


# ------------------------------------------------------------------ reconstruct
def _is_uniformish(s: SamplingSet) -> bool:
    """gs_main.cpp:98-106"""
    if s.dim != 1 or s.size() < 3:
        return False
    c = s.coords
    gap = c[1] - c[0]
    return bool(np.all(np.abs((c[2:] - c[1:-1]) - gap) <= 1e-12))


def cmd_reconstruct(a) -> int:
    if a.weighted and a.unweighted:
        raise UsageError("--weighted and --unweighted are mutually exclusive")
    s = gsio.read_frequency_file(a.freq_file)
    data = gsio.read_sample_file(a.sample_file)
    gsio.require_same_count(s, data)
    family_p(a.family)  # DomainError for an unknown family, before any work
    weighted = (a.bandwidth is not None and not _is_uniformish(s)) if not (a.weighted or a.unweighted) \
        else bool(a.weighted)
    opt = Freq2WaveOptions(bandwidth=a.bandwidth)
    if weighted:
        region = a.bandwidth if a.bandwidth is not None else 0.0
        if region <= 0.0:
            region = float(np.max(np.abs(s.coords)))
        opt.weights = inputs.voronoi_weights(s.dim, s.coords, region)
    t0 = time.perf_counter()
    op = freq2wave(s, a.family, a.scale_J, opt)
    init_seconds = time.perf_counter() - t0
    t0 = time.perf_counter()
    x, st = solve_least_squares(op, data, SolveOptions(max_iterations=a.max_iter, tolerance=a.tol))
    solve_seconds = time.perf_counter() - t0
    gsio.write_coefficient_file(a.output, gsio.CoefficientFile(s.dim, a.family, a.scale_J, x))
    side = {"iterations": st.iterations, "converged": st.converged, "residual": st.residual,
            "weighted": weighted, "init_seconds": init_seconds, "solve_seconds": solve_seconds}
    with open(a.output + ".stats.json", "w") as f:
        f.write(json.dumps(side, indent=2) + "\n")
    print(f"iterations {st.iterations} residual {st.residual:g}" + ("" if st.converged else " (not converged)"))
    return 0 if st.converged else 6


# ------------------------------------------------------------------ bench (bench.cpp)
# name, dim, family, J, pattern, m_param, epsilon, eta, turns, bandwidth (bench.cpp:40-50)
REGISTRY = [
    ("uniform1d", 1, "db4", 12, "uniform", 8192, 0.5, 0.0, 0, 0.0),
    ("jitter1d", 1, "db4", 11, "jitter", 5463, 0.36, 0.09, 0, 0.0),
    ("uniform2d", 2, "db4", 8, "uniform", 512, 0.5, 0.0, 0, 0.0),
    ("jitter2d", 2, "db4", 5, "jitter", 162, 0.19, 0.045, 0, 0.0),
    ("spiral", 2, "db4", 5, "spiral", 27681, 0.0, 0.0, 27, 15.8),
]


def bench_sampling_set(problem, scale: float, seed: int):
    """bench.cpp:53-80 -> (SamplingSet, J)"""
    name, dim, fam, J0, pattern, m_param, eps0, eta0, turns, bw = problem
    if not (scale > 0):
        raise DomainError("scale must be positive")
    J = J0 + int(_llround(math.log2(scale)))
    n_old, n_new = 1 << J0, 1 << J
    m = int(_llround(m_param * scale))
    if m < 1:
        raise DomainError("scale leaves no sample points")
    shrink = n_new / n_old
    if pattern == "uniform":
        eps = eps0 * (m_param / m) * shrink
        return SamplingSet(dim, inputs.gen_grid(m, eps, dim)), J
    if pattern == "jitter":
        eps = eps0 * (m_param / m) * shrink
        eta = eta0 * (eps / eps0)
        return SamplingSet(dim, inputs.gen_jitter(m, eps, eta, seed, dim)), J
    ppt = m / turns
    return SamplingSet(2, inputs.gen_spiral(turns, ppt, bw * shrink)), J


def _llround(v: float) -> int:
    return int(math.floor(v + 0.5)) if v >= 0 else -int(math.floor(-v + 0.5))


def run_bench(name: str, scale=1.0, seed=20160613, warmups=1, repeats=5, solve_options=None):
    """bench.cpp:82-136: median init / solve seconds over `repeats` rounds."""
    prob = next((p for p in REGISTRY if p[0] == name), None)
    if prob is None:
        raise DomainError(f"unknown benchmark problem: {name}")
    if repeats < 1:
        raise DomainError("repeats must be >= 1")
    s, J = bench_sampling_set(prob, scale, seed)
    inits, solves = [], []
    rec = {"problem": name, "rows": 0, "cols": 0, "iterations": 0}
    for rnd in range(warmups + repeats):
        t0 = time.perf_counter()
        op = freq2wave(s, prob[2], J)
        init = time.perf_counter() - t0
        truth = inputs.seeded_coefficients(op.cols(), seed)
        data = apply_forward(op, truth)
        t0 = time.perf_counter()
        _, st = solve_least_squares(op, data, solve_options)
        solve = time.perf_counter() - t0
        if rnd >= warmups:
            inits.append(init)
            solves.append(solve)
            rec["iterations"] = st.iterations
        rec["rows"], rec["cols"] = op.rows(), op.cols()
        op.close()
    rec["init_seconds"] = float(np.median(inits))
    rec["solve_seconds"] = float(np.median(solves))
    rec["seconds_per_iteration"] = rec["solve_seconds"] / rec["iterations"] if rec["iterations"] > 0 else 0.0
    return rec


def append_bench_csv(path, rec) -> None:
    """bench.cpp:138-150"""
    fresh = not os.path.exists(path) or os.path.getsize(path) == 0
    try:
        out = open(path, "a")
    except OSError:
        from . import FileFormatError
        raise FileFormatError(f"cannot open bench report: {path}") from None
    with out:
        if fresh:
            out.write("problem,rows,cols,init_seconds,solve_seconds,iterations,seconds_per_iteration\n")
        out.write("%s,%d,%d,%.6f,%.6f,%d,%.6f\n" % (rec["problem"], rec["rows"], rec["cols"], rec["init_seconds"],
                                                   rec["solve_seconds"], rec["iterations"],
                                                   rec["seconds_per_iteration"]))


def cmd_bench(a) -> int:
    rec = run_bench(a.problem, a.scale, a.seed, 1, a.repeats)
    append_bench_csv(a.report, rec)
    print("%s %dx%d init %.3fs solve %.3fs iters %d s/iter %.4f" % (
        rec["problem"], rec["rows"], rec["cols"], rec["init_seconds"], rec["solve_seconds"], rec["iterations"],
        rec["seconds_per_iteration"]))
    return 0


def cmd_evaluate(a) -> int:
    """gs_main.cpp:179-198: real part of the coefficients -> weval -> CSV / PGM."""
    from . import dyadic
    cf = gsio.read_coefficient_file(a.coefficient_file)
    real = np.ascontiguousarray(cf.values.real)
    if cf.dim == 1:
        gsio.write_evaluation_csv(a.output, dyadic.weval_1d(real, cf.family, cf.J, a.resolution))
    else:
        gsio.write_evaluation_pgm(a.output, dyadic.weval_2d(real, cf.family, cf.J, a.resolution))
    print(f"wrote {a.output}")
    return 0


# ------------------------------------------------------------------ parser (gs_main.cpp:217-291)
def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="gs", description="generalized sampling pipeline (B200 operator)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("gen", help="generate a sampling pattern")
    g.add_argument("kind", help="grid | jitter | spiral")
    g.add_argument("--M", type=int, default=0)
    g.add_argument("--epsilon", type=float, default=1.0)
    g.add_argument("--eta", type=float, default=0.0)
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("--turns", type=int, default=1)
    g.add_argument("--points-per-turn", type=float, default=0.0)
    g.add_argument("--bandwidth", type=float, default=1.0)
    g.add_argument("--dim", type=int, default=1)
    g.add_argument("-o", "--output", required=True)
    g.add_argument("--format", default="csv")
    g.add_argument("--truncated-cosine-samples", default="")
    w = sub.add_parser("weights", help="Voronoi weights and density")
    w.add_argument("freq_file")
    w.add_argument("--bandwidth", type=float, required=True)
    w.add_argument("-o", "--output", default="")
    r = sub.add_parser("reconstruct", help="least-squares reconstruction")
    r.add_argument("freq_file")
    r.add_argument("sample_file")
    r.add_argument("--family", required=True)
    r.add_argument("--scale-J", type=int, required=True)
    r.add_argument("--bandwidth", type=float, default=None)
    r.add_argument("--weighted", action="store_true")
    r.add_argument("--unweighted", action="store_true")
    r.add_argument("--tol", type=float, default=1e-10)
    r.add_argument("--max-iter", type=int, default=0)
    r.add_argument("-o", "--output", required=True)
    e = sub.add_parser("evaluate", help="evaluate coefficients on a dyadic grid")
    e.add_argument("coefficient_file")
    e.add_argument("--resolution", type=int, required=True)
    e.add_argument("-o", "--output", required=True)
    b = sub.add_parser("bench", help="run a registry benchmark problem")
    b.add_argument("problem", help="uniform1d | jitter1d | uniform2d | jitter2d | spiral")
    b.add_argument("--scale", type=float, default=1.0)
    b.add_argument("--seed", type=int, default=20160613)
    b.add_argument("--repeats", type=int, default=5)
    b.add_argument("--report", default="bench.csv")
    return ap


_CMDS = {"gen": cmd_gen, "weights": cmd_weights, "reconstruct": cmd_reconstruct, "evaluate": cmd_evaluate,
         "bench": cmd_bench}


def main(argv=None) -> int:
    ap = build_parser()
    try:
        a = ap.parse_args(argv)
    except SystemExit as ex:  # CLI11 parse errors exit 2 (gs_main.cpp:281-283)
        return 0 if ex.code == 0 else 2
    try:
        return _CMDS[a.cmd](a)
    except Error as ex:
        print(f"error: {ex}", file=sys.stderr)
        return ex.exit_code
    except Exception as ex:  # gs_main.cpp:287-290
        print(f"error: {ex}", file=sys.stderr)
        return 1
