"""Generate the CGLS config-parity fixtures (tests/golden/cgls_*.npz).

The oracle (oracle/gs_oracle.cpp, test infrastructure) runs each config's own
CGLS iteration count on the config's seeded inputs (harness
conventions of bench.py: problem_inputs / coeffs_and_noise) with the
tol = 1e-300 idiom of the reference's test_solver.cpp:46, so the iterate after
exactly K iterations (solver.cpp:70-88) is what the GPU must reproduce.

Stored per config (tests/test_gpu_cgls_configs.py reads them; the oracle is
not run at test time -- C4 takes ~25 min on one core):
  x        the oracle iterate after K iterations (complex128, full)
  history  its relative normal-equation residual per iteration (K + 1)
  b_idx / b_val / b_norm   a sample of the oracle's data vector b = T x_true
           + noise and its norm (the GPU test builds b with its own T and
           checks it against these first)
  coords_sha / weights_sha  SHA-256 of the input arrays (the GPU box rebuilds
           them with the same generators; identical bytes are asserted)
  sens     ||x_K(b (1 + 1e-15 r)) - x_K(b)|| / ||x_K(b)||: how far the
           oracle's own iterate moves under a roundoff-sized data
           perturbation (the CG roundoff floor of the problem)

Usage: python tools/gen_cgls_fixtures.py c3 | c4 | c5:0 | c5:85 | ...
(each config in its own process; they are independent).
      python tools/gen_cgls_fixtures.py --checkpoints 10,25,50 c4
stores the oracle iterates after those (shorter) iteration counts instead
(cgls_c4_ckpt.npz): how the GPU / oracle gap grows with the iteration count
on an ill-conditioned config.
"""
import hashlib
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (harness: inputs, seeds, iteration counts)
import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def b_sample_idx(M):
    head = np.arange(min(64, M))
    stride = np.linspace(0, M - 1, 1024).astype(np.int64)
    return np.unique(np.concatenate([head, stride]))


def checkpoints(spec, ks):
    workload, _, b = spec.partition(":")
    b = int(b or 0)
    t0 = time.time()
    dim, p, J, c, mu, bw, sig = bench.problem_inputs(workload, b, bench.ProductGen())
    op_u = oracle.Op(dim, p, J, c, bandwidth=bw)
    x_true, noise = bench.coeffs_and_noise(b, op_u.cols, op_u.rows, sig)
    data = op_u.forward(x_true) + noise
    del op_u
    op = oracle.Op(dim, p, J, c, weights=mu, bandwidth=bw)
    res = {}

    def run(k):
        res[k] = op.solve(data, max_iterations=k, tolerance=1e-300)[0]

    ths = [threading.Thread(target=run, args=(k,)) for k in ks]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    name = f"cgls_{workload}_ckpt.npz"
    np.savez(os.path.join(OUT, name), iters=np.array(ks), **{f"x{k}": res[k] for k in ks})
    print(f"{spec}: checkpoints {ks} in {time.time() - t0:.0f} s -> {name}", flush=True)


def op_sensitivity(spec):
    """The oracle's iterate moved by a last-bit perturbation of the OPERATOR:
    the Voronoi weights mu (folded into the rows as sqrt(mu)) scaled by
    (1 + 2^-52 r), r = +-1 -- a 1-ulp change of every row of T, the size of
    the rounding differences between any two implementations of T."""
    workload, _, b = spec.partition(":")
    b = int(b or 0)
    iters = bench.CONFIG_ITERS[workload]
    t0 = time.time()
    dim, p, J, c, mu, bw, sig = bench.problem_inputs(workload, b, bench.ProductGen())
    op_u = oracle.Op(dim, p, J, c, bandwidth=bw)
    x_true, noise = bench.coeffs_and_noise(b, op_u.cols, op_u.rows, sig)
    data = op_u.forward(x_true) + noise
    del op_u
    rng = np.random.default_rng(2)
    mu2 = mu * (1 + 2.0 ** -52 * rng.choice([-1.0, 1.0], mu.size))
    res = {}

    def run(key, m):
        res[key] = oracle.Op(dim, p, J, c, weights=m, bandwidth=bw).solve(data, max_iterations=iters,
                                                                          tolerance=1e-300)[0]

    ths = [threading.Thread(target=run, args=("a", mu)), threading.Thread(target=run, args=("b", mu2))]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    name = f"cgls_{workload}_opsens.npz"
    sens = oracle.rel_error(res["b"], res["a"])
    np.savez(os.path.join(OUT, name), sens_op=sens, iters=iters)
    print(f"{spec}: operator sensitivity (1-ulp row weights) after {iters} iterations {sens:.3e}, "
          f"{time.time() - t0:.0f} s -> {name}", flush=True)


def main(spec):
    workload, _, b = spec.partition(":")
    b = int(b or 0)
    iters = bench.CONFIG_ITERS[workload]
    t0 = time.time()
    dim, p, J, c, mu, bw, sig = bench.problem_inputs(workload, b, bench.ProductGen())
    op_u = oracle.Op(dim, p, J, c, bandwidth=bw)
    x_true, noise = bench.coeffs_and_noise(b, op_u.cols, op_u.rows, sig)
    data = op_u.forward(x_true) + noise
    del op_u
    op = oracle.Op(dim, p, J, c, weights=mu, bandwidth=bw)
    print(f"{spec}: inputs + operators {time.time() - t0:.0f} s", flush=True)
    rng = np.random.default_rng(1)
    pert = data * (1 + 1e-15 * (rng.standard_normal(data.size) + 1j * rng.standard_normal(data.size)))
    res = {}

    def run(key, rhs):
        res[key] = op.solve(rhs, max_iterations=iters, tolerance=1e-300)

    ths = [threading.Thread(target=run, args=("x", data)), threading.Thread(target=run, args=("p", pert))]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    x, st = res["x"]
    xp, _ = res["p"]
    assert st["iterations"] == iters, st["iterations"]
    idx = b_sample_idx(data.size)
    name = f"cgls_{workload}" + (f"_b{b}" if workload == "c5" else "") + ".npz"
    np.savez(os.path.join(OUT, name), x=x, history=np.asarray(st["history"]), b_idx=idx, b_val=data[idx],
             b_norm=np.linalg.norm(data), coords_sha=sha(c), weights_sha=sha(mu) if mu is not None else "",
             sens=oracle.rel_error(xp, x), iters=iters, workload=workload, problem=b,
             x_true_err=oracle.rel_error(x, x_true))
    print(f"{spec}: {iters} iterations, sens {oracle.rel_error(xp, x):.2e}, |x-x_true|/|x_true| "
          f"{oracle.rel_error(x, x_true):.2e}, total {time.time() - t0:.0f} s -> {name}", flush=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--op-sensitivity":
        for s in args[1:]:
            op_sensitivity(s)
    elif args and args[0] == "--checkpoints":
        ks = [int(v) for v in args[1].split(",")]
        for s in args[2:]:
            checkpoints(s, ks)
    else:
        for s in args:
            main(s)
