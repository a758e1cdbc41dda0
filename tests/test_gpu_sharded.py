"""Sample-sharded CGLS in the library: the
loop stays on the GPU and the two per-iteration sums (||q||^2 and the
adjoint partials T_g* r_g) are NCCL allreduces the library issues on its
stream.  One GPU here: a world-size-1 communicator runs the same code path
(the NCCL sum of one rank is the identity), checked against the oracle and
the unsharded solve; the row-block decomposition itself (sum of the shards'
adjoints = the full adjoint) is checked with two shard operators on the
same GPU.  The multi-rank plumbing is covered on CPU (tests/test_distributed_gloo.py)."""
import math

import numpy as np
import pytest

import oracle
from oracle import rel_error

pytestmark = pytest.mark.gpu


def rc(n, rng):
    return (rng.standard_normal(n) + 1j * rng.standard_normal(n)) / math.sqrt(2)


def spiral_problem():
    c = oracle.gen_spiral(16, 256.0, 32.0)  # 4096 points, C4 geometry at 1/256 the size
    mu = oracle.voronoi(2, c, 32.0)
    return c, mu


def test_sharded_world1_matches_oracle_and_unsharded():
    import paper_1607_04091_b200 as gs
    from paper_1607_04091_b200.distributed import Communicator, ShardedSession, solve_least_squares_sharded
    rng = np.random.default_rng(3)
    c, mu = spiral_problem()
    ref = oracle.Op(2, 4, 5, c, weights=mu, bandwidth=32.0)
    raw = oracle.Op(2, 4, 5, c, bandwidth=32.0).forward(rc(1024, rng)) + 1e-3 * rc(c.size // 2, rng)
    op = gs.freq2wave(gs.SamplingSet(2, c), "db4", 5, bandwidth=32.0, weights=mu)
    comm = Communicator(1, 0, Communicator.unique_id(), device=0)
    xs, st = solve_least_squares_sharded(op, comm, raw, max_iterations=15, tolerance=1e-300)
    xu, su = gs.solve_least_squares(op, raw, max_iterations=15, tolerance=1e-300)
    xr, sr = ref.solve(raw, max_iterations=15, tolerance=1e-300)
    e_ref, e_uns = rel_error(xs, xr), rel_error(xs, xu)
    print(f"sharded(world 1) vs oracle {e_ref:.2e}, vs unsharded {e_uns:.2e}")
    assert st.iterations == 15 and e_ref <= 1e-8 and e_uns <= 1e-10
    assert np.allclose(st.history, sr["history"], rtol=1e-6)
    # split session: begin / step / result
    s = ShardedSession(op, comm, raw, history_capacity=20)
    s.step(15)
    xb, sb = s.result()
    assert rel_error(xb, xs) <= 1e-14
    comm.close()


def test_row_blocks_sum_to_the_operator():
    """T* r = sum_g T_g* r_g and T p = [T_g p] for two contiguous shards."""
    import paper_1607_04091_b200 as gs
    from paper_1607_04091_b200.distributed import shard_range
    rng = np.random.default_rng(4)
    c, mu = spiral_problem()
    M = c.size // 2
    full = gs.freq2wave(gs.SamplingSet(2, c), "db4", 5, bandwidth=32.0, weights=mu)
    r, p = rc(M, rng), rc(1024, rng)
    parts, rows = [], []
    for g in range(2):
        lo, hi = shard_range(M, g, 2)
        sh = gs.freq2wave(gs.SamplingSet(2, c[2 * lo:2 * hi]), "db4", 5, bandwidth=32.0, weights=mu[lo:hi])
        parts.append(gs.apply_adjoint(sh, r[lo:hi]))
        rows.append(gs.apply_forward(sh, p))
    assert rel_error(parts[0] + parts[1], gs.apply_adjoint(full, r)) <= 1e-13
    assert rel_error(np.concatenate(rows), gs.apply_forward(full, p)) <= 1e-13
