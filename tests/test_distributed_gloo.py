"""Sample-sharded CGLS (paper_1607_04091_b200/distributed.py, SURVEY 8(e) C4
row) on CPU: world_size 2 over gloo, each rank owning half of the samples of a
weighted 2D db4 problem with the oracle as its local operator.  The sharded
iterate must equal the single-process solve (solver.cpp:19-91) to roundoff,
with the same residual history and iteration count."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    c = oracle.gen_jitter(24, 0.5, 0.2, 4242, 2)
    K = float(np.max(np.abs(c)))
    mu = oracle.voronoi(2, c, K)
    rng = np.random.default_rng(7)
    M = c.size // 2
    b = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    return c, mu, K, b


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1607_04091_b200.distributed import cgls_sharded, shard_range, torch_collectives
    c, mu, K, b = _problem()
    M = c.size // 2
    lo, hi = shard_range(M, rank, world)
    op = oracle.Op(2, 4, 4, c[2 * lo:2 * hi], weights=mu[lo:hi], bandwidth=K)
    b_loc = torch.from_numpy(np.sqrt(mu[lo:hi]) * b[lo:hi])
    fwd = lambda x: torch.from_numpy(op.forward(x.numpy()))  # noqa: E731
    adj = lambda y: torch.from_numpy(op.adjoint(y.numpy()))  # noqa: E731
    allreduce_sum, norm2 = torch_collectives()
    x0 = torch.zeros(op.cols, dtype=torch.complex128)
    x, st = cgls_sharded(fwd, adj, b_loc, x0, allreduce_sum, norm2, 12, 1e-300)
    if rank == 0:
        q.put((x.numpy(), st.iterations, list(st.history)))
    dist.destroy_process_group()


def test_sharded_cgls_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    x, its, hist = q.get(timeout=300)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    c, mu, K, b = _problem()
    ref = oracle.Op(2, 4, 4, c, weights=mu, bandwidth=K)
    xr, sr = ref.solve(b, max_iterations=12, tolerance=1e-300)
    assert its == sr["iterations"] == 12
    assert oracle.rel_error(x, xr) < 1e-10
    assert np.allclose(hist, sr["history"], rtol=1e-9)
