"""GPU Voronoi density-compensation weights: the 2D cells on
the device equal the host harness's bit for bit (same routine, no FMA
contraction) at the C5 input size and on a C4-geometry spiral, and the reference's O(M^2) clip
(oracle restatement of weights.cpp:59-70) to roundoff on small sets; the
reference's input checks (range, duplicates) raise DomainError."""
import time

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def test_gpu_weights_equal_host_at_config_sizes():
    from paper_1607_04091_b200 import inputs
    import bench
    # C5 at full size; the C4 spiral geometry at 1/16 of its points (its dense
    # arms make the full 2^20-point case a minutes-long host fallback)
    for name, c, K in (("C5 problem 0", oracle.gen_jitter(512, 0.5, 0.2, bench.SEED, 2), None),
                       ("spiral (C4 geometry, 2^16 points)", oracle.gen_spiral(16, 4096.0, 128.0), 128.0)):
        K = K or float(np.max(np.abs(c)))
        t = time.perf_counter()
        g = inputs.voronoi_weights(2, c, K, device=0)
        tg = time.perf_counter() - t
        t = time.perf_counter()
        h = inputs.voronoi_weights(2, c, K)
        th = time.perf_counter() - t
        print(f"{name}: {c.size // 2} cells, GPU {tg:.3f} s, host {th:.3f} s, identical {np.array_equal(g, h)}")
        assert np.array_equal(g, h)


def test_gpu_weights_vs_reference_clip_and_checks():
    from paper_1607_04091_b200 import DomainError, inputs
    for n, seed in ((20, 1), (33, 2)):
        c = oracle.gen_jitter(n, 0.5, 0.2, seed, 2)
        K = float(np.max(np.abs(c)))
        a, b = oracle.voronoi(2, c, K), inputs.voronoi_weights(2, c, K, device=0)
        assert np.max(np.abs(a - b) / a) < 1e-11
    with pytest.raises(DomainError):
        inputs.voronoi_weights(2, np.array([0.0, 0.0, 0.0, 0.0]), 1.0, device=0)
    with pytest.raises(DomainError):
        inputs.voronoi_weights(2, np.array([0.0, 0.0, 2.0, 0.0]), 1.0, device=0)
