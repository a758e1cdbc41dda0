"""Input harness vs the oracle: the reference's pattern generators reproduce
bit-for-bit, and the fast exact Voronoi weights equal the reference's
O(M^2) half-plane clipping (weights.cpp:59-70) to roundoff."""
import numpy as np
import pytest

import oracle


def inp():
    from paper_1607_04091_b200 import inputs
    return inputs


def test_patterns_bit_identical():
    I = inp()
    assert np.array_equal(I.gen_grid(1024, 1.0), oracle.gen_grid(1024, 1.0))
    assert np.array_equal(I.gen_grid(16, 0.5, 2), oracle.gen_grid(16, 0.5, 2))
    assert np.array_equal(I.gen_jitter(4096, 0.5, 0.2, 20160613), oracle.gen_jitter(4096, 0.5, 0.2, 20160613))
    assert np.array_equal(I.gen_jitter(64, 0.5, 0.2, 7, 2), oracle.gen_jitter(64, 0.5, 0.2, 7, 2))
    assert np.array_equal(I.gen_spiral(4, 300.0, 50.0), oracle.gen_spiral(4, 300.0, 50.0))


@pytest.mark.parametrize("case", ["jitter", "spiral", "random"])
def test_fast_voronoi_matches_reference_clipping(case):
    I = inp()
    rng = np.random.default_rng(3)
    if case == "jitter":
        c = oracle.gen_jitter(40, 0.5, 0.2, 99, 2)
    elif case == "spiral":
        c = oracle.gen_spiral(6, 250.0, 40.0)
    else:
        c = rng.uniform(-5, 5, 2 * 1200)
    K = float(np.max(np.abs(c))) * 1.01
    want = oracle.voronoi(2, c, K)
    got = I.voronoi_weights(2, c, K, threads=4)
    assert np.max(np.abs(got - want) / want) < 1e-10
    assert abs(got.sum() - 4 * K * K) < 1e-9 * 4 * K * K


def test_voronoi_1d_and_errors():
    I = inp()
    c = oracle.gen_jitter(4096, 0.5, 0.2, 20160613)
    K = float(np.max(np.abs(c)))
    assert np.allclose(I.voronoi_weights(1, c, K), oracle.voronoi(1, c, K), rtol=0, atol=1e-12)
    import paper_1607_04091_b200 as gs
    with pytest.raises(gs.DomainError):
        I.voronoi_weights(2, np.array([0.0, 0.0, 0.0, 0.0]), 1.0)
    with pytest.raises(gs.DomainError):
        I.voronoi_weights(2, np.array([0.0, 2.0]), 1.0)


def test_oracle_bucketed_voronoi_matches_reference_clip():
    """oracle.voronoi_fast (the CPU legs' weights for the 2^18-2^20-point
    configs) gives the reference loop's cells (weights.cpp:59-70) to roundoff."""
    import numpy as np
    import oracle
    for n, seed in ((17, 3), (40, 11)):
        c = oracle.gen_jitter(n, 0.5, 0.2, seed, 2)
        K = float(np.max(np.abs(c)))
        a, b = oracle.voronoi(2, c, K), oracle.voronoi_fast(2, c, K)
        assert np.max(np.abs(a - b) / a) < 1e-11
    s = oracle.gen_spiral(3, 200.0, 16.0)
    a, b = oracle.voronoi(2, s, 16.0), oracle.voronoi_fast(2, s, 16.0)
    assert np.max(np.abs(a - b) / a) < 1e-11
