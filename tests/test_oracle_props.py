"""Oracle self-consistency at sizes the CPU finishes in seconds."""

import numpy as np
import pytest


def test_generator_seed_determinism_and_shape(oracle):
    cfg = oracle.web_config(8.0)
    a = oracle.gen_edges(cfg, 20000, 5)
    b = oracle.gen_edges(cfg, 20000, 5)
    c = oracle.gen_edges(cfg, 20000, 6)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert not np.array_equal(a[1], c[1][: a[1].size]) or a[1].size != c[1].size
    deg, total = oracle.gen_degrees(cfg, 200000, 1)
    assert abs((deg == 0).mean() - 0.15) < 0.01
    assert abs(deg.mean() - 8.0) < 0.3
    assert deg.max() <= 5000 * 3


def test_uniform_generator_profile(oracle):
    deg, total = oracle.gen_degrees(oracle.uniform_config(10), 10000, 3)
    assert deg.max() <= 10 and abs((deg == 0).mean() - 1 / 11) < 0.02
    src, dst = oracle.gen_edges(oracle.uniform_config(10), 10000, 3)
    assert not np.any(src == dst)


@pytest.mark.parametrize("n", [2, 3, 5, 17, 1000, 4097])
def test_feistel_is_a_bijection(oracle, n):
    perm = [oracle.feistel(x, n, 11) for x in range(n)]
    assert sorted(perm) == list(range(n))


def test_parallel_sweep_agrees_with_sequential(oracle):
    cfg = oracle.web_config(8.0)
    src, dst = oracle.gen_edges(cfg, 3000, 9)
    off, tgt, _ = oracle.csr_build(3000, src, dst, clean=True)
    seq = oracle.run_seq(off, tgt, 0.85, 1e-10, "sweep")
    for policy in (0, 1, 2):  # exhaust, geometric, adaptive
        par = oracle.run_psweep(off, tgt, 0.85, 1e-10, policy=policy, decay=0.75 if policy == 2 else 0.5)
        assert np.abs(par.rank - seq.rank).sum() <= 2e-10
        assert par.residual <= 1e-10 * 0.15


def test_signed_resume_in_oracle(oracle):
    """Negative fluid diffuses with the same rule (update.py:77-102 path)."""
    rng = np.random.default_rng(3)
    n = 200
    src = rng.integers(0, n, 800)
    dst = rng.integers(0, n, 800)
    off, tgt, _ = oracle.csr_build(n, src, dst, clean=True)
    f = oracle.init_fluid(n)
    f[::7] *= -1.0
    r = oracle.run_seq(off, tgt, 0.85, 1e-10, "sweep", fluid=f)
    p = oracle.run_psweep(off, tgt, 0.85, 1e-10, fluid=f)
    assert np.abs(r.history - p.history).sum() <= 2e-10
