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


def test_csr_merge_is_clean_union(oracle):
    """csr_merge(clean CSR, extra edges) == build_clean_edges + from_edges of the concatenation
    (graph.py:183-200; csr_build is pinned to the reference's goldens)."""
    rng = np.random.default_rng(8)
    for _ in range(20):
        n = int(rng.integers(2, 300))
        s1, d1 = rng.integers(0, n, 4 * n), rng.integers(0, n, 4 * n)
        off, tgt, _ = oracle.csr_build(n, s1, d1, clean=True)
        m2 = int(rng.integers(0, 3 * n))
        s2, d2 = rng.integers(0, n, m2), rng.integers(0, n, m2)
        moff, mtgt, mst = oracle.csr_merge(n, off, tgt, s2, d2)
        src = np.concatenate([np.repeat(np.arange(n), np.diff(off)), s2])
        dst = np.concatenate([tgt, d2])
        coff, ctgt, cst = oracle.csr_build(n, src, dst, clean=True)
        assert np.array_equal(moff, coff) and np.array_equal(mtgt, ctgt)
        assert mst[0] == cst[0] and mst[2] == int((s2 == d2).sum())
        assert mst[1] == m2 - mst[2] - (cst[0] - tgt.size)


@pytest.mark.parametrize("kind,n,seed", [("uniform", 10_000, 1234), ("web8", 200_000, 2), ("web16", 200_000, 0)])
def test_exact_size_generator(oracle, kind, n, seed):
    """Fill rounds redraw the slots cleaning dropped until the configured out-degrees exist as
    distinct edges (ref gen.py:66-110 draws until the target count of distinct links exists);
    the result is the clean build of all draws, every round reproducible from its streams."""
    cfg = {"uniform": oracle.uniform_config(10), "web8": oracle.web_config(8.0),
           "web16": oracle.web_config(16.0)}[kind]
    off, tgt, rep = oracle.gen_graph_exact(cfg, n, seed)
    deg, total = oracle.gen_degrees(cfg, n, seed)
    got = np.diff(off)
    assert np.all(got <= deg) and rep["target_links"] == total
    assert rep["unfilled"] == total - tgt.size <= 1e-3 * total
    src = np.repeat(np.arange(n, dtype=np.uint32), got)
    assert not np.any(src == tgt)
    # rows strictly ascending (unique)
    assert np.all((np.diff(tgt.astype(np.int64)) > 0) | (np.diff(src.astype(np.int64)) > 0))
    # replay: the union of every round's draws, cleaned once, is the same graph
    s0, d0 = oracle.gen_edges_round(cfg, n, seed, 0, deg)
    o, t, _ = oracle.csr_build(n, s0, d0, clean=True)
    allsrc, alldst = [s0], [d0]
    for r in range(1, rep["rounds"] + 1):
        deficit = (deg.astype(np.int64) - np.diff(o)).astype(np.uint32)
        sr, dr = oracle.gen_edges_round(cfg, n, seed, r, deficit, o, t)
        allsrc.append(sr)
        alldst.append(dr)
        o, t, _ = oracle.csr_merge(n, o, t, sr, dr)
    co, ct, _ = oracle.csr_build(n, np.concatenate(allsrc), np.concatenate(alldst), clean=True)
    assert np.array_equal(co, off) and np.array_equal(ct, tgt)
