"""Batched personalized PageRank (BASELINE config 4) against the reference run per column."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,B,k", [(3000, 64, 10), (20_000, 16, 10), (500, 7, 3)])
def test_batched_ppr_matches_per_column_reference(cuda, oracle, n, B, k):
    from paper_1202_6158_b200 import ppr
    src, dst = oracle.gen_edges(oracle.web_config(8.0), n, 5)
    off, tgt, _ = oracle.csr_build(n, src, dst, clean=True)
    g = cuda.SparseGraph(n, off, tgt.astype(np.int32))
    seeds = ppr.config4_seeds(n, B, k, seed=3)
    rank, stats, resid = ppr.personalized_pagerank(g, seeds, target_error=1e-11)
    rank = rank.cpu().numpy()
    assert max(resid) <= 1e-11 * 0.15
    for c in range(B):
        v = np.zeros(n)
        np.add.at(v, seeds[c].astype(np.int64), 1.0 / k)
        ref = oracle.run_seq(off, tgt, 0.85, 1e-13, "sweep", teleport=v).rank
        assert np.abs(rank[:, c] - ref).sum() <= 1e-9, c


def test_batched_ppr_rejects_bad_batch(cuda):
    from paper_1202_6158_b200 import ppr
    g = cuda.SparseGraph.from_edges(3, [0, 1], [1, 2])
    with pytest.raises(ValueError):
        ppr.BatchedPPR(g, 65)
    with pytest.raises(ValueError):
        ppr.BatchedPPR(g, 2, mode="scatter")


def test_batched_ppr_counters_one_sweep(cuda):
    """One row visit counts once (not once per lane): on a chain 0->1->...->n-1 the first
    sweep (theta = the seeds' fluid) diffuses exactly the k seed rows, one edge each."""
    from paper_1202_6158_b200 import ppr
    n = 1000
    g = cuda.SparseGraph.from_edges(n, np.arange(n - 1), np.arange(1, n))
    seeds = np.array([[10, 300, 600]], dtype=np.uint32)
    p = ppr.BatchedPPR(g, 1, target_error=1e-9, max_sweeps=1)
    try:
        _, stats, _ = p.solve(seeds)
    finally:
        p.close()
    assert stats.sweeps == 1
    assert stats.diffusions == 3
    assert stats.elementary_steps == 3


def test_batched_ppr_counters_bounded(cuda, oracle):
    """Whole solve: every sweep visits each row at most once, so diffusions <= n * sweeps and
    elementary_steps <= m * sweeps; every visited row pushes all its edges."""
    from paper_1202_6158_b200 import ppr
    n, B = 5000, 64
    src, dst = oracle.gen_edges(oracle.uniform_config(10), n, 9)
    off, tgt, _ = oracle.csr_build(n, src, dst, clean=True)
    g = cuda.SparseGraph(n, off, tgt.astype(np.int32))
    _, stats, _ = ppr.personalized_pagerank(g, ppr.config4_seeds(n, B, 10, seed=1), target_error=1e-9)
    assert 0 < stats.diffusions <= n * stats.sweeps
    assert 0 < stats.elementary_steps <= int(tgt.size) * stats.sweeps
    # mean out-degree 5 (uniform 0..10): the visited rows average close to it
    assert 2.0 <= stats.elementary_steps / stats.diffusions <= 10.0


@pytest.mark.parametrize("n,B", [(4000, 64), (2500, 5)])
def test_batched_ppr_pull_and_push_agree(cuda, oracle, n, B):
    """The pull formulation (take + pull over the transposed CSR, no atomics) and the
    push formulation (red.add scatter) reach the same per-column ranks, and the pull
    matches the reference run per column."""
    mode = "pull"
    from paper_1202_6158_b200 import ppr
    src, dst = oracle.gen_edges(oracle.web_config(8.0), n, 11)
    off, tgt, _ = oracle.csr_build(n, src, dst, clean=True)
    g = cuda.SparseGraph(n, off, tgt.astype(np.int32))
    seeds = ppr.config4_seeds(n, B, 10, seed=4)
    r_pull, s_pull, res_pull = ppr.personalized_pagerank(g, seeds, target_error=1e-11, mode=mode)
    r_push, s_push, res_push = ppr.personalized_pagerank(g, seeds, target_error=1e-11, mode="push")
    assert max(res_pull) <= 1e-11 * 0.15 and max(res_push) <= 1e-11 * 0.15
    r_pull, r_push = r_pull.cpu().numpy(), r_push.cpu().numpy()
    for c in range(B):
        assert np.abs(r_pull[:, c] - r_push[:, c]).sum() <= 2e-9, c
    v = np.zeros(n)
    np.add.at(v, seeds[0].astype(np.int64), 1.0 / 10)
    ref = oracle.run_seq(off, tgt, 0.85, 1e-13, "sweep", teleport=v).rank
    assert np.abs(r_pull[:, 0] - ref).sum() <= 1e-9
    # every visited row pushes all its edges in both formulations
    assert 0 < s_pull.diffusions and 0 < s_pull.elementary_steps <= int(tgt.size) * s_pull.sweeps


def test_batched_ppr_pull_is_deterministic(cuda, oracle):
    """No atomics on the pull path: two solves give bit-identical histories (the hub rows'
    segments are added in a fixed order)."""
    import torch
    from paper_1202_6158_b200 import ppr
    n = 3000
    src, dst = oracle.gen_edges(oracle.web_config(8.0), n, 2)
    off, tgt, _ = oracle.csr_build(n, src, dst, clean=True)
    g = cuda.SparseGraph(n, off, tgt.astype(np.int32))
    seeds = ppr.config4_seeds(n, 8, 10, seed=6)
    p = ppr.BatchedPPR(g, 8, target_error=1e-10, mode="pull")
    try:
        p.solve(seeds)
        h1 = p.history.clone()
        p.solve(seeds)
        assert torch.equal(h1, p.history)
    finally:
        p.close()


def test_batched_ppr_pull_hub_rows(cuda, oracle):
    """A star-heavy graph whose hub rows have more than 1024 (and more than 2048) parents,
    so the pull splits them into segments: the ranks still match the push formulation."""
    from paper_1202_6158_b200 import ppr
    n = 6000
    rng = np.random.default_rng(1)
    src = np.concatenate([np.arange(n), np.arange(n), rng.integers(0, n, 4 * n)])
    dst = np.concatenate([np.full(n, 7), np.full(n, 4242), rng.integers(0, n, 4 * n)])
    off, tgt, _ = oracle.csr_build(n, src.astype(np.uint32), dst.astype(np.uint32), clean=True)
    g = cuda.SparseGraph(n, off, tgt.astype(np.int32))
    seeds = ppr.config4_seeds(n, 4, 10, seed=2)
    a, _, ra = ppr.personalized_pagerank(g, seeds, target_error=1e-11, mode="pull")
    b, _, rb = ppr.personalized_pagerank(g, seeds, target_error=1e-11, mode="push")
    assert max(ra) <= 1e-11 * 0.15 and max(rb) <= 1e-11 * 0.15
    a, b = a.cpu().numpy(), b.cpu().numpy()
    for c in range(4):
        assert np.abs(a[:, c] - b[:, c]).sum() <= 2e-9, c


@pytest.mark.parametrize("hot", ["0", "1", "32"])
def test_batched_ppr_hot_rows(cuda, oracle, monkeypatch, hot):
    """The push formulation sums the pushes into the highest in-degree rows in a
    per-block shared-memory table (FR_PP_HOT rows, default 16); with 0, 1 or 32 such
    rows every column matches the reference run with its teleport vector."""
    from paper_1202_6158_b200 import ppr
    monkeypatch.setenv("FR_PP_HOT", hot)
    n, B = 5000, 6
    src, dst = oracle.gen_edges(oracle.web_config(8.0), n, 21)
    off, tgt, _ = oracle.csr_build(n, src, dst, clean=True)
    g = cuda.SparseGraph(n, off, tgt.astype(np.int32))
    seeds = ppr.config4_seeds(n, B, 10, seed=8)
    rank, _, resid = ppr.personalized_pagerank(g, seeds, target_error=1e-11)
    assert max(resid) <= 1e-11 * 0.15
    rank = rank.cpu().numpy()
    for c in range(B):
        v = np.zeros(n)
        np.add.at(v, seeds[c].astype(np.int64), 1.0 / 10)
        ref = oracle.run_seq(off, tgt, 0.85, 1e-13, "sweep", teleport=v).rank
        assert np.abs(rank[:, c] - ref).sum() <= 1e-9, c
