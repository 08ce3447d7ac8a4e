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
