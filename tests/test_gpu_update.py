"""Incremental update on the device (reference update.py; PAPER Theorem 3.4)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
D = 0.85


def random_graph(cuda, rng, n, max_out=4, dangling_frac=0.3):
    dangling = rng.random(n) < dangling_frac
    src, dst = [], []
    for j in range(n):
        if dangling[j]:
            continue
        k = min(int(rng.integers(1, max_out + 1)), n - 1)
        t = rng.choice(n - 1, size=k, replace=False)
        t = t + (t >= j)
        src += [j] * k
        dst += t.tolist()
    if not src:
        src, dst = [0], [1]
    return cuda.SparseGraph.from_edges(n, src, dst)


def dense(g):
    off, tgt = g.host_csr()
    P = np.zeros((g.n, g.n))
    for j in range(g.n):
        kids = tgt[off[j]:off[j + 1]]
        if kids.size:
            P[kids, j] = 1.0 / kids.size
    return P


def single_edit(cuda, rng, g):
    while True:
        s, t = int(rng.integers(0, g.n)), int(rng.integers(0, g.n))
        if s != t:
            break
    if g.has_edge(s, t):
        return cuda.GraphDelta(added=[], removed=[(s, t)])
    return cuda.GraphDelta(added=[(s, t)], removed=[])


def test_signed_fluid_and_delta(cuda):
    from paper_1202_6158_b200.update import SignedFluid, delta_fluid
    sf = SignedFluid.from_net(torch.tensor([0.5, -0.2, 0.0], dtype=torch.float64))
    assert sf.pos.tolist() == [0.5, 0.0, 0.0] and sf.neg.tolist() == [0.0, 0.2, 0.0]
    g = cuda.SparseGraph.from_edges(3, [0], [1])
    g2 = cuda.apply_delta(g, cuda.GraphDelta(added=[(0, 2)], removed=[]))
    sf = delta_fluid(g, g2, np.array([0.3, 0.1, 0.2]), D)
    assert float(sf.pos[2]) == pytest.approx(D * 0.3 / 2)
    assert float(sf.neg[1]) == pytest.approx(D * 0.3 / 2)
    assert delta_fluid(g, g, np.array([0.3, 0.1, 0.2]), D).l1() == 0.0


def test_theorem_3_4_identity(cuda):
    from paper_1202_6158_b200 import update
    rng = np.random.default_rng(105)
    for _ in range(6):
        n = int(rng.integers(4, 21))
        g = random_graph(cuda, rng, n)
        params = cuda.DiffusionParams(target_error=1e-12)
        state = cuda.init(g, params)
        cuda.run(g, params, cuda.make_scheduler("sweep"), state=state)
        h_old = state.history.cpu().numpy().copy()
        g2 = cuda.apply_delta(g, single_edit(cuda, rng, g))
        new_state, _ = update.resume_state(state, g2, params, cuda.make_scheduler("sweep"))
        p_new, p_old = dense(g2), dense(g)
        expected = np.linalg.solve(np.eye(n) - D * p_new, D * (p_new - p_old) @ h_old)
        assert np.abs((new_state.history.cpu().numpy() - h_old) - expected).max() <= 1e-8


def test_resume_matches_fresh_run(cuda):
    from paper_1202_6158_b200 import update
    rng = np.random.default_rng(7)
    params = cuda.DiffusionParams(target_error=1e-9)
    for _ in range(12):
        n = int(rng.integers(10, 201))
        g = random_graph(cuda, rng, n)
        state = cuda.init(g, params)
        cuda.run(g, params, cuda.make_scheduler("sweep"), state=state)
        g2 = cuda.apply_delta(g, single_edit(cuda, rng, g))
        resumed, _ = update.resume(state, g2, params, cuda.make_scheduler("sweep"))
        fresh, _ = cuda.run(g2, params, cuda.make_scheduler("sweep"))
        assert float(np.abs(resumed - fresh).sum()) <= 2 * params.target_error


def test_resume_with_hub_rows_on_the_owned_graph_path(cuda, oracle, monkeypatch):
    """Signed fluid through the CUDA-graph owned path of a large graph whose rows with >= 2048
    children are pushed one sweep late (deferred hub rows, their in-flight fluid counted in the
    exact residual checks): the resumed rank matches a fresh solve of the edited graph."""
    from paper_1202_6158_b200 import update
    monkeypatch.setenv("FR_SMALL", "0")
    n = 150_000
    src, dst = oracle.gen_edges(oracle.web_config(8.0), n, 5)
    rng = np.random.default_rng(9)
    hubs = [11, 70_000, 149_000]
    src = np.concatenate([src] + [np.full(2500, h, dtype=np.uint32) for h in hubs])
    dst = np.concatenate([dst] + [rng.choice(n, 2500, replace=False).astype(np.uint32) for _ in hubs])
    off, tgt, _ = oracle.csr_build(n, src, dst, clean=True)
    g = cuda.SparseGraph(n, torch.as_tensor(off), torch.as_tensor(tgt.astype(np.int32)))
    sched = cuda.make_scheduler("sweep", policy="adaptive", sweep_decay=0.6, degree_exponent=0.85,
                                edge_frac=0.2, kernel_path="owned")
    params = cuda.DiffusionParams(target_error=1e-10)
    state = cuda.init(g, params)
    cuda.run(g, params, sched, state=state)
    # edit: 40 new edges out of a hub row and 40 random ones, 20 removals
    added = [(hubs[0], int(t)) for t in rng.choice(n, 40, replace=False) if int(t) != hubs[0]
             and not g.has_edge(hubs[0], int(t))]
    added += [(int(s), int(t)) for s, t in rng.integers(0, n, (40, 2)) if s != t and not g.has_edge(int(s), int(t))]
    removed = []
    for e in rng.choice(tgt.size, 20, replace=False):
        s = int(np.searchsorted(off, e, side="right") - 1)
        removed.append((s, int(tgt[e])))
    g2 = cuda.apply_delta(g, cuda.GraphDelta(added=sorted(set(added)), removed=sorted(set(removed))))
    resumed, _ = update.resume(state, g2, params, sched)
    fresh, _ = cuda.run(g2, params, sched)
    assert float(np.abs(resumed - fresh).sum()) <= 4 * params.target_error
