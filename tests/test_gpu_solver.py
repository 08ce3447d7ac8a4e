"""Device diffusion solver vs the reference (goldens) and the oracle.

Tolerances (fp64): the device sweep stops when the fluid mass R satisfies
R/(1-d) <= target_error; the unnormalized history is then within
target_error of the limit in L1 (PAPER Theorem 3.2), so two normalized ranks
from runs at target T differ by at most ~2T/|h|_1.  Tests run at T <= 1e-10
and assert L1 <= 1e-9 (the north-star bound) against the reference's own
normalized rank.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
KINDS = ("sweep", "max", "per", "rand", "op", "op2")
L1_FP64 = 1e-9


def graph_from(cuda, off, tgt):
    return cuda.SparseGraph(off.size - 1, torch.as_tensor(off), torch.as_tensor(tgt.astype(np.int32)))


def l1(a, b):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else a
    return float(np.abs(a - b).sum())


@pytest.mark.parametrize("path", ["fused", "binned", "owned", "fused-graph", "owned-graph"])
@pytest.mark.parametrize("kind", KINDS)
def test_small_graphs_match_reference(cuda, golden_small, oracle, monkeypatch, kind, path):
    """Every selection rule on the reference's small graphs; "-graph" forces the multi-block
    sweep kernels (FR_SMALL=0) that these sizes would otherwise hand to the single-block solve."""
    if path.endswith("-graph"):
        monkeypatch.setenv("FR_SMALL", "0")
        path = path[:-6]
    for tag in golden_small["tags"]:
        tag = str(tag)
        g = graph_from(cuda, golden_small[f"{tag}_off"], golden_small[f"{tag}_tgt"])
        tel = golden_small[f"{tag}_teleport"] if f"{tag}_teleport" in golden_small else None
        params = cuda.DiffusionParams(damping=0.85, teleport=tel, target_error=1e-11)
        rank, trace = cuda.run(g, params, cuda.make_scheduler(kind, seed=3, kernel_path=path))
        # the reference's own rank at a tight target (the oracle is bit-exact with it,
        # test_oracle_golden.py); the goldens themselves were taken at 1e-9..1e-10
        truth = oracle.run_seq(golden_small[f"{tag}_off"], golden_small[f"{tag}_tgt"], 0.85, 1e-14,
                               "sweep", teleport=tel).rank
        assert l1(rank, truth) <= L1_FP64 / 10, (tag, kind)
        golden = golden_small[f"{tag}_sweep_rank"]
        h1 = float(np.abs(oracle.run_seq(golden_small[f"{tag}_off"], golden_small[f"{tag}_tgt"], 0.85, 1e-14,
                                         "sweep", teleport=tel).history).sum())
        assert l1(rank, golden) <= 2 * float(golden_small[f"{tag}_target_error"]) / h1 + L1_FP64 / 10
        assert trace.rows[-1].residual <= 1e-11 * 0.15


@pytest.mark.parametrize("path", ["fused", "binned", "owned"])
def test_config1_matches_reference(cuda, golden_configs, path):
    """BASELINE config 1: 10k uniform graph, residual < 1e-10, fp64."""
    g = graph_from(cuda, golden_configs["cfg1_off"], golden_configs["cfg1_tgt"])
    for policy, decay in (("exhaust", 0.5), ("geometric", 0.5), ("geometric", 0.9)):
        rank, trace = cuda.run(g, cuda.DiffusionParams(target_error=1e-10),
                               cuda.make_scheduler("sweep", policy=policy, sweep_decay=decay, kernel_path=path))
        assert l1(rank, golden_configs["cfg1_sweep_rank"]) <= L1_FP64
        assert trace.rows[-1].residual <= 1e-10 * 0.15


def test_web_graph_matches_reference(cuda, golden_configs):
    g = graph_from(cuda, golden_configs["web5k_off"], golden_configs["web5k_tgt"])
    rank, _ = cuda.run(g, cuda.DiffusionParams(target_error=1e-10), cuda.make_scheduler("sweep"))
    assert l1(rank, golden_configs["web5k_sweep_rank"]) <= L1_FP64


def test_sweep_counters_match_parallel_oracle(cuda, oracle):
    """Same selection schedule as the oracle's restatement of the device sweep."""
    src, dst = oracle.gen_edges(oracle.web_config(8.0), 20_000, 8)
    off, tgt, _ = oracle.csr_build(20_000, src, dst, clean=True)
    g = graph_from(cuda, off, tgt)
    for policy, code in (("exhaust", 0), ("geometric", 1)):
        ref = oracle.run_psweep(off, tgt, 0.85, 1e-10, policy=code)
        state = cuda.init(g, cuda.DiffusionParams(target_error=1e-10))
        rank, trace = cuda.run(g, cuda.DiffusionParams(target_error=1e-10),
                               cuda.make_scheduler("sweep", policy=policy, kernel_path="binned"), state=state)
        assert l1(rank, ref.rank) <= 2e-10
        # the selected sets can differ only through last-bit rounding near theta
        assert abs(state.sweeps - ref.sweeps) <= max(2, ref.sweeps // 50)
        assert abs(state.elementary_steps - ref.elementary_steps) <= 0.02 * ref.elementary_steps


@pytest.mark.parametrize("path", ["fused", "binned", "owned"])
def test_fp32_fluid_variant(cuda, golden_configs, path):
    """fp32 fluid / fp64 history: stated tolerance 1e-6 L1 against the fp64 reference."""
    g = graph_from(cuda, golden_configs["web5k_off"], golden_configs["web5k_tgt"])
    rank, trace = cuda.run(g, cuda.DiffusionParams(target_error=1e-9),
                           cuda.make_scheduler("sweep", kernel_path=path), fluid_dtype=torch.float32)
    assert l1(rank, golden_configs["web5k_sweep_rank"]) <= 1e-6


def test_power_iteration_matches_oracle(cuda, golden_small, oracle):
    for tag in golden_small["tags"]:
        tag = str(tag)
        g = graph_from(cuda, golden_small[f"{tag}_off"], golden_small[f"{tag}_tgt"])
        tel = golden_small[f"{tag}_teleport"] if f"{tag}_teleport" in golden_small else None
        te = float(golden_small[f"{tag}_target_error"])
        x, trace = cuda.power_iterate(g, cuda.DiffusionParams(teleport=tel, target_error=te))
        assert l1(x, golden_small[f"{tag}_mat_iter_rank"]) <= 1e-12, tag
        assert trace.rows[-1].diffusions == int(golden_small[f"{tag}_mat_iter_iters"]), tag


def test_power_iteration_long_rows(cuda, oracle):
    """In-degree hubs exercise the split-row SpMV path."""
    src, dst = oracle.gen_edges(oracle.web_config(8.0), 200_000, 12)
    off, tgt, _ = oracle.csr_build(200_000, src, dst, clean=True)
    g = graph_from(cuda, off, tgt)
    assert int(g.in_degree.max()) > 2048
    x, trace = cuda.power_iterate(g, cuda.DiffusionParams(target_error=1e-10))
    ox, iters, _ = oracle.power_iterate(off, tgt, 0.85, 1e-10)
    assert l1(x, ox) <= 1e-11
    assert abs(trace.rows[-1].diffusions - iters) <= 1
    rank, _ = cuda.run(g, cuda.DiffusionParams(target_error=1e-10), cuda.make_scheduler("sweep"))
    assert l1(rank, ox) <= 2e-9


def test_power_iteration_row_tiles(cuda, oracle):
    """The row-tile SpMV at its edges: in-degrees exactly at and just above the long-row
    split (1024 / 1025), a row with every other node as parent, tiles without edges, and
    n not a multiple of the 32-row tile."""
    rng = np.random.default_rng(4)
    n = 5003
    src, dst = [], []
    for t, k in ((0, n - 1), (1, 1024), (2, 1025), (3, 31)):
        par = rng.choice(np.setdiff1d(np.arange(n), [t]), size=k, replace=False)
        src.extend(par.tolist())
        dst.extend([t] * k)
    extra = rng.integers(64, n, (2, 3000))  # nodes 4..63 receive nothing: edge-free tiles
    keep = extra[0] != extra[1]
    src.extend(extra[0][keep].tolist())
    dst.extend(extra[1][keep].tolist())
    off, tgt, _ = oracle.csr_build(n, np.array(src, dtype=np.uint32), np.array(dst, dtype=np.uint32), clean=True)
    g = graph_from(cuda, off, tgt)
    x, trace = cuda.power_iterate(g, cuda.DiffusionParams(target_error=1e-12))
    ox, iters, _ = oracle.power_iterate(off, tgt, 0.85, 1e-12)
    assert l1(x, ox) <= 1e-13
    assert abs(trace.rows[-1].diffusions - iters) <= 1


def test_single_node_diffuse_bit_exact(cuda, golden_small, oracle):
    """engine.diffuse on the device equals the reference step (distinct targets: no reordering)."""
    tag = "rg3"
    off, tgt = golden_small[f"{tag}_off"], golden_small[f"{tag}_tgt"]
    g = graph_from(cuda, off, tgt)
    params = cuda.DiffusionParams()
    state = cuda.init(g, params)
    f = oracle.init_fluid(g.n)
    h = np.zeros(g.n)
    for i in [0, 3, 1, 3, 7, 2, 0]:
        i %= g.n
        cuda.diffuse(state, i)
        sent = f[i]
        if sent != 0.0:
            f[i] = 0.0
            h[i] += sent
            deg = off[i + 1] - off[i]
            if deg:
                f[tgt[off[i]:off[i + 1]]] += sent * (0.85 / deg)
    assert np.array_equal(state.fluid.cpu().numpy(), f)
    assert np.array_equal(state.history.cpu().numpy(), h)


def test_conservation_identity_mid_run(cuda, oracle):
    """Theorem 3.1 after a partial run: H + F = F0 + d P H (stored, uncompleted P)."""
    src, dst = oracle.gen_edges(oracle.web_config(8.0), 5000, 21)
    off, tgt, _ = oracle.csr_build(5000, src, dst, clean=True)
    g = graph_from(cuda, off, tgt)
    params = cuda.DiffusionParams(target_error=1e-12)
    state = cuda.init(g, params)
    f0 = state.fluid.cpu().numpy().copy()
    cuda.run(g, params, cuda.make_scheduler("sweep", policy="geometric", sweep_decay=0.9), state=state, max_sweeps=7)
    torch.cuda.synchronize()
    h = state.history.cpu().numpy()
    f = state.fluid.cpu().numpy()
    deg = np.diff(off)
    src_e = np.repeat(np.arange(g.n), deg)
    push = np.zeros(g.n)
    np.add.at(push, tgt.astype(np.int64), h[src_e] / deg[src_e])
    assert np.abs(h + f - f0 - 0.85 * push).max() <= 1e-15
    assert state.sweeps == 7
    # the fused kernel's exact fluid mass equals the run's residual bookkeeping
    assert abs(f.sum() - state.residual) <= 1e-15


def test_bound_equals_true_error_without_dangling(cuda):
    rng = np.random.default_rng(15)
    n = 300
    src, dst = [], []
    for j in range(n):
        t = rng.choice(n - 1, size=3, replace=False)
        t = t + (t >= j)
        src += [j] * 3
        dst += t.tolist()
    g = cuda.SparseGraph.from_edges(n, src, dst)
    params = cuda.DiffusionParams(target_error=1e-6)
    state = cuda.init(g, params)
    cuda.run(g, params, cuda.make_scheduler("sweep"), state=state, max_sweeps=5)
    P = np.zeros((n, n))
    P[np.array(dst), np.array(src)] = 1.0 / 3
    truth = np.linalg.solve(np.eye(n) - 0.85 * P, 0.15 * np.full(n, 1.0 / n))
    dist = np.abs(truth - state.history.cpu().numpy()).sum()
    assert dist == pytest.approx(cuda.error_bound(state), abs=1e-12)


def test_zero_edge_graph_converges_to_teleport(cuda):
    g = cuda.SparseGraph.from_edges(3, [], [])
    v = np.array([0.2, 0.3, 0.5])
    rank, _ = cuda.run(g, cuda.DiffusionParams(teleport=v), cuda.make_scheduler("sweep"))
    assert np.allclose(rank, v, atol=1e-12)


def test_undamped_diagnostic_mode(cuda):
    g = cuda.SparseGraph.from_edges(2, [0, 1], [1, 0])
    with pytest.raises(ValueError):
        cuda.run(g, cuda.DiffusionParams(damping=1.0), cuda.make_scheduler("max"))
    rank, trace = cuda.run(g, cuda.DiffusionParams(damping=1.0), cuda.make_scheduler("sweep"), max_diffusions=500)
    assert trace.rows[-1].diffusions >= 500
    assert np.allclose(rank, [0.5, 0.5], atol=2e-3)


def test_signed_fluid_resume(cuda, oracle):
    rng = np.random.default_rng(3)
    n = 400
    off, tgt, _ = oracle.csr_build(n, rng.integers(0, n, 1600), rng.integers(0, n, 1600), clean=True)
    g = graph_from(cuda, off, tgt)
    f = oracle.init_fluid(n)
    f[::7] *= -1.0
    params = cuda.DiffusionParams(target_error=1e-11)
    state = cuda.init_from_fluid(g, params, f)
    assert state.signed
    cuda.run(g, params, cuda.make_scheduler("sweep"), state=state)
    ref = oracle.run_seq(off, tgt, 0.85, 1e-11, "sweep", fluid=f)
    assert l1(state.history, ref.history) <= 1e-10


def test_host_buffer_entry_point(cuda, golden_configs):
    """fr_pagerank_host: the reference-facing one-call path from host buffers."""
    import ctypes
    from paper_1202_6158_b200 import _lib
    off = np.ascontiguousarray(golden_configs["cfg1_off"])
    tgt = np.ascontiguousarray(golden_configs["cfg1_tgt"])
    n = off.size - 1
    cfg = cuda.make_scheduler("sweep").solver_config(cuda.DiffusionParams(target_error=1e-10))
    rank = np.empty(n)
    stats = _lib.SolveStats()
    _lib.check(_lib.lib.fr_pagerank_host(n, tgt.size, off.ctypes.data, tgt.ctypes.data, None, ctypes.byref(cfg),
                                         rank.ctypes.data, ctypes.byref(stats)))
    assert l1(rank, golden_configs["cfg1_sweep_rank"]) <= L1_FP64


@pytest.mark.parametrize("n,mean", [(5_000, 8.0), (300_000, 12.0)])
def test_host_buffer_entry_point_teleport(cuda, oracle, n, mean):
    """fr_pagerank_host with a personalized teleport (params.teleport, engine.py:56-62,
    149-159) against the oracle run with the same V; bad vectors are rejected like
    DiffusionParams.validate (engine.py:47-54)."""
    import ctypes
    from paper_1202_6158_b200 import _lib
    src, dst = oracle.gen_edges(oracle.web_config(mean), n, 23)
    off, tgt, _ = oracle.csr_build(n, src, dst, clean=True)
    rng = np.random.default_rng(5)
    v = np.zeros(n)
    v[rng.choice(n, 50, replace=False)] = rng.uniform(0.5, 1.5, 50)
    v /= v.sum()
    params = cuda.DiffusionParams(target_error=1e-10, teleport=v)
    cfg = cuda.make_scheduler("sweep", policy="adaptive", sweep_decay=0.6, edge_frac=0.2,
                              degree_exponent=0.65).solver_config(params)
    rank = np.empty(n)
    stats = _lib.SolveStats()
    _lib.check(_lib.lib.fr_pagerank_host(n, tgt.size, off.ctypes.data, tgt.ctypes.data, v.ctypes.data,
                                         ctypes.byref(cfg), rank.ctypes.data, ctypes.byref(stats)))
    ref = oracle.run_seq(off, tgt, 0.85, 1e-12, "sweep", teleport=v).rank
    assert l1(rank, ref) <= L1_FP64
    uniform = oracle.run_seq(off, tgt, 0.85, 1e-10, "sweep").rank
    assert l1(rank, uniform) > 1e-3  # the teleport was used
    for bad in (v * 1.001, np.where(np.arange(n) == 0, -1e-3, v)):
        bad = np.ascontiguousarray(bad)
        with pytest.raises(ValueError):
            _lib.check(_lib.lib.fr_pagerank_host(n, tgt.size, off.ctypes.data, tgt.ctypes.data, bad.ctypes.data,
                                                 ctypes.byref(cfg), rank.ctypes.data, ctypes.byref(stats)))


@pytest.mark.parametrize("hot_slots,warm_slots", [(-1, -1), (0, -1), (7, 0), (0, 0), (-1, 5000)])
def test_hot_slot_aggregation(cuda, oracle, hot_slots, warm_slots):
    """Shared-memory aggregation of pushes into in-degree hubs keeps exact conservation."""
    src, dst = oracle.gen_edges(oracle.web_config(8.0), 200_000, 31)
    off, tgt, _ = oracle.csr_build(200_000, src, dst, clean=True)
    g = graph_from(cuda, off, tgt)
    params = cuda.DiffusionParams(target_error=1e-10)
    sched = cuda.make_scheduler("sweep", policy="geometric", sweep_decay=0.9, hot_slots=hot_slots,
                                warm_slots=warm_slots)
    state = cuda.init(g, params)
    rank, trace = cuda.run(g, params, sched, state=state)
    ref = oracle.run_seq(off, tgt, 0.85, 1e-11, "sweep").rank
    assert l1(rank, ref) <= 2e-10
    assert state.residual <= 1e-10 * 0.15


def test_host_buffer_entry_point_with_hubs(cuda, oracle):
    """fr_pagerank_host on a web graph whose in-degree hubs get shared-memory / warm slots:
    the slot preparation must be ordered after the host-to-device copies."""
    import ctypes
    from paper_1202_6158_b200 import _lib
    n = 300_000
    src, dst = oracle.gen_edges(oracle.web_config(12.0), n, 17)
    off, tgt, _ = oracle.csr_build(n, src, dst, clean=True)
    cfg = cuda.make_scheduler("sweep", policy="geometric", sweep_decay=0.9).solver_config(
        cuda.DiffusionParams(target_error=1e-10))
    for _ in range(2):
        rank = np.empty(n)
        stats = _lib.SolveStats()
        _lib.check(_lib.lib.fr_pagerank_host(n, tgt.size, off.ctypes.data, tgt.ctypes.data, None, ctypes.byref(cfg),
                                             rank.ctypes.data, ctypes.byref(stats)))
        ref = oracle.run_seq(off, tgt, 0.85, 1e-11, "sweep").rank
        assert l1(rank, ref) <= 1e-9


@pytest.mark.parametrize("beta", [0.5, 1.0])
@pytest.mark.parametrize("path", ["fused", "binned", "owned"])
def test_degree_exponent_sweep(cuda, oracle, monkeypatch, beta, path):
    """Degree-scaled sweep score |f|(out+1)^-beta (PAPER sec. 4.3) converges to the same rank.
    (The multi-block sweep kernels: the single-block small-graph solve diffuses pushes within
    the sweep and does less work than the parallel restatement, test_small_graph_single_launch.)"""
    monkeypatch.setenv("FR_SMALL", "0")
    src, dst = oracle.gen_edges(oracle.web_config(12.0), 50_000, 23)
    off, tgt, _ = oracle.csr_build(50_000, src, dst, clean=True)
    g = graph_from(cuda, off, tgt)
    sched = cuda.make_scheduler("sweep", policy="geometric", sweep_decay=0.9, degree_exponent=beta, kernel_path=path)
    rank, trace = cuda.run(g, cuda.DiffusionParams(target_error=1e-10), sched)
    ref = oracle.run_seq(off, tgt, 0.85, 1e-12, "sweep").rank
    assert l1(rank, ref) <= 1e-9
    # the oracle's restatement of the same schedule does the same amount of work
    deg = np.diff(off).astype(np.float64)
    p = oracle.run_psweep(off, tgt, 0.85, 1e-10, policy=1, decay=0.9, weight=(deg + 1) ** -beta)
    assert abs(trace.rows[-1].elementary_steps - p.elementary_steps) <= 0.15 * p.elementary_steps


@pytest.mark.parametrize("damping", [0.85, 0.99])
@pytest.mark.parametrize("path", ["fused", "binned", "owned"])
def test_adaptive_theta(cuda, oracle, monkeypatch, damping, path):
    """Adaptive theta (edges per sweep steered to edge_frac*m) converges to the same rank,
    and its sweep/edge counts follow the oracle's restatement of the rule (multi-block kernels)."""
    monkeypatch.setenv("FR_SMALL", "0")
    src, dst = oracle.gen_edges(oracle.web_config(12.0), 50_000, 29)
    off, tgt, _ = oracle.csr_build(50_000, src, dst, clean=True)
    g = graph_from(cuda, off, tgt)
    sched = cuda.make_scheduler("sweep", policy="adaptive", sweep_decay=0.75, degree_exponent=0.65,
                                kernel_path=path)
    rank, trace = cuda.run(g, cuda.DiffusionParams(damping=damping, target_error=1e-10), sched)
    ref = oracle.run_seq(off, tgt, damping, 1e-12, "sweep").rank
    assert l1(rank, ref) <= 1e-9
    deg = np.diff(off).astype(np.float64)
    p = oracle.run_psweep(off, tgt, damping, 1e-10, policy=2, decay=0.75, weight=(deg + 1) ** -0.65,
                          edge_frac=0.2)
    assert abs(trace.rows[-1].elementary_steps - p.elementary_steps) <= 0.2 * p.elementary_steps
    assert abs(trace.rows[-1].sweeps - p.sweeps) <= max(3, 0.2 * p.sweeps)


@pytest.mark.parametrize("fluid", ["fp64", "fp32"])
def test_wide_index_kernel(cuda, oracle, monkeypatch, fluid):
    """The 64-bit-offset sweep kernel (taken when m >= 2^32 or n >= 2^31) on a test-sized graph
    (FR_FORCE_WIDE=1 skips the narrow offset copy): same rank, same work as the narrow kernel."""
    monkeypatch.setenv("FR_FORCE_WIDE", "1")
    src, dst = oracle.gen_edges(oracle.web_config(12.0), 200_000, 37)
    off, tgt, _ = oracle.csr_build(200_000, src, dst, clean=True)
    g = graph_from(cuda, off, tgt)
    # fp32 fluid: a 1e-8 target (its stated rank tolerance is 1e-6); near 1e-10 the
    # fp32 rounding floor makes the number of sweeps vary from run to run
    fp32 = fluid == "fp32"
    params = cuda.DiffusionParams(target_error=1e-8 if fp32 else 1e-10)
    sched = cuda.make_scheduler("sweep", policy="adaptive", sweep_decay=0.7, degree_exponent=0.65,
                                edge_frac=0.15)
    dtype = torch.float32 if fp32 else torch.float64
    rank, trace = cuda.run(g, params, sched, fluid_dtype=dtype)
    ref = oracle.run_seq(off, tgt, 0.85, 1e-12, "sweep").rank
    tol = 1e-6 if fp32 else 1e-9
    assert l1(rank, ref) <= tol
    monkeypatch.delenv("FR_FORCE_WIDE")
    rank2, trace2 = cuda.run(g, params, sched, fluid_dtype=dtype)
    assert l1(rank2, ref) <= tol
    if not fp32:
        e1, e2 = trace.rows[-1].elementary_steps, trace2.rows[-1].elementary_steps
        assert abs(e1 - e2) <= 0.15 * e2


@pytest.mark.parametrize("chunk", ["256", "1024", "16384"])
@pytest.mark.parametrize("fluid", ["fp64", "fp32"])
def test_owned_chunk_sizes(cuda, oracle, monkeypatch, chunk, fluid):
    """Owned-chunk sweep (shared-memory sums of in-chunk pushes, Gauss-Seidel take): the rank
    does not depend on the chunk size, i.e. on which pushes stay in shared memory and which
    leave the chunk through F."""
    monkeypatch.setenv("FR_OWN_CHUNK", chunk)
    src, dst = oracle.gen_edges(oracle.web_config(12.0), 200_000, 41)
    off, tgt, _ = oracle.csr_build(200_000, src, dst, clean=True)
    g = graph_from(cuda, off, tgt)
    fp32 = fluid == "fp32"
    params = cuda.DiffusionParams(target_error=1e-8 if fp32 else 1e-10)
    sched = cuda.make_scheduler("sweep", policy="adaptive", sweep_decay=0.7, degree_exponent=0.65,
                                edge_frac=0.15, kernel_path="owned")
    state = cuda.init(g, params, fluid_dtype=torch.float32 if fp32 else torch.float64)
    rank, trace = cuda.run(g, params, sched, state=state)
    ref = oracle.run_seq(off, tgt, 0.85, 1e-12, "sweep").rank
    assert l1(rank, ref) <= (1e-6 if fp32 else 1e-9)
    assert state.residual <= params.target_error * (1 - params.damping)


def test_owned_conservation(cuda, oracle, monkeypatch):
    """Owned path with small chunks (many pushes leave the chunk, the rest are summed in shared
    memory and flushed): exact conservation after a partial run (Theorem 3.1:
    H + F = F0 + d P H), and repeated full solves on fresh states."""
    monkeypatch.setenv("FR_OWN_CHUNK", "256")
    monkeypatch.setenv("FR_SMALL", "0")  # n = 100k would otherwise take the single-block solve
    src, dst = oracle.gen_edges(oracle.web_config(8.0), 100_000, 43)
    off, tgt, _ = oracle.csr_build(100_000, src, dst, clean=True)
    g = graph_from(cuda, off, tgt)
    sched = cuda.make_scheduler("sweep", policy="adaptive", sweep_decay=0.7, degree_exponent=0.65,
                                edge_frac=0.15, kernel_path="owned")
    params = cuda.DiffusionParams(target_error=1e-12)
    state = cuda.init(g, params)
    f0 = state.fluid.cpu().numpy().copy()
    cuda.run(g, params, sched, state=state, max_sweeps=7)
    torch.cuda.synchronize()
    h = state.history.cpu().numpy()
    f = state.fluid.cpu().numpy()
    deg = np.diff(off)
    src_e = np.repeat(np.arange(g.n), deg)
    push = np.zeros(g.n)
    np.add.at(push, tgt.astype(np.int64), h[src_e] / deg[src_e])
    assert np.abs(h + f - f0 - 0.85 * push).max() <= 1e-15
    assert state.sweeps == 7
    params = cuda.DiffusionParams(target_error=1e-10)
    ref = oracle.run_seq(off, tgt, 0.85, 1e-12, "sweep").rank
    for _ in range(2):  # the second solve starts from the counters the first one left
        state = cuda.init(g, params)
        rank, _ = cuda.run(g, params, sched, state=state)
        assert l1(rank, ref) <= 1e-9
        assert state.residual <= 1e-10 * 0.15


@pytest.mark.parametrize("small", ["1", "0"])
def test_small_graph_single_launch(cuda, oracle, monkeypatch, small):
    """n <= 2^17: the whole solve runs as one single-block launch (FR_SMALL=0 forces the
    graph of sweep kernels); both match the reference and keep conservation exact."""
    monkeypatch.setenv("FR_SMALL", small)
    src, dst = oracle.gen_edges(oracle.web_config(8.0), 60_000, 47)
    off, tgt, _ = oracle.csr_build(60_000, src, dst, clean=True)
    g = graph_from(cuda, off, tgt)
    sched = cuda.make_scheduler("sweep", policy="adaptive", sweep_decay=0.7, degree_exponent=0.65, edge_frac=0.15)
    params = cuda.DiffusionParams(target_error=1e-12)
    state = cuda.init(g, params)
    f0 = state.fluid.cpu().numpy().copy()
    cuda.run(g, params, sched, state=state, max_sweeps=5)
    h = state.history.cpu().numpy()
    f = state.fluid.cpu().numpy()
    deg = np.diff(off)
    src_e = np.repeat(np.arange(g.n), deg)
    push = np.zeros(g.n)
    np.add.at(push, tgt.astype(np.int64), h[src_e] / deg[src_e])
    assert np.abs(h + f - f0 - 0.85 * push).max() <= 1e-15
    assert state.sweeps == 5
    params = cuda.DiffusionParams(target_error=1e-10)
    rank, trace = cuda.run(g, params, sched)
    ref = oracle.run_seq(off, tgt, 0.85, 1e-12, "sweep").rank
    assert l1(rank, ref) <= 1e-9
    assert trace.rows[-1].residual <= 1e-10 * 0.15
    # no more work than the parallel restatement of the schedule (pushes within a sweep
    # only let fluid merge before it moves on)
    p = oracle.run_psweep(off, tgt, 0.85, 1e-10, policy=2, decay=0.7, weight=(deg + 1.0) ** -0.65,
                          edge_frac=0.15)
    assert trace.rows[-1].elementary_steps <= 1.05 * p.elementary_steps


@pytest.mark.parametrize("path,small", [("owned", "1"), ("owned", "0"), ("fused", "0")])
def test_signed_fluid_residual_refresh(cuda, oracle, monkeypatch, path, small):
    """Signed fluid whose pushes cancel: the true |F|_1 falls much faster than the incremental
    estimate R - (1-d)|sent|, so without the reference's periodic exact refresh (every n
    diffusions, engine.py:331-333) the loop would sweep on until the fluid underflows. The
    device re-derives R every n diffusions and stops at the target like the reference."""
    monkeypatch.setenv("FR_SMALL", small)
    n = 4000
    src = np.repeat(np.arange(n), 2)
    dst = (src + np.tile([1, 2], n)) % n
    g = cuda.SparseGraph.from_edges(n, src, dst)
    f0 = np.where(np.arange(n) % 2 == 0, 1.0, -1.0) / n
    params = cuda.DiffusionParams(target_error=1e-10)
    sched = cuda.make_scheduler("sweep", policy="geometric", sweep_decay=0.7, kernel_path=path)
    state = cuda.init_from_fluid(g, params, f0)
    assert state.signed
    cuda.run(g, params, sched, state=state)
    assert state.residual <= 1e-10 * 0.15
    assert state.sweeps < 400, state.sweeps
    off, tgt, _ = oracle.csr_build(n, src.astype(np.uint32), dst.astype(np.uint32), clean=False)
    ref = oracle.run_seq(off, tgt, 0.85, 1e-13, "sweep", fluid=f0)
    assert l1(state.history, ref.history) <= 2e-10


@pytest.mark.parametrize("defer", ["1", "0"])
def test_owned_deferred_hub_rows(cuda, oracle, monkeypatch, defer):
    """Rows with >= 2048 children: in the CUDA-graph loop of the owned path they are queued by
    one sweep and pushed by the next sweep's blocks (FR_HUB_DEFER, default on), the last
    sweep's by a drain after the loop.  Exact conservation after a budget stop (nothing left
    in flight) and the rank of a full solve against the oracle."""
    monkeypatch.setenv("FR_HUB_DEFER", defer)
    monkeypatch.setenv("FR_SMALL", "0")
    n = 150_000
    src, dst = oracle.gen_edges(oracle.web_config(8.0), n, 47)
    rng = np.random.default_rng(3)
    hubs = [17, 40_000, 90_001, 149_990]
    src = np.concatenate([src] + [np.full(3000, h, dtype=np.uint32) for h in hubs])
    dst = np.concatenate([dst] + [rng.choice(n, 3000, replace=False).astype(np.uint32) for _ in hubs])
    off, tgt, _ = oracle.csr_build(n, src, dst, clean=True)
    assert (np.diff(off)[hubs] >= 2048).all()
    g = graph_from(cuda, off, tgt)
    sched = cuda.make_scheduler("sweep", policy="adaptive", sweep_decay=0.6, degree_exponent=0.85,
                                edge_frac=0.2, kernel_path="owned")
    params = cuda.DiffusionParams(target_error=1e-12)
    state = cuda.init(g, params)
    f0 = state.fluid.cpu().numpy().copy()
    cuda.run(g, params, sched, state=state, max_sweeps=6)
    torch.cuda.synchronize()
    h = state.history.cpu().numpy()
    f = state.fluid.cpu().numpy()
    deg = np.diff(off)
    src_e = np.repeat(np.arange(g.n), deg)
    push = np.zeros(g.n)
    np.add.at(push, tgt.astype(np.int64), h[src_e] / deg[src_e])
    assert np.abs(h + f - f0 - 0.85 * push).max() <= 1e-15
    assert state.sweeps == 6
    params = cuda.DiffusionParams(target_error=1e-10)
    ref = oracle.run_seq(off, tgt, 0.85, 1e-12, "sweep").rank
    rank, _ = cuda.run(g, params, sched)
    assert l1(rank, ref) <= 1e-9


def _shape_graph(n, degs, rng):
    """Rows with the given out-degree pattern (cycled over the nodes); targets near the row."""
    deg = np.resize(np.asarray(degs, dtype=np.int64), n)
    src = np.repeat(np.arange(n, dtype=np.uint32), deg)
    # distinct targets per row: a random start, then consecutive ids (wrapping), never the row itself
    start = rng.integers(1, n - deg.max() - 1, size=n)
    k = np.arange(src.size) - np.repeat(np.cumsum(deg) - deg, deg)
    dst = ((src.astype(np.int64) + np.repeat(start, deg) + k) % n).astype(np.uint32)
    return src, dst


@pytest.mark.parametrize("shape", ["ones", "lane31", "full96", "big_small", "sparse", "mixed"])
def test_owned_row_search_shapes(cuda, oracle, monkeypatch, shape):
    """k_sweep_own finds the row of an edge position from a REDUX.OR mask of the row heads in
    each 32-position window over the lane-compacted active rows.  Degree patterns that put the
    heads on the window boundaries: every row one edge (32 heads per window), one active row per
    tile in the last lane, tiles of exactly 96 / 192 edges (whole batches), rows just under
    the hub threshold next to one-edge rows (windows without heads, thousands of positions),
    mostly dangling rows, and a mixed pattern -- conservation after a partial run, then the
    rank against the oracle."""
    monkeypatch.setenv("FR_SMALL", "0")
    monkeypatch.setenv("FR_OWN_CHUNK", "256")
    rng = np.random.default_rng(11)
    n = 40_000
    degs = {
        "ones": [1],
        "lane31": [0] * 31 + [37],
        "full96": [3] * 32 + [6] * 32,
        "big_small": [2047, 1, 0, 1, 2040, 1, 1, 33],
        "sparse": [0, 0, 0, 5, 0, 0, 0, 0, 0, 64, 0],
        "mixed": [31, 32, 33, 1, 0, 95, 96, 97, 2, 0, 0, 191, 192, 193, 7],
    }[shape]
    src, dst = _shape_graph(n, degs, rng)
    off, tgt, _ = oracle.csr_build(n, src, dst, clean=True)
    g = graph_from(cuda, off, tgt)
    sched = cuda.make_scheduler("sweep", policy="adaptive", sweep_decay=0.6, degree_exponent=0.85,
                                edge_frac=0.2, kernel_path="owned")
    params = cuda.DiffusionParams(target_error=1e-12)
    state = cuda.init(g, params)
    f0 = state.fluid.cpu().numpy().copy()
    cuda.run(g, params, sched, state=state, max_sweeps=5)
    torch.cuda.synchronize()
    h = state.history.cpu().numpy()
    f = state.fluid.cpu().numpy()
    deg = np.diff(off)
    src_e = np.repeat(np.arange(g.n), deg)
    push = np.zeros(g.n)
    np.add.at(push, tgt.astype(np.int64), h[src_e] / deg[src_e])
    assert np.abs(h + f - f0 - 0.85 * push).max() <= 1e-15
    params = cuda.DiffusionParams(target_error=1e-10)
    rank, _ = cuda.run(g, params, sched)
    ref = oracle.run_seq(off, tgt, 0.85, 1e-13, "sweep").rank
    assert l1(rank, ref) <= 1e-9
