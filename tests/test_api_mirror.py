"""The reference package's own behavioural checks, restated against this package's API.

Each class follows a test group of the reference (tests/test_engine.py and
tests/test_graph.py of fluidrank): parameter validation, init, single-node
diffusion arithmetic, full runs against a dense direct solve, the error
bound, pull-style collect, the convergence trace, edge-list parsing and graph
deltas.  Parsing and validation errors are raised on the host before any
device work, so those run without a GPU; everything else is marked gpu.
Known, documented difference: run() takes the device selection rules of
make_scheduler (and the reference class names), not arbitrary Python
scheduler objects.
"""

import io

import numpy as np
import pytest
import torch

D = 0.85


# ---------------------------------------------------------------- helpers (test-side math)
def random_edges(rng, n, max_out=4, dangling_frac=0.3):
    """Random simple digraph as (src, dst) lists, roughly dangling_frac of nodes without out-links."""
    dangling = rng.random(n) < dangling_frac
    src, dst = [], []
    for j in range(n):
        if dangling[j]:
            continue
        k = min(int(rng.integers(1, max_out + 1)), n - 1)
        t = rng.choice(n - 1, size=k, replace=False)
        t = t + (t >= j)
        src += [j] * k
        dst += [int(x) for x in t]
    if not src:
        src, dst = [0], [1]
    return src, dst


def dense_p(n, src, dst):
    """Column-stochastic P with P[i, j] = 1/outdeg(j); dangling columns zero."""
    p = np.zeros((n, n))
    deg = np.bincount(np.asarray(src, dtype=np.int64), minlength=n)
    for s, t in zip(src, dst):
        p[t, s] = 1.0 / deg[s]
    return p


def solve_unnormalized(n, src, dst, d=D, v=None):
    v = np.full(n, 1.0 / n) if v is None else v
    return np.linalg.solve(np.eye(n) - d * dense_p(n, src, dst), (1 - d) * v)


def solve_pagerank(n, src, dst, d=D, v=None):
    """Direct solve with dangling columns completed by the teleport vector."""
    v = np.full(n, 1.0 / n) if v is None else v
    p = dense_p(n, src, dst)
    deg = np.bincount(np.asarray(src, dtype=np.int64), minlength=n)
    for j in np.nonzero(deg == 0)[0]:
        p[:, j] = v
    return np.linalg.solve(np.eye(n) - d * p, (1 - d) * v)


def host(x):
    return x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


# ---------------------------------------------------------------- CPU: validation and parsing
class TestParams:
    def test_defaults_valid(self):
        from paper_1202_6158_b200 import DiffusionParams
        DiffusionParams().validate(5)

    @pytest.mark.parametrize("damping", [0.0, -0.1, 1.5])
    def test_bad_damping(self, damping):
        from paper_1202_6158_b200 import DiffusionParams
        with pytest.raises(ValueError):
            DiffusionParams(damping=damping).validate()

    def test_teleport_must_normalize(self):
        from paper_1202_6158_b200 import DiffusionParams
        with pytest.raises(ValueError):
            DiffusionParams(teleport=np.array([0.5, 0.6])).validate(2)
        with pytest.raises(ValueError):
            DiffusionParams(teleport=np.array([1.5, -0.5])).validate(2)

    def test_teleport_length_checked(self):
        from paper_1202_6158_b200 import DiffusionParams
        with pytest.raises(ValueError):
            DiffusionParams(teleport=np.array([1.0])).validate(2)

    def test_bad_target(self):
        from paper_1202_6158_b200 import DiffusionParams
        with pytest.raises(ValueError):
            DiffusionParams(target_error=0.0).validate()


class TestSchedulerChoices:
    def test_unknown_kind_policy_decay(self):
        from paper_1202_6158_b200 import make_scheduler
        with pytest.raises(ValueError):
            make_scheduler("nope")
        with pytest.raises(ValueError):
            make_scheduler("sweep", policy="nope")
        with pytest.raises(ValueError):
            make_scheduler("sweep", sweep_decay=1.0)
        with pytest.raises(ValueError):
            make_scheduler("sweep", degree_exponent=-1.0)
        with pytest.raises(ValueError):
            make_scheduler("sweep", policy="adaptive", edge_frac=0.0)

    def test_reference_class_names(self):
        from paper_1202_6158_b200 import sched
        assert sched.GreedyScheduler().kind == "max"
        assert sched.RoundRobinScheduler().kind == "per"
        assert sched.RandomScheduler(seed=3).kind == "rand"
        assert sched.ThresholdSweepScheduler().kind == "sweep"
        assert sched.DegreeScaledScheduler().kind == "op"
        assert sched.DegreeScaledScheduler(use_in_degree=False).kind == "op2"


class TestSchedulerProtocol:
    """run() takes reference scheduler objects (sched.py:16-161) by their kind and knobs."""

    def test_reference_objects_map_to_device_rules(self):
        from paper_1202_6158_b200.engine import device_schedule

        class ThresholdSweepScheduler:  # the reference class's public attributes
            kind = "sweep"

            def __init__(self, decay=0.5):
                self.decay = decay

            def next(self, state, graph):
                raise AssertionError("the device rule replaces next()")

        class RandomScheduler:
            kind = "rand"

            def __init__(self, seed=0):
                self.seed = seed

        s = device_schedule(ThresholdSweepScheduler(decay=0.9))
        assert (s.kind, s.decay) == ("sweep", 0.9)
        r = device_schedule(RandomScheduler(seed=11))
        assert (r.kind, r.seed) == ("rand", 11)

        class DegreeScaled:
            kind = "op2"

        assert device_schedule(DegreeScaled()).kind == "op2"

    def test_custom_next_and_rejection(self):
        from paper_1202_6158_b200.engine import device_schedule

        class Custom:
            def next(self, state, graph):
                return 0

        assert device_schedule(Custom()) is None
        with pytest.raises(TypeError):
            device_schedule(object())


class TestTraceObject:
    def test_csv_header_and_rows(self):
        from paper_1202_6158_b200 import ConvergenceTrace
        t = ConvergenceTrace()
        t.append(0, 0, 0.15, 1.0)
        t.append(10, 3, 0.01, 0.066, true_error=0.05)
        buf = io.StringIO()
        t.write_csv(buf)
        lines = buf.getvalue().strip().splitlines()
        assert lines[0] == "elementary_steps,diffusions,residual,bound,true_error"
        assert len(lines) == 3
        assert t.steps_to_error(0.1) == 10 and t.steps_to_error(0.01) is None


class TestParseErrors:
    """Malformed input is rejected by the host parser before any device work."""

    def load(self, lines, **kw):
        from paper_1202_6158_b200 import load_edge_list
        return load_edge_list(io.StringIO("\n".join(lines) + "\n"), **kw)

    def test_prefixed_forced_on_pairs_fails(self):
        from paper_1202_6158_b200 import GraphFormatError
        with pytest.raises(GraphFormatError):
            self.load(["0 1"], format="prefixed")

    def test_malformed_line_reports_number(self):
        from paper_1202_6158_b200 import GraphFormatError
        with pytest.raises(GraphFormatError) as err:
            self.load(["0 1", "zap"])
        assert err.value.line == 2

    def test_negative_id(self):
        from paper_1202_6158_b200 import GraphFormatError
        with pytest.raises(GraphFormatError):
            self.load(["0 -1"])

    def test_id_overflow(self):
        from paper_1202_6158_b200 import GraphFormatError
        with pytest.raises(GraphFormatError) as err:
            self.load([f"0 {2 ** 63}"])
        assert "overflow" in str(err.value)

    def test_empty_input(self):
        from paper_1202_6158_b200 import GraphFormatError
        with pytest.raises(GraphFormatError):
            self.load([""])

    def test_bad_delta_line(self):
        from paper_1202_6158_b200 import GraphFormatError, load_delta
        with pytest.raises(GraphFormatError):
            load_delta(io.StringIO("* 1 2\n"))

    def test_overlapping_delta_rejected(self):
        from paper_1202_6158_b200 import DeltaError, GraphDelta
        with pytest.raises(DeltaError):
            GraphDelta(added=[(0, 1)], removed=[(0, 1)])


# ---------------------------------------------------------------- GPU: engine
@pytest.fixture
def two_cycle(cuda):
    return cuda.SparseGraph.from_edges(2, [0, 1], [1, 0])


@pytest.fixture
def chain_with_dangling(cuda):
    return cuda.SparseGraph.from_edges(2, [0], [1])


@pytest.mark.gpu
class TestInit:
    def test_uniform_two_nodes(self, cuda, two_cycle):
        s = cuda.init(two_cycle, cuda.DiffusionParams())
        assert np.allclose(host(s.fluid), [0.075, 0.075], atol=1e-15, rtol=0)
        assert s.residual == pytest.approx(0.15, abs=1e-15)
        assert not host(s.history).any()
        assert s.diffusions == 0 and s.elementary_steps == 0

    def test_single_node(self, cuda):
        g = cuda.SparseGraph.from_edges(1, [], [])
        s = cuda.init(g, cuda.DiffusionParams(damping=0.5, teleport=np.array([1.0])))
        assert host(s.fluid)[0] == 0.5 and s.residual == 0.5

    @pytest.mark.parametrize("n", [1, 3, 17])
    def test_initial_mass(self, cuda, n):
        g = cuda.SparseGraph.from_edges(n, [0] if n > 1 else [], [1] if n > 1 else [])
        s = cuda.init(g, cuda.DiffusionParams())
        assert host(s.fluid).sum() == pytest.approx(1 - D, abs=1e-15)


@pytest.mark.gpu
class TestDiffuse:
    def test_two_cycle_arithmetic(self, cuda, two_cycle):
        s = cuda.init(two_cycle, cuda.DiffusionParams())
        cuda.diffuse(s, 0)
        f, h = host(s.fluid), host(s.history)
        assert f[0] == 0.0 and f[1] == pytest.approx(0.075 + 0.06375, abs=1e-15)
        assert h[0] == pytest.approx(0.075, abs=1e-15) and h[1] == 0.0
        assert s.residual == pytest.approx(0.15 - 0.075 * 0.15, abs=1e-15)
        assert s.elementary_steps == 1 and s.diffusions == 1

    def test_dangling_absorbs_everything(self, cuda, chain_with_dangling):
        s = cuda.init(chain_with_dangling, cuda.DiffusionParams())
        r0 = s.residual
        cuda.diffuse(s, 1)
        assert host(s.history)[1] == pytest.approx(0.075, abs=1e-15)
        assert s.residual == pytest.approx(r0 - 0.075, abs=1e-15)
        assert s.elementary_steps == 0

    def test_empty_node_is_noop(self, cuda, two_cycle):
        s = cuda.init(two_cycle, cuda.DiffusionParams())
        s.fluid[0] = 0.0
        snap = (host(s.fluid).copy(), host(s.history).copy(), s.residual, s.diffusions, s.elementary_steps)
        cuda.diffuse(s, 0)
        assert np.array_equal(host(s.fluid), snap[0]) and np.array_equal(host(s.history), snap[1])
        assert (s.residual, s.diffusions, s.elementary_steps) == snap[2:]

    def test_out_of_range(self, cuda, two_cycle):
        s = cuda.init(two_cycle, cuda.DiffusionParams())
        with pytest.raises(IndexError):
            cuda.diffuse(s, 2)


@pytest.mark.gpu
class TestRun:
    def test_two_cycle_symmetric(self, cuda, two_cycle):
        rank, _ = cuda.run(two_cycle, cuda.DiffusionParams(), cuda.sched.GreedyScheduler())
        assert np.allclose(host(rank), [0.5, 0.5], atol=1e-8)

    def test_chain_matches_completed_solve(self, cuda, chain_with_dangling):
        params = cuda.DiffusionParams()
        rank, _ = cuda.run(chain_with_dangling, params, cuda.sched.GreedyScheduler())
        truth = solve_pagerank(2, [0], [1])
        assert truth[0] == pytest.approx(0.5 / 1.425, abs=1e-12)  # hand check: 1.425 x0 = 0.5
        assert np.abs(host(rank) - truth).sum() < 2 * params.target_error

    def test_unnormalized_history_bound(self, cuda):
        rng = np.random.default_rng(21)
        params = cuda.DiffusionParams(target_error=1e-9)
        for _ in range(5):
            src, dst = random_edges(rng, 30)
            g = cuda.SparseGraph.from_edges(30, src, dst)
            s = cuda.init(g, params)
            cuda.run(g, params, cuda.make_scheduler("sweep"), state=s)
            assert np.abs(host(s.history) - solve_unnormalized(30, src, dst)).sum() <= params.target_error * 1.01

    def test_matches_dense_solve_small_graphs(self, cuda):
        rng = np.random.default_rng(33)
        params = cuda.DiffusionParams(target_error=1e-10)
        for _ in range(10):
            n = int(rng.integers(2, 50))
            src, dst = random_edges(rng, n)
            g = cuda.SparseGraph.from_edges(n, src, dst)
            rank, _ = cuda.run(g, params, cuda.sched.GreedyScheduler())
            assert np.abs(host(rank) - solve_pagerank(n, src, dst)).sum() < 1e-9

    def test_schedule_independence(self, cuda):
        rng = np.random.default_rng(4)
        src, dst = random_edges(rng, 60)
        g = cuda.SparseGraph.from_edges(60, src, dst)
        params = cuda.DiffusionParams(target_error=1e-9)
        rules = [cuda.sched.GreedyScheduler(), cuda.sched.RoundRobinScheduler(), cuda.sched.RandomScheduler(seed=9),
                 cuda.make_scheduler("sweep"), cuda.make_scheduler("op"), cuda.make_scheduler("op2"),
                 cuda.make_scheduler("sweep", policy="adaptive", sweep_decay=0.7, degree_exponent=0.65)]
        ranks = [host(cuda.run(g, params, r)[0]) for r in rules]
        for a in ranks:
            for b in ranks:
                assert np.abs(a - b).sum() <= 2 * params.target_error

    def test_conservation_every_step(self, cuda):
        rng = np.random.default_rng(7)
        params = cuda.DiffusionParams()
        for _ in range(3):
            src, dst = random_edges(rng, 25)
            g = cuda.SparseGraph.from_edges(25, src, dst)
            p = dense_p(25, src, dst)
            s = cuda.init(g, params)
            f0 = host(s.fluid).copy()
            rr = cuda.sched.RoundRobinScheduler()
            for _ in range(150):
                cuda.diffuse(s, rr.next(s, g))
                gap = host(s.history) + host(s.fluid) - f0 - D * p @ host(s.history)
                assert np.abs(gap).max() <= 1e-10 * 25

    def test_history_monotone_residual_decreasing(self, cuda):
        rng = np.random.default_rng(8)
        src, dst = random_edges(rng, 20)
        g = cuda.SparseGraph.from_edges(20, src, dst)
        s = cuda.init(g, cuda.DiffusionParams())
        rs = cuda.sched.RandomScheduler(seed=3)
        prev_h, prev_r = host(s.history).copy(), s.residual
        for _ in range(150):
            i = rs.next(s, g)
            had = host(s.fluid)[i] > 0
            cuda.diffuse(s, i)
            assert np.all(host(s.history) >= prev_h)
            if had:
                assert s.residual < prev_r
            prev_h, prev_r = host(s.history).copy(), s.residual

    def test_greedy_fluid_decay(self, cuda):
        """Every greedy step removes at least the (1-d)/n share of the fluid mass."""
        rng = np.random.default_rng(9)
        for _ in range(3):
            src, dst = random_edges(rng, 30)
            g = cuda.SparseGraph.from_edges(30, src, dst)
            s = cuda.init(g, cuda.DiffusionParams())
            gr = cuda.sched.GreedyScheduler()
            shrink = 1 - (1 - D) / 30
            prev = host(s.fluid).sum()
            for _ in range(100):
                cuda.diffuse(s, gr.next(s, g))
                total = host(s.fluid).sum()
                assert total <= prev * shrink + 1e-12
                prev = total
                if total == 0.0:
                    break


@pytest.mark.gpu
class TestErrorBound:
    def test_starts_at_one(self, cuda, two_cycle):
        assert cuda.error_bound(cuda.init(two_cycle, cuda.DiffusionParams())) == pytest.approx(1.0, abs=1e-15)

    def test_at_convergence(self, cuda, two_cycle):
        params = cuda.DiffusionParams()
        s = cuda.init(two_cycle, params)
        cuda.run(two_cycle, params, cuda.sched.GreedyScheduler(), state=s)
        assert cuda.error_bound(s) <= params.target_error

    def test_tracks_fluid_mass_exactly(self, cuda):
        rng = np.random.default_rng(14)
        src, dst = random_edges(rng, 30, dangling_frac=0.0)
        g = cuda.SparseGraph.from_edges(30, src, dst)
        s = cuda.init(g, cuda.DiffusionParams())
        rr = cuda.sched.RoundRobinScheduler()
        for step in range(120):
            cuda.diffuse(s, rr.next(s, g))
            if step % 17 == 0:
                assert cuda.error_bound(s) == pytest.approx(host(s.fluid).sum() / (1 - D), rel=1e-12)


@pytest.mark.gpu
class TestCollect:
    def test_fixed_point_preserved(self, cuda):
        rng = np.random.default_rng(18)
        src, dst = random_edges(rng, 15)
        g = cuda.SparseGraph.from_edges(15, src, dst)
        truth = solve_unnormalized(15, src, dst)
        s = cuda.init(g, cuda.DiffusionParams())
        s.history = torch.as_tensor(truth, device=s.fluid.device).clone()
        for i in range(15):
            cuda.collect(s, i)
            assert host(s.history)[i] == pytest.approx(truth[i], abs=1e-14)

    def test_isolated_node(self, cuda):
        g = cuda.SparseGraph.from_edges(1, [], [])
        s = cuda.init(g, cuda.DiffusionParams(damping=0.5, teleport=np.array([1.0])))
        cuda.collect(s, 0)
        assert host(s.history)[0] == 0.5

    def test_converged_run_is_fixed_point(self, cuda):
        rng = np.random.default_rng(19)
        src, dst = random_edges(rng, 40)
        g = cuda.SparseGraph.from_edges(40, src, dst)
        params = cuda.DiffusionParams(target_error=1e-10)
        s = cuda.init(g, params)
        cuda.run(g, params, cuda.make_scheduler("sweep"), state=s)
        before = host(s.history).copy()
        for i in range(40):
            cuda.collect(s, i)
        assert np.abs(host(s.history) - before).max() < 1e-8

    def test_out_of_range(self, cuda, two_cycle):
        s = cuda.init(two_cycle, cuda.DiffusionParams())
        with pytest.raises(IndexError):
            cuda.collect(s, 5)


@pytest.mark.gpu
class TestTrace:
    def test_csv_shape(self, cuda, two_cycle):
        _, trace = cuda.run(two_cycle, cuda.DiffusionParams(), cuda.sched.GreedyScheduler(), trace_every=1)
        buf = io.StringIO()
        trace.write_csv(buf)
        lines = buf.getvalue().strip().splitlines()
        assert lines[0] == "elementary_steps,diffusions,residual,bound,true_error"
        assert len(lines) == len(trace.rows) + 1
        steps = [r.elementary_steps for r in trace.rows]
        assert steps == sorted(steps)

    def test_true_error_column(self, cuda, two_cycle):
        params = cuda.DiffusionParams()
        _, trace = cuda.run(two_cycle, params, cuda.sched.GreedyScheduler(), trace_every=1,
                            reference=np.array([0.5, 0.5]))
        assert trace.rows[-1].true_error <= params.target_error
        assert trace.steps_to_error(1.0) is not None

    @pytest.mark.parametrize("small", ["1", "0"])
    def test_sampled_true_errors(self, cuda, monkeypatch, small):
        """trace_every + reference (engine.py:265-277, 334-336): sampled rows at least
        trace_every diffusions apart, each with the device-measured true L1 error."""
        monkeypatch.setenv("FR_SMALL", small)
        from oracle import oracle as O
        O.build()
        n = 5000
        src, dst = O.gen_edges(O.web_config(8.0), n, 4)
        off, tgt, _ = O.csr_build(n, src, dst, clean=True)
        g = cuda.SparseGraph(n, off, tgt.astype(np.int32))
        truth = O.run_seq(off, tgt, 0.85, 1e-14, "sweep").rank
        params = cuda.DiffusionParams(target_error=1e-10)
        rank, trace = cuda.run(g, params, cuda.make_scheduler("sweep", policy="geometric", sweep_decay=0.7),
                               trace_every=n // 2, reference=truth)
        rows = trace.rows
        assert len(rows) >= 4
        assert all(b.diffusions - a.diffusions >= n // 2 for a, b in zip(rows[1:-2], rows[2:-1]))
        errs = [r.true_error for r in rows[1:]]
        assert all(e is not None for e in errs)
        assert errs[-1] == pytest.approx(float(np.abs(rank - truth).sum()), abs=1e-15)
        assert errs[-1] <= 1e-9 and errs[0] > errs[-1]
        assert trace.sweep_rows and len(trace.sweep_rows) >= len(rows) - 2

    def test_custom_scheduler_runs_reference_loop(self, cuda, two_cycle):
        """A scheduler with only next(state, graph) is driven node by node (engine.py:289-336)."""
        class Alternate:
            def __init__(self):
                self.k = 0

            def next(self, state, graph):
                self.k += 1
                return self.k % graph.n

        params = cuda.DiffusionParams(target_error=1e-6)
        rank, trace = cuda.run(two_cycle, params, Alternate(), trace_every=1)
        assert np.abs(rank - 0.5).sum() <= 2e-6
        assert len(trace.rows) > 10 and trace.rows[-1].bound <= 1e-6

    def test_custom_scheduler_starvation(self, cuda):
        """A scheduler that keeps picking an empty node raises StarvationError (engine.py:304-312)."""
        class Stuck:
            def next(self, state, graph):
                return 2

        g = cuda.SparseGraph.from_edges(3, [0, 1], [1, 0])
        params = cuda.DiffusionParams(teleport=np.array([0.5, 0.5, 0.0]))
        with pytest.raises(cuda.StarvationError):
            cuda.run(g, params, Stuck())

    def test_signed_state_residual(self, cuda):
        g = cuda.SparseGraph.from_edges(2, [0, 1], [1, 0])
        s = cuda.init_from_fluid(g, cuda.DiffusionParams(), np.array([0.5, -0.25]))
        assert s.signed and s.residual == 0.75


# ---------------------------------------------------------------- GPU: graph
def load_lines(cuda, lines, **kw):
    return cuda.load_edge_list(io.StringIO("\n".join(lines) + "\n"), **kw)


@pytest.mark.gpu
class TestLoadEdgeList:
    def test_two_cycle(self, cuda):
        g = load_lines(cuda, ["0 1", "1 0"])
        assert g.n == 2 and g.edge_count == 2 and g.dangling_count == 0

    def test_dedup_and_self_loop(self, cuda):
        g = load_lines(cuda, ["0 1", "0 1", "1 1"])
        assert g.n == 2 and g.edge_count == 1 and list(g.dangling) == [1]
        assert (g.report.duplicates_dropped, g.report.self_loops_dropped, g.report.edges_seen) == (1, 1, 3)

    def test_comments_and_blank_lines(self, cuda):
        assert load_lines(cuda, ["# header", "% other", "", "0 1", "1 0"]).edge_count == 2

    def test_first_appearance_compaction(self, cuda):
        g = load_lines(cuda, ["5 3", "3 7"])
        assert g.original_ids == [5, 3, 7]
        assert g.has_edge(0, 1) and g.has_edge(1, 2)

    def test_prefixed_format(self, cuda):
        g = load_lines(cuda, ["n 10 http://a", "n 20 http://b", "n 30", "e 10 20", "e 20 30"])
        assert g.n == 3 and g.edge_count == 2
        assert g.labels[0] == "http://a" and g.original_ids == [10, 20, 30]

    def test_node_only_prefixed_input_is_all_dangling(self, cuda):
        g = load_lines(cuda, ["n 1", "n 2"])
        assert g.n == 2 and g.edge_count == 0 and g.dangling_count == 2

    def test_dump_load_round_trip(self, cuda):
        rng = np.random.default_rng(3)
        src, dst = random_edges(rng, 40)
        g = cuda.SparseGraph.from_edges(40, src, dst)
        buf = io.StringIO()
        cuda.dump_edge_list(g, buf)
        g2 = cuda.load_edge_list(io.StringIO(buf.getvalue()))

        def edges(gr):
            s, t = gr.edge_arrays()
            ids = gr.original_ids
            return {(ids[int(a)], ids[int(b)]) for a, b in zip(host(s), host(t))}
        assert edges(g) == edges(g2)

    def test_canonical_bytes_stable(self, cuda):
        from paper_1202_6158_b200.graph import canonical_bytes
        g = load_lines(cuda, ["0 1", "1 0", "1 2"])
        assert canonical_bytes(g) == canonical_bytes(g)


@pytest.mark.gpu
class TestColumn:
    def test_malformed_csr_rejected(self, cuda):
        """A caller-supplied CSR is validated once on the device before any kernel indexes it."""
        with pytest.raises(ValueError):
            cuda.SparseGraph(2, np.array([0, 1, 3]), np.array([1, 0]))  # off[n] != len(targets)
        with pytest.raises(ValueError):
            cuda.SparseGraph(3, np.array([0, 2, 1, 2]), np.array([1, 2]))  # decreasing offsets
        with pytest.raises(ValueError):
            cuda.SparseGraph(2, np.array([0, 1, 2]), np.array([1, 2]))  # target >= n
        with pytest.raises(ValueError):
            cuda.SparseGraph(2, np.array([1, 1, 2]), np.array([1, 0]))  # off[0] != 0
        g = cuda.SparseGraph(2, np.array([0, 1, 2]), np.array([1, 0]))
        assert g.edge_count == 2

    def test_two_cycle(self, cuda, two_cycle):
        assert two_cycle.column(0) == [(1, 1.0)]

    def test_star_weights(self, cuda):
        g = cuda.SparseGraph.from_edges(5, [0, 0, 0, 0], [1, 2, 3, 4])
        assert g.column(0) == [(1, 0.25), (2, 0.25), (3, 0.25), (4, 0.25)]

    def test_dangling_column_empty(self, cuda, chain_with_dangling):
        assert chain_with_dangling.column(1) == []

    def test_out_of_range(self, cuda, two_cycle):
        with pytest.raises(IndexError):
            two_cycle.column(2)
        with pytest.raises(IndexError):
            two_cycle.column(-1)

    def test_column_sums_and_degrees(self, cuda):
        rng = np.random.default_rng(11)
        src, dst = random_edges(rng, 60)
        g = cuda.SparseGraph.from_edges(60, src, dst)
        out_deg, in_deg = host(g.out_degree), host(g.in_degree)
        assert out_deg.sum() == in_deg.sum() == g.edge_count
        for j in range(60):
            col = g.column(j)
            assert out_deg[j] == len(col)
            if col:
                assert abs(sum(w for _, w in col) - 1.0) < 1e-12


@pytest.mark.gpu
class TestDelta:
    def test_add_edge(self, cuda):
        g = cuda.SparseGraph.from_edges(2, [0], [1])
        g2 = cuda.apply_delta(g, cuda.GraphDelta(added=[(1, 0)], removed=[]))
        assert g2.has_edge(1, 0) and g2.dangling_count == 0

    def test_remove_edge_makes_dangling(self, cuda, two_cycle):
        g2 = cuda.apply_delta(two_cycle, cuda.GraphDelta(added=[], removed=[(1, 0)]))
        assert list(g2.dangling) == [1]

    def test_round_trip(self, cuda):
        rng = np.random.default_rng(5)
        src, dst = random_edges(rng, 30)
        g = cuda.SparseGraph.from_edges(30, src, dst)
        s, t = g.edge_arrays()
        removed = [(int(a), int(b)) for a, b in zip(host(s)[:3], host(t)[:3])]
        added = next([(0, k)] for k in range(1, g.n) if not g.has_edge(0, k) and (0, k) not in removed)
        delta = cuda.GraphDelta(added=added, removed=removed)
        g3 = cuda.apply_delta(cuda.apply_delta(g, delta), delta.inverse())
        assert np.array_equal(host(g.out_offsets), host(g3.out_offsets))
        assert np.array_equal(host(g.out_targets), host(g3.out_targets))

    def test_rejections(self, cuda, two_cycle):
        with pytest.raises(cuda.DeltaError):
            cuda.apply_delta(two_cycle, cuda.GraphDelta(added=[], removed=[(0, 0)]))
        with pytest.raises(cuda.DeltaError):
            cuda.apply_delta(two_cycle, cuda.GraphDelta(added=[(0, 1)], removed=[]))

    def test_column_weights_rescale(self, cuda):
        g = cuda.SparseGraph.from_edges(3, [0], [1])
        g2 = cuda.apply_delta(g, cuda.GraphDelta(added=[(0, 2)], removed=[]))
        assert g2.column(0) == [(1, 0.5), (2, 0.5)]

    def test_load_delta_maps_original_ids(self, cuda):
        g = load_lines(cuda, ["5 3", "3 7"])
        delta = cuda.load_delta(io.StringIO("+ 7 5\n- 5 3\n"), graph=g)
        assert delta.added == [(2, 0)] and delta.removed == [(0, 1)]

    def test_delta_columns(self, cuda, two_cycle):
        assert cuda.delta_columns(two_cycle, two_cycle) == []
        g = cuda.SparseGraph.from_edges(6, [3], [1])
        assert cuda.delta_columns(g, cuda.apply_delta(g, cuda.GraphDelta(added=[(3, 2)], removed=[]))) == [3]
        assert cuda.delta_columns(g, cuda.apply_delta(
            g, cuda.GraphDelta(added=[(5, 1)], removed=[(3, 1)]))) == [3, 5]
        with pytest.raises(ValueError):
            cuda.delta_columns(two_cycle, cuda.SparseGraph.from_edges(3, [0], [1]))
