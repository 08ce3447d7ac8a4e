"""Fluid-diffusion ranking engine on the GPU (mirror of fluidrank/engine.py).

Same names, argument meaning and errors as the reference; the state vectors
live in HBM as torch tensors and run() drives the device sweep solver of
csrc/fr_diffuse.cu (whole convergence loop inside one CUDA graph).  The
returned rank is a numpy float64 vector like the reference's; pass
``as_tensor=True`` to keep it on the device.
"""

from __future__ import annotations

import csv
import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check, lib, ptr, require_device, stream_ptr
from .sched import KINDS, DeviceSchedule


class StarvationError(RuntimeError):
    """A scheduler kept selecting empty nodes while fluid remained."""


class ParamsMismatchError(ValueError):
    """Two run phases were configured with incompatible parameters."""


@dataclass
class DiffusionParams:
    """Damping, teleport distribution and stopping threshold (engine.py:29-69).

    teleport=None means uniform 1/N; damping=1.0 only with a diffusion budget.
    """

    damping: float = 0.85
    teleport: object = None
    target_error: float = 1e-8

    def validate(self, n=None):
        if not 0.0 < self.damping <= 1.0:
            raise ValueError(f"damping must be in (0, 1], got {self.damping}")
        if self.target_error <= 0.0:
            raise ValueError(f"target_error must be positive, got {self.target_error}")
        if self.teleport is not None:
            v = torch.as_tensor(self.teleport, dtype=torch.float64)
            if n is not None and tuple(v.shape) != (n,):
                raise ValueError(f"teleport length {tuple(v.shape)} does not match n={n}")
            if bool((v < 0.0).any()):
                raise ValueError("teleport vector has negative entries")
            total = float(v.sum())
            if abs(total - 1.0) > 1e-12:
                raise ValueError(f"teleport vector sums to {total!r}, expected 1")

    def teleport_vector(self, n, device=None):
        device = device or require_device()
        if self.teleport is None:
            return torch.full((n,), 1.0 / n, dtype=torch.float64, device=device)
        v = torch.as_tensor(self.teleport, dtype=torch.float64).to(device)
        if tuple(v.shape) != (n,):
            raise ValueError(f"teleport length {tuple(v.shape)} does not match n={n}")
        return v.clone()

    def matches(self, other):
        if (self.teleport is None) != (other.teleport is None):
            return False
        same_v = self.teleport is None or torch.equal(
            torch.as_tensor(self.teleport, dtype=torch.float64).cpu(),
            torch.as_tensor(other.teleport, dtype=torch.float64).cpu())
        return self.damping == other.damping and self.target_error == other.target_error and same_v


@dataclass
class TraceRow:
    elementary_steps: int
    diffusions: int
    residual: float
    bound: float | None
    true_error: float | None = None
    sweeps: int = 0
    theta: float | None = None


class ConvergenceTrace:
    """Sampled convergence history (one row per device sweep), CSV-serializable."""

    FIELDS = ("elementary_steps", "diffusions", "residual", "bound", "true_error")

    def __init__(self):
        self.rows = []
        self.sweep_rows = []  # device runs: (elementary_steps, diffusions, residual, bound) per sweep

    def append(self, elementary_steps, diffusions, residual, bound, true_error=None, sweeps=0, theta=None):
        self.rows.append(TraceRow(int(elementary_steps), int(diffusions), float(residual),
                                  None if bound is None else float(bound), true_error, int(sweeps), theta))

    def write_csv(self, sink):
        close = False
        if isinstance(sink, (str, bytes)) or hasattr(sink, "__fspath__"):
            sink = open(sink, "w", encoding="utf-8", newline="")
            close = True
        try:
            writer = csv.writer(sink)
            writer.writerow(self.FIELDS)
            for r in self.rows:
                writer.writerow([r.elementary_steps, r.diffusions, f"{r.residual:.17g}",
                                 "" if r.bound is None else f"{r.bound:.17g}",
                                 "" if r.true_error is None else f"{r.true_error:.17g}"])
        finally:
            if close:
                sink.close()

    def steps_to_error(self, threshold):
        for r in self.rows:
            if r.true_error is not None and r.true_error <= threshold:
                return r.elementary_steps
        return None

    def __len__(self):
        return len(self.rows)


@dataclass
class DiffusionState:
    """Fluid, history, residual and counters; vectors are device tensors."""

    fluid: torch.Tensor
    history: torch.Tensor
    residual: float
    diffusions: int = 0
    elementary_steps: int = 0
    signed: bool = False
    graph: object = None
    params: DiffusionParams = None
    sweeps: int = 0

    def fluid_magnitude(self):
        return self.fluid.abs() if self.signed else self.fluid

    def exact_residual(self):
        out = ctypes.c_double(0.0)
        check(lib.fr_abs_sum(self.fluid.numel(), ptr(self.fluid), int(self.fluid.dtype == torch.float32),
                             ctypes.byref(out), stream_ptr()))
        return out.value


def _fluid_fp32(dtype):
    if dtype in (None, torch.float64):
        return False
    if dtype == torch.float32:
        return True
    raise ValueError(f"fluid dtype must be float64 or float32, got {dtype}")


def init(graph, params, fluid_dtype=torch.float64):
    """Fresh state: fluid = (1-d)*teleport, history = 0 (engine.py:149-159)."""
    params.validate(graph.n)
    dev = require_device()
    fp32 = _fluid_fp32(fluid_dtype)
    fluid = torch.empty(graph.n, dtype=torch.float32 if fp32 else torch.float64, device=dev)
    history = torch.empty(graph.n, dtype=torch.float64, device=dev)
    tel = None if params.teleport is None else params.teleport_vector(graph.n, dev)
    check(lib.fr_init_state(graph.n, float(params.damping), ptr(tel), ptr(fluid), int(fp32), ptr(history),
                            stream_ptr()))
    state = DiffusionState(fluid=fluid, history=history, residual=0.0, graph=graph, params=params)
    state.residual = state.exact_residual()
    return state


def init_from_fluid(graph, params, fluid, history=None, fluid_dtype=torch.float64):
    """State seeded with an arbitrary (possibly signed) fluid (engine.py:162-172)."""
    params.validate(graph.n)
    dev = require_device()
    fp32 = _fluid_fp32(fluid_dtype)
    f = torch.as_tensor(fluid, dtype=torch.float64).to(dev).clone()
    if tuple(f.shape) != (graph.n,):
        raise ValueError(f"fluid length {tuple(f.shape)} does not match n={graph.n}")
    if fp32:
        f = f.to(torch.float32)
    h = (torch.zeros(graph.n, dtype=torch.float64, device=dev) if history is None
         else torch.as_tensor(history, dtype=torch.float64).to(dev).clone())
    signed = bool((f < 0.0).any())
    state = DiffusionState(fluid=f, history=h, residual=0.0, signed=signed, graph=graph, params=params)
    state.residual = state.exact_residual() if signed else float(f.sum(dtype=torch.float64))
    return state


def diffuse(state, i, graph=None, params=None):
    """Diffuse node i once (engine.py:175-199); a node without fluid is a no-op."""
    graph = state.graph if graph is None else graph
    params = state.params if params is None else params
    if not 0 <= i < graph.n:
        raise IndexError(f"node {i} out of range")
    if state.fluid.dtype != torch.float64:
        raise ValueError("single-node diffuse works on float64 fluid")
    sent = ctypes.c_double(0.0)
    check(lib.fr_diffuse_node(graph.n, ptr(graph.out_offsets), ptr(graph.out_targets), ptr(state.fluid),
                              ptr(state.history), int(i), float(params.damping), ctypes.byref(sent),
                              stream_ptr()))
    s = sent.value
    if s == 0.0:
        return state
    deg = int(graph.out_offsets[i + 1] - graph.out_offsets[i])
    if deg:
        state.residual -= abs(s) * (1.0 - params.damping)
        state.elementary_steps += deg
    else:
        state.residual -= abs(s)
    state.diffusions += 1
    return state


def error_bound(state, params=None):
    """Upper bound on the L1 distance of history to its limit (engine.py:202-211)."""
    params = state.params if params is None else params
    if params.damping >= 1.0:
        return math.inf
    return state.residual / (1.0 - params.damping)


def collect(state, i, graph=None, params=None):
    """Pull-style recompute of one history entry (engine.py:214-232)."""
    graph = state.graph if graph is None else graph
    params = state.params if params is None else params
    if not 0 <= i < graph.n:
        raise IndexError(f"node {i} out of range")
    v = float(params.teleport[i]) if params.teleport is not None else 1.0 / graph.n
    in_off, in_src = graph.reverse_csr()
    lo, hi = int(in_off[i]), int(in_off[i + 1])
    pulled = 0.0
    if hi > lo:
        par = in_src[lo:hi].to(torch.int64)
        pulled = float((state.history[par] / graph.out_degree[par].to(torch.float64)).sum())
    state.history[i] = (1.0 - params.damping) * v + params.damping * pulled
    return state.history


class Solver:
    """A device solver bound to (graph, state, rule): fr_solver_* of the C ABI.

    Reusable: run() diffuses from the current state to the target each call.
    """

    def __init__(self, graph, state, scheduler, params=None, max_sweeps=0, max_diffusions=None,
                 trace_cap=1 << 16):
        params = state.params if params is None else params
        self.graph, self.state, self.scheduler, self.params = graph, state, scheduler, params
        self.fp32 = state.fluid.dtype == torch.float32
        self._weights = scheduler.weights(graph).contiguous() if scheduler.needs_weights() else None
        cfg = scheduler.solver_config(params, self.fp32, max_sweeps, max_diffusions)
        self.cfg = cfg
        handle = ctypes.c_void_p()
        check(lib.fr_solver_create(graph.n, graph.edge_count, ptr(graph.out_offsets), ptr(graph.out_targets),
                                   ptr(self._weights), ptr(state.fluid), ptr(state.history), ctypes.byref(cfg),
                                   int(trace_cap), stream_ptr(), ctypes.byref(handle)))
        self.handle = handle
        self.trace_cap = trace_cap

    def run(self, profiled=False):
        stats = _lib.SolveStats()
        if profiled:
            ms = (ctypes.c_double * 5)()
            launches = (ctypes.c_int64 * 5)()
            check(lib.fr_solver_run_profiled(self.handle, stream_ptr(), ctypes.byref(stats), ms, launches))
            self.kernel_ms = list(ms)
            self.kernel_launches = list(launches)
        else:
            check(lib.fr_solver_run(self.handle, stream_ptr(), ctypes.byref(stats)))
        return stats

    def trace_rows(self):
        rows = (_lib.TraceRow * self.trace_cap)()
        length = ctypes.c_int64(0)
        check(lib.fr_solver_trace(self.handle, rows, self.trace_cap, ctypes.byref(length), stream_ptr()))
        return [rows[k] for k in range(min(length.value, self.trace_cap))]

    def close(self):
        if self.handle:
            lib.fr_solver_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _normalized(history):
    rank = torch.empty_like(history)
    check(lib.fr_normalize(history.numel(), ptr(history), ptr(rank), None, stream_ptr()))
    return rank


def _true_error(history, ref):
    """|history/|history|_1 - ref|_1 on the device (engine.py:269-274); None before any mass."""
    out = ctypes.c_double(0.0)
    check(lib.fr_l1_error(history.numel(), ptr(history), ptr(ref), ctypes.byref(out), stream_ptr()))
    return out.value if float(history.abs().sum()) > 0.0 else None


def device_schedule(scheduler):
    """The device sweep rule for a scheduler object, or None for a custom next() rule.

    Accepts this package's DeviceSchedule and any object carrying the reference's
    ``kind`` attribute (sched.py:16-161: the reference classes, with their ``decay``
    and ``seed``); objects without a known kind but with next(state, graph) are
    driven one node at a time like the reference loop (engine.py:297).
    """
    if isinstance(scheduler, DeviceSchedule):
        return scheduler
    kind = getattr(scheduler, "kind", None)
    if kind in KINDS:
        kw = {}
        if kind == "sweep":
            kw["decay"] = float(getattr(scheduler, "decay", 0.5))
        if kind == "rand":
            seed = getattr(scheduler, "seed", 0)
            kw["seed"] = int(seed) if isinstance(seed, (int, np.integer)) else 0
        return DeviceSchedule(kind, **kw)
    if callable(getattr(scheduler, "next", None)):
        return None
    raise TypeError(f"scheduler {scheduler!r} has neither a known kind ({', '.join(KINDS)}) nor next(state, graph)")


def _output(rank, as_tensor):
    return rank if as_tensor else rank.cpu().numpy()


def _run_custom(graph, params, scheduler, state, trace, threshold, trace_every, ref, max_diffusions):
    """engine.py:289-336 for a scheduler with only next(state, graph): the reference
    loop, one device diffusion per selection, with its starvation bookkeeping."""
    n, d = graph.n, params.damping
    stamp = np.zeros(n, dtype=np.int64)
    epoch, distinct_empty, empty_streak, streak_cap = 1, 0, 0, 64 * n
    next_trace = state.diffusions + trace_every
    next_refresh = state.diffusions + n

    def sample():
        err = None if ref is None else _true_error(state.history, ref)
        trace.append(state.elementary_steps, state.diffusions, state.residual,
                     None if d >= 1.0 else state.residual / (1.0 - d), err, sweeps=state.sweeps)

    while True:
        if state.residual <= threshold:
            state.residual = state.exact_residual()
            if state.residual <= threshold:
                break
        if max_diffusions is not None and state.diffusions >= max_diffusions:
            break
        i = int(scheduler.next(state, graph))
        before = state.diffusions
        diffuse(state, i, graph, params)
        if state.diffusions == before:  # the node held no fluid
            empty_streak += 1
            if stamp[i] != epoch:
                stamp[i] = epoch
                distinct_empty += 1
            if distinct_empty >= n or empty_streak >= streak_cap:
                state.residual = state.exact_residual()
                if state.residual <= threshold:
                    break
                raise StarvationError(
                    f"scheduler made {empty_streak} empty selections covering {distinct_empty} nodes while "
                    f"bound {error_bound(state, params):.3g} exceeds target {params.target_error:.3g}")
            continue
        empty_streak = distinct_empty = 0
        epoch += 1
        if state.diffusions >= next_refresh:
            state.residual = state.exact_residual()
            next_refresh = state.diffusions + n
        if state.diffusions >= next_trace:
            sample()
            next_trace = state.diffusions + trace_every


def run(graph, params, scheduler, trace_every=None, reference=None, max_diffusions=None, state=None,
        fluid_dtype=torch.float64, max_sweeps=0, as_tensor=False):
    """Diffuse until residual/(1-d) <= target_error (engine.py:240-341).

    Returns (rank, trace): rank is the history renormalized to sum one, a numpy
    float64 vector like the reference's (``as_tensor=True``: the device tensor,
    no copy).  The device solves whole sweeps, so trace rows are sampled at
    sweep ends: a row once the diffusion count has advanced by trace_every
    (default n, as the reference) since the last one, plus the first and last
    rows; ``trace.sweep_rows`` keeps one row per sweep.  With ``reference`` (a
    normalized rank vector) every sampled row carries the true L1 error, taken
    on the device at that sweep (fr_solver_run_sampled).  With damping=1.0
    max_diffusions is required.
    """
    params.validate(graph.n)
    d = params.damping
    n = graph.n
    if d >= 1.0 and max_diffusions is None:
        raise ValueError("undamped diagnostic mode requires max_diffusions")
    sched = device_schedule(scheduler)
    if state is None:
        state = init(graph, params, fluid_dtype=fluid_dtype)
    trace_every = n if trace_every is None else max(1, int(trace_every))
    ref = None
    if reference is not None:
        ref = torch.as_tensor(np.asarray(reference, dtype=np.float64) if not isinstance(reference, torch.Tensor)
                              else reference, dtype=torch.float64).to(state.history.device).contiguous()
        if tuple(ref.shape) != (n,):
            raise ValueError(f"reference length {tuple(ref.shape)} does not match n={n}")
    trace = ConvergenceTrace()

    def bound(r):
        return None if d >= 1.0 else r / (1.0 - d)

    err0 = None if ref is None else _true_error(state.history, ref)
    trace.append(state.elementary_steps, state.diffusions, state.residual, bound(state.residual), err0,
                 sweeps=state.sweeps)
    if sched is None:
        _run_custom(graph, params, scheduler, state, trace, params.target_error * (1.0 - d), trace_every, ref,
                    max_diffusions)
        state.residual = state.exact_residual()
    else:
        solver = Solver(graph, state, sched, params, max_sweeps=max_sweeps,
                        max_diffusions=None if max_diffusions is None else max_diffusions - state.diffusions)
        try:
            if ref is None:
                stats = solver.run()
                errs = None
            else:
                stats = _lib.SolveStats()
                check(lib.fr_solver_run_sampled(solver.handle, stream_ptr(), ptr(ref), int(trace_every),
                                                ctypes.byref(stats)))
                errs = (ctypes.c_double * solver.trace_cap)()
                check(lib.fr_solver_trace_errors(solver.handle, errs, solver.trace_cap, stream_ptr()))
            base_steps, base_diff, base_sweeps = state.elementary_steps, state.diffusions, state.sweeps
            next_trace = base_diff + trace_every
            for k, r in enumerate(solver.trace_rows()):
                steps, diffs = base_steps + r.elementary_steps, base_diff + r.diffusions
                row = (steps, diffs, r.residual, bound(r.residual))
                trace.sweep_rows.append(row)
                if diffs >= next_trace:
                    e = None if errs is None or math.isnan(errs[k]) else float(errs[k])
                    trace.append(*row, e, sweeps=base_sweeps + r.sweeps, theta=r.theta)
                    next_trace = diffs + trace_every
        finally:
            solver.close()
        state.elementary_steps += int(stats.elementary_steps)
        state.diffusions += int(stats.diffusions)
        state.sweeps += int(stats.sweeps)
        state.residual = float(stats.residual)
    rank = _normalized(state.history)
    err = None if ref is None else float((rank - ref).abs().sum())
    # the final sample (engine.py:338-340), with the exact residual: it restates a
    # row already taken at the same diffusion count
    if trace.rows and trace.rows[-1].diffusions == state.diffusions:
        trace.rows.pop()
    trace.append(state.elementary_steps, state.diffusions, state.residual, bound(state.residual), err,
                 sweeps=state.sweeps)
    return _output(rank, as_tensor), trace
