"""Power iteration (MAT-ITER) on the GPU: mirror of fluidrank/baseline.py:20-56.

The matrix-vector product is the pull CSR SpMV of csrc/fr_spmv.cu over the
transposed graph; the whole iteration loop runs inside one CUDA graph.
The online ranker (OPIC, baseline.py:59-186) is not on the accelerated path.
"""

from __future__ import annotations

import ctypes

import torch

from ._lib import check, lib, ptr, require_device, stream_ptr
from .engine import ConvergenceTrace


class PowerIteration:
    """fr_power_* handle bound to one graph and teleport vector."""

    def __init__(self, graph, params):
        dev = require_device()
        self.graph = graph
        in_off, in_src = graph.reverse_csr()
        self._tel = None if params.teleport is None else params.teleport_vector(graph.n, dev).contiguous()
        handle = ctypes.c_void_p()
        check(lib.fr_power_create(graph.n, graph.edge_count, ptr(graph.out_offsets), ptr(in_off), ptr(in_src),
                                  float(params.damping), ptr(self._tel), stream_ptr(), ctypes.byref(handle)))
        self.handle = handle

    def run(self, target_error, max_iterations=1_000_000):
        x = torch.empty(self.graph.n, dtype=torch.float64, device=self.graph.out_offsets.device)
        iters = ctypes.c_int64(0)
        diff = ctypes.c_double(0.0)
        rc = lib.fr_power_run(self.handle, float(target_error), int(max_iterations), ptr(x), ctypes.byref(iters),
                              ctypes.byref(diff), stream_ptr())
        if rc == 6:
            raise RuntimeError(f"no convergence within {max_iterations} iterations")
        check(rc)
        return x, int(iters.value), float(diff.value)

    def run_profiled(self, target_error, max_iterations=1_000_000):
        """Same iterations launched from the host with CUDA events: (x, iterations, rows_ms,
        hubs_ms, rest_ms) summed over the iterations (roofline report): short rows with
        their update, hub rows regrouped by source block (slices and long segments), and
        the hub rows' update with the stopping rule."""
        x = torch.empty(self.graph.n, dtype=torch.float64, device=self.graph.out_offsets.device)
        iters = ctypes.c_int64(0)
        ms = (ctypes.c_double * 4)()
        check(lib.fr_power_run_profiled(self.handle, float(target_error), int(max_iterations), ptr(x),
                                        ctypes.byref(iters), ms, stream_ptr()))
        self.last_profile_ms = {"short_rows": ms[0], "hub_slices": ms[1], "hub_segments": ms[2], "rest": ms[3]}
        return x, int(iters.value), ms[0], ms[1] + ms[2], ms[3]

    def close(self):
        if self.handle:
            lib.fr_power_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def power_iterate(graph, params, target_error=None, trace_every=1, reference=None, max_iterations=1_000_000,
                  as_tensor=False):
    """Power iteration with dangling mass folded back through the teleport.

    Stops when |X_n - X_{n-1}|_1 * d/(1-d) <= target_error (params.target_error
    by default).  Returns (rank, trace): rank is a numpy vector like the
    reference's (``as_tensor=True``: the device tensor); each iteration costs L
    elementary steps.  The loop runs on the device, so the trace holds the
    final row.
    """
    params.validate(graph.n)
    d = params.damping
    if d >= 1.0:
        raise ValueError("power iteration requires damping < 1")
    if target_error is None:
        target_error = params.target_error
    pi = PowerIteration(graph, params)
    try:
        x, iters, diff = pi.run(target_error, max_iterations)
    finally:
        pi.close()
    trace = ConvergenceTrace()
    err = None
    if reference is not None:
        ref = torch.as_tensor(reference, dtype=torch.float64).to(x.device)
        err = float((x - ref).abs().sum())
    trace.append(iters * graph.edge_count, iters, diff, diff * d / (1.0 - d), err)
    return (x if as_tensor else x.cpu().numpy()), trace
