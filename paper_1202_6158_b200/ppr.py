"""Batched personalized PageRank by fluid diffusion (BASELINE.json config 4).

Each of B <= 64 personalization vectors V_c (uniform over k seed nodes) is an
independent instance of the reference's run() with teleport = V_c
(engine.py:240-341); on the device the B instances share one sweep: fluid and
history are n x B row-major fp64 arrays, every edge visit scatters a B-wide
vector, and each column stops at its own residual target.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import check, lib, ptr, require_device, stream_ptr


def config4_seeds(n, B=64, k=10, seed=0):
    """B personalization vectors, each uniform over k seed nodes drawn at random (config 4)."""
    rng = np.random.default_rng(seed)
    return np.stack([rng.choice(n, size=k, replace=False) for _ in range(B)]).astype(np.uint32)


class BatchedPPR:
    """fr_ppr_* handle: graph + (n x B) state, reusable across solves."""

    MODES = ("push", "pull")

    def __init__(self, graph, B, damping=0.85, target_error=1e-9, decay=0.6, max_sweeps=0, mode="push"):
        """mode "push" (default, fastest): every edge visit scatters the row with
        red.global.add; "pull": take + pull over the transposed CSR (no atomics,
        bit-reproducible, Jacobi within a sweep: more sweeps)."""
        if mode not in self.MODES:
            raise ValueError(f"mode must be one of {sorted(self.MODES)}, got {mode!r}")
        if not 1 <= B <= 64:
            raise ValueError(f"B must be in [1, 64], got {B}")
        dev = require_device()
        self.graph, self.B = graph, int(B)
        self.damping, self.target_error = float(damping), float(target_error)
        self.fluid = torch.zeros((graph.n, B), dtype=torch.float64, device=dev)
        self.history = torch.zeros((graph.n, B), dtype=torch.float64, device=dev)
        cfg = _lib.SolverConfig()
        cfg.damping, cfg.target_error, cfg.decay = self.damping, self.target_error, float(decay)
        cfg.max_sweeps = int(max_sweeps)
        handle = ctypes.c_void_p()
        check(lib.fr_ppr_create(graph.n, graph.edge_count, ptr(graph.out_offsets), ptr(graph.out_targets), B,
                                ptr(self.fluid), ptr(self.history), ctypes.byref(cfg), stream_ptr(),
                                ctypes.byref(handle)))
        self.handle = handle
        self.mode = mode
        if mode == "pull":
            in_off, in_src = graph.reverse_csr()
            check(lib.fr_ppr_set_pull(self.handle, ptr(in_off), ptr(in_src)))

    def solve(self, seeds):
        """seeds: (B, k) node ids.  Returns (rank n x B device tensor, stats, column residuals)."""
        s = torch.as_tensor(np.ascontiguousarray(seeds, dtype=np.uint32).astype(np.int64), device=self.fluid.device)
        if s.dim() != 2 or s.shape[0] != self.B:
            raise ValueError(f"seeds must have shape ({self.B}, k)")
        if bool((s < 0).any()) or bool((s >= self.graph.n).any()):
            raise ValueError("seed node out of range")
        s32 = s.to(torch.int32).contiguous()
        check(lib.fr_ppr_init(self.graph.n, self.B, ptr(s32), int(s.shape[1]), self.damping, ptr(self.fluid),
                              ptr(self.history), stream_ptr()))
        stats = _lib.SolveStats()
        resid = (ctypes.c_double * self.B)()
        check(lib.fr_ppr_run(self.handle, stream_ptr(), ctypes.byref(stats), resid))
        rank = torch.empty_like(self.history)
        check(lib.fr_ppr_normalize(self.graph.n, self.B, ptr(self.history), ptr(rank), stream_ptr()))
        return rank, stats, list(resid)

    def close(self):
        if self.handle:
            lib.fr_ppr_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def personalized_pagerank(graph, seeds, damping=0.85, target_error=1e-9, decay=0.6, mode="push"):
    """Rank vectors (n x B) for B seed sets (B x k), one batched device solve."""
    seeds = np.asarray(seeds)
    p = BatchedPPR(graph, seeds.shape[0], damping, target_error, decay, mode=mode)
    try:
        rank, stats, resid = p.solve(seeds)
    finally:
        p.close()
    return rank, stats, resid
