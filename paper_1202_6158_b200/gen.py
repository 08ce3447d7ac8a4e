"""Seeded synthetic graphs generated on the device (BASELINE.json configs).

Two generators, both bit-identical to the specification in
oracle/fr_oracle.c (tests/test_gen.py checks it):
  uniform  config 1: out-degree uniform in {0..max_out}, uniform targets
  web      configs 2-5: power-law out-degree (exponent 2.1, max 5000)
           rescaled to a mean, 15 % dangling, 70 % of targets within
           +-window ids, 30 % Zipf(1.0) over a keyed permutation of ids
The edge list is turned into a CSR by the device builder in clean mode
(duplicates collapsed, self-loops dropped -- the reference loader's
semantics, graph.py:183-200).  The BASELINE graphs (baseline_graph) then
redraw the dropped slots in fill rounds until the configured out-degrees
exist as distinct edges (the reference generator's "draw until the target
number of distinct links exists", gen.py:66-110).
The paper's own section-4.1 generator (reference gen.py) is a sequential
numpy rejection sampler and is not on the accelerated path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import check, lib, ptr, require_device, stream_ptr
from .graph import SparseGraph, csr_build


def uniform_config(max_out=10):
    return _lib.GenConfig(kind=0, max_out=max_out)


def web_config(mean_degree=8.0, alpha=2.1, max_degree=5000, window=1000, dangling_frac=0.15,
               local_frac=0.7, zipf_s=1.0):
    return _lib.GenConfig(kind=1, mean_degree=mean_degree, alpha=alpha, max_degree=max_degree,
                          window=window, dangling_frac=dangling_frac, local_frac=local_frac, zipf_s=zipf_s)


# BASELINE.json configs (index = position in "configs")
CONFIGS = {
    1: dict(n=10_000, cfg=lambda: uniform_config(10), target_error=1e-10),
    2: dict(n=1_000_000, cfg=lambda: web_config(8.0), target_error=1e-9),
    3: dict(n=20_000_000, cfg=lambda: web_config(10.0), target_error=1e-9),
    4: dict(n=1_000_000, cfg=lambda: web_config(8.0), target_error=1e-9),
    5: dict(n=100_000_000, cfg=lambda: web_config(16.0), target_error=1e-9),
}


def gen_degrees(cfg, n, seed):
    """Configured out-degree (slot count) of every node: device int32 tensor, total."""
    dev = require_device()
    deg = torch.empty(n, dtype=torch.int32, device=dev)
    total = ctypes.c_int64(0)
    check(lib.fr_gen_degrees(ctypes.byref(cfg), n, seed, ptr(deg), ctypes.byref(total), stream_ptr()))
    return deg, int(total.value)


def draw_edges(cfg, n, seed, deg, total, round=0, off=None, tgt=None):
    """Source-major draws for deg[u] slots of every node u (fill round `round`; (off, tgt)
    the clean graph so far)."""
    dev = deg.device
    src = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    dst = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    check(lib.fr_gen_edges_round(ctypes.byref(cfg), n, seed, int(round), ptr(deg), ptr(off), ptr(tgt), ptr(src),
                                 ptr(dst), stream_ptr()))
    return src[:total], dst[:total]


def generate_edges(cfg, n, seed):
    """Device edge list (src, dst) as int32 tensors holding uint32 ids (the base draw)."""
    deg, m = gen_degrees(cfg, n, seed)
    return draw_edges(cfg, n, seed, deg, m, 0)


@dataclass(frozen=True)
class GenReport:
    slots: int            # edges drawn (all rounds)
    realized_links: int   # after dedup / self-loop removal
    duplicates: int       # draws dropped as duplicates (all rounds)
    self_loops: int       # draws dropped as self-loops (all rounds)
    dangling: int
    seed: int
    target_links: int = 0  # configured out-degrees summed
    rounds: int = 0        # fill rounds after the base draw (exact mode)
    unfilled: int = 0      # target_links - realized_links


MAX_FILL_ROUNDS = 32


def generate(cfg, n, seed=0, exact=False, max_rounds=MAX_FILL_ROUNDS):
    """(SparseGraph, GenReport) for a generator config, built on the device.

    exact=False: the base draw, cleaned (duplicates collapsed, self-loops
    dropped, graph.py:183-200).  exact=True: the slots that cleaning dropped are
    redrawn in fill rounds (fr_gen_edges_round) until every node has its
    configured out-degree in distinct edges -- as the reference generator draws
    until the target number of distinct links exists (gen.py:66-110); a node
    whose window and Zipf mass cannot supply them within max_rounds keeps the
    deficit (reported as unfilled).
    """
    deg, total = gen_degrees(cfg, n, seed)
    src, dst = draw_edges(cfg, n, seed, deg, total, 0)
    off, tgt, (L, dups, loops) = csr_build(n, src, dst, clean=True)
    del src, dst
    torch.cuda.empty_cache()
    slots, rounds = total, 0
    if exact:
        deg64 = deg.to(torch.int64)
        for r in range(1, max_rounds + 1):
            deficit = deg64 - torch.diff(off)
            need = int(deficit.sum())
            if need == 0:
                break
            d32 = deficit.to(torch.int32)
            s2, d2 = draw_edges(cfg, n, seed, d32, need, r, off, tgt)
            # clean union of the graph so far with the redraws: one device CSR build
            rows = torch.repeat_interleave(torch.arange(n, dtype=torch.int32, device=off.device), torch.diff(off))
            src = torch.cat([rows, s2])
            del rows, s2
            dst = torch.cat([tgt, d2])
            del off, tgt, d2, d32, deficit
            # the builder allocates from the CUDA stream-ordered pool: hand torch's cached
            # blocks back first (config 5: 1.6B edges, ~13 GB per edge-list copy)
            torch.cuda.empty_cache()
            off, tgt, (L, rd, rl) = csr_build(n, src, dst, clean=True)
            del src, dst
            torch.cuda.empty_cache()
            slots += need
            dups += rd
            loops += rl
            rounds = r
    g = SparseGraph(n, off, tgt, _trusted=True)
    rep = GenReport(slots=slots, realized_links=L, duplicates=dups, self_loops=loops, dangling=g.dangling_count,
                    seed=seed, target_links=total, rounds=rounds, unfilled=total - L)
    return g, rep


def baseline_graph(config_index, seed=0, n=None, exact=True):
    """The graph of BASELINE.json config 1..5 (n may be overridden to scale it): the
    configured out-degrees realised as distinct edges (exact=True, see generate)."""
    spec = CONFIGS[config_index]
    return generate(spec["cfg"](), spec["n"] if n is None else n, seed, exact=exact)


def degree_report(graph):
    """Exact in/out degree histograms as {degree: count} (gen.py:113-120)."""
    out_hist = torch.bincount(graph.out_degree).cpu().numpy()
    in_hist = torch.bincount(graph.in_degree).cpu().numpy()
    return {"out": {int(d): int(c) for d, c in enumerate(out_hist) if c},
            "in": {int(d): int(c) for d, c in enumerate(in_hist) if c}}
