"""Seeded synthetic graphs generated on the device (BASELINE.json configs).

Two generators, both bit-identical to the specification in
oracle/fr_oracle.c (tests/test_gen.py checks it):
  uniform  config 1: out-degree uniform in {0..max_out}, uniform targets
  web      configs 2-5: power-law out-degree (exponent 2.1, max 5000)
           rescaled to a mean, 15 % dangling, 70 % of targets within
           +-window ids, 30 % Zipf(1.0) over a keyed permutation of ids
The edge list is turned into a CSR by the device builder in clean mode
(duplicates collapsed, self-loops dropped -- the reference loader's
semantics, graph.py:183-200), so the realised edge count is reported.
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


def generate_edges(cfg, n, seed):
    """Device edge list (src, dst) as int32 tensors holding uint32 ids."""
    dev = require_device()
    deg = torch.empty(n, dtype=torch.int32, device=dev)
    total = ctypes.c_int64(0)
    check(lib.fr_gen_degrees(ctypes.byref(cfg), n, seed, ptr(deg), ctypes.byref(total), stream_ptr()))
    m = int(total.value)
    src = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    dst = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    check(lib.fr_gen_edges(ctypes.byref(cfg), n, seed, ptr(deg), ptr(src), ptr(dst), stream_ptr()))
    return src[:m], dst[:m]


@dataclass(frozen=True)
class GenReport:
    slots: int            # edges drawn
    realized_links: int   # after dedup / self-loop removal
    duplicates: int
    self_loops: int
    dangling: int
    seed: int


def generate(cfg, n, seed=0):
    """(SparseGraph, GenReport) for a generator config, built on the device."""
    src, dst = generate_edges(cfg, n, seed)
    off, tgt, (L, dups, loops) = csr_build(n, src, dst, clean=True)
    del src, dst
    g = SparseGraph(n, off, tgt, _trusted=True)
    rep = GenReport(slots=L + dups + loops, realized_links=L, duplicates=dups, self_loops=loops,
                    dangling=g.dangling_count, seed=seed)
    return g, rep


def baseline_graph(config_index, seed=0, n=None):
    """The graph of BASELINE.json config 1..5 (n may be overridden to scale it)."""
    spec = CONFIGS[config_index]
    return generate(spec["cfg"](), spec["n"] if n is None else n, seed)


def degree_report(graph):
    """Exact in/out degree histograms as {degree: count} (gen.py:113-120)."""
    out_hist = torch.bincount(graph.out_degree).cpu().numpy()
    in_hist = torch.bincount(graph.in_degree).cpu().numpy()
    return {"out": {int(d): int(c) for d, c in enumerate(out_hist) if c},
            "in": {int(d): int(c) for d, c in enumerate(in_hist) if c}}
