"""Batched personalized PageRank timing on BASELINE config 3 (1M-node web graph,
mean out-degree 8, 64 vectors x 10 seeds, d=0.85, each column to L1 residual
1e-9).  Development tool; bench.py carries the same leg in its JSON line."""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1202_6158_b200 as fr  # noqa: E402
from paper_1202_6158_b200 import gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--mean", type=float, default=8.0)
ap.add_argument("--B", type=int, default=64)
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--decay", default="0.9")
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()

g, _ = gen.generate(gen.web_config(args.mean), args.n, 0)
seeds = fr.config4_seeds(args.n, args.B, args.k, seed=0)
for decay in [float(x) for x in args.decay.split(",")]:
    p = fr.BatchedPPR(g, args.B, 0.85, 1e-9, decay)
    best = None
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        rank, stats, resid = p.solve(seeds)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    colsum = rank.sum(0)
    print(f"decay={decay}: {best / 1e3:.4f} s  sweeps={stats.sweeps} node_visits={stats.diffusions:.3e} "
          f"edges={stats.elementary_steps:.3e} edge_columns/s={stats.elementary_steps * args.B / (best / 1e3):.3e} "
          f"max_col_resid={max(resid):.2e} colsum_err={float((colsum - 1).abs().max()):.1e}", flush=True)
    p.close()
