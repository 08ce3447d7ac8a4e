"""Batched-PPR profiling driver (BASELINE configs[3]): the exact config-4 graph, 64
personalization vectors x 10 seeds, one warm-up and one profiled solve.  Under ncu use
--graph-profiling graph (the solve is one CUDA graph with a while node).  Not a benchmark."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1202_6158_b200 as fr  # noqa: E402
from paper_1202_6158_b200 import gen  # noqa: E402

import argparse  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--local-frac", type=float, default=None, help="generator local fraction (diagnostic graphs)")
ap.add_argument("--mode", default="push", help="push | pull | hybrid")
ap.add_argument("--decays", default="0.6", help="comma-separated theta decays, one timed solve each")
args = ap.parse_args()
if args.local_frac is None:
    g, _ = gen.baseline_graph(4)
else:
    g, _ = gen.generate(gen.web_config(8.0, local_frac=args.local_frac), 1_000_000, 0, exact=True)
seeds = fr.config4_seeds(g.n, 64, 10, seed=0)
for dec in [float(x) for x in args.decays.split(",")]:
    p = fr.BatchedPPR(g, 64, 0.85, 1e-9, decay=dec, mode=args.mode)
    p.solve(seeds)
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rank, st, res = p.solve(seeds)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"n={g.n} L={g.edge_count} decay {dec} time {min(ts):.2f} ms (of {len(ts)}) sweeps={st.sweeps} "
          f"row_visits={st.diffusions} edge_visits={st.elementary_steps} pushes={st.hub_edges} "
          f"max_residual={max(res):.2e}")
