"""Power-iteration SpMV profiling driver: the exact config-5 graph, its transpose,
and host-launched iterations (so ncu can select k_pi_rows / k_pi_segs by name).
Prints per-iteration kernel times.  Development tool; not a benchmark."""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1202_6158_b200 as fr  # noqa: E402
from paper_1202_6158_b200 import gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000_000)
ap.add_argument("--mean", type=float, default=16.0)
ap.add_argument("--iters", type=int, default=0, help="iteration cap (0: to the 1e-9 rule)")
ap.add_argument("--reps", type=int, default=1)
args = ap.parse_args()

g, _ = gen.generate(gen.web_config(args.mean), args.n, 0, exact=True)
g.reverse_csr()
pi = fr.PowerIteration(g, fr.DiffusionParams(target_error=1e-9))
pi.run_profiled(1e-9, 2)  # warm-up
for _ in range(args.reps):
    x, it, rows, segs, rest = pi.run_profiled(1e-9, args.iters or 1_000_000)
    L = g.edge_count
    print(f"n={g.n} L={L} iterations={it} per iteration: short rows {rows / it:.3f} ms  hub rows {segs / it:.3f} ms  "
          f"rest {rest / it:.3f} ms  spmv GB/s (12 B/edge + 40 B/row) "
          f"{(12 * L + 40 * g.n) / ((rows + segs + rest) / it / 1e3) / 1e9:.0f}  "
          + "  ".join(f"{k} {v / it:.3f}" for k, v in pi.last_profile_ms.items()))
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
pi.run(1e-9)
e0.record()
x2, it2, _ = pi.run(1e-9)
e1.record()
torch.cuda.synchronize()
print(f"graph-launched solve: {e0.elapsed_time(e1):.1f} ms, {it2} iterations, |x - x_profiled|_1 = "
      f"{float((x2 - x).abs().sum()):.2e}")
