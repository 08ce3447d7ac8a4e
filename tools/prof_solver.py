"""Profiling driver: build a web graph on the device and run one host-launched
(sweep-by-sweep) solve so ncu can select kernels by name.  Not a benchmark."""

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1202_6158_b200 as fr  # noqa: E402
from paper_1202_6158_b200 import gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000_000)
ap.add_argument("--mean", type=float, default=16.0)
ap.add_argument("--policy", default="adaptive")
ap.add_argument("--edge-frac", type=float, default=0.2)
ap.add_argument("--decay", type=float, default=0.6)
ap.add_argument("--fluid", default="fp64")
ap.add_argument("--path", default="owned")
ap.add_argument("--hot-slots", type=int, default=0)
ap.add_argument("--block-min", type=int, default=0)
ap.add_argument("--beta", type=float, default=0.85)
ap.add_argument("--warm-slots", type=int, default=0)
ap.add_argument("--graph", action="store_true", help="run the CUDA-graph path instead")
ap.add_argument("--local-frac", type=float, default=0.7)
ap.add_argument("--window", type=int, default=1000)
args = ap.parse_args()

g, rep = gen.generate(gen.web_config(args.mean, local_frac=args.local_frac, window=args.window), args.n, 0, exact=True)
params = fr.DiffusionParams(target_error=1e-9)
state = fr.init(g, params, fluid_dtype=torch.float32 if args.fluid == "fp32" else torch.float64)
solver = fr.Solver(g, state, fr.make_scheduler("sweep", policy=args.policy, sweep_decay=args.decay, kernel_path=args.path, hot_slots=args.hot_slots, warm_slots=args.warm_slots,
                                                     block_min_degree=args.block_min,
                                                     degree_exponent=args.beta, edge_frac=args.edge_frac), params)
t = time.perf_counter()
st = solver.run(profiled=not args.graph)
torch.cuda.synchronize()
print(f"n={args.n} L={g.edge_count} sweeps={st.sweeps} diffusions={st.diffusions} "
      f"edges={st.elementary_steps} residual={st.residual:.3e} wall={time.perf_counter() - t:.3f}s")
if not args.graph:
    print("kernel ms", [round(x, 2) for x in solver.kernel_ms], "launches", solver.kernel_launches)
