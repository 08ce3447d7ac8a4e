"""Sweep-kernel A/B: build the config-5 web graph once on the device, then time
full CUDA-graph solves (residual target 1e-9) for each variant
"path[:ENV=VAL[:ENV=VAL...]]" (e.g. fused, owned:FR_OWN_CHUNK=8192), and the
rank L1 of each against the first variant.  Development tool; not a benchmark."""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1202_6158_b200 as fr  # noqa: E402
from paper_1202_6158_b200 import _lib, gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000_000)
ap.add_argument("--mean", type=float, default=16.0)
ap.add_argument("--damping", type=float, default=0.85)
ap.add_argument("--decay", type=float, default=0.6)
ap.add_argument("--beta", type=float, default=0.85)
ap.add_argument("--edge-frac", type=float, default=0.2)
ap.add_argument("--policy", default="adaptive")
ap.add_argument("--fluid", default="fp64")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--hot-slots", type=int, default=0)
ap.add_argument("--block-min", type=int, default=0)
ap.add_argument("--warm-slots", type=int, default=0)
ap.add_argument("variants", nargs="+")
args = ap.parse_args()

g, _ = gen.generate(gen.web_config(args.mean), args.n, 0, exact=True)
fp32 = args.fluid == "fp32"
params = fr.DiffusionParams(damping=args.damping, target_error=1e-9)
first = None
for v in args.variants:
    parts = v.split(":")
    path, env = parts[0], dict(p.split("=", 1) for p in parts[1:])
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    state = fr.init(g, params, fluid_dtype=torch.float32 if fp32 else torch.float64)
    sched = fr.make_scheduler("sweep", policy=args.policy, sweep_decay=args.decay, degree_exponent=args.beta,
                              edge_frac=args.edge_frac, kernel_path=path, hot_slots=args.hot_slots,
                              block_min_degree=args.block_min, warm_slots=args.warm_slots)
    solver = fr.Solver(g, state, sched, params)
    for k, o in old.items():
        if o is None:
            os.environ.pop(k)
        else:
            os.environ[k] = o
    times = []
    for rep in range(args.reps):
        _lib.check(_lib.lib.fr_init_state(g.n, args.damping, None, _lib.ptr(state.fluid), int(fp32),
                                          _lib.ptr(state.history), _lib.stream_ptr()))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        st = solver.run()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    h = state.history.to(torch.float64)
    rank = h / h.sum()
    if first is None:
        first = rank.clone()
    l1 = float((rank - first).abs().sum())
    print(f"{v}: best {min(times):.4f} s  (all {' '.join(f'{t:.4f}' for t in times)})  sweeps={st.sweeps} "
          f"edges={st.elementary_steps:.4e} diffusions={st.diffusions:.4e} residual={st.residual:.2e} "
          f"l1_vs_first={l1:.2e}", flush=True)
    del solver, state
