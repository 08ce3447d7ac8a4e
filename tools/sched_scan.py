"""Schedule scan: build the config-5 web graph once on the device, then time a
full CUDA-graph solve (residual target 1e-9) for each (damping, decay, beta).
Development tool for choosing the theta schedule; not a benchmark."""

import argparse
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1202_6158_b200 as fr  # noqa: E402
from paper_1202_6158_b200 import _lib, gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000_000)
ap.add_argument("--mean", type=float, default=16.0)
ap.add_argument("--damping", default="0.85")
ap.add_argument("--decay", default="0.75")
ap.add_argument("--beta", default="0.65")
ap.add_argument("--policy", default="geometric")
ap.add_argument("--edge-frac", default="0.2")
ap.add_argument("--fluid", default="fp64")
ap.add_argument("--path", default="fused")
args = ap.parse_args()

g, _ = gen.generate(gen.web_config(args.mean), args.n, 0, exact=True)
fl = [float(x) for x in args.damping.split(",")]
dl = [float(x) for x in args.decay.split(",")]
bl = [float(x) for x in args.beta.split(",")]
el = [float(x) for x in args.edge_frac.split(",")]
fp32 = args.fluid == "fp32"
for damping, decay, beta, ef in itertools.product(fl, dl, bl, el):
    params = fr.DiffusionParams(damping=damping, target_error=1e-9)
    state = fr.init(g, params, fluid_dtype=torch.float32 if fp32 else torch.float64)
    sched = fr.make_scheduler("sweep", policy=args.policy, sweep_decay=decay, degree_exponent=beta, edge_frac=ef,
                              kernel_path=args.path)
    solver = fr.Solver(g, state, sched, params)
    best = None
    for rep in range(2):
        _lib.check(_lib.lib.fr_init_state(g.n, damping, None, _lib.ptr(state.fluid), int(fp32),
                                          _lib.ptr(state.history), _lib.stream_ptr()))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        st = solver.run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    print(f"d={damping} decay={decay} beta={beta} edge_frac={ef}: {best / 1e3:.4f} s  sweeps={st.sweeps} "
          f"edges={st.elementary_steps:.3e} residual={st.residual:.2e}", flush=True)
    del solver, state
