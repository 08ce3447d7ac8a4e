"""Fixed per-sweep cost of k_sweep: a solve whose fluid sits on a handful of
nodes selects almost nothing per sweep, so each sweep is the bare scan of
F and the row offsets over all n nodes (plus the per-sweep small kernels).
Development tool."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1202_6158_b200 as fr  # noqa: E402
from paper_1202_6158_b200 import gen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
beta = float(sys.argv[2]) if len(sys.argv) > 2 else 0.65
g, _ = gen.generate(gen.web_config(16.0), n, 0)
params = fr.DiffusionParams(target_error=1e-300)
f0 = torch.zeros(n, dtype=torch.float64)
f0[:: n // 4] = 0.25
for sweeps in (10, 60):
    state = fr.init_from_fluid(g, params, f0)
    sched = fr.make_scheduler("sweep", policy="geometric", sweep_decay=0.999, degree_exponent=beta)
    solver = fr.Solver(g, state, sched, params, max_sweeps=sweeps)
    solver.run()
    state2 = fr.init_from_fluid(g, params, f0)
    solver2 = fr.Solver(g, state2, sched, params, max_sweeps=sweeps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    st = solver2.run(profiled=bool(os.environ.get("PROF")))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{sweeps} sweeps: {ms:.2f} ms ({ms / sweeps:.3f} ms/sweep incl. setup)  edges={st.elementary_steps} "
          f"diffusions={st.diffusions}", flush=True)
    solver.close()
    solver2.close()
