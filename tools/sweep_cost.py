"""Per-sweep cost model from the device trace: fit t_sweep = a + b * edges over
the sweeps of one CUDA-graph solve (bench defaults, config 5)."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1202_6158_b200 as fr  # noqa: E402
from paper_1202_6158_b200 import _lib, gen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
path = sys.argv[2] if len(sys.argv) > 2 else "fused"
every = int(sys.argv[3]) if len(sys.argv) > 3 else 0
g, _ = gen.generate(gen.web_config(16.0), n, 0)
params = fr.DiffusionParams(target_error=1e-9)
state = fr.init(g, params)
sched = fr.make_scheduler("sweep", policy="adaptive", sweep_decay=0.6, degree_exponent=0.65, edge_frac=0.2,
                           kernel_path=path)
solver = fr.Solver(g, state, sched, params, trace_cap=1 << 12)
for rep in range(2):
    _lib.check(_lib.lib.fr_init_state(g.n, 0.85, None, _lib.ptr(state.fluid), 0, _lib.ptr(state.history),
                                      _lib.stream_ptr()))
    st = solver.run()
    torch.cuda.synchronize()
rows = solver.trace_rows()
t = np.array([r.t_ns for r in rows], dtype=np.float64) * 1e-6
e = np.array([r.elementary_steps for r in rows], dtype=np.float64)
d = np.array([r.diffusions for r in rows], dtype=np.float64)
dt, de, dd = np.diff(t), np.diff(e), np.diff(d)
A = np.stack([np.ones_like(de), de / 1e6, dd / 1e6], 1)
coef, *_ = np.linalg.lstsq(A, dt, rcond=None)
pred = A @ coef
print(f"sweeps={len(dt)} total={dt.sum():.1f} ms  fit: {coef[0]:.3f} ms/sweep + {coef[1]:.5f} ms/M edges "
      f"+ {coef[2]:.5f} ms/M diffusions  (r2={1 - ((dt - pred) ** 2).sum() / ((dt - dt.mean()) ** 2).sum():.3f})")
print(f"fixed part {coef[0] * len(dt):.1f} ms, edge part {coef[1] * de.sum() / 1e6:.1f} ms, "
      f"diffusion part {coef[2] * dd.sum() / 1e6:.1f} ms")
for k in range(0, len(dt), every or max(1, len(dt) // 12)):
    print(f"  sweep {k:3d}: {dt[k]:.3f} ms  edges {de[k] / 1e6:8.1f} M  diffusions {dd[k] / 1e6:6.1f} M")
