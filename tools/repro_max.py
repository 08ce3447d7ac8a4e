"""Repro of fuzz case (seed 13, case 5): max rule, decay 0.9, d = 0.99, n = 300k web graph; the
residual after a budget of sweeps for each path / precision."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1202_6158_b200 as fr  # noqa: E402
from oracle import oracle  # noqa: E402

n, seed = 300_000, 494253
src, dst = oracle.gen_edges(oracle.web_config(4.0), n, seed)
off, tgt, _ = oracle.csr_build(n, src, dst, clean=True)
g = fr.SparseGraph(n, torch.as_tensor(off), torch.as_tensor(tgt.astype(np.int32)))
for path in ("fused", "owned"):
    for fp32 in (False, True):
        for budget in (1000, 10000, 100000, 400000):
            params = fr.DiffusionParams(damping=0.99, target_error=1e-8)
            sched = fr.make_scheduler("max", seed=seed & 0xFFFF, policy="adaptive", sweep_decay=0.9, kernel_path=path)
            state = fr.init(g, params, fluid_dtype=torch.float32 if fp32 else torch.float64)
            try:
                fr.run(g, params, sched, state=state, max_sweeps=budget)
            except Exception as e:  # noqa: BLE001
                print("exc", repr(e)[:100])
            f = state.fluid.double()
            print(f"{path} {'fp32' if fp32 else 'fp64'} budget={budget}: sweeps={state.sweeps} diffusions={state.diffusions} "
                  f"residual_est={state.residual:.3e} exact={float(f.abs().sum()):.3e} max|f|={float(f.abs().max()):.3e} "
                  f"nonzero={int((f != 0).sum())}", flush=True)
            if state.residual <= 1e-8 * 0.01:
                break
