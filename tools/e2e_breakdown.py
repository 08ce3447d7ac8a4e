"""Where the host-buffer entry point (fr_pagerank_host) spends its time on
config 5: H2D of the CSR, solver setup (slot classes, encoded columns, narrow
offsets, graph instantiation), the solve, normalize + D2H.  Development tool."""

import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1202_6158_b200 as fr  # noqa: E402
from paper_1202_6158_b200 import _lib, gen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
g, _ = gen.generate(gen.web_config(16.0), n, 0)
L = g.edge_count
h_off = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
h_tgt = torch.empty(L, dtype=torch.int32, pin_memory=True)
h_off.copy_(g.out_offsets)
h_tgt.copy_(g.out_targets)
h_rank = torch.empty(n, dtype=torch.float64, pin_memory=True)
params = fr.DiffusionParams(target_error=1e-9)
sched = fr.make_scheduler("sweep", policy="adaptive", sweep_decay=0.6, degree_exponent=0.65, edge_frac=0.2)
cfg = sched.solver_config(params)


def timed(fn, reps=3):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best


d_off = torch.empty_like(g.out_offsets)
d_tgt = torch.empty_like(g.out_targets)
t_h2d = timed(lambda: (d_off.copy_(h_off, non_blocking=True), d_tgt.copy_(h_tgt, non_blocking=True)))
d_rank = torch.empty(n, dtype=torch.float64, device="cuda")
t_d2h = timed(lambda: h_rank.copy_(d_rank, non_blocking=True))
state = fr.init(g, params)


def setup_only():
    s = fr.Solver(g, state, sched, params)
    s.close()


t_setup = timed(setup_only)
solver = fr.Solver(g, state, sched, params)


def solve():
    _lib.check(_lib.lib.fr_init_state(n, 0.85, None, _lib.ptr(state.fluid), 0, _lib.ptr(state.history),
                                      _lib.stream_ptr()))
    solver.run()


t_solve = timed(solve)
solver.close()
stats = _lib.SolveStats()
t_e2e = timed(lambda: _lib.check(_lib.lib.fr_pagerank_host(n, L, h_off.data_ptr(), h_tgt.data_ptr(), None,
                                                           ctypes.byref(cfg), h_rank.data_ptr(),
                                                           ctypes.byref(stats))))
print(f"H2D {t_h2d * 1e3:.1f} ms ({(h_off.numel() * 8 + h_tgt.numel() * 4) / t_h2d / 1e9:.1f} GB/s)  "
      f"setup {t_setup * 1e3:.1f} ms  solve {t_solve * 1e3:.1f} ms  D2H {t_d2h * 1e3:.1f} ms  "
      f"sum {1e3 * (t_h2d + t_setup + t_solve + t_d2h):.1f} ms  |  fr_pagerank_host {t_e2e * 1e3:.1f} ms")
