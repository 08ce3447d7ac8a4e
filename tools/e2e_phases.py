"""Time the phases of the host-buffer path (H2D, solver setup, solve, D2H) on config 5 (tools/)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1202_6158_b200 as fr  # noqa: E402
from paper_1202_6158_b200 import _lib, gen  # noqa: E402

g, _ = gen.generate(gen.web_config(16.0), 100_000_000, 0)
n, L = g.n, g.edge_count
h_off = torch.empty(n + 1, dtype=torch.int64, pin_memory=True).copy_(g.out_offsets)
h_tgt = torch.empty(L, dtype=torch.int32, pin_memory=True).copy_(g.out_targets)
params = fr.DiffusionParams(target_error=1e-9)
sched = fr.make_scheduler("sweep", policy="geometric", sweep_decay=0.9)
for rep in range(2):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    d_off = h_off.to("cuda", non_blocking=True)
    d_tgt = h_tgt.to("cuda", non_blocking=True)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    g2 = fr.SparseGraph(n, d_off, d_tgt)
    state = fr.init(g2, params)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    solver = fr.Solver(g2, state, sched, params)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    st = solver.run()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    rank = torch.empty_like(state.history)
    _lib.check(_lib.lib.fr_normalize(n, _lib.ptr(state.history), _lib.ptr(rank), None, _lib.stream_ptr()))
    h_rank = rank.cpu()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    solver.close()
    names = ["h2d", "state init", "solver setup", "solve", "normalize+d2h"]
    print(" ".join(f"{nm}={1000 * (t[i + 1] - t[i]):.1f}ms" for i, nm in enumerate(names)))
    cfg = sched.solver_config(params)
    hs = _lib.SolveStats()
    hr = torch.empty(n, dtype=torch.float64, pin_memory=True)
    t0 = time.perf_counter()
    _lib.check(_lib.lib.fr_pagerank_host(n, L, h_off.data_ptr(), h_tgt.data_ptr(), ctypes.byref(cfg), hr.data_ptr(),
                                         ctypes.byref(hs)))
    print(f"fr_pagerank_host total {1000 * (time.perf_counter() - t0):.1f} ms")
