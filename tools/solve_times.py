"""Per-solve device times of the graph path, repeated in one process (variance study; tools/)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1202_6158_b200 as fr  # noqa: E402
from paper_1202_6158_b200 import _lib, gen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
g, _ = gen.generate(gen.web_config(16.0), n, 0)
params = fr.DiffusionParams(target_error=1e-9)
state = fr.init(g, params)
solver = fr.Solver(g, state, fr.make_scheduler("sweep", policy="geometric", sweep_decay=0.9), params)
times = []
for k in range(10):
    _lib.check(_lib.lib.fr_init_state(n, 0.85, None, _lib.ptr(state.fluid), 0, _lib.ptr(state.history),
                                      _lib.stream_ptr()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = solver.run()
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
    print(f"solve {k}: {times[-1]:.1f} ms sweeps={st.sweeps} edges={st.elementary_steps}", flush=True)
    rows = solver.trace_rows()
    dt = [(rows[j].t_ns - rows[j - 1].t_ns) / 1e6 for j in range(1, len(rows))]
    q = len(dt) // 4
    print("   per-sweep ms by quarter:", [round(sum(dt[i * q:(i + 1) * q]), 1) for i in range(4)],
          "max sweep %.2f ms at %d" % (max(dt), dt.index(max(dt)) + 1))
