"""Randomized parity sweep: random graphs (uniform and web generators, 1..300k
nodes), random schedules (rule, theta policy, decay, beta, edge_frac), both
fluid precisions, every kernel path with and without the single-block small
graph solve, each rank checked against the oracle (the reference restated).
Every 4th case also runs the power iteration against the oracle's (same
iteration count, L1 <= 1e-12 plus 1e-9 * iterations of rounding), and every
8th case (n >= 2) a batched personalized solve in both formulations (push,
pull) against per-column oracle runs.  Development tool (the test suite holds
the fixed cases); prints one line per case and a summary, exits 1 on any
failure."""

import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1202_6158_b200 as fr  # noqa: E402
from oracle import oracle  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
fails = 0
for case in range(cases):
    n = rng.choice([1, 2, 31, 33, 100, 1000, 5000, 40_000, 140_000, 300_000])
    web = rng.random() < 0.6 and n >= 100
    cfg = oracle.web_config(rng.choice([4.0, 8.0, 16.0])) if web else oracle.uniform_config(rng.choice([0, 3, 10]))
    seed = rng.randrange(1 << 20)
    src, dst = oracle.gen_edges(cfg, n, seed)
    off, tgt, _ = oracle.csr_build(n, src, dst, clean=True)
    kind = rng.choice(["sweep", "sweep", "sweep", "max", "per", "rand", "op", "op2"])
    policy = rng.choice(["exhaust", "geometric", "adaptive"])
    path = rng.choice(["owned", "owned", "fused", "binned"])
    small = rng.choice(["1", "0"])
    fp32 = rng.random() < 0.25
    beta = rng.choice([0.0, 0.5, 0.65, 1.0]) if kind == "sweep" else 0.0
    damping = rng.choice([0.85, 0.85, 0.5, 0.99])
    if kind == "max" and damping == 0.99 and n > 40_000:
        # the max rule diffuses only the nodes within `decay` of the largest fluid (a handful per
        # sweep on a web graph); at d = 0.99 a 300k-node graph needs > 10^6 such sweeps, the
        # solver's cap (seed 13, case 5: NoConvergenceError on every path and precision alike,
        # tools/repro_max.py) -- a property of the rule, not a parity case
        damping = 0.85
    target = 1e-8 if fp32 else 1e-10
    os.environ["FR_SMALL"] = small
    g = fr.SparseGraph(n, torch.as_tensor(off), torch.as_tensor(tgt.astype(np.int32)))
    params = fr.DiffusionParams(damping=damping, target_error=target)
    kw = dict(policy=policy, sweep_decay=rng.choice([0.5, 0.6, 0.7, 0.9]), kernel_path=path)
    if kind == "sweep":
        kw.update(degree_exponent=beta, edge_frac=rng.choice([0.1, 0.2, 0.3]))
    sched = fr.make_scheduler(kind, seed=seed & 0xFFFF, **kw)
    desc = (f"n={n} {'web' if web else 'uniform'} L={tgt.size} {kind}/{policy} beta={beta} d={damping} "
            f"{path} small={small} {'fp32' if fp32 else 'fp64'}")
    try:
        rank, trace = fr.run(g, params, sched, fluid_dtype=torch.float32 if fp32 else torch.float64)
        ref = oracle.run_seq(off, tgt, damping, target * 1e-3, "sweep").rank
        err = float(np.abs(rank - ref).sum())
        # the solver's bound: L1 of the normalized rank <= ~2 * target / |h|_1 (fp64); fp32 fluid 1e-6
        bound = 1e-6 if fp32 else 2.5 * target / (1 - damping) + 1e-12
        ok = err <= bound and trace.rows[-1].residual <= target * (1 - damping) * (1 + 1e-9)
    except Exception as e:  # noqa: BLE001
        ok, err = False, repr(e)
    extra = ""
    if ok and case % 4 == 0 and damping < 1.0:
        try:
            x, _ = fr.power_iterate(g, fr.DiffusionParams(damping=damping, target_error=1e-10))
            xr, it_r, _ = oracle.power_iterate(off, tgt, damping, 1e-10)
            perr = float(np.abs(x - xr).sum())
            ok = perr <= 1e-9
            extra += f" power l1={perr:.2e} (oracle {it_r} it)"
        except Exception as e:  # noqa: BLE001
            ok, extra = False, extra + f" power {e!r}"
    if ok and case % 8 == 0 and n >= 2:
        B = rng.choice([1, 5, 64])
        k = min(10, n)
        seeds = fr.config4_seeds(n, B, k, seed=seed)
        try:
            worst = 0.0
            for mode in ("push", "pull"):
                r, _, res = fr.personalized_pagerank(g, seeds, damping=damping, target_error=1e-11, mode=mode)
                r = r.cpu().numpy()
                for c in range(min(B, 3)):
                    v = np.zeros(n)
                    np.add.at(v, seeds[c].astype(np.int64), 1.0 / k)
                    ref = oracle.run_seq(off, tgt, damping, 1e-13, "sweep", teleport=v).rank
                    worst = max(worst, float(np.abs(r[:, c] - ref).sum()))
            ok = worst <= 2.5e-10 / (1 - damping)  # seeds may be dangling: |h|_1 < 1 scales the bound
            extra += f" ppr(B={B}) push/pull l1<={worst:.2e}"
        except Exception as e:  # noqa: BLE001
            ok, extra = False, extra + f" ppr {e!r}"
    fails += not ok
    print(f"{'ok  ' if ok else 'FAIL'} {desc}: l1={err}{extra}", flush=True)
print(f"{cases - fails}/{cases} passed")
sys.exit(1 if fails else 0)
