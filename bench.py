"""Benchmark: D-iteration PageRank on one B200 per rank (BASELINE.json metric).

metric  edges diffused/s and time to L1 residual 1e-9 (100M nodes), % of HBM peak
step    one full solve: init F=(1-d)/N, H=0; device sweeps until the fluid mass
        R satisfies R/(1-d) <= 1e-9; normalize the history into the rank.
value   elementary steps (edges diffused, PAPER sec. 4.2) of all ranks / max-over-ranks
        device time, with the graph resident in HBM.
e2e     the same metric through the C-ABI host-buffer entry fr_pagerank_host:
        H2D of the CSR from pinned memory, solve, D2H of the rank, per step.
Multi-GPU: the solve does not shard (one graph per GPU, BASELINE north star),
so --gpus N runs N independent replicas ("replicas only", scaling = weak).

--impl reference times the reference algorithm's CPU implementation (the
oracle port of engine.run + ThresholdSweepScheduler, bit-exact with the
reference) on the same config-5 graph (built by the oracle's generator, bit-
exact with the device's), each step a bounded sample: the sequential run from
the initial state for a fixed diffusion budget.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "edges diffused/s and time to L1 residual 1e-9 (100M nodes), % of HBM peak"
UNIT = "edges/s"

WORKLOADS = {
    # BASELINE.json configs[4]: N=100M, ~1.6B edges (mean out-degree 16), int64 offsets, uint32 columns
    5: dict(n=100_000_000, mean=16.0, damping=0.85, target=1e-9,
            name="config5: web graph N=100M, mean out-degree 16 (power law 2.1, 15% dangling, "
                 "70% local +-1000 / 30% Zipf(1.0)), d=0.85, fp64, L1 residual 1e-9"),
    3: dict(n=20_000_000, mean=10.0, damping=0.85, target=1e-9,
            name="config3: web graph N=20M, mean out-degree 10, d=0.85, fp64, L1 residual 1e-9"),
    2: dict(n=1_000_000, mean=8.0, damping=0.85, target=1e-9,
            name="config2: web graph N=1M, mean out-degree 8, d=0.85, fp64, L1 residual 1e-9"),
}
CPU_SAMPLE_DIFFUSIONS = 250_000_000  # repo arm's cpu_baseline: ~15 s of sequential ALGO-REF on config 5
REF_STEP_DIFFUSIONS = 40_000_000     # --impl reference: ~2.5 s per step


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return world, rank, local


def reduce_max(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------------ CPU baseline
def cpu_sample(off, tgt, damping, target, budget, graph_name):
    """Reference algorithm (oracle port, bit-exact with fluidrank.engine.run + ThresholdSweepScheduler)
    on the benchmarked graph itself, from the initial state for `budget` diffusions (one host core:
    the algorithm is sequential).  Only the C solve is timed."""
    from oracle import oracle as O
    O.build()
    r = O.run_seq(off, tgt, damping, target, "sweep", max_diffusions=budget)
    return {"value": r.elementary_steps / r.seconds, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": (f"{graph_name}: sequential ALGO-REF + ThresholdSweepScheduler (oracle/fr_oracle.c, "
                       f"bit-exact with the reference) from the initial state, first {budget:,} diffusions: "
                       f"{r.elementary_steps:,} edges in {r.seconds:.2f} s"),
            "seconds": r.seconds, "elementary_steps": r.elementary_steps, "diffusions": r.diffusions}


def cpu_full_solve(off, tgt, damping, target, graph_name):
    """One complete sequential reference solve to the target (time to residual on the host)."""
    from oracle import oracle as O
    O.build()
    r = O.run_seq(off, tgt, damping, target, "sweep")
    return {"graph": graph_name, "time_to_residual_s": r.seconds, "edges": r.elementary_steps,
            "edges_per_s": r.elementary_steps / r.seconds, "diffusions": r.diffusions,
            "final_residual": r.residual, "cores": 1, "kind": "port",
            "algorithm": "sequential ALGO-REF + ThresholdSweepScheduler(decay 0.5), oracle/fr_oracle.c"}


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    from oracle import oracle as O
    O.build()
    w = WORKLOADS[args.config]
    n = args.n or w["n"]
    t0 = time.perf_counter()
    off, tgt, rep = O.gen_graph_exact(O.web_config(w["mean"]), n, args.seed)
    t_graph = time.perf_counter() - t0
    name = f"{w['name']} (exact-size graph: {tgt.size:,} edges; seed {args.seed})"
    for _ in range(args.warmup):
        cpu_sample(off, tgt, w["damping"], w["target"], REF_STEP_DIFFUSIONS, name)
    secs, steps = 0.0, 0
    for _ in range(args.steps):
        smp = cpu_sample(off, tgt, w["damping"], w["target"], REF_STEP_DIFFUSIONS, name)
        secs += smp["seconds"]
        steps += smp["elementary_steps"]
    value = steps / secs
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * secs / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": w["name"], "n": n, "edges": int(tgt.size), "seed": args.seed,
                       "graph": "oracle.gen_graph_exact (bit-exact with the device generator)",
                       "graph_build_s": t_graph,
                       "step": (f"sequential ALGO-REF + ThresholdSweepScheduler from the initial state for "
                                f"{REF_STEP_DIFFUSIONS:,} diffusions (a bounded sample of one solve)"),
                       "parallelism": "1 host core (sequential algorithm)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port", "sample": smp["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm
def algorithmic_bytes(n, sweeps, diffusions, edges, hub_edges, fp32, narrow=False):
    """Algorithmic (compulsory) bytes of the fused sweep over one solve.

    k_sweep, per sweep:       every node's fluid (8 B, 4 for fp32) + row offset (8 B; 4 B
                              for the solver's narrow copy when m < 2^32 and n < 2^31)
             per diffusion:   fluid write-back of the take (8/4 B) + history read+write (16 B)
             per pushed edge: column index (4 B) + the target's fluid value (8/4 B),
                              counted once per edge as in SpMV accounting
    k_push_block (hubs), per hub edge: 4 + 8/4 B.
    """
    fb = 4 if fp32 else 8
    ob = 4 if narrow else 8
    own_edges = edges - hub_edges
    sweep_b = sweeps * n * (fb + ob) + diffusions * (fb + 16) + own_edges * (4 + fb)
    hub_b = hub_edges * (4 + fb)
    return sweep_b, hub_b


BYTES_PER_EDGE_DOC = ("12 B per pushed edge (4 B column index + 8 B target fluid), plus 12 B per node per sweep "
                      "(8 B fluid + 4 B narrow row offset scan; 16 B when m >= 2^32) and 24 B per diffusion "
                      "(take write-back + history r/w)")


def run_ours(args, world, rank, local):
    import ctypes

    import numpy as np
    import torch

    import paper_1202_6158_b200 as fr
    from paper_1202_6158_b200 import _lib, gen

    w = dict(WORKLOADS[args.config])
    if args.n:
        w["n"] = args.n
    n = w["n"]
    dev = torch.device("cuda", local)
    t0 = time.perf_counter()
    # the exact-size graph: base draw, cleaned, fill rounds redrawing the dropped slots
    g, grep_ = gen.generate(gen.web_config(w["mean"]), n, args.seed, exact=True)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    off, tgt = g.out_offsets, g.out_targets
    L = g.edge_count
    torch.cuda.empty_cache()
    fp32 = args.fluid == "fp32"
    params = fr.DiffusionParams(damping=w["damping"], target_error=w["target"])
    sched = fr.make_scheduler("sweep", policy=args.policy, sweep_decay=args.decay,
                              thread_max_degree=args.thread_max, block_min_degree=args.block_min,
                              kernel_path=args.path, hot_slots=args.hot_slots,
                              warm_slots=args.warm_slots, degree_exponent=args.beta, edge_frac=args.edge_frac)
    state = fr.init(g, params, fluid_dtype=torch.float32 if fp32 else torch.float64)
    solver = fr.Solver(g, state, sched, params, trace_cap=1 << 16)
    rank_out = torch.empty(n, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        _lib.check(_lib.lib.fr_init_state(n, params.damping, None, _lib.ptr(state.fluid), int(fp32),
                                          _lib.ptr(state.history), _lib.stream_ptr()))
        st = solver.run()
        _lib.check(_lib.lib.fr_normalize(n, _lib.ptr(state.history), _lib.ptr(rank_out), None,
                                         _lib.stream_ptr()))
        return st

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    edges = 0
    sweeps = []
    stats = []
    for _ in range(args.steps):
        st = step()
        edges += st.elementary_steps
        sweeps.append(st.sweeps)
        stats.append(st)
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    barrier(world)
    ms = ev0.elapsed_time(ev1)
    ms_max = reduce_max(ms, world)
    edges_all = reduce_sum(float(edges), world)
    value = edges_all / (ms_max / 1000.0)
    ms_per_step = ms_max / args.steps
    last = stats[-1]
    rows = solver.trace_rows()
    # our kernels in the timed region: init (1) + graph prologue (2) + per sweep (owned: sweep, fold,
    # finalize, guarded mass pass, guarded check = 5, its hub rows pushed inside the next sweep;
    # fused: + hub = 6; binned: 5) + owned: hub drain and fold after the loop (2) + exact residual (2)
    # + normalize (3)
    per_sweep = 6 if args.path == "fused" else 5
    after_loop = 2 if args.path == "owned" and os.environ.get("FR_HUB_DEFER", "1") != "0" else 0
    if args.path == "owned" and not after_loop:
        per_sweep = 6
    launches = sum(1 + 2 + per_sweep * s + after_loop + 2 + 3 for s in sweeps)

    # correctness guard for the measured run: stopping rule met, rank normalized
    assert last.residual <= params.target_error * (1 - params.damping) * 1.0000001, last.residual
    rsum = float(rank_out.sum())
    assert abs(rsum - 1.0) < 1e-9, rsum

    # ---- per-kernel roofline: same solve, launched sweep by sweep with events
    _lib.check(_lib.lib.fr_init_state(n, params.damping, None, _lib.ptr(state.fluid), int(fp32),
                                      _lib.ptr(state.history), _lib.stream_ptr()))
    pst = solver.run(profiled=True)
    kms, kl = solver.kernel_ms, solver.kernel_launches
    peak, peak_kind = load_peaks()
    if args.path != "binned":
        narrow = L < (1 << 32) and n < (1 << 31)  # the solver's narrow row-offset copy (fr_diffuse.cu setup)
        sweep_b, hub_b = algorithmic_bytes(n, pst.sweeps, pst.diffusions, pst.elementary_steps, pst.hub_edges, fp32,
                                           narrow)
        sweep_name = "k_sweep_own" if args.path == "owned" else "k_sweep"
        classes = {sweep_name: (kms[0], kl[0], sweep_b), "k_push_block": (kms[3], kl[3], hub_b)}
    else:
        fb = 4 if fp32 else 8
        classes = {"k_select": (kms[0], kl[0], pst.sweeps * n * fb + pst.diffusions * (fb + 16 + 16 + 4 + fb)),
                   "k_push_thread+k_push_warp+k_push_block": (kms[1] + kms[2] + kms[3], kl[1],
                                                             pst.elementary_steps * (4 + fb))}
    dom = max(classes, key=lambda k: classes[k][0])
    dms, dl, db = classes[dom]
    avg_ms = dms / dl if dl else 0.0
    achieved = (db / dl) / (avg_ms / 1000.0) / 1e9 if dl and avg_ms else 0.0
    traffic = None
    ncu_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(ncu_path):
        try:
            traffic = json.load(open(ncu_path)).get(dom)
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": dom,
                "peak_source": ("measured copy bandwidth, MEASURED_PEAKS.json hbm_gbs" if peak_kind == "measured"
                                else "fallback 6.65 TB/s (B200_PROFILING.md)"),
                "bytes_per_launch": db / dl if dl else 0, "avg_launch_ms": avg_ms,
                "share_of_step": round(dms / sum(kms), 4) if sum(kms) else None,
                "kernel_ms": {"select_or_sweep": kms[0], "push_thread": kms[1], "push_warp": kms[2],
                              "push_block": kms[3], "fold_finalize_check": kms[4]},
                "launches": {"select_or_sweep": kl[0], "push_block": kl[3]},
                "algorithmic_bytes_definition": BYTES_PER_EDGE_DOC,
                "algorithmic_bytes_per_diffused_edge": round(sum(c[2] for c in classes.values())
                                                              / max(1, pst.elementary_steps), 2),
                "timing": "sweep-by-sweep host launches with CUDA events on the launching stream"}

    # ---- the fp32-fluid / fp64-history variant on the same graph (stated tolerance 1e-6 L1)
    fp32_leg = None
    if not fp32 and not args.no_fp32:
        st32 = fr.init(g, params, fluid_dtype=torch.float32)
        sol32 = fr.Solver(g, st32, sched, params, trace_cap=16)
        sol32.run()  # warm-up
        _lib.check(_lib.lib.fr_init_state(n, params.damping, None, _lib.ptr(st32.fluid), 1, _lib.ptr(st32.history),
                                          _lib.stream_ptr()))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s32 = sol32.run()
        e1.record(stream)
        torch.cuda.synchronize()
        t32 = reduce_max(e0.elapsed_time(e1), world) / 1000.0
        r32 = st32.history / st32.history.sum()
        fp32_leg = {"time_to_residual_s": t32, "edges": s32.elementary_steps, "sweeps": s32.sweeps,
                    "edges_per_s": reduce_sum(float(s32.elementary_steps), world) / t32,
                    "rank_l1_vs_fp64": float((r32 - rank_out).abs().sum()), "stated_tolerance": 1e-6}
        sol32.close()
        del st32, r32
        torch.cuda.empty_cache()

    # ---- the same solve with the plain |f| score (beta = 0): more edges, more time
    plain = None
    if args.beta != 0.0 and not args.no_plain:
        sched0 = fr.make_scheduler("sweep", policy=args.policy, sweep_decay=args.decay, kernel_path=args.path,
                                   hot_slots=args.hot_slots, warm_slots=args.warm_slots, degree_exponent=0.0,
                                   edge_frac=args.edge_frac)
        st0 = fr.init(g, params, fluid_dtype=torch.float32 if fp32 else torch.float64)
        sol0 = fr.Solver(g, st0, sched0, params, trace_cap=16)
        sol0.run()
        _lib.check(_lib.lib.fr_init_state(n, params.damping, None, _lib.ptr(st0.fluid), int(fp32),
                                          _lib.ptr(st0.history), _lib.stream_ptr()))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s0 = sol0.run()
        e1.record(stream)
        torch.cuda.synchronize()
        t0s = reduce_max(e0.elapsed_time(e1), world) / 1000.0
        plain = {"degree_exponent": 0.0, "time_to_residual_s": t0s, "edges": s0.elementary_steps,
                 "edges_per_s": reduce_sum(float(s0.elementary_steps), world) / t0s, "sweeps": s0.sweeps}
        sol0.close()
        del st0

    # ---- the in-repo comparison solver on the same graph: power iteration (MAT-ITER,
    # baseline.py:20-56) to its own stopping rule |x_n - x_{n-1}|_1 d/(1-d) <= 1e-9
    power = None
    if not args.no_power:
        t0 = time.perf_counter()
        g.reverse_csr()
        torch.cuda.synchronize()
        t_tr = time.perf_counter() - t0
        pi = fr.PowerIteration(g, params)
        pi.run(w["target"])  # warm-up (graph instantiation)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        x_pi, iters, diff = pi.run(w["target"])
        e1.record(stream)
        torch.cuda.synchronize()
        t_pi = reduce_max(e0.elapsed_time(e1), world) / 1000.0
        # SpMV roofline: the same iterations host-launched with events around the SpMV
        _, it_p, rows_ms, segs_ms, rest_ms = pi.run_profiled(w["target"])
        spmv_ms = rows_ms + segs_ms + rest_ms
        # per iteration: 4 B source index + 8 B gathered z per edge; per row 8 B in-offset,
        # x read + write, 1/outdeg, z write (the update is fused into the row kernels;
        # the uniform teleport is not stored)
        spmv_bytes = 12 * L + 40 * n
        spmv_ach = spmv_bytes / (spmv_ms / it_p / 1000.0) / 1e9
        power = {"time_s": t_pi, "iterations": iters, "edges": iters * L, "edges_per_s": iters * L / t_pi,
                 "transpose_build_s": t_tr, "rank_l1_vs_diffusion": float((x_pi - rank_out).abs().sum()),
                 "stopping_rule": "|x_n - x_{n-1}|_1 * d/(1-d) <= 1e-9 (baseline.py:52)",
                 "roofline": {"bound": "hbm", "kernel": "k_pi_rows + k_pi_segs + k_pi_hub_update (pull SpMV "
                                                        "with the update fused)",
                              "achieved": round(spmv_ach, 1), "peak": load_peaks()[0], "unit": "GB/s",
                              "frac": round(spmv_ach / load_peaks()[0], 4),
                              "bytes_per_iteration": spmv_bytes, "avg_iteration_ms": spmv_ms / it_p,
                              "short_rows_ms": rows_ms / it_p, "hub_rows_by_source_block_ms": segs_ms / it_p,
                              "hub_update_check_ms": rest_ms / it_p,
                              "algorithmic_bytes_definition": "12 B per edge (4 B source index + 8 B gathered "
                                                              "x/deg) + 40 B per row (8 B in-offset, x read and "
                                                              "write, 1/outdeg, x/deg write)",
                              "timing": "host-launched iterations, CUDA events around the iteration's kernels"},
                 "vs_diffusion_time": t_pi / (ms_per_step / 1000.0)}
        pi.close()
        del x_pi
        g._reverse = None
        torch.cuda.empty_cache()

    # ---- the slow-convergence case of the same config (BASELINE config 5: d=0.99)
    d099 = None
    if not args.no_d099:
        p99 = fr.DiffusionParams(damping=0.99, target_error=w["target"])
        st99 = fr.init(g, p99, fluid_dtype=torch.float32 if fp32 else torch.float64)
        # the slow-convergence case has its own scanned schedule optimum
        sched99 = fr.make_scheduler("sweep", policy=args.policy, sweep_decay=args.decay99, kernel_path=args.path,
                                    hot_slots=args.hot_slots, warm_slots=args.warm_slots,
                                    degree_exponent=args.beta, edge_frac=args.edge_frac99)
        sol99 = fr.Solver(g, st99, sched99, p99, trace_cap=16)
        sol99.run()  # warm-up (graph instantiation, first touch)
        _lib.check(_lib.lib.fr_init_state(n, 0.99, None, _lib.ptr(st99.fluid), int(fp32), _lib.ptr(st99.history),
                                          _lib.stream_ptr()))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s99 = sol99.run()
        e1.record(stream)
        torch.cuda.synchronize()
        t99 = reduce_max(e0.elapsed_time(e1), world) / 1000.0
        d099 = {"damping": 0.99, "decay": args.decay99, "edge_frac": args.edge_frac99,
                "time_to_residual_s": t99, "edges": s99.elementary_steps,
                "edges_per_s": reduce_sum(float(s99.elementary_steps), world) / t99, "sweeps": s99.sweeps,
                "final_residual": s99.residual}
        sol99.close()
        del st99

    # ---- the other single-solve BASELINE configs (1: N=10k uniform, 2: N=1M web,
    # 3: N=20M web in fp64 and fp32 fluid), same schedule, graph resident
    others = None
    c3_host = None  # host CSR of config 3 for the CPU reference solve
    if not args.no_configs:
        others = {}
        for k in (1, 2, 3):
            gk, rk = gen.baseline_graph(k, seed=args.seed)
            if k == 3 and not args.no_cpu_c3 and rank == 0:
                c3_host = (gk.out_offsets.cpu().numpy(), gk.out_targets.cpu().numpy().view(np.uint32))
            pk = fr.DiffusionParams(damping=0.85, target_error=gen.CONFIGS[k]["target_error"])
            leg = {"n": gk.n, "edges": gk.edge_count, "target_error": pk.target_error}
            ranks = {}
            for fl in (("fp64", "fp32") if k == 3 else ("fp64",)):
                f32 = fl == "fp32"
                sk = fr.init(gk, pk, fluid_dtype=torch.float32 if f32 else torch.float64)
                solk = fr.Solver(gk, sk, sched, pk, trace_cap=16)
                best = None
                for _ in range(3):  # first run: graph instantiation and first touch
                    _lib.check(_lib.lib.fr_init_state(gk.n, 0.85, None, _lib.ptr(sk.fluid), int(f32),
                                                      _lib.ptr(sk.history), _lib.stream_ptr()))
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    stk = solk.run()
                    e1.record(stream)
                    torch.cuda.synchronize()
                    tk = reduce_max(e0.elapsed_time(e1), world) / 1000.0
                    best = tk if best is None else min(best, tk)
                ranks[fl] = sk.history / sk.history.sum()
                leg[fl] = {"time_to_residual_s": best, "sweeps": stk.sweeps, "edges": stk.elementary_steps,
                           "edges_per_s": stk.elementary_steps / best, "final_residual": stk.residual}
                solk.close()
                del sk
            if "fp32" in ranks:
                leg["fp32"]["rank_l1_vs_fp64"] = float((ranks["fp32"] - ranks["fp64"]).abs().sum())
                leg["fp32"]["stated_tolerance"] = 1e-6
            others["config%d" % k] = leg
            del gk, ranks
            torch.cuda.empty_cache()

    # ---- batched personalized PageRank (BASELINE configs[3]): 1M-node web graph,
    # 64 personalization vectors x 10 seeds, every column to L1 residual 1e-9
    ppr = None
    if not args.no_ppr:
        g4, _ = gen.baseline_graph(4, seed=args.seed)
        seeds = fr.config4_seeds(g4.n, 64, 10, seed=args.seed)
        pp = fr.BatchedPPR(g4, 64, 0.85, w["target"])
        pp.solve(seeds)  # warm-up (graph instantiation)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rank4, st4, res4 = pp.solve(seeds)
        e1.record(stream)
        torch.cuda.synchronize()
        t4 = reduce_max(e0.elapsed_time(e1), world) / 1000.0
        colsum = float((rank4.sum(0) - 1.0).abs().max())
        peak = load_peaks()[0]
        # algorithmic bytes: every sweep scans the n x B fluid rows (8 B x B each); a row visit
        # takes the row (8 B x B) and adds it to the history (16 B x B); an edge visit reads its
        # 4 B column index and scatters one 8 B red.add per non-zero column value (pushes)
        Bc = 64
        ppr_bytes = (st4.sweeps * g4.n * 8 * Bc + st4.diffusions * 24 * Bc + st4.elementary_steps * 4
                     + st4.hub_edges * 8)
        ppr_ach = ppr_bytes / t4 / 1e9
        ppr_roof = {"bound": "hbm", "achieved": round(ppr_ach, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(ppr_ach / peak, 4), "column_pushes": st4.hub_edges,
                    "pushes_per_s": st4.hub_edges / t4,
                    "l2_atomic_envelope_per_s": {"l2_resident": 2.0e11, "local_window_streamed": 8.0e10,
                                                 "uniform_800MB": 2.3e10, "source": "tools/red_probe.cu (DESIGN.md)"},
                    "algorithmic_bytes_definition": "8 B x 64 per row per sweep (scan) + 24 B x 64 per row visit "
                                                    "(take, history r/w) + 4 B per edge visit + 8 B per pushed "
                                                    "column value",
                    "timing": "whole solve, CUDA events (k_ppr_sweep dominates)"}
        try:
            pt = json.load(open(os.path.join(ROOT, "profiles", "r02_ppr_traffic.json")))
            ppr_roof["traffic"] = pt["dram_bytes_per_solve"]
            ppr_roof["traffic_note"] = "ncu DRAM bytes of one whole solve (graph profiling), profiles/r02_ppr_traffic.json"
        except Exception:
            ppr_roof["traffic"] = None
        ppr = {"roofline": ppr_roof,"workload": "BASELINE configs[3]: N=1M web graph (mean out-degree 8, %d edges), 64 vectors x 10 "
                           "seeds, d=0.85, each column to L1 residual 1e-9, n x 64 fp64 row-major state" % g4.edge_count,
               "time_s": t4, "sweeps": st4.sweeps, "row_visits": st4.diffusions, "edge_visits": st4.elementary_steps,
               "column_pushes": st4.hub_edges,
               "max_column_residual": max(res4), "max_column_sum_error": colsum, "decay": 0.6,
               "timing": "one fr_ppr_init + fr_ppr_run + normalize, CUDA events"}
        pp.close()
        del rank4, g4
        torch.cuda.empty_cache()

    # ---- end to end through the C ABI from pinned host buffers
    h_off = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
    h_tgt = torch.empty(L, dtype=torch.int32, pin_memory=True)
    h_off.copy_(off)
    h_tgt.copy_(tgt)
    h_rank = torch.empty(n, dtype=torch.float64, pin_memory=True)
    cfgc = sched.solver_config(params, fp32)
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    hs = _lib.SolveStats()
    # one untimed call: the first one grows the device memory pool
    _lib.check(_lib.lib.fr_pagerank_host(n, L, h_off.data_ptr(), h_tgt.data_ptr(), None, ctypes.byref(cfgc),
                                         h_rank.data_ptr(), ctypes.byref(hs)))
    e2e_edges = 0
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        _lib.check(_lib.lib.fr_pagerank_host(n, L, h_off.data_ptr(), h_tgt.data_ptr(), None, ctypes.byref(cfgc),
                                             h_rank.data_ptr(), ctypes.byref(hs)))
        e2e_edges += hs.elementary_steps
    e2e_s = time.perf_counter() - t0
    e2e_s = reduce_max(e2e_s, world)
    e2e_edges = reduce_sum(float(e2e_edges), world)
    rank_err = float((h_rank.to(dev) - rank_out).abs().sum())
    # both runs stop at residual/(1-d) <= 1e-9, so their normalized ranks agree to ~2e-9 / |h|_1
    # (fp32 fluid: within its stated 1e-6 tolerance)
    tol = 1e-6 if fp32 else 1e-8
    assert rank_err <= tol, f"host-buffer path disagrees with the resident run: L1 {rank_err:.3e}"

    line = None
    if rank == 0:
        cpu = None
        if not args.no_cpu:
            # the reference algorithm on the benchmarked graph itself (host copy of the device CSR)
            cpu = cpu_sample(h_off.numpy(), h_tgt.numpy().view(np.uint32), w["damping"], w["target"],
                             CPU_SAMPLE_DIFFUSIONS, f"{w['name']} (this run's graph, {L:,} edges)")
        cpu_c3 = None
        if c3_host is not None:
            cpu_c3 = cpu_full_solve(c3_host[0], c3_host[1], 0.85, gen.CONFIGS[3]["target_error"],
                                    "config3: N=20M web graph, mean out-degree 10 (the other_configs.config3 graph)")
            if others:
                cpu_c3["gpu_speedup_time_to_residual"] = (cpu_c3["time_to_residual_s"]
                                                           / others["config3"]["fp64"]["time_to_residual_s"])
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32-fluid/f64-history" if fp32 else "f64", "data": "synthetic",
            "config": {"workload": w["name"], "n": n, "edges": L, "edges_configured": grep_.target_links,
                       "edges_unfilled": grep_.unfilled, "fill_rounds": grep_.rounds,
                       "edge_slots_drawn": grep_.slots, "duplicates_dropped": grep_.duplicates,
                       "self_loops_dropped": grep_.self_loops, "damping": w["damping"],
                       "target_error": w["target"], "policy": args.policy, "decay": args.decay,
                       "edge_frac": args.edge_frac if args.policy == "adaptive" else None,
                       "kernel_path": args.path, "hot_slots": args.hot_slots, "warm_slots": args.warm_slots,
                       "degree_exponent": args.beta,
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                       "l2": "inputs larger than L2 (CSR %.1f GB >> 126 MB)" % ((8 * (n + 1) + 4 * L) / 1e9)},
            "time_to_residual_s": ms_per_step / 1000.0,
            "sweeps_per_solve": last.sweeps, "diffusions_per_solve": last.diffusions,
            "edges_per_solve": last.elementary_steps, "final_residual": last.residual,
            "graph_build_s": t_gen,
            "solver_setup": ("fr_solver_create (slot classes from a sampled in-degree, encoded column copy, "
                             "narrow offsets) runs once before the timed solves: the graph stays resident and "
                             "is solved many times; e2e includes it on every call"),
            "e2e": {"value": e2e_edges / e2e_s, "unit": UNIT,
                    "h2d_bytes_per_step": 8 * (n + 1) + 4 * L, "d2h_bytes_per_step": 8 * n,
                    "seconds_per_step": e2e_s / e2e_steps, "steps": e2e_steps,
                    "rank_l1_vs_resident_run": rank_err},
            "gpu_launches": launches,
            "d099": d099,
            "plain_score_schedule": plain,
            "fp32_fluid": fp32_leg,
            "power_iteration": power,
            "ppr": ppr, "other_configs": others,
            "roofline": roofline,
            "cpu_baseline": None if cpu is None else {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "cpu_config3_full_solve": cpu_c3,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    barrier(world)
    solver.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, default=5, choices=sorted(WORKLOADS))
    ap.add_argument("--n", type=int, default=0, help="override node count (scaled workload)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--policy", default="adaptive", choices=("exhaust", "geometric", "adaptive"))
    ap.add_argument("--decay", type=float, default=0.6, help="theta decay per sweep (adaptive: nominal)")
    ap.add_argument("--edge-frac", type=float, default=0.2,
                    help="adaptive theta: target edges pushed per sweep as a fraction of m")
    ap.add_argument("--decay99", type=float, default=0.7, help="the d=0.99 leg's nominal decay")
    ap.add_argument("--edge-frac99", type=float, default=0.15, help="the d=0.99 leg's edge_frac")
    ap.add_argument("--path", default="owned", choices=("fused", "binned", "owned"))
    ap.add_argument("--hot-slots", type=int, default=0, help="0 default (2048), -1 off")
    ap.add_argument("--warm-slots", type=int, default=0, help="0 default (2^21), -1 off")
    ap.add_argument("--beta", type=float, default=0.85, help="degree exponent of the sweep score")
    ap.add_argument("--fluid", default="fp64", choices=("fp64", "fp32"))
    ap.add_argument("--thread-max", type=int, default=0)
    ap.add_argument("--block-min", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cpu-c3", action="store_true", help="skip the full sequential CPU solve of config 3")
    ap.add_argument("--no-d099", action="store_true", help="skip the d=0.99 solve")
    ap.add_argument("--no-ppr", action="store_true", help="skip the batched PPR (configs[3]) solve")
    ap.add_argument("--no-plain", action="store_true", help="skip the beta=0 comparison solve")
    ap.add_argument("--no-fp32", action="store_true", help="skip the fp32-fluid comparison solve")
    ap.add_argument("--no-power", action="store_true", help="skip the power-iteration comparison")
    ap.add_argument("--no-configs", action="store_true", help="skip BASELINE configs 1-3")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        rc = run_reference(args, world, rank)
    else:
        rc = run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
