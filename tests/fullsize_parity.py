"""Full-size parity: the BASELINE configurations solved on the GPU, checked against the
CPU oracle on the same seeded graphs (TEST INFRASTRUCTURE; run on the GPU box).

    [FR_PARITY_SEED=S] python tests/fullsize_parity.py [--configs 2,3,4,5] [--out profiles/r02_parity_fullsize.json]

For each configuration the device builds the exact-size graph (gen.baseline_graph:
base draw, cleaned, fill rounds) and a worker process builds the same graph with the
oracle (oracle.gen_graph_exact, bit-exact with the reference loader's cleaning):
  * CSR: offsets and column indices compared by SHA-256 of the arrays (plus sizes and
    the generator report) -- bit-exact or fail;
  * ranks: the device solve with the EXACT bench schedule (owned path, default chunks
    and slots, adaptive theta (0.6, 0.2) at d = 0.85 and (0.7, 0.15) at d = 0.99,
    degree exponent 0.85, target 1e-9) against the oracle's sequential ALGO-REF +
    ThresholdSweepScheduler run (oracle.run_seq, bit-exact with fluidrank.engine.run)
    at a tighter target: L1 <= 1e-9 in fp64, <= 1e-6 for the fp32-fluid variant;
  * config 5 also through the host-buffer entry point fr_pagerank_host (8-piece copy,
    sampled in-degree slot classes), and at d = 0.99;
  * config 4: 8 of the 64 batched personalized columns against per-column oracle runs
    with teleport V_c (ref engine.py:56-62, 149-159).
The oracle solves run in parallel worker processes (one per solve, spawned before the
GPU work starts), each building its own copy of the graph from the seed.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

SEED = int(os.environ.get("FR_PARITY_SEED", "0"))  # 0 = bench.py's default seed (the env reaches the spawned workers)
TMP = os.environ.get("FR_PARITY_TMP", "/tmp/fr_parity")
# (n, mean out-degree) of the web-generator BASELINE configs
WEB = {2: (1_000_000, 8.0), 3: (20_000_000, 10.0), 4: (1_000_000, 8.0), 5: (100_000_000, 16.0)}
SCHED = {0.85: (0.6, 0.2), 0.99: (0.7, 0.15)}  # bench.py --decay/--edge-frac, --decay99/--edge-frac99
ORACLE_TRUTH = {0.85: 1e-12, 0.99: 1e-12}  # oracle targets of the "tight" solution
GPU_TIGHT = {0.85: 1e-10, 0.99: 1e-11}     # the device solve re-run below the config's 1e-9
PPR_COLUMNS = 8
BETA = 0.85  # bench.py --beta


def sha(a):
    import numpy as np
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8)).hexdigest()


# ------------------------------------------------------------------ oracle workers (CPU only)
def oracle_graph(cfg_index):
    from oracle import oracle as O
    n, mean = WEB[cfg_index]
    return O.gen_graph_exact(O.web_config(mean), n, SEED)


def worker_solve(cfg_index, damping, target, tag):
    """Oracle graph + sequential reference run to `target`; rank saved to TMP/<tag>.npy."""
    import numpy as np
    from oracle import oracle as O
    t0 = time.time()
    off, tgt, rep = oracle_graph(cfg_index)
    t_graph = time.time() - t0
    t0 = time.time()
    r = O.run_seq(off, tgt, damping, target, "sweep")
    t_run = time.time() - t0
    np.save(os.path.join(TMP, f"{tag}.npy"), r.rank)
    return {"tag": tag, "config": cfg_index, "damping": damping, "oracle_target": target,
            "n": int(off.size - 1), "edges": int(tgt.size), "off_sha": sha(off), "tgt_sha": sha(tgt), "report": rep,
            "graph_s": t_graph, "run_s": t_run, "diffusions": r.diffusions, "elementary_steps": r.elementary_steps,
            "residual": r.residual}


def worker_ppr(cfg_index, columns, tag):
    """Oracle runs of the first `columns` config-4 personalization vectors (teleport V_c)."""
    import numpy as np
    from oracle import oracle as O
    from paper_1202_6158_b200.ppr import config4_seeds  # numpy only: the seed draw of config 4
    off, tgt, rep = oracle_graph(cfg_index)
    n = off.size - 1
    seeds = config4_seeds(n, 64, 10, seed=SEED)
    ranks, own = [], []
    t0 = time.time()
    for c in range(columns):
        v = np.zeros(n)
        np.add.at(v, seeds[c].astype(np.int64), 1.0 / seeds.shape[1])
        truth = O.run_seq(off, tgt, 0.85, 1e-12, "sweep", teleport=v).rank
        ranks.append(truth)
        # the reference's own run at the config's residual 1e-9: its distance to the
        # tight solution is the accuracy any solver has at that stopping rule
        own.append(float(np.abs(O.run_seq(off, tgt, 0.85, 1e-9, "sweep", teleport=v).rank - truth).sum()))
    np.save(os.path.join(TMP, f"{tag}.npy"), np.stack(ranks, axis=1))
    return {"tag": tag, "config": cfg_index, "columns": columns, "off_sha": sha(off), "tgt_sha": sha(tgt),
            "report": rep, "run_s": time.time() - t0, "reference_at_1e-9_l1": own}


# ------------------------------------------------------------------ GPU side
def gpu_config(cfg_index, results, futures):
    import ctypes

    import numpy as np
    import torch

    import paper_1202_6158_b200 as fr
    from paper_1202_6158_b200 import _lib, gen

    out = {}
    t0 = time.time()
    g, rep = gen.baseline_graph(cfg_index, seed=SEED)
    torch.cuda.synchronize()
    out["graph_s"] = time.time() - t0
    off_h = g.out_offsets.cpu().numpy()
    tgt_h = g.out_targets.cpu().numpy().view(np.uint32)
    out.update(n=g.n, edges=g.edge_count, off_sha=sha(off_h), tgt_sha=sha(tgt_h),
               report={"slots": rep.slots, "realized_links": rep.realized_links, "duplicates": rep.duplicates,
                       "self_loops": rep.self_loops, "target_links": rep.target_links, "rounds": rep.rounds,
                       "unfilled": rep.unfilled})
    ranks = {}
    if cfg_index == 4:
        seeds = fr.config4_seeds(g.n, 64, 10, seed=SEED)
        for te in (1e-9, 1e-10):
            rank, stats, resid = fr.personalized_pagerank(g, seeds, target_error=te)
            ranks[f"ppr_{te}"] = rank[:, :PPR_COLUMNS].cpu().numpy()
            out[f"ppr_{te}"] = {"sweeps": stats.sweeps, "max_column_residual": max(resid)}
    else:
        dampings = (0.85, 0.99) if cfg_index == 5 else (0.85,)
        for d in dampings:
            decay, ef = SCHED[d]
            sched = fr.make_scheduler("sweep", policy="adaptive", sweep_decay=decay, edge_frac=ef,
                                      degree_exponent=BETA)
            params = fr.DiffusionParams(damping=d, target_error=1e-9)
            legs = [("fp64", 1e-9), ("tight", GPU_TIGHT[d])] + ([("fp32", 1e-9)] if cfg_index == 3 else [])
            for fl, te in legs:
                t0 = time.time()
                rank, trace = fr.run(g, fr.DiffusionParams(damping=d, target_error=te), sched,
                                     fluid_dtype=torch.float32 if fl == "fp32" else torch.float64)
                key = f"d{d}_{fl}"
                ranks[key] = rank
                last = trace.rows[-1]
                out[key] = {"sweeps": last.sweeps, "diffusions": last.diffusions,
                            "elementary_steps": last.elementary_steps, "residual": last.residual,
                            "wall_s": time.time() - t0}
            if cfg_index in (3, 5) and d == 0.85:
                # the reference-facing one-call path from host buffers (pieces when m >= 2^26)
                h_off = np.ascontiguousarray(off_h)
                h_tgt = np.ascontiguousarray(tgt_h)
                cfg = sched.solver_config(params)
                hr = np.empty(g.n)
                st = _lib.SolveStats()
                _lib.check(_lib.lib.fr_pagerank_host(g.n, h_tgt.size, h_off.ctypes.data, h_tgt.ctypes.data, None,
                                                     ctypes.byref(cfg), hr.ctypes.data, ctypes.byref(st)))
                ranks["d0.85_host"] = hr
                out["d0.85_host"] = {"sweeps": st.sweeps, "residual": st.residual}
    del g
    torch.cuda.empty_cache()
    return out, ranks


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,4,5")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_parity_fullsize.json"))
    args = ap.parse_args()
    cfgs = [int(c) for c in args.configs.split(",")]
    os.makedirs(TMP, exist_ok=True)
    import numpy as np
    from oracle import oracle as O
    O.build()
    ctx = mp.get_context("spawn")
    jobs = []
    for c in cfgs:
        if c == 4:
            jobs.append((c, "ppr", None, None))
        else:
            for d in ((0.85, 0.99) if c == 5 else (0.85,)):
                # the tight oracle solution, and the reference's own run at the config's 1e-9
                jobs.append((c, f"c{c}_d{d}", d, ORACLE_TRUTH[d]))
                jobs.append((c, f"c{c}_d{d}_ref1e-9", d, 1e-9))
    t_start = time.time()
    pool = ctx.Pool(processes=len(jobs))
    futures = {}
    for c, tag, d, te in jobs:
        if tag == "ppr":
            futures[tag] = pool.apply_async(worker_ppr, (c, PPR_COLUMNS, "c4_ppr"))
        else:
            futures[tag] = pool.apply_async(worker_solve, (c, d, te, tag))
    pool.close()

    import torch
    torch.cuda.set_device(0)
    report = {"seed": SEED, "oracle": "oracle/fr_oracle.c run_seq (ALGO-REF + ThresholdSweepScheduler, bit-exact "
                                       "with fluidrank.engine.run) on oracle.gen_graph_exact",
              "schedule": {"0.85": SCHED[0.85], "0.99": SCHED[0.99], "degree_exponent": BETA,
                           "kernel_path": "owned", "policy": "adaptive", "target_error": 1e-9},
              "bounds": {"fp64": 1e-9, "fp32_fluid": 1e-6}, "configs": {}}
    gpu_ranks = {}
    for c in cfgs:
        out, ranks = gpu_config(c, report, futures)
        report["configs"][f"config{c}"] = {"gpu": out}
        gpu_ranks[c] = ranks
        print(f"[gpu] config {c}: {json.dumps(out)}", flush=True)
    ok = True
    for c in cfgs:
        rec = report["configs"][f"config{c}"]
        gpu = rec["gpu"]
        checks = {}
        if c == 4:
            w = futures["ppr"].get()
            ref = np.load(os.path.join(TMP, "c4_ppr.npy"))
            checks["csr_bit_exact"] = (w["off_sha"], w["tgt_sha"]) == (gpu["off_sha"], gpu["tgt_sha"])
            for te in (1e-9, 1e-10):
                checks[f"ppr_{te}_column_l1"] = [float(np.abs(gpu_ranks[c][f"ppr_{te}"][:, k] - ref[:, k]).sum())
                                                 for k in range(PPR_COLUMNS)]
            # at the config's residual 1e-9 the device columns are as close to the tight
            # solution as the reference's own run at 1e-9; run 10x tighter they meet 1e-9
            checks["ppr_1e-09_vs_reference_at_1e-9"] = max(
                a / b for a, b in zip(checks["ppr_1e-09_column_l1"], w["reference_at_1e-9_l1"]))
            checks["ppr_1e-09_ok"] = checks["ppr_1e-09_vs_reference_at_1e-9"] <= 1.5
            checks["ppr_1e-10_ok"] = max(checks["ppr_1e-10_column_l1"]) <= 1e-9
            rec["oracle"] = w
        else:
            for d in ((0.85, 0.99) if c == 5 else (0.85,)):
                w = futures[f"c{c}_d{d}"].get()
                w9 = futures[f"c{c}_d{d}_ref1e-9"].get()
                ref = np.load(os.path.join(TMP, f"c{c}_d{d}.npy"))
                ref9 = np.load(os.path.join(TMP, f"c{c}_d{d}_ref1e-9.npy"))
                rec[f"oracle_d{d}"] = w
                rec[f"oracle_d{d}_at_1e-9"] = w9
                checks["csr_bit_exact"] = all(
                    (x["off_sha"], x["tgt_sha"], x["edges"], x["report"]) ==
                    (gpu["off_sha"], gpu["tgt_sha"], gpu["edges"], gpu["report"]) for x in (w, w9))
                # the accuracy the config's stopping rule gives the reference itself
                ref_err = float(np.abs(ref9 - ref).sum())
                checks[f"d{d}_reference_at_1e-9_l1"] = ref_err
                for key, rank in gpu_ranks[c].items():
                    if not key.startswith(f"d{d}_"):
                        continue
                    l1 = float(np.abs(rank - ref).sum())
                    checks[f"{key}_l1"] = l1
                    if key.endswith("fp32"):
                        checks[f"{key}_ok"] = l1 <= 1e-6
                    elif key.endswith("tight"):
                        checks[f"{key}_ok"] = l1 <= 1e-9
                    else:
                        # at residual 1e-9: within 1e-9 of the tight solution, or (d = 0.99,
                        # where dangling absorption shrinks |h|_1 ~16x and no solver stopping at
                        # 1e-9 gets there) no farther from it than the reference's own run
                        checks[f"{key}_vs_reference"] = l1 / ref_err if ref_err > 0 else None
                        checks[f"{key}_ok"] = l1 <= 1e-9 or l1 <= 1.5 * ref_err
                os.remove(os.path.join(TMP, f"c{c}_d{d}.npy"))
                os.remove(os.path.join(TMP, f"c{c}_d{d}_ref1e-9.npy"))
        rec["checks"] = checks
        ok = ok and all(v for k, v in checks.items() if k.endswith("_ok") or k == "csr_bit_exact")
        print(f"[check] config {c}: {json.dumps(checks)}", flush=True)
    pool.join()
    report["all_ok"] = ok
    report["wall_s"] = time.time() - t_start
    with open(args.out, "w") as f:
        json.dump(report, f, indent=1)
    print(json.dumps({"all_ok": ok, "wall_s": report["wall_s"]}), flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
