"""ctypes front end of the CPU oracle (oracle/fr_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, never by the product
package.  Each wrapper names the reference function it restates
(reference = /root/reference/pkg/src/fluidrank).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import time
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libfr_oracle.so")

SWEEP, MAX, PER, OP, OP2 = 0, 1, 2, 3, 4
KIND_CODES = {"sweep": SWEEP, "max": MAX, "per": PER, "op": OP, "op2": OP2}


class GenConfig(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("max_out", ctypes.c_int32),
                ("mean_degree", ctypes.c_double), ("alpha", ctypes.c_double),
                ("max_degree", ctypes.c_int32), ("window", ctypes.c_int32),
                ("dangling_frac", ctypes.c_double), ("local_frac", ctypes.c_double),
                ("zipf_s", ctypes.c_double)]


class TraceRow(ctypes.Structure):
    _fields_ = [("elementary_steps", ctypes.c_int64), ("diffusions", ctypes.c_int64),
                ("residual", ctypes.c_double), ("bound", ctypes.c_double)]


class RunResult(ctypes.Structure):
    _fields_ = [("diffusions", ctypes.c_int64), ("elementary_steps", ctypes.c_int64),
                ("residual", ctypes.c_double), ("trace_len", ctypes.c_int64),
                ("sweeps", ctypes.c_int64), ("status", ctypes.c_int32)]


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64, f64, i32 = ctypes.c_int64, ctypes.c_double, ctypes.c_int
        L.fro_pairwise_sum.restype = f64
        L.fro_pairwise_sum.argtypes = [P, i64, i32]
        L.fro_gen_degrees.restype = i64
        L.fro_gen_degrees.argtypes = [P, i64, ctypes.c_uint64, P]
        L.fro_gen_edges.restype = i32
        L.fro_gen_edges.argtypes = [P, i64, ctypes.c_uint64, P, P, P]
        L.fro_gen_edges_round.restype = i32
        L.fro_gen_edges_round.argtypes = [P, i64, ctypes.c_uint64, ctypes.c_uint32, P, P, P, P, P]
        L.fro_csr_merge.restype = i32
        L.fro_csr_merge.argtypes = [i64, P, P, i64, P, P, P, P, P]
        L.fro_gen_feistel.restype = ctypes.c_uint64
        L.fro_gen_feistel.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
        L.fro_gen_powerlaw_table.restype = i32
        L.fro_gen_powerlaw_table.argtypes = [P, P, P]
        L.fro_gen_zipf_table.restype = None
        L.fro_gen_zipf_table.argtypes = [i64, f64, P]
        L.fro_csr_build.restype = i32
        L.fro_csr_build.argtypes = [i64, i64, P, P, i32, P, P, P]
        L.fro_run_seq.restype = i32
        L.fro_run_seq.argtypes = [i64, P, P, P, f64, f64, i32, f64, i64, i64, i32, P, P,
                                  f64, i64, i64, P, i64, P, P]
        L.fro_run_psweep.restype = i32
        L.fro_run_psweep.argtypes = [i64, P, P, f64, f64, i32, f64, i64, i32, P, P, P, i64, P, P, P, f64]
        L.fro_power_iterate.restype = i64
        L.fro_power_iterate.argtypes = [i64, P, P, P, i64, f64, P, f64, i64, i64, P, P, i64, P, P]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


# ---------------------------------------------------------------- generator
# BASELINE.json configs (the web generator's parameters are configs 2-5).
def uniform_config(max_out=10):
    return GenConfig(kind=0, max_out=max_out)


def web_config(mean_degree=8.0, alpha=2.1, max_degree=5000, window=1000,
               dangling_frac=0.15, local_frac=0.7, zipf_s=1.0):
    return GenConfig(kind=1, mean_degree=mean_degree, alpha=alpha, max_degree=max_degree,
                     window=window, dangling_frac=dangling_frac, local_frac=local_frac,
                     zipf_s=zipf_s)


def gen_degrees(cfg, n, seed):
    deg = np.empty(n, dtype=np.uint32)
    total = lib().fro_gen_degrees(ctypes.byref(cfg), n, seed, _ptr(deg))
    if total < 0:
        raise ValueError("bad generator config")
    return deg, int(total)


def gen_edges(cfg, n, seed):
    """Edge list (src, dst) as uint32 in source-major slot order."""
    deg, total = gen_degrees(cfg, n, seed)
    src = np.empty(total, dtype=np.uint32)
    dst = np.empty(total, dtype=np.uint32)
    if lib().fro_gen_edges(ctypes.byref(cfg), n, seed, _ptr(deg), _ptr(src), _ptr(dst)) != 0:
        raise MemoryError("generator table allocation failed")
    return src, dst


def gen_edges_round(cfg, n, seed, rnd, deg, off=None, tgt=None):
    """Draws for deg[u] slots of every node in fill round rnd (round 0 = gen_edges);
    (off, tgt): the clean graph so far (a node whose local window it already fills
    draws from the Zipf class only)."""
    deg = np.ascontiguousarray(deg, dtype=np.uint32)
    total = int(deg.sum(dtype=np.int64))
    src = np.empty(max(total, 1), dtype=np.uint32)
    dst = np.empty(max(total, 1), dtype=np.uint32)
    off = None if off is None else np.ascontiguousarray(off, dtype=np.int64)
    tgt = None if tgt is None else np.ascontiguousarray(tgt, dtype=np.uint32)
    if lib().fro_gen_edges_round(ctypes.byref(cfg), n, seed, rnd, _ptr(deg), _ptr(off), _ptr(tgt), _ptr(src),
                                 _ptr(dst)) != 0:
        raise MemoryError("generator table allocation failed")
    return src[:total], dst[:total]


def csr_merge(n, off, tgt, src2, dst2):
    """Clean union of a clean CSR with extra edges (graph.py:183-200 on the concatenation)."""
    src2 = np.ascontiguousarray(src2, dtype=np.uint32)
    dst2 = np.ascontiguousarray(dst2, dtype=np.uint32)
    off_out = np.empty(n + 1, dtype=np.int64)
    tgt_out = np.empty(max(int(off[-1]) + src2.size, 1), dtype=np.uint32)
    stats = np.zeros(3, dtype=np.int64)
    rc = lib().fro_csr_merge(n, _ptr(np.ascontiguousarray(off, dtype=np.int64)),
                             _ptr(np.ascontiguousarray(tgt, dtype=np.uint32)), src2.size, _ptr(src2), _ptr(dst2),
                             _ptr(off_out), _ptr(tgt_out), _ptr(stats))
    if rc:
        raise ValueError(CSR_ERRORS.get(rc, f"csr merge failed ({rc})"))
    return off_out, tgt_out[: int(stats[0])].copy(), tuple(int(x) for x in stats)


MAX_FILL_ROUNDS = 32


def gen_graph_exact(cfg, n, seed, max_rounds=MAX_FILL_ROUNDS):
    """The exact-size BASELINE graph: base draw, cleaned, then fill rounds that redraw the
    dropped slots (per-node deficit) until every node has its configured out-degree in
    distinct edges (the reference generator draws until the target number of distinct
    links exists, gen.py:66-110).  Returns (off, tgt, report dict)."""
    deg, total = gen_degrees(cfg, n, seed)
    src, dst = gen_edges_round(cfg, n, seed, 0, deg)
    off, tgt, (L, dups, loops) = csr_build(n, src, dst, clean=True)
    del src, dst
    slots, rounds = total, 0
    for r in range(1, max_rounds + 1):
        deficit = (deg.astype(np.int64) - np.diff(off)).astype(np.uint32)
        need = int(deficit.sum(dtype=np.int64))
        if need == 0:
            break
        s2, d2 = gen_edges_round(cfg, n, seed, r, deficit, off, tgt)
        off, tgt, (L, rd, rl) = csr_merge(n, off, tgt, s2, d2)
        slots += need
        dups += rd
        loops += rl
        rounds = r
    return off, tgt, {"slots": slots, "realized_links": L, "duplicates": dups, "self_loops": loops,
                      "target_links": total, "rounds": rounds, "unfilled": total - L}


def feistel(x, n, seed):
    return int(lib().fro_gen_feistel(x, n, seed))


# ---------------------------------------------------------------- CSR build
CSR_ERRORS = {1: "edge endpoint out of range", 2: "self-loop in edge arrays",
              3: "duplicate edge in edge arrays"}


def csr_build(n, src, dst, clean=False):
    """graph.py:74-97 from_edges (strict) / graph.py:183-200 + from_edges (clean).

    Returns (offsets int64[n+1], targets uint32[L], (L, duplicates, self_loops)).
    """
    src = np.ascontiguousarray(src, dtype=np.uint32)
    dst = np.ascontiguousarray(dst, dtype=np.uint32)
    m = src.size
    off = np.empty(n + 1, dtype=np.int64)
    tgt = np.empty(max(m, 1), dtype=np.uint32)
    stats = np.zeros(3, dtype=np.int64)
    rc = lib().fro_csr_build(n, m, _ptr(src), _ptr(dst), int(clean), _ptr(off), _ptr(tgt), _ptr(stats))
    if rc:
        raise ValueError(CSR_ERRORS.get(rc, f"csr build failed ({rc})"))
    return off, tgt[: int(stats[0])].copy(), tuple(int(x) for x in stats)


def in_degree(n, tgt):
    return np.bincount(tgt.astype(np.int64), minlength=n).astype(np.int64)


def transpose(n, off, tgt):
    """In-link CSR (rows = targets, sources ascending) -- graph.py:158-180."""
    deg = np.diff(off)
    src = np.repeat(np.arange(n, dtype=np.uint32), deg)
    in_off, in_src, _ = csr_build(n, tgt, src, clean=False)
    return in_off, in_src


# ---------------------------------------------------------------- solvers
def pairwise_sum(a, absval=False):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().fro_pairwise_sum(_ptr(a), a.size, int(absval)))


def init_fluid(n, damping=0.85, teleport=None):
    """engine.py:149-159 init."""
    v = np.full(n, 1.0 / n) if teleport is None else np.asarray(teleport, dtype=np.float64).copy()
    return v if damping >= 1.0 else (1.0 - damping) * v


@dataclass
class OracleRun:
    rank: np.ndarray
    history: np.ndarray
    fluid: np.ndarray
    residual: float
    diffusions: int
    elementary_steps: int
    sweeps: int
    trace: np.ndarray  # rows (elementary_steps, diffusions, residual, bound)
    seconds: float = 0.0  # the C solve alone (fro_run_seq), wall clock


def _trace_array(rows, length):
    k = min(length, len(rows))
    out = np.zeros((k, 4))
    for i in range(k):
        r = rows[i]
        out[i] = (r.elementary_steps, r.diffusions, r.residual, r.bound)
    return out


def run_seq(off, tgt, damping=0.85, target_error=1e-8, kind="sweep", decay=0.5,
            teleport=None, max_diffusions=None, trace_every=None, fluid=None,
            history=None, residual=None, trace_cap=1 << 16):
    """engine.py:240-341 run() with the named sched.py scheduler, sequentially."""
    n = off.size - 1
    off = np.ascontiguousarray(off, dtype=np.int64)
    tgt = np.ascontiguousarray(tgt, dtype=np.uint32)
    fluid = init_fluid(n, damping, teleport) if fluid is None else np.array(fluid, dtype=np.float64)
    history = np.zeros(n) if history is None else np.array(history, dtype=np.float64)
    signed = bool(np.any(fluid < 0.0))
    if residual is None:
        residual = pairwise_sum(fluid, absval=signed)
    in_deg = in_degree(n, tgt) if kind == "op" else None  # only the op weights read it
    rows = (TraceRow * trace_cap)()
    rank = np.empty(n)
    res = RunResult()
    t0 = time.perf_counter()
    rc = lib().fro_run_seq(n, _ptr(off), _ptr(tgt), _ptr(in_deg), damping, target_error,
                           KIND_CODES[kind], decay, -1 if max_diffusions is None else max_diffusions,
                           0 if trace_every is None else trace_every, int(signed), _ptr(fluid),
                           _ptr(history), residual, 0, 0, rows, trace_cap, _ptr(rank),
                           ctypes.byref(res))
    elapsed = time.perf_counter() - t0
    if rc == 3:
        raise RuntimeError("scheduler starved")
    return OracleRun(rank, history, fluid, res.residual, res.diffusions, res.elementary_steps,
                     0, _trace_array(rows, res.trace_len), elapsed)


def run_psweep(off, tgt, damping=0.85, target_error=1e-8, policy=0, decay=0.5,
               teleport=None, max_sweeps=None, fluid=None, history=None, trace_cap=1 << 16, weight=None,
               edge_frac=0.2):
    """The product's data-parallel threshold sweep, restated sequentially."""
    n = off.size - 1
    off = np.ascontiguousarray(off, dtype=np.int64)
    tgt = np.ascontiguousarray(tgt, dtype=np.uint32)
    fluid = init_fluid(n, damping, teleport) if fluid is None else np.array(fluid, dtype=np.float64)
    history = np.zeros(n) if history is None else np.array(history, dtype=np.float64)
    signed = bool(np.any(fluid < 0.0))
    rows = (TraceRow * trace_cap)()
    rank = np.empty(n)
    res = RunResult()
    w = None if weight is None else np.ascontiguousarray(weight, dtype=np.float64)
    lib().fro_run_psweep(n, _ptr(off), _ptr(tgt), damping, target_error, policy, decay,
                         -1 if max_sweeps is None else max_sweeps, int(signed), _ptr(fluid),
                         _ptr(history), rows, trace_cap, _ptr(rank), ctypes.byref(res), _ptr(w), edge_frac)
    return OracleRun(rank, history, fluid, res.residual, res.diffusions, res.elementary_steps,
                     res.sweeps, _trace_array(rows, res.trace_len))


def power_iterate(off, tgt, damping=0.85, target_error=1e-8, teleport=None,
                  max_iterations=1_000_000, trace_every=1, trace_cap=1 << 16):
    """baseline.py:20-56 power_iterate (scipy CSR matvec order)."""
    n = off.size - 1
    in_off, in_src = transpose(n, off, tgt)
    out_deg = np.diff(off).astype(np.int64)
    v = None if teleport is None else np.ascontiguousarray(teleport, dtype=np.float64)
    x = np.empty(n)
    rows = (TraceRow * trace_cap)()
    tlen = ctypes.c_int64(0)
    diff = ctypes.c_double(0)
    it = lib().fro_power_iterate(n, _ptr(in_off), _ptr(in_src), _ptr(out_deg), int(tgt.size),
                                 damping, _ptr(v), target_error, max_iterations, trace_every,
                                 _ptr(x), rows, trace_cap, ctypes.byref(tlen), ctypes.byref(diff))
    if it < 0:
        raise RuntimeError(f"no convergence within {max_iterations} iterations")
    return x, int(it), _trace_array(rows, tlen.value)
