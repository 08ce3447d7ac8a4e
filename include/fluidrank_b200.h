/*
 * fluidrank_b200.h -- C ABI of the B200-native fluid-diffusion (D-iteration)
 * PageRank solver.  This is the drop-in boundary: the Python host package
 * paper_1202_6158_b200 binds exactly these symbols through ctypes, and any
 * other host language binds them the same way.
 *
 * Conventions
 *   d_*     device pointers (CUDA global memory of the current device)
 *   h_*     host pointers
 *   stream  a cudaStream_t passed as void* (NULL = legacy default stream)
 *   return  FR_OK (0) or an FR_ERR_* code; fr_last_error() gives the
 *           thread-local message of the last failure.
 *   Nodes are dense ids 0..n-1 with n < 2^32; row offsets are int64, column
 *   indices uint32 (the BASELINE config-5 layout: 64-bit offsets, 32-bit
 *   indices).
 *
 * Each entry point names the reference interface it replaces
 * (reference = pkg/src/fluidrank/ of arxiv/paper_1202_6158).
 */
#ifndef FLUIDRANK_B200_H
#define FLUIDRANK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 3: fr_power_run_profiled fills 4 timings (was 3); fr_ppr_set_pull added */
#define FR_ABI_VERSION 3

enum fr_status {
    FR_OK = 0,
    FR_ERR_RANGE = 1,          /* edge endpoint out of range      (graph.py:86-87) */
    FR_ERR_SELF_LOOP = 2,      /* self-loop in edge arrays        (graph.py:88-89) */
    FR_ERR_DUPLICATE = 3,      /* duplicate edge in edge arrays   (graph.py:92-94) */
    FR_ERR_ARG = 4,            /* invalid argument                                 */
    FR_ERR_CUDA = 5,           /* CUDA runtime failure                             */
    FR_ERR_NO_CONVERGENCE = 6, /* sweep budget exhausted above the target          */
    FR_ERR_NO_DEVICE = 7       /* no CUDA device visible                           */
};

const char *fr_last_error(void);
int fr_abi_version(void);
/* Number of SMs of the current device (148 on B200); 0 when none. */
int fr_device_sms(void);

/* ------------------------------------------------------------------ */
/* Synthetic graphs (BASELINE.json configs).  kind 0 = "uniform"       */
/* (config 1), kind 1 = "web" (configs 2-5).  Bit-identical to the     */
/* specification in oracle/fr_oracle.c (fro_gen_*).                    */
/* ------------------------------------------------------------------ */
typedef struct fr_gen_config {
    int32_t kind;
    int32_t max_out;       /* uniform: out-degree uniform in {0..max_out} */
    double mean_degree;    /* web: mean out-degree after rescaling        */
    double alpha;          /* web: out-degree power-law exponent          */
    int32_t max_degree;    /* web: power-law truncation                   */
    int32_t window;        /* web: local targets within +-window ids      */
    double dangling_frac;  /* web: fraction of zero out-degree nodes      */
    double local_frac;     /* web: fraction of local targets              */
    double zipf_s;         /* web: Zipf exponent of non-local targets     */
} fr_gen_config;

/* Per-node slot counts; *h_total = sum (edge-list length). */
int fr_gen_degrees(const fr_gen_config *cfg, int64_t n, uint64_t seed, uint32_t *d_deg,
                   int64_t *h_total, void *stream);
/* Source-major edge list (src[e], dst[e]), e < h_total of fr_gen_degrees. */
int fr_gen_edges(const fr_gen_config *cfg, int64_t n, uint64_t seed, const uint32_t *d_deg,
                 uint32_t *d_src, uint32_t *d_dst, void *stream);
/* Fill round `round` of the exact-size graph (round 0 = fr_gen_edges): d_deg is
 * the per-node deficit left by cleaning (duplicates / self-loops dropped) and
 * (d_offsets, d_targets) the clean graph so far (NULL in round 0); the draws
 * come from fresh per-round streams, and a node whose local window the graph
 * already completes draws from the Zipf class only.  Repeating draw -> clean
 * union until no deficit is left realises the configured out-degrees as
 * distinct edges, as the reference generator draws until the target count of
 * distinct links exists (gen.py:66-110). */
int fr_gen_edges_round(const fr_gen_config *cfg, int64_t n, uint64_t seed, uint32_t round,
                       const uint32_t *d_deg, const int64_t *d_offsets, const uint32_t *d_targets,
                       uint32_t *d_src, uint32_t *d_dst, void *stream);

/* ------------------------------------------------------------------ */
/* CSR construction on the device.                                     */
/* Replaces graph.py:74-97 SparseGraph.from_edges (clean = 0: rejects  */
/* out-of-range ids, self-loops and duplicates with FR_ERR_*), and     */
/* graph.py:183-200 build_clean_edges + from_edges (clean = 1: drops   */
/* self-loops, collapses duplicates).  Children of each node are       */
/* sorted ascending, exactly as the reference's lexsort.               */
/* d_offsets: n+1 int64; d_targets: capacity m.                        */
/* h_stats[3] = {edges kept L, duplicates dropped, self-loops dropped}.*/
/* ------------------------------------------------------------------ */
int fr_csr_build(int64_t n, int64_t m, const uint32_t *d_src, const uint32_t *d_dst, int32_t clean,
                 int64_t *d_offsets, uint32_t *d_targets, int64_t *h_stats, void *stream);
/* graph.py:62 in_degree = bincount(out_targets). */
int fr_in_degree(int64_t n, int64_t m, const uint32_t *d_targets, int64_t *d_in_degree, void *stream);

/* ------------------------------------------------------------------ */
/* Diffusion state.                                                    */
/* ------------------------------------------------------------------ */
/* engine.py:149-159 init / 162-172 init_from_fluid: fluid =
 * (1-damping)*teleport (teleport NULL = uniform 1/n; damping >= 1 keeps
 * the teleport itself), history = 0.  fluid_fp32 selects a float fluid. */
int fr_init_state(int64_t n, double damping, const double *d_teleport, void *d_fluid,
                  int32_t fluid_fp32, double *d_history, void *stream);
/* engine.py:175-199 diffuse(state, i): one node; *h_sent = fluid taken. */
int fr_diffuse_node(int64_t n, const int64_t *d_offsets, const uint32_t *d_targets, double *d_fluid,
                    double *d_history, int64_t node, double damping, double *h_sent, void *stream);
/* sum |x| (engine.py:145-146 exact_residual, 202-211 error_bound). */
int fr_abs_sum(int64_t n, const void *d_x, int32_t x_fp32, double *h_sum, void *stream);
/* engine.py:235-237 _normalized: rank = history / sum|history|. */
int fr_normalize(int64_t n, const double *d_history, double *d_rank, double *h_total, void *stream);
/* engine.py:269-274 sample(): true error |history/|history|_1 - reference|_1. */
int fr_l1_error(int64_t n, const double *d_history, const double *d_reference, double *h_err, void *stream);

/* ------------------------------------------------------------------ */
/* Data-parallel threshold-sweep solver: engine.py:240-341 run() with  */
/* the schedules of sched.py (sweep 69-113, max 16-25, per 52-66,      */
/* rand 28-49, op/op2 116-144) lifted to whole-frontier sweeps.  The   */
/* convergence loop runs on the device (CUDA graph while-node).        */
/* ------------------------------------------------------------------ */
enum fr_select {
    FR_SELECT_SWEEP = 0, /* |f| >= theta                                  */
    FR_SELECT_MAX = 1,   /* |f| >= decay * (max |f| of the previous sweep) */
    FR_SELECT_PER = 2,   /* every node holding fluid (Jacobi cycle)       */
    FR_SELECT_RAND = 3,  /* each fluid-holding node with prob. rand_frac  */
    FR_SELECT_OP = 4,    /* |f| * score_weight >= theta (weights 1/((in+1)(out+1))) */
    FR_SELECT_OP2 = 5    /* |f| * score_weight >= theta (weights 1/(out+1))         */
};
enum fr_theta_policy {
    FR_THETA_EXHAUST = 0,   /* decay only after a sweep that finds nothing (sched.py:101-108) */
    FR_THETA_GEOMETRIC = 1, /* decay after every sweep (PAPER sec. 4.2)                       */
    FR_THETA_ADAPTIVE = 2   /* theta steered so a sweep pushes ~ edge_frac * m edges:
                               theta *= decay * sqrt(pushed / (edge_frac * m)), clamped   */
};

typedef struct fr_solver_config {
    double damping;           /* d                                     */
    double target_error;      /* stop when residual <= target*(1-d)    */
    double decay;             /* theta decay factor (sched.py:79)      */
    double rand_frac;         /* FR_SELECT_RAND selection probability  */
    double edge_frac;         /* FR_THETA_ADAPTIVE: target pushed edges per sweep / m (<= 0: 0.2) */
    int64_t max_sweeps;       /* sweep budget (<= 0: 1e6)              */
    int64_t max_diffusions;   /* stop once this many diffusions ran (<= 0: none);
                                 required when damping == 1 (engine.py:256-257) */
    int32_t select;           /* enum fr_select                         */
    int32_t policy;           /* enum fr_theta_policy                   */
    int32_t fluid_fp32;       /* 1: float fluid, double history         */
    int32_t thread_max_degree;/* bins: deg <= this -> thread per node (0 = default 8)   */
    int32_t block_min_degree; /* deg >= this -> block per node (0 = default 2048)       */
    uint32_t seed;            /* FR_SELECT_RAND                          */
    int32_t kernel_path;      /* 0: fused warp-tile sweep (select, take and push in one
                                    kernel; hubs block-per-node) -- default of a zeroed config
                                 1: binned queues (select kernel, then thread / warp /
                                    block-per-node push kernels)
                                 2: owned chunks (as 0, but a block owns a chunk of
                                    consecutive nodes: in-chunk pushes are summed in shared
                                    memory and diffused in the same sweep; FR_OWN_CHUNK
                                    nodes, default 2048) -- the Python mirror's default */
    int32_t hot_slots;        /* fused path: pushes into the hot_slots highest in-degree
                                 nodes are summed per block in shared memory first
                                 (0 = default: 2048, owned path 512; max 2048; -1 = off) */
    double degree_exponent;   /* FR_SELECT_SWEEP score = |f| * (out_degree + 1)^-degree_exponent
                                 (0 = |f|, the reference sweep; 1 = the op2 weight of
                                 sched.py:131-138; PAPER sec. 4.3 ALGO-OP2)          */
    int32_t warm_slots;       /* fused path: pushes into the next warm_slots highest
                                 in-degree nodes go to a compact L2-resident array that
                                 is folded back into F after every sweep
                                 (0 = default 2^19, max 2^24, -1 = off)             */
} fr_solver_config;

typedef struct fr_trace_row {
    int64_t elementary_steps; /* edges diffused so far                 */
    int64_t diffusions;       /* node diffusions so far                */
    int64_t sweeps;
    double residual;          /* fluid mass left (R of ALGO-REF)       */
    double theta;             /* threshold used by this sweep          */
    int64_t t_ns;             /* device clock (%globaltimer) at the end of the sweep */
} fr_trace_row;

typedef struct fr_solve_stats {
    int64_t diffusions;
    int64_t elementary_steps;
    int64_t sweeps;
    double residual;          /* exact sum |F| after the run           */
    double theta;
    int64_t trace_len;
    int64_t hub_edges;        /* edges pushed by the hub (block-per-node) kernel */
} fr_solve_stats;

typedef struct fr_solver fr_solver;

/* Binds a graph, a state (d_fluid / d_history, updated in place) and a
 * configuration; builds the device-side loop once.  d_score_weight: per-node
 * score multiplier for FR_SELECT_OP / OP2 (else NULL).  trace_cap: per-sweep
 * rows kept on the device. */
int fr_solver_create(int64_t n, int64_t m, const int64_t *d_offsets, const uint32_t *d_targets,
                     const double *d_score_weight, void *d_fluid, double *d_history,
                     const fr_solver_config *cfg, int64_t trace_cap, void *stream,
                     fr_solver **out);
/* Diffuses from the current state until residual <= target*(1-d).
 * An explicit budget (max_sweeps / max_diffusions > 0) stops quietly, like the
 * reference's max_diffusions; FR_ERR_NO_CONVERGENCE means the implicit 1e6
 * sweep cap ran out above the target. */
int fr_solver_run(fr_solver *s, void *stream, fr_solve_stats *h_stats);
int fr_solver_trace(fr_solver *s, fr_trace_row *h_rows, int64_t cap, int64_t *h_len, void *stream);
/* Same computation as fr_solver_run, but launched sweep by sweep from the
 * host with CUDA events around every kernel (for the roofline report; not
 * the timed path).  Per kernel class k (0 select, 1 thread-bin push,
 * 2 warp-bin push, 3 block-bin push, 4 finalize): h_ms[k] = summed device
 * time, h_launches[k] = launches. */
int fr_solver_run_profiled(fr_solver *s, void *stream, fr_solve_stats *h_stats, double *h_ms,
                           int64_t *h_launches);
/* engine.py:240-341 run(..., trace_every, reference): the same solve as
 * fr_solver_run, sweeps launched from the host; after every sweep that brings
 * the diffusion count past the next multiple of trace_every, the true L1
 * error |h/|h|_1 - reference|_1 of that trace row is recorded (engine.py:
 * 269-277, 334-336).  Diagnostic path (one host sync per sweep). */
int fr_solver_run_sampled(fr_solver *s, void *stream, const double *d_reference, int64_t trace_every,
                          fr_solve_stats *h_stats);
/* True errors of the last sampled run, one per trace row (NaN: not sampled). */
int fr_solver_trace_errors(fr_solver *s, double *h_err, int64_t cap, void *stream);
int fr_solver_destroy(fr_solver *s);

/* ------------------------------------------------------------------ */
/* Power iteration (MAT-ITER): baseline.py:20-56 power_iterate on a  */
/* pull CSR SpMV over the transposed graph (graph.py:158-180).         */
/* ------------------------------------------------------------------ */
typedef struct fr_power fr_power;
int fr_power_create(int64_t n, int64_t m, const int64_t *d_out_offsets, const int64_t *d_in_offsets,
                    const uint32_t *d_in_sources, double damping, const double *d_teleport,
                    void *stream, fr_power **out);
/* x <- teleport, iterate until |x_n - x_{n-1}|_1 * d/(1-d) <= target_error. */
int fr_power_run(fr_power *p, double target_error, int64_t max_iterations, double *d_x,
                 int64_t *h_iterations, double *h_diff, void *stream);
/* Same iterations launched from the host with CUDA events (roofline report, not
 * the timed path), summed over the iterations (h_ms: 4 doubles): h_ms[0] =
 * short-row SpMV tiles with their rows' update, h_ms[1] = hub rows (in-degree >
 * 1024) by source block, h_ms[2] = long hub slices, h_ms[3] = the rest (hub
 * rows' update, stopping rule). */
int fr_power_run_profiled(fr_power *p, double target_error, int64_t max_iterations, double *d_x,
                          int64_t *h_iterations, double *h_ms, void *stream);
int fr_power_destroy(fr_power *p);

/* ------------------------------------------------------------------ */
/* Batched personalized PageRank (BASELINE config 4): B <= 64 teleport */
/* vectors diffuse together; fluid/history are n x B row-major fp64.   */
/* Each column c is engine.py:240-341 run() with teleport V_c; column  */
/* c stops once its residual <= target*(1-d) (checked exactly).        */
/* ------------------------------------------------------------------ */
typedef struct fr_ppr fr_ppr;
/* F[s, c] += (1-d)/k for each of the k seeds s of column c (V_c uniform over
 * its seeds, repeated seeds accumulate), H = 0.  d_seeds: B x k uint32. */
int fr_ppr_init(int64_t n, int32_t B, const uint32_t *d_seeds, int32_t k, double damping, double *d_fluid,
                double *d_history, void *stream);
/* cfg: damping, target_error, decay (geometric theta), max_sweeps. */
int fr_ppr_create(int64_t n, int64_t m, const int64_t *d_offsets, const uint32_t *d_targets, int32_t B,
                  double *d_fluid, double *d_history, const fr_solver_config *cfg, void *stream, fr_ppr **out);
/* h_col_residual (B): exact final residual of each column.  h_stats:
 * diffusions = row visits, elementary_steps = edge visits, hub_edges = column
 * values scattered (one red.add each; zero pushes are skipped). */
int fr_ppr_run(fr_ppr *p, void *stream, fr_solve_stats *h_stats, double *h_col_residual);
/* Pull formulation (no atomics, bit-reproducible): the selected rows' pushes are
 * written once and every node sums those of its selected parents over the
 * transposed CSR (d_in_offsets int64[n+1], d_in_sources uint32[m], graph.py
 * to_matrix(); the arrays must stay valid while the handle is used).  Jacobi
 * within a sweep, so more sweeps than the default push (red.add scatter); the
 * same fixed point per column. */
int fr_ppr_set_pull(fr_ppr *p, const int64_t *d_in_offsets, const uint32_t *d_in_sources);
int fr_ppr_destroy(fr_ppr *p);
/* rank[:, c] = history[:, c] / sum |history[:, c]|. */
int fr_ppr_normalize(int64_t n, int32_t B, const double *d_history, double *d_rank, void *stream);

/* ------------------------------------------------------------------ */
/* One call from host buffers (the reference-facing end-to-end path):  */
/* H2D of the CSR, device solve, D2H of the normalized rank.           */
/* engine.py:240-341 run(graph, params, scheduler) -> rank.            */
/* h_teleport: n doubles, params.teleport (engine.py:56-62, 149-159);  */
/* NULL = uniform 1/n.  Rejected like DiffusionParams.validate         */
/* (engine.py:47-54) when negative or not summing to 1 within 1e-12.   */
/* ------------------------------------------------------------------ */
int fr_pagerank_host(int64_t n, int64_t m, const int64_t *h_offsets, const uint32_t *h_targets,
                     const double *h_teleport, const fr_solver_config *cfg, double *h_rank,
                     fr_solve_stats *h_stats);

#ifdef __cplusplus
}
#endif
#endif /* FLUIDRANK_B200_H */
