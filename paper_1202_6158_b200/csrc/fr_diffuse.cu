// fr_diffuse.cu -- data-parallel threshold-sweep D-iteration on the device.
//
// Reference semantics: engine.py:240-341 run() driving the ALGO-REF diffusion
// step (engine.py:315-329; PAPER sec. 2.2 / 3.3) under a node-selection rule
// (sched.py).  Because H_n + F_n = F_0 + dP H_n holds for ANY selection order
// (PAPER Theorem 3.1), a whole frontier of nodes can diffuse at once.
//
// Owned path (kernel_path = 2, the Python default), one sweep:
//   k_sweep_own    block of 4 warps per chunk of 2048 consecutive nodes, chunks
//                  taken in order from one counter, tiles of the chunk claimed
//                  one at a time; per tile as k_sweep below, except that pushes
//                  into the block's own chunk are summed in shared memory and
//                  taken by the chunk's later tiles in the same sweep
//                  (Gauss-Seidel), the rest flushed to F at the chunk end; odd
//                  sweeps run backwards; rows with >= t2 children are queued and,
//                  in the CUDA-graph loop, pushed by the next sweep's blocks
//                  between their chunks (the last sweep's by a k_push_block drain
//                  after the loop; host-launched sweeps run k_push_block after
//                  each sweep); then k_fold, k_finalize
//
// Fused path (kernel_path = 0), one sweep:
//   k_sweep        warp per tile of 32 consecutive nodes, tiles taken in order
//                  from segmented counters: scan F and the row offsets, select
//                  (|f| * (deg+1)^-beta >= theta, or the other rules), take the
//                  loaded fluid with red.add(F_i, -f) and red.add(H_i, f), then
//                  push f*d/deg over the tile's compacted edge space (hot
//                  targets summed in shared memory, warm targets into the
//                  L2-resident Fw); rows with >= t2 children are queued
//   k_push_block   block per queued hub row, adjacency streamed into shared
//                  memory by cp.async.bulk through a 3-stage mbarrier ring
//   k_fold         Fw back into F
//   k_finalize     fixed-order reduction of the block partials, counters,
//                  trace row, theta schedule, loop condition
//   k_mass_partials / k_mass_check   (guarded) exact sum |F| before stopping
//
// Binned path (kernel_path = 1, the north star's literal degree bins):
//   k_select       coalesced scan, take, block-scan enqueue into three bins
//   k_push_thread  thread per node    (deg <= thread_max_degree)
//   k_push_warp    warp per node      (128-bit coalesced column loads)
//   k_push_block   block per hub node (as above), then k_fold, k_finalize
//
// The sweep loop is a CUDA-graph while-node: the host launches one graph per
// solve and waits once; there is no per-sweep host round trip.
#include <math.h>
#include <stdlib.h>

#include <climits>
#include <cstddef>

#include <algorithm>
#include <type_traits>
#include <vector>

#include "fr_common.cuh"

namespace fr {

static constexpr int SEL_NT = 256;
static constexpr int SEL_IT = 4;
static constexpr long long SEL_TILE = SEL_NT * SEL_IT;
static constexpr int FIN_NT = 256;
static constexpr int BLK_NT = 512;
static constexpr int BLK_CHUNK = 2048;  // uint32 column indices per stage (8 KB)
static constexpr int BLK_STAGES = 3;
static constexpr int SW_MAX_SEGS = 256;
static constexpr int SEG_PAD = 16;  // u64 per counter: one 128-byte line per segment counter

struct SolveCtl {
    double theta;       // threshold of the next sweep
    double residual;    // mass - absorbed after the last sweep
    double last_max;    // max score seen by the last select pass
    double mass0;       // exact mass at the start of the solve
    u64 diffusions, steps, sweeps;
    u64 hub_steps;      // edges pushed by the block-per-node hub kernel
    u64 trace_len;
    u32 qcount[3];
    u32 stop;
    u32 need_check;     // fused path: incremental residual crossed the target, verify exactly
    u32 is_signed;      // the starting fluid had negative entries (an incremental-update resume)
    double exact;       // sum |F| after the run (fr_solver_run)
    u64 next_refresh;   // signed fluid: re-derive the residual exactly once diffusions reach this
    u64 next_trace;     // sampled runs: record the true error once diffusions reach this
    // everything above is the header copied back after a run
    u64 seg_next[SW_MAX_SEGS * SEG_PAD];  // fused path: in-order tile counters, one 128 B line each
    // owned path in a graph (hub_defer): hub rows queued in sweep s (queue s & 1) are
    // pushed by the blocks of sweep s + 1 between their chunks, the last sweep's by a
    // drain after the loop
    u32 hub_cnt[2], hub_next[2];
};

enum { PATH_FUSED = 0, PATH_BINNED = 1, PATH_OWNED = 2 };
// the fused and owned paths share the residual bookkeeping, hub queue and graph shape
__host__ __device__ __forceinline__ bool fused_like(int path) { return path != PATH_BINNED; }

template <typename FT>
struct SweepArgs {
    FT *F;
    double *H;
    const u64 *off;
    const u32 *off32;      // narrow copy of off when m < 2^32 and n < 2^31 (fused path), else null
    const u32 *tgt;
    const double *weight;  // score multiplier (op/op2) or null
    SolveCtl *ctl;
    u32 *qnode[3];
    FT *qval[3];
    double *part_mass, *part_abs, *part_max;
    u64 *part_steps, *part_sel, *part_hsteps;
    const u32 *slot_node;  // slot -> node for the hot and warm classes (fused path)
    FT *Fw;                // compact fluid of the slotted nodes, folded into F every sweep
    u32 nhot;              // slots [0, nhot): shared-memory aggregated
    u32 nslots;            // slots [nhot, nslots): red.add into the L2-resident Fw
    fr_trace_row *trace;
    long long n, m;
    long long trace_cap;
    long long max_sweeps;
    long long max_diffusions;
    double d, thr, decay, rand_frac;
    double edge_frac;  // FR_THETA_ADAPTIVE target: pushed edges per sweep / m
    float beta;  // degree exponent: score = |f| * (out_degree + 1)^-beta (0: plain |f|)
    u32 t0, t2;  // deg <= t0 -> thread bin; deg >= t2 -> block bin
    int select, policy;
    u32 seed;
    int path;
    int segs;    // fused path: in-order segments (<= SW_MAX_SEGS)
    u32 chunk;   // fused path: tiles per reservation
    u32 own_ch;  // owned path: nodes per block-owned chunk (power of two)
    u32 own_rev;  // owned path: odd sweeps run in descending node order
    int hub_defer;  // owned path in a graph: hub rows pushed one sweep later by the sweep kernel (SolveCtl::hub_cnt)
    u32 hub_stride;  // entries per parity of the deferred hub queue (qnode[2] / qval[2])

    // sampled runs (fr_solver_run_sampled, single-block path): true L1 error of the
    // normalized history against ref every trace_every diffusions, into true_err[row]
    const double *ref;
    long long trace_every;
    double *true_err;

    int in_graph;
    cudaGraphConditionalHandle cond;
};

// (deg + 1)^-beta on the SFU (two MUFU ops, no denormal fix-ups: deg + 1 >= 1
// and the result is >= 2^-32 for beta <= 1); the score only orders nodes, so
// float precision suffices.  Every kernel uses this one function, so the
// selection is consistent between the sweep, the mass pass and the binned path.
__device__ __forceinline__ double deg_weight(float beta, unsigned long long deg) {
    float l, w;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"((float)deg + 1.0f));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(w) : "f"(-beta * l));
    return (double)w;
}

__device__ __forceinline__ u64 hmix(u64 z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static constexpr u32 HOT_FLAG = 0x80000000u;
#ifndef FR_BLK_COLD
#define FR_BLK_COLD 1
#endif

// ------------------------------------------------------------------ prologue
// Exact sum |F| and max score.  guarded: only when the fused path asked for a check.
template <typename FT>
__global__ void __launch_bounds__(SEL_NT) k_mass_partials(SweepArgs<FT> a, int guarded) {
    __shared__ double sm[SEL_NT / 32];
    if (guarded && !a.ctl->need_check) return;
    double mass = 0.0, mx = 0.0, neg = 0.0;
    if (a.hub_defer) {
        // hub rows taken by the last sweep and not pushed yet: d*f each, |q| * deg
        const u32 par = (u32)((a.ctl->sweeps + 1) & 1);
        const u32 cnt = a.ctl->hub_cnt[par];
        for (u32 q = blockIdx.x * SEL_NT + threadIdx.x; q < cnt; q += gridDim.x * SEL_NT) {
            const u32 node = a.qnode[2][par * a.hub_stride + q];
            mass += fabs((double)a.qval[2][par * a.hub_stride + q]) * (double)(a.off[node + 1] - a.off[node]);
        }
    }
    for (long long i = blockIdx.x * (long long)SEL_NT + threadIdx.x; i < a.n; i += (long long)gridDim.x * SEL_NT) {
        const double f = (double)a.F[i];
        const double af = fabs(f);
        mass += af;
        neg = fmin(neg, f);
        double score = a.weight ? af * a.weight[i] : af;
        if (a.beta != 0.0f) score = af * deg_weight(a.beta, a.off[i + 1] - a.off[i]);
        mx = fmax(mx, score);
    }
    const double bm = block_sum<SEL_NT>(mass, sm);
    const double bx = block_max<SEL_NT>(mx, sm);
    const double bn = -block_max<SEL_NT>(-neg, sm);
    if (threadIdx.x == 0) {
        a.part_mass[blockIdx.x] = bm;
        a.part_max[blockIdx.x] = bx;
        a.part_abs[blockIdx.x] = bn;  // most negative fluid (the prologue's signed test)
    }
}

template <typename FT>
__global__ void __launch_bounds__(FIN_NT) k_prologue(SweepArgs<FT> a, int nparts) {
    __shared__ double sm[FIN_NT / 32];
    double mass = 0.0, mx = 0.0, neg = 0.0;
    for (int p = threadIdx.x; p < nparts; p += FIN_NT) {
        mass += a.part_mass[p];
        mx = fmax(mx, a.part_max[p]);
        neg = fmin(neg, a.part_abs[p]);
    }
    mass = block_sum<FIN_NT>(mass, sm);
    mx = block_max<FIN_NT>(mx, sm);
    neg = -block_max<FIN_NT>(-neg, sm);
    if (threadIdx.x == 0) {
        SolveCtl *c = a.ctl;
        c->theta = mx;  // sched.py:89-90: threshold starts at the max fluid
        c->last_max = mx;
        c->residual = mass;
        c->mass0 = mass;
        c->is_signed = neg < 0.0 ? 1u : 0u;
        c->next_refresh = c->diffusions + (u64)a.n;
        c->qcount[0] = c->qcount[1] = c->qcount[2] = 0;
        for (int q = 0; q < SW_MAX_SEGS; q++) c->seg_next[q * SEG_PAD] = 0;
        c->stop = (mass <= a.thr || mass == 0.0) ? 1u : 0u;
        if (a.in_graph) cudaGraphSetConditional(a.cond, c->stop ? 0u : 1u);
    }
}

// Fused path: exact check of the stopping rule once the incremental residual
// says we are done (engine.py:290-293 re-derives the residual the same way).
template <typename FT>
__global__ void __launch_bounds__(FIN_NT) k_mass_check(SweepArgs<FT> a, int nparts) {
    __shared__ double sm[FIN_NT / 32];
    SolveCtl *c = a.ctl;
    if (!c->need_check) return;
    double mass = 0.0;
    for (int p = threadIdx.x; p < nparts; p += FIN_NT) mass += a.part_mass[p];
    mass = block_sum<FIN_NT>(mass, sm);
    if (threadIdx.x == 0) {
        c->residual = mass;
        c->need_check = 0;
        const bool done = mass <= a.thr || mass == 0.0 || c->stop;
        c->stop = done ? 1u : 0u;
        if (a.in_graph) cudaGraphSetConditional(a.cond, done ? 0u : 1u);
    }
}

// ------------------------------------------------------------------ hot targets
// Zipf in-degree hubs receive a large share of all pushes; red.global.add on
// one address serialises in its L2 slice (~0.7 G ops/s measured, tools/
// red_probe.cu), so pushes into the HOT_SLOTS highest in-degree nodes are
// summed per block in shared memory and flushed once per block.  The solver
// keeps a private copy of the column indices in which such targets carry
// HOT_FLAG | slot (slot_node[slot] = node id).
static constexpr int HOT_SLOTS = 2048;
static constexpr u32 WARM_SLOTS = 2u << 20;    // cap unit: up to 8x this many warm slots
static constexpr u32 WARM_DEFAULT = 1u << 19;  // 4 MB of fp64 fluid: best on config 5 (0.5M-16M scanned)
// Slots exist only when n <= 2^31 (prepare_slots), so a set HOT_FLAG bit can
// only mean a slot when nslots != 0; without slots every target is a node id.
template <typename FT>
__device__ __forceinline__ void push_one(FT *__restrict__ F, FT *__restrict__ Fw, FT *hot_acc, u32 nhot, u32 t,
                                         FT v, bool slotted = true) {
    if (slotted && (t & HOT_FLAG)) {
        const u32 sl = t & ~HOT_FLAG;
        if (sl < nhot) atomicAdd(hot_acc + sl, v);  // shared memory
        else red_add(Fw + sl, v);                  // compact, L2-resident
    } else {
        red_add(F + t, v);
    }
}

// push_one for a pusher far from its targets (hub rows): unslotted targets more
// than 4096 ids from the source get the L2 evict-first hint (random lines)
template <typename FT>
__device__ __forceinline__ void push_far(FT *__restrict__ F, FT *__restrict__ Fw, FT *hot_acc, u32 nhot, u32 t,
                                         FT v, bool slotted, u32 node, u64 pol) {
#if FR_BLK_COLD
    if (!(slotted && (t & HOT_FLAG)) && (t - node + 4096u) > 8192u) {
        red_add_hint(F + t, v, pol);
        return;
    }
#endif
    push_one(F, Fw, hot_acc, nhot, t, v, slotted);
}

template <typename FT>
__device__ __forceinline__ void hot_clear(FT *hot_acc, u32 nhot, int nt) {
    for (u32 s = threadIdx.x; s < nhot; s += nt) hot_acc[s] = (FT)0;
}

template <typename FT>
__device__ __forceinline__ void hot_flush(FT *__restrict__ Fw, const FT *hot_acc, u32 nhot, int nt) {
    for (u32 s = threadIdx.x; s < nhot; s += nt) {
        const FT x = hot_acc[s];
        if (x != (FT)0) red_add(Fw + s, x);
    }
}

// Moves the fluid gathered in Fw back to the slotted nodes (runs alone, after
// every push of the sweep), so F is complete when the next sweep starts.
template <typename FT>
__global__ void __launch_bounds__(256) k_fold(SweepArgs<FT> a) {
    for (u32 s = blockIdx.x * blockDim.x + threadIdx.x; s < a.nslots; s += gridDim.x * blockDim.x) {
        const FT v = a.Fw[s];
        if (v != (FT)0) {
            a.F[a.slot_node[s]] += v;
            a.Fw[s] = (FT)0;
        }
    }
}

// ------------------------------------------------------------------ fused sweep (default path)
#ifndef FR_SW_NT
#define FR_SW_NT 256
#endif
#ifndef FR_SW_UNROLL
#define FR_SW_UNROLL 2
#endif
#ifndef FR_PF_LANES
#define FR_PF_LANES 3  // 5: also the history lines (measured neutral)
#endif
#ifndef FR_SW_PF
#define FR_SW_PF 3
#endif
static constexpr int SW_NT = FR_SW_NT;
static constexpr int SW_PF = FR_SW_PF;  // L2 prefetch distance in tiles
static constexpr int SW_UNROLL = FR_SW_UNROLL;
static constexpr int DSC_TAB = 256;  // tabulated d/deg in k_sweep


__device__ __forceinline__ double take_fluid(double *p) {
    return __longlong_as_double((long long)atomicExch(reinterpret_cast<unsigned long long *>(p), 0ull));
}
__device__ __forceinline__ float take_fluid(float *p) { return atomicExch(p, 0.0f); }

__device__ __forceinline__ u32 warp_sum_u32(u32 v) { return __reduce_add_sync(0xffffffffu, v); }

// One warp per tile of 32 consecutive nodes, one sweep per launch:
//   * coalesced load of F and of the row offsets of the next tile into
//     registers (and an L2 prefetch of a tile further ahead);
//   * a selected node takes exactly the fluid value the scan loaded with a
//     fire-and-forget red.add(F_i, -f); pushes of other warps that raced
//     with the scan stay in F for the next sweep (conservation is exact,
//     PAPER Theorem 3.1 holds for any split of the fluid); H_i += f likewise;
//   * the active (non-hub) rows of the tile form one compacted edge space
//     (warp prefix scan of their degrees); each lane takes edge p of a batch,
//     finds its row by a 5-step shuffle binary search, and SW_UNROLL column
//     loads per lane are in flight (two register batches, ping-ponged) ahead
//     of the red.global.add of sent*d/deg into F (hot / warm targets to
//     shared memory / Fw);
//   * hub rows (deg >= t2) are queued for the block-per-node kernel.
#ifndef FR_SW_MINB
#define FR_SW_MINB 4
#endif

// WIDE = false: 32-bit node / tile indices and the narrow row offsets (off32)
// -- fewer registers and instructions per tile, half the offset traffic.
template <typename FT, bool WIDE>
__global__ void __launch_bounds__(SW_NT, FR_SW_MINB) k_sweep(SweepArgs<FT> a) {
    using OT = typename std::conditional<WIDE, u64, u32>::type;  // row offsets
    using IT = typename std::conditional<WIDE, long long, u32>::type;  // node / tile indices
    const OT *__restrict__ offp = WIDE ? (const OT *)a.off : (const OT *)a.off32;
    __shared__ double red_sm[SW_NT / 32];
    __shared__ u64 red_sm64[SW_NT / 32];
    __shared__ FT hot_acc[HOT_SLOTS];
    constexpr u32 FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const SolveCtl *c = a.ctl;
    const double theta = c->theta;
    const u64 sweep = c->sweeps;
    const double keep_frac = 1.0 - a.d;
    double absorbed = 0.0, mx = 0.0;
    u64 steps = 0, nsel = 0, hsteps = 0;
    const IT ntiles = (IT)((a.n + 31) >> 5);
    const IT nn = (IT)a.n;
    const u32 *__restrict__ tgt = a.tgt;
    FT *__restrict__ F = a.F;
    hot_clear(hot_acc, a.nhot, SW_NT);
    // d/deg for the common small degrees (bit-identical to the division below)
    __shared__ double dsc_sm[DSC_TAB];
    for (int q = threadIdx.x; q < DSC_TAB; q += SW_NT) dsc_sm[q] = q ? a.d / (double)q : 0.0;
    __syncthreads();
    // In-order scheduling: the tiles are split into SW_SEGS contiguous segments,
    // each with its own counter; a warp takes SW_CHUNK consecutive tiles of its
    // segment at a time and moves on to the next segment when its own is done.
    // Every segment therefore has one tight moving front, so the fluid lines
    // that neighbouring sources push into (local targets) are hit while they
    // are still in L2 instead of being refilled (tools/red_probe.cu: in-order
    // chunks reach the minimum DRAM traffic, free-running warps ~1.8x it).
    const int SW_SEGS = a.segs;
    const u32 SW_CHUNK = a.chunk;
    const IT seg_tiles = (ntiles + SW_SEGS - 1) / SW_SEGS;
    int seg = (int)((blockIdx.x * (SW_NT / 32) + (threadIdx.x >> 5)) % SW_SEGS), misses = 0;
    IT chunk_end = 0;
    // the next chunk is reserved one chunk ahead, so the counter's atomic
    // round trip overlaps the current chunk's work
    unsigned long long pend = 0;
    auto issue_grab = [&]() {
        if (lane == 0) pend = atomicAdd(&a.ctl->seg_next[seg * SEG_PAD], (unsigned long long)SW_CHUNK);
    };
    auto grab = [&](IT &t) -> bool {
        for (;;) {
            const unsigned long long k = __shfl_sync(FULL, pend, 0);
            // segments past the last tile are empty (s1 == s0; never wraps)
            const IT s0 = (IT)seg * seg_tiles < ntiles ? (IT)seg * seg_tiles : ntiles;
            const IT s1 = s0 + seg_tiles < ntiles ? s0 + seg_tiles : ntiles;
            if (k < (unsigned long long)(s1 - s0)) {
                t = s0 + (IT)k;
                chunk_end = t + SW_CHUNK < s1 ? t + SW_CHUNK : s1;
                misses = 0;
                issue_grab();
                return true;
            }
            seg = (seg + 1) % SW_SEGS;
            if (++misses >= SW_SEGS) return false;
            issue_grab();
        }
    };
    issue_grab();
    IT tile = 0;
    bool have = grab(tile);
    // software pipeline: fluid and row offsets of the next tile are in flight
    // while the current tile is processed
    FT f_cur = (FT)0;
    OT lo_cur = 0, end_cur = 0;
    auto load_tile = [&](IT t, FT &fo, OT &loo, OT &endo) {
        const IT b = t << 5, i = b + lane;
        const bool v = i < nn;
        loo = offp[v ? i : nn];
        endo = lane == 31 ? offp[b + 32 < nn ? b + 32 : nn] : (OT)0;
        fo = v ? F[i] : (FT)0;
    };
    if (have) load_tile(tile, f_cur, lo_cur, end_cur);
    while (have) {
        IT nxt = tile + 1;
        const bool have_nx = nxt < chunk_end ? true : grab(nxt);
        FT f_nx = (FT)0;
        OT lo_nx = 0, end_nx = 0;
        if (have_nx) load_tile(nxt, f_nx, lo_nx, end_nx);
        {
            // warm L2 with the fluid and offsets of a tile further ahead in the chunk
            // (no registers held), so the register prefetch above hits L2
            // lanes 0, 1: the tile's two 128 B fluid lines (fp64), lane 2: its
            // offsets, lanes 3, 4: its history lines (the history red.adds of
            // the ~half of the nodes a sweep selects would otherwise miss L2)
            const IT pf = tile + SW_PF;
            if (pf < chunk_end && lane < FR_PF_LANES) {
                const IT j = (pf << 5) + (lane & 1) * 16;
                const void *pa = lane < 2 ? (const void *)(F + j)
                                 : lane == 2 ? (const void *)(offp + j)
                                             : (const void *)(a.H + (pf << 5) + (lane - 3) * 16);
                if (j < nn) asm volatile("prefetch.global.L2 [%0];" ::"l"(pa));
            }
        }

        const IT i = (tile << 5) + lane;
        const bool valid = i < nn;
        const OT lo = lo_cur;
        OT hi = __shfl_down_sync(FULL, lo, 1);
        if (lane == 31) hi = end_cur;
        const u32 deg = (u32)(hi - lo);
        const FT f = f_cur;
        const double af = fabs((double)f);
        double score = (a.weight && valid) ? af * a.weight[i] : af;
        if (a.beta != 0.0f) score = af * deg_weight(a.beta, deg);
        mx = fmax(mx, score);
        bool sel;
        if (a.select == FR_SELECT_PER) sel = true;
        else if (a.select == FR_SELECT_RAND)
            sel = (double)(hmix(((u64)a.seed << 40) ^ (sweep << 32) ^ hmix((u64)i)) >> 11) * 0x1.0p-53 < a.rand_frac;
        else sel = score >= theta;
        sel = sel && valid && f != (FT)0;
        const bool big = deg >= a.t2;
        const bool act = sel && !big && deg > 0;
        // take exactly the fluid already loaded: a fire-and-forget subtraction
        // (fluid pushed here since the load stays in F for the next sweep), so
        // nothing below waits on a round trip (an atomicExch + H load did)
        FT sent = (FT)0;
        if (sel) {
            sent = f;
            red_add(F + i, -f);
        }
        // compacted edge space of the active rows of this tile
        const u32 adeg = act ? deg : 0u;
        u32 incl = adeg;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 t = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += t;
        }
        const u32 start = incl - adeg;
        const u32 total = __shfl_sync(FULL, incl, 31);
        // two register-resident batches (named, never indexed at run time, so
        // they stay in registers and the column loads stay in flight)
        u32 tvA[SW_UNROLL], tvB[SW_UNROLL];
        int rvA[SW_UNROLL], rvB[SW_UNROLL];
        auto issue = [&](u32 (&tv)[SW_UNROLL], int (&rv)[SW_UNROLL], u32 c0) {
#pragma unroll
            for (int u = 0; u < SW_UNROLL; u++) {
                // lanes past the end re-read the last column (same line, no
                // extra traffic): an unconditional load lands straight in its
                // register, a predicated one forced a copy that waited on it
                const u32 p0 = c0 + (u32)(u * 32 + lane);
                const u32 p = p0 < total ? p0 : total - 1;
                int r = 0;
#pragma unroll
                for (int s2 = 16; s2 > 0; s2 >>= 1) {
                    const u32 v = __shfl_sync(FULL, start, r + s2);
                    if (v <= p) r += s2;
                }
                const OT rlo = __shfl_sync(FULL, lo, r);
                const u32 rs = __shfl_sync(FULL, start, r);
                rv[u] = p0 < total ? r : -1;
                tv[u] = __ldg(tgt + rlo + (p - rs));
            }
        };
        if (total) issue(tvA, rvA, 0);
        // fluid-to-history swap in registers, push value, counters
        double pv = 0.0;
        if (sel) {
            const double as = fabs((double)sent);
            red_add(a.H + i, (double)sent);
            nsel++;
            if (deg == 0) {
                absorbed += as;  // dangling: all of it leaves (PAPER sec. 3.3)
            } else {
                absorbed += as * keep_frac;
                steps += deg;
                pv = (double)sent * (deg < DSC_TAB ? dsc_sm[deg] : a.d / (double)deg);  // sent*(d/deg), engine.py:321
            }
        }
        const FT pvf = (FT)pv;
        // hubs -> block-per-node kernel
        const bool hub = sel && big;
        const u32 hmask = __ballot_sync(FULL, hub);
        if (hmask) {
            u32 hb = 0;
            const int leader = __ffs(hmask) - 1;
            if (lane == leader) hb = atomicAdd(&a.ctl->qcount[2], (u32)__popc(hmask));
            hb = __shfl_sync(FULL, hb, leader);
            if (hub) {
                const u32 q = hb + __popc(hmask & ((1u << lane) - 1u));
                a.qnode[2][q] = (u32)i;
                a.qval[2][q] = pvf;
                hsteps += deg;
            }
        }
        // scatter, one batch of 32*SW_UNROLL edges in flight ahead of the reds
        auto scatter = [&](const u32 (&tv)[SW_UNROLL], const int (&rv)[SW_UNROLL]) {
#pragma unroll
            for (int u = 0; u < SW_UNROLL; u++) {
                const int r = rv[u];
                const FT v = __shfl_sync(FULL, pvf, r < 0 ? 0 : r);
                if (r >= 0) push_one(F, a.Fw, hot_acc, a.nhot, tv[u], v, a.nslots != 0);
            }
        };
        constexpr u32 STEP = 32 * SW_UNROLL;
        for (u32 c0 = 0; c0 < total; c0 += 2 * STEP) {
            // batch A (in flight) is scattered while batch B loads, then the roles swap
            if (c0 + STEP < total) issue(tvB, rvB, c0 + STEP);
            scatter(tvA, rvA);
            if (c0 + STEP >= total) break;
            if (c0 + 2 * STEP < total) issue(tvA, rvA, c0 + 2 * STEP);
            scatter(tvB, rvB);
        }
        f_cur = f_nx;
        lo_cur = lo_nx;
        end_cur = end_nx;
        tile = nxt;
        have = have_nx;
    }
    __syncthreads();
    hot_flush(a.Fw, hot_acc, a.nhot, SW_NT);
    const double ba = block_sum<SW_NT>(absorbed, red_sm);
    const double bx = block_max<SW_NT>(mx, red_sm);
    const u64 bs = block_sum_u64<SW_NT>(steps, red_sm64);
    const u64 bn = block_sum_u64<SW_NT>(nsel, red_sm64);
    const u64 bh = block_sum_u64<SW_NT>(hsteps, red_sm64);
    if (threadIdx.x == 0) {
        a.part_hsteps[blockIdx.x] = bh;
        a.part_abs[blockIdx.x] = ba;
        a.part_max[blockIdx.x] = bx;
        a.part_steps[blockIdx.x] = bs;
        a.part_sel[blockIdx.x] = bn;
        a.part_mass[blockIdx.x] = 0.0;
    }
}

// ------------------------------------------------------------------ owned-chunk sweep (kernel_path = 2)
// Block per chunk of own_ch consecutive nodes (2048 with 128 threads: fewer
// nodes in flight per chunk make the Gauss-Seidel below stronger), chunks
// taken in order from one counter.  70% of the generator's edges land within
// +-1000 ids of their source, so most pushes of a chunk stay inside it: those are summed in a
// shared-memory copy of the chunk's fluid (acc) instead of red.global.add in
// L2, and a node reached by such pushes before its own tile is scanned
// diffuses them in the same sweep (Gauss-Seidel within the chunk; PAPER
// Theorem 3.1 allows any order).  A selected node's take leaves -F_i in acc, so
// at the end of the chunk one coalesced red.add per non-zero node both removes
// the taken fluid from F and adds what was pushed there afterwards.  Pushes that
// leave the chunk, and the slotted hot/warm targets, are handled as in k_sweep.
#ifndef FR_OWN_NT
#define FR_OWN_NT 128
#endif
#ifndef FR_OWN_MINB
#define FR_OWN_MINB 9  // 9 blocks x 4 warps per SM: <= 56 registers (the 64-bit-index variant keeps 8)
#endif
#ifndef FR_OWN_PF
#define FR_OWN_PF 2  // L2 prefetch distance in warp rounds
#endif
#ifndef FR_OWN_PF_LANES
#define FR_OWN_PF_LANES 3  // lanes 0, 1: fluid lines, 2: offsets, 3, 4: history lines
#endif
#ifndef FR_OWN_UNROLL
#define FR_OWN_UNROLL 3  // column loads in flight per lane and batch (k_sweep: FR_SW_UNROLL)
#endif
#ifndef FR_COLD_HINT
#define FR_COLD_HINT 1
#endif
#ifndef FR_OWN_SKIPSCAN
#define FR_OWN_SKIPSCAN 0
#endif
#ifndef FR_OWN_BULKPF
#define FR_OWN_BULKPF 1  // one bulk L2 prefetch of the chunk's fluid and offsets (0: per-tile prefetches)
#endif

#ifndef FR_OWN_RSEARCH
#define FR_OWN_RSEARCH 1  // row of an edge position from a REDUX/VOTE head mask over lane-compacted rows (0: 5-step shuffle search)
#endif

#ifndef FR_OWN_UNISCAT
#define FR_OWN_UNISCAT 3  // scatter: one shared-memory add (chunk + hot tables), one global red.add (warm + near); 3: the global adds predicated
#endif

#ifndef FR_OWN_TAKEACC
#define FR_OWN_TAKEACC 1  // the take leaves -f in acc (one exchange); the chunk flush subtracts it from F
#endif

static constexpr int OWN_NT = FR_OWN_NT;
static constexpr int OWN_UNROLL = FR_OWN_UNROLL;
static_assert(OWN_UNROLL * 6 <= 32, "packed row indices");
static constexpr int OWN_NW = OWN_NT / 32;

__device__ __forceinline__ double take_shared(double *p) {
    return __longlong_as_double((long long)atomicExch(reinterpret_cast<unsigned long long *>(p), 0ull));
}
__device__ __forceinline__ float take_shared(float *p) { return atomicExch(p, 0.0f); }
// exchange: returns what was pending and leaves x
__device__ __forceinline__ double swap_shared(double *p, double x) {
    return __longlong_as_double((long long)atomicExch(reinterpret_cast<unsigned long long *>(p),
                                                      (unsigned long long)__double_as_longlong(x)));
}
__device__ __forceinline__ float swap_shared(float *p, float x) { return atomicExch(p, x); }

// Deferred hub rows (hub_defer): the whole block claims one row queued by the
// previous sweep and pushes it (128 threads over its columns, as k_push_block;
// hot targets into the block's table).  Returns false when none is left.
template <typename FT>
__device__ bool own_hub_row(const SweepArgs<FT> &a, FT *hot_acc, u64 sweep) {
    __shared__ u32 hub_sm;
    const u32 par = (u32)((sweep + 1) & 1);  // the queue of sweep - 1
    SolveCtl *c = a.ctl;
    if (threadIdx.x == 0) {
        const u32 cnt = c->hub_cnt[par];
        u32 k = ~0u;
        if (c->hub_next[par] < cnt) {
            k = atomicAdd(&c->hub_next[par], 1u);
            if (k >= cnt) k = ~0u;
        }
        hub_sm = k;
    }
    __syncthreads();
    const u32 k = hub_sm;
    __syncthreads();  // hub_sm is read by every thread before the next call writes it
    if (k == ~0u) return false;
    const u32 q = k + par * a.hub_stride;
    const u32 node = a.qnode[2][q];
    const FT v = a.qval[2][q];
    const u64 lo = a.off[node], hi = a.off[node + 1];
    const u64 pol = FR_BLK_COLD ? policy_evict_first() : 0ull;
    const bool slotted = a.nslots != 0;
#pragma unroll 4
    for (u64 e = lo + threadIdx.x; e < hi; e += OWN_NT)
        push_far(a.F, a.Fw, hot_acc, a.nhot, __ldg(a.tgt + e), v, slotted, node, pol);
    return true;
}

template <typename FT, bool WIDE>
__global__ void __launch_bounds__(OWN_NT, WIDE ? 8 : FR_OWN_MINB) k_sweep_own(SweepArgs<FT> a) {
    using OT = typename std::conditional<WIDE, u64, u32>::type;
    using IT = typename std::conditional<WIDE, long long, u32>::type;
    const OT *__restrict__ offp = WIDE ? (const OT *)a.off : (const OT *)a.off32;
    extern __shared__ __align__(16) unsigned char own_smem[];
    FT *acc = reinterpret_cast<FT *>(own_smem);  // [own_ch]: the chunk's incoming fluid
    FT *hot_acc = acc + a.own_ch;                // [nhot]
    __shared__ double red_sm[OWN_NT / 32];
    __shared__ u64 red_sm64[OWN_NT / 32];
    __shared__ double dsc_sm[DSC_TAB];
    __shared__ u64 chunk_sm[2];
    __shared__ u32 tile_ctr[2];  // next unclaimed tile of the chunk (double-buffered by chunk parity)
    constexpr u32 FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const SolveCtl *c = a.ctl;
    const double theta = c->theta;
    const u64 sweep = c->sweeps;
    const double keep_frac = 1.0 - a.d;
    double absorbed = 0.0, mx = 0.0;
    // per-thread counters: 32-bit on the narrow path (a thread sees < 2^32 edges per sweep there)
    using CT = typename std::conditional<WIDE, u64, u32>::type;
    CT steps = 0, nsel = 0, hsteps = 0;
    const bool slotted = a.nslots != 0;
    const u32 CH = a.own_ch;
    const IT nn = (IT)a.n;
    const u32 *__restrict__ tgt = a.tgt;
    FT *__restrict__ F = a.F;
#if FR_COLD_HINT
    const u64 cold_pol = policy_evict_first();
#endif
    u32 lemask = (2u << lane) - 1u;  // lanes at or below this one
#if FR_OWN_UNISCAT > 3
    asm volatile("mov.u32 %0, %0;" : "+r"(lemask));  // kept in a register
#endif
#if FR_OWN_UNISCAT
    u32 sbase = (u32)__cvta_generic_to_shared(acc);
    asm volatile("mov.u32 %0, %0;" : "+r"(sbase));  // kept in a register (else re-derived at every add)
    u32 fmask = a.nslots != 0 ? HOT_FLAG : 0u;
    u32 hot_end = a.own_ch + a.nhot;
#if FR_OWN_UNISCAT > 1
    asm volatile("mov.u32 %0, %0;" : "+r"(fmask));
    asm volatile("mov.u32 %0, %0;" : "+r"(hot_end));
#endif
#endif
    for (u32 q = threadIdx.x; q < CH; q += OWN_NT) acc[q] = (FT)0;
    hot_clear(hot_acc, a.nhot, OWN_NT);
    for (int q = threadIdx.x; q < DSC_TAB; q += OWN_NT) dsc_sm[q] = q ? a.d / (double)q : 0.0;
    const u64 nchunks = ((u64)a.n + CH - 1) / CH;
    const bool rev = (sweep & 1) && a.own_rev;
    for (u32 it = 0;; it++) {
        if (threadIdx.x == 0) {
            chunk_sm[it & 1] = atomicAdd(&a.ctl->seg_next[0], 1ull);
            tile_ctr[it & 1] = OWN_NW;  // warp w starts on tile w, then claims tiles in order
        }
        __syncthreads();  // chunk id visible; the previous chunk's flush is complete
        const u64 ch0 = chunk_sm[it & 1];
        if (ch0 >= nchunks) break;
        // odd sweeps run backwards (chunks and the tiles inside them): a node then
        // sees this sweep's pushes from the nodes behind it in the id order as well
        // as, the sweep before, those ahead of it (symmetric Gauss-Seidel)
        const u64 ch = rev ? nchunks - 1 - ch0 : ch0;
        const IT base = (IT)(ch * CH);
        const u32 len = (u32)((u64)a.n - (u64)base < CH ? (u64)a.n - (u64)base : CH);
        const u32 ntl = (len + 31) >> 5;
        auto tmap = [&](u32 lt) -> u32 { return rev ? ntl - 1 - lt : lt; };
#if FR_OWN_BULKPF
        if (threadIdx.x == 0) {
            // the chunk's fluid and row offsets into L2 by two bulk prefetches (16 B granules)
            const u32 fb = (len * (u32)sizeof(FT) + 15u) & ~15u;
            const u32 ob = ((len + 1) * (u32)sizeof(OT) + 15u) & ~15u;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(F + base), "r"(fb) : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(offp + base), "r"(ob) : "memory");
        }
#endif
        FT f_cur = (FT)0;
        OT lo_cur = 0, end_cur = 0;
        auto load_tile = [&](u32 lt, FT &fo, OT &loo, OT &endo) {
            const IT b = base + (IT)(tmap(lt) << 5), i = b + lane;
            const bool v = i < nn;
            loo = offp[v ? i : nn];
            endo = lane == 31 ? offp[b + 32 < nn ? b + 32 : nn] : (OT)0;
            fo = v ? F[i] : (FT)0;
        };
        // tiles are claimed one at a time (the tiles of a chunk differ widely in
        // edge work), so the warps reach the flush barrier together
        u32 *ctr = &tile_ctr[it & 1];
        u32 lt = warp;
        if (lt < ntl) load_tile(lt, f_cur, lo_cur, end_cur);
        while (lt < ntl) {
            u32 lnx = 0;
            if (lane == 0) lnx = atomicAdd(ctr, 1u);
            lnx = __shfl_sync(FULL, lnx, 0);
            FT f_nx = (FT)0;
            OT lo_nx = 0, end_nx = 0;
            if (lnx < ntl) load_tile(lnx, f_nx, lo_nx, end_nx);
            if (!FR_OWN_BULKPF) {
                const u32 pf = lnx + FR_OWN_PF * OWN_NW;
                if (pf < ntl && lane < FR_OWN_PF_LANES) {
                    const IT j = base + (IT)(tmap(pf) << 5) + (lane & 1) * 16;
                    const void *pa = lane < 2 ? (const void *)(F + j)
                                     : lane == 2 ? (const void *)(offp + j)
                                                 : (const void *)(a.H + j);
                    if (j < nn) asm volatile("prefetch.global.L2 [%0];" ::"l"(pa));
                }
            }
            const u32 li = (tmap(lt) << 5) + lane;
            const IT i = base + (IT)li;
            const bool valid = li < len;
            const OT lo = lo_cur;
            OT hi = __shfl_down_sync(FULL, lo, 1);
            if (lane == 31) hi = end_cur;
            const u32 deg = (u32)(hi - lo);
            const FT fg = f_cur;
            const FT pend = valid ? acc[li] : (FT)0;  // pushed here earlier in this chunk
            const FT f = fg + pend;
            const double af = fabs((double)f);
            double score = (a.weight && valid) ? af * a.weight[i] : af;
            if (a.beta != 0.0f) score = af * deg_weight(a.beta, deg);
            mx = fmax(mx, score);
            bool sel;
            if (a.select == FR_SELECT_PER) sel = true;
            else if (a.select == FR_SELECT_RAND)
                sel = (double)(hmix(((u64)a.seed << 40) ^ (sweep << 32) ^ hmix((u64)i)) >> 11) * 0x1.0p-53 < a.rand_frac;
            else sel = score >= theta;
            sel = sel && valid && f != (FT)0;
            const bool big = deg >= a.t2;
            const bool act = sel && !big && deg > 0;
            // take: one shared-memory exchange returns what was pushed here earlier in
            // this chunk and leaves -fg in its place (other warps of the block keep
            // adding to it); the chunk flush then subtracts the taken global fluid
            // from F together with the later pushes in its one red.add per node, so
            // the take costs no global operation of its own.  F_i keeps fg until the
            // flush: only this block reads the chunk's F during the sweep.
            FT sent = (FT)0;
            if (sel) {
#if FR_OWN_TAKEACC
                const FT ps = swap_shared(acc + li, -fg);
#else
                const FT ps = pend != (FT)0 ? take_shared(acc + li) : (FT)0;
                if (fg != (FT)0) red_add(F + i, -fg);
#endif
                sent = fg + ps;
            }
            const u32 adeg = act ? deg : 0u;
            u32 incl = adeg;
#if FR_OWN_SKIPSCAN
            // a tile with nothing to push skips the scan (sparse sweeps)
            const u32 total = __reduce_add_sync(FULL, adeg);
            if (total)
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const u32 t = __shfl_up_sync(FULL, incl, o);
                    if (lane >= o) incl += t;
                }
            const u32 start = incl - adeg;
#else
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u32 t = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += t;
            }
            const u32 start = incl - adeg;
            const u32 total = __shfl_sync(FULL, incl, 31);
#endif
            // column batches: the targets in registers, each lane's row (r + 1, 0 = past
            // the end) packed 6 bits per batch slot into one register
            u32 tvA[OWN_UNROLL], tvB[OWN_UNROLL], tvC[OWN_UNROLL];
            u32 rvA = 0, rvB = 0, rvC = 0;
#if FR_OWN_RSEARCH
            // The active rows are compacted into the low lanes (lane k holds the k-th
            // active row: its start in the edge space and lo - start, the base its
            // columns are addressed from), so their starts are strictly increasing and
            // the row of the 32 positions of a window follows from one REDUX.OR of the
            // row heads inside the window, one VOTE for the rows at or before it and a
            // POPC per lane -- no shuffles (they share the L1 data pipe with the
            // shared-memory atomics, the busiest unit of this kernel).
            const u32 amask = __ballot_sync(FULL, act);
            const u32 na = (u32)__popc(amask);
            int csrc = 0;  // lane of the (lane + 1)-th active row: the largest x with popc(amask below x) <= lane
#pragma unroll
            for (int s2 = 16; s2 > 0; s2 >>= 1) {
                const int x = csrc + s2;
                if ((u32)__popc(amask & ((1u << x) - 1u)) <= (u32)lane) csrc = x;
            }
            const u32 cst0 = __shfl_sync(FULL, start, csrc);
            const u32 cstart = (u32)lane < na ? cst0 : 0xffffffffu;
            const OT cbase = __shfl_sync(FULL, (OT)(lo - (OT)start), csrc);
            auto issue = [&](u32 (&tv)[OWN_UNROLL], u32 &rv, u32 c0) {
                rv = 0;
#pragma unroll
                for (int u = 0; u < OWN_UNROLL; u++) {
                    const u32 w0 = c0 + (u32)(u * 32);
                    const u32 t = cstart - w0;  // 1..31: this row's head lies inside the window
                    const u32 heads = __reduce_or_sync(FULL, (t - 1u < 31u) ? (1u << t) : 0u);
                    const u32 nb = (u32)__popc(__ballot_sync(FULL, cstart <= w0));  // >= 1: the first row starts at 0
                    const u32 p0 = w0 + (u32)lane;
                    const bool in = p0 < total;
                    const u32 p = in ? p0 : total - 1;
                    const u32 r = in ? nb + (u32)__popc(heads & lemask) - 1u : na - 1u;
                    const OT cb = __shfl_sync(FULL, cbase, (int)r);
                    rv |= (in ? r + 1u : 0u) << (6 * u);
                    tv[u] = __ldg(tgt + (cb + (OT)p));
                }
            };
#else
            auto issue = [&](u32 (&tv)[OWN_UNROLL], u32 &rv, u32 c0) {
                rv = 0;
#pragma unroll
                for (int u = 0; u < OWN_UNROLL; u++) {
                    const u32 p0 = c0 + (u32)(u * 32 + lane);
                    const u32 p = p0 < total ? p0 : total - 1;
                    int r = 0;
#pragma unroll
                    for (int s2 = 16; s2 > 0; s2 >>= 1) {
                        const u32 v = __shfl_sync(FULL, start, r + s2);
                        if (v <= p) r += s2;
                    }
                    const OT rlo = __shfl_sync(FULL, lo, r);
                    const u32 rs = __shfl_sync(FULL, start, r);
                    rv |= (p0 < total ? (u32)(r + 1) : 0u) << (6 * u);
                    tv[u] = __ldg(tgt + rlo + (p - rs));
                }
            };
#endif
            constexpr u32 STEP = 32 * OWN_UNROLL;
            // two batches in flight before the first scatter
            if (total) issue(tvA, rvA, 0);
            if (total > STEP) issue(tvB, rvB, STEP);
            double pv = 0.0;
            if (sel) {
                const double as = fabs((double)sent);
                red_add(a.H + i, (double)sent);
                nsel++;
                if (deg == 0) {
                    absorbed += as;  // dangling: all of it leaves (PAPER sec. 3.3)
                } else {
                    absorbed += as * keep_frac;
                    steps += deg;
                    pv = (double)sent * (deg < DSC_TAB ? dsc_sm[deg] : a.d / (double)deg);  // engine.py:321
                }
            }
            const FT pvf = (FT)pv;
#if FR_OWN_RSEARCH
            const FT spv = __shfl_sync(FULL, pvf, csrc);  // push value of the lane's compacted row
#else
            const FT spv = pvf;
#endif
            const bool hub = sel && big;
            const u32 hmask = __ballot_sync(FULL, hub);
            if (hmask) {
                u32 hb = 0;
                const int leader = __ffs(hmask) - 1;
                if (lane == leader) hb = atomicAdd(a.hub_defer ? &a.ctl->hub_cnt[sweep & 1] : &a.ctl->qcount[2],
                                                   (u32)__popc(hmask));
                hb = __shfl_sync(FULL, hb, leader);
                if (hub) {
                    const u32 q = hb + __popc(hmask & ((1u << lane) - 1u)) +
                                  (a.hub_defer ? (u32)(sweep & 1) * a.hub_stride : 0u);
                    a.qnode[2][q] = (u32)i;
                    a.qval[2][q] = pvf;
                    hsteps += deg;
                }
            }
            const u32 ubase = (u32)base;
            auto scatter = [&](const u32 (&tv)[OWN_UNROLL], const u32 rv) {
#pragma unroll
                for (int u = 0; u < OWN_UNROLL; u++) {
                    const int r = (int)((rv >> (6 * u)) & 63u) - 1;
                    const FT v = __shfl_sync(FULL, spv, r < 0 ? 0 : r);
                    if (r >= 0) {
                        const u32 t = tv[u];
                        const u32 lt2 = t - ubase;
#if FR_OWN_UNISCAT
                        // two destinations in shared memory (the chunk table, the hot table right
                        // behind it) share one add; the warm and the near unslotted global targets
                        // share one red.add; the cold ones keep their own (uniform policy operand)
                        const u32 tf = t & fmask;  // != 0: a slotted target
                        const u32 sl = t ^ tf;     // its slot, or the node id itself
                        const u32 idx = tf ? CH + sl : lt2;
#if FR_OWN_UNISCAT > 2 && FR_COLD_HINT
                        // the global adds predicated (no branch around them), then the shared-memory lanes
                        const bool sh = idx < (tf ? hot_end : len);
                        const bool cold = !tf && (lt2 + 4096u) > CH + 8192u;
                        red_add_pred2((tf ? a.Fw : F) + sl, v, cold_pol, !sh && !cold, !sh && cold);
                        if (sh) shared_red_add(sbase + idx * (u32)sizeof(FT), v);
                        continue;
#endif
                        if (idx < (tf ? hot_end : len)) shared_red_add(sbase + idx * (u32)sizeof(FT), v);
#if FR_COLD_HINT
                        else if (!tf && (lt2 + 4096u) > CH + 8192u) red_add_hint(F + t, v, cold_pol);
#endif
                        else red_add((tf ? a.Fw : F) + sl, v);
                        continue;
#endif
                        if (!(slotted && (t & HOT_FLAG)) && lt2 < len) atomicAdd(acc + lt2, v);  // inside the chunk
#if FR_COLD_HINT
                        else if (!(slotted && (t & HOT_FLAG)) && (t - ubase + 4096u) > CH + 8192u)
                            red_add_hint(F + t, v, cold_pol);  // far, unslotted: do not displace the front
#endif
                        else push_one(F, a.Fw, hot_acc, a.nhot, t, v, slotted);
                    }
                }
            };
            // three rotating batches (named, so they stay in registers): two are in
            // flight while the third is scattered
            for (u32 c0 = 0; c0 < total; c0 += 3 * STEP) {
                if (c0 + 2 * STEP < total) issue(tvC, rvC, c0 + 2 * STEP);
                scatter(tvA, rvA);
                if (c0 + STEP >= total) break;
                if (c0 + 3 * STEP < total) issue(tvA, rvA, c0 + 3 * STEP);
                scatter(tvB, rvB);
                if (c0 + 2 * STEP >= total) break;
                if (c0 + 4 * STEP < total) issue(tvB, rvB, c0 + 4 * STEP);
                scatter(tvC, rvC);
            }
            f_cur = f_nx;
            lo_cur = lo_nx;
            end_cur = end_nx;
            lt = lnx;
        }
        __syncthreads();  // every push into acc of this chunk is done
        for (u32 q = threadIdx.x; q < len; q += OWN_NT) {
            const FT x = acc[q];
            if (x != (FT)0) {
                red_add(F + base + q, x);
                acc[q] = (FT)0;
            }
        }
        if (a.hub_defer) own_hub_row(a, hot_acc, sweep);  // one hub row of the previous sweep per chunk
    }
    if (a.hub_defer)
        while (own_hub_row(a, hot_acc, sweep)) {
        }
    hot_flush(a.Fw, hot_acc, a.nhot, OWN_NT);
    const double ba = block_sum<OWN_NT>(absorbed, red_sm);
    const double bx = block_max<OWN_NT>(mx, red_sm);
    const u64 bs = block_sum_u64<OWN_NT>((u64)steps, red_sm64);
    const u64 bn = block_sum_u64<OWN_NT>((u64)nsel, red_sm64);
    const u64 bh = block_sum_u64<OWN_NT>((u64)hsteps, red_sm64);
    if (threadIdx.x == 0) {
        a.part_hsteps[blockIdx.x] = bh;
        a.part_abs[blockIdx.x] = ba;
        a.part_max[blockIdx.x] = bx;
        a.part_steps[blockIdx.x] = bs;
        a.part_sel[blockIdx.x] = bn;
        a.part_mass[blockIdx.x] = 0.0;
    }
}

// ------------------------------------------------------------------ S: select + take + enqueue
template <typename FT>
__global__ void __launch_bounds__(SEL_NT) k_select(SweepArgs<FT> a) {
    __shared__ u64 scan_sm[SEL_NT / 32 + 1];
    __shared__ u64 qbase[3];
    __shared__ double red_sm[SEL_NT / 32];
    __shared__ u64 red_sm64[SEL_NT / 32];
    const SolveCtl *c = a.ctl;
    const double theta = c->theta;
    const u64 sweep = c->sweeps;
    const double keep_frac = 1.0 - a.d;
    double mass = 0.0, absorbed = 0.0, mx = 0.0;
    u64 steps = 0, nsel = 0;
    const long long ntiles = (a.n + SEL_TILE - 1) / SEL_TILE;
    constexpr u64 M21 = (1ull << 21) - 1;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        u32 e_node[SEL_IT];
        FT e_val[SEL_IT];
        int e_bin[SEL_IT];
        u64 packed = 0;
#pragma unroll
        for (int it = 0; it < SEL_IT; it++) {
            const long long i = tile * SEL_TILE + it * SEL_NT + threadIdx.x;
            e_bin[it] = -1;
            if (i < a.n) {
                const FT f = a.F[i];
                const double af = fabs((double)f);
                mass += af;
                double score = a.weight ? af * a.weight[i] : af;
                if (a.beta != 0.0f) score = af * deg_weight(a.beta, a.off[i + 1] - a.off[i]);
                mx = fmax(mx, score);
                bool sel;
                if (a.select == FR_SELECT_PER) sel = true;
                else if (a.select == FR_SELECT_RAND)
                    sel = (double)(hmix(((u64)a.seed << 40) ^ (sweep << 32) ^ hmix((u64)i)) >> 11) * 0x1.0p-53 < a.rand_frac;
                else sel = score >= theta;
                if (sel && f != (FT)0) {
                    const u64 lo = a.off[i], hi = a.off[i + 1];
                    const u64 deg = hi - lo;
                    a.F[i] = (FT)0;
                    a.H[i] += (double)f;
                    nsel++;
                    if (deg == 0) {
                        absorbed += af;  // dangling: all of it leaves (PAPER sec. 3.3)
                    } else {
                        absorbed += af * keep_frac;
                        steps += deg;
                        const int bin = deg <= a.t0 ? 0 : (deg < a.t2 ? 1 : 2);
                        e_bin[it] = bin;
                        e_node[it] = (u32)i;
                        e_val[it] = (FT)((double)f * (a.d / (double)deg));  // sent*(d/deg), engine.py:321
                        packed += 1ull << (21 * bin);
                    }
                }
            }
        }
        u64 tot;
        const u64 excl = block_excl_scan<SEL_NT>(packed, scan_sm, &tot);
        if (threadIdx.x < 3) {
            const u32 cnt = (u32)((tot >> (21 * threadIdx.x)) & M21);
            qbase[threadIdx.x] = cnt ? atomicAdd(&a.ctl->qcount[threadIdx.x], cnt) : 0u;
        }
        __syncthreads();
        if (packed) {
            u64 pos[3] = {qbase[0] + (excl & M21), qbase[1] + ((excl >> 21) & M21), qbase[2] + ((excl >> 42) & M21)};
#pragma unroll
            for (int it = 0; it < SEL_IT; it++) {
                const int b = e_bin[it];
                if (b >= 0) {
                    const u64 p = pos[b]++;
                    a.qnode[b][p] = e_node[it];
                    a.qval[b][p] = e_val[it];
                }
            }
        }
        __syncthreads();
    }
    const double bm = block_sum<SEL_NT>(mass, red_sm);
    const double ba = block_sum<SEL_NT>(absorbed, red_sm);
    const double bx = block_max<SEL_NT>(mx, red_sm);
    const u64 bs = block_sum_u64<SEL_NT>(steps, red_sm64);
    const u64 bn = block_sum_u64<SEL_NT>(nsel, red_sm64);
    if (threadIdx.x == 0) {
        a.part_mass[blockIdx.x] = bm;
        a.part_abs[blockIdx.x] = ba;
        a.part_max[blockIdx.x] = bx;
        a.part_steps[blockIdx.x] = bs;
        a.part_sel[blockIdx.x] = bn;
    }
}

// ------------------------------------------------------------------ P: push kernels
template <typename FT>
__global__ void __launch_bounds__(256) k_push_thread(SweepArgs<FT> a) {
    __shared__ FT hot_acc[HOT_SLOTS];
    const u32 cnt = a.ctl->qcount[0];
    const u32 *__restrict__ qn = a.qnode[0];
    const FT *__restrict__ qv = a.qval[0];
    hot_clear(hot_acc, a.nhot, 256);
    __syncthreads();
    for (u32 e = blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += gridDim.x * blockDim.x) {
        const u32 node = qn[e];
        const FT v = qv[e];
        const u64 lo = a.off[node], hi = a.off[node + 1];
        for (u64 k = lo; k < hi; k++) push_one(a.F, a.Fw, hot_acc, a.nhot, __ldg(a.tgt + k), v, a.nslots != 0);
    }
    __syncthreads();
    hot_flush(a.Fw, hot_acc, a.nhot, 256);
}

template <typename FT>
__global__ void __launch_bounds__(256) k_push_warp(SweepArgs<FT> a) {
    __shared__ FT hot_acc[HOT_SLOTS];
    const u32 cnt = a.ctl->qcount[1];
    const int lane = threadIdx.x & 31;
    hot_clear(hot_acc, a.nhot, 256);
    __syncthreads();
    const u32 nwarps = gridDim.x * (blockDim.x >> 5);
    const uint4 *tgt4 = reinterpret_cast<const uint4 *>(a.tgt);
    for (u32 e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); e < cnt; e += nwarps) {
        const u32 node = a.qnode[1][e];
        const FT v = a.qval[1][e];
        const u64 lo = a.off[node], hi = a.off[node + 1];
        const u64 a0 = min(hi, (lo + 3) & ~3ull);
        const u64 a1 = max(a0, hi & ~3ull);
        if (lo + lane < a0) push_one(a.F, a.Fw, hot_acc, a.nhot, __ldg(a.tgt + lo + lane), v, a.nslots != 0);
        if (a1 + lane < hi) push_one(a.F, a.Fw, hot_acc, a.nhot, __ldg(a.tgt + a1 + lane), v, a.nslots != 0);
        for (u64 q = (a0 >> 2) + lane; q < (a1 >> 2); q += 32) {
            const uint4 t = ld_stream_u4(tgt4 + q);
            push_one(a.F, a.Fw, hot_acc, a.nhot, t.x, v, a.nslots != 0);
            push_one(a.F, a.Fw, hot_acc, a.nhot, t.y, v, a.nslots != 0);
            push_one(a.F, a.Fw, hot_acc, a.nhot, t.z, v, a.nslots != 0);
            push_one(a.F, a.Fw, hot_acc, a.nhot, t.w, v, a.nslots != 0);
        }
    }
    __syncthreads();
    hot_flush(a.Fw, hot_acc, a.nhot, 256);
}

// Block per hub node.  The 16-byte-aligned body of the adjacency row streams
// through a BLK_STAGES-deep ring of shared-memory chunks filled by the bulk
// copy engine (cp.async.bulk -> UBLKCP), so column-index loads overlap the
// red.global.add scatter of the previous chunks.
template <typename FT>
__global__ void __launch_bounds__(BLK_NT) k_push_block(SweepArgs<FT> a) {
    __shared__ __align__(128) u32 stage[BLK_STAGES][BLK_CHUNK];
    __shared__ __align__(8) u64 bar[BLK_STAGES];
    __shared__ FT hot_acc[HOT_SLOTS];
    // hub_defer: the drain after the loop, over the rows the last sweep queued
    const u32 par = (u32)((a.ctl->sweeps + 1) & 1);
    const u32 cnt = a.hub_defer ? a.ctl->hub_cnt[par] : a.ctl->qcount[2];
    const u32 qoff = a.hub_defer ? par * a.hub_stride : 0u;
    if (blockIdx.x >= cnt) return;
    const u64 pol = FR_BLK_COLD ? policy_evict_first() : 0ull;
    if (threadIdx.x == 0) {
        for (int s = 0; s < BLK_STAGES; s++) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    hot_clear(hot_acc, a.nhot, BLK_NT);
    __syncthreads();
    u32 seq = 0;  // chunks consumed by this block so far (slot = seq % STAGES, parity = (seq / STAGES) & 1)
    for (u32 e = blockIdx.x; e < cnt; e += gridDim.x) {
        const u32 node = a.qnode[2][qoff + e];
        const FT v = a.qval[2][qoff + e];
        const u64 lo = a.off[node], hi = a.off[node + 1];
        const u64 a0 = min(hi, (lo + 3) & ~3ull);
        const u64 a1 = max(a0, hi & ~3ull);
        if (lo + threadIdx.x < a0)
            push_far(a.F, a.Fw, hot_acc, a.nhot, __ldg(a.tgt + lo + threadIdx.x), v, a.nslots != 0, node, pol);
        if (a1 + threadIdx.x < hi)
            push_far(a.F, a.Fw, hot_acc, a.nhot, __ldg(a.tgt + a1 + threadIdx.x), v, a.nslots != 0, node, pol);
        const u64 body = a1 - a0;
        const u32 nch = (u32)((body + BLK_CHUNK - 1) / BLK_CHUNK);
        if (threadIdx.x == 0) {
            for (u32 c = 0; c < nch && c < BLK_STAGES - 1; c++) {
                const u32 s = (seq + c) % BLK_STAGES;
                const u32 len = (u32)min((u64)BLK_CHUNK, body - (u64)c * BLK_CHUNK);
                mbar_expect_tx(&bar[s], len * 4);
                bulk_load(stage[s], a.tgt + a0 + (u64)c * BLK_CHUNK, len * 4, &bar[s]);
            }
        }
        for (u32 c = 0; c < nch; c++) {
            if (threadIdx.x == 0 && c + BLK_STAGES - 1 < nch) {
                const u32 cc = c + BLK_STAGES - 1;
                const u32 s = (seq + cc) % BLK_STAGES;
                const u32 len = (u32)min((u64)BLK_CHUNK, body - (u64)cc * BLK_CHUNK);
                mbar_expect_tx(&bar[s], len * 4);
                bulk_load(stage[s], a.tgt + a0 + (u64)cc * BLK_CHUNK, len * 4, &bar[s]);
            }
            const u32 s = (seq + c) % BLK_STAGES;
            mbar_wait(&bar[s], ((seq + c) / BLK_STAGES) & 1u);
            const u32 len = (u32)min((u64)BLK_CHUNK, body - (u64)c * BLK_CHUNK);
            const u32 *sp = stage[s];
#pragma unroll 4
            for (u32 k = threadIdx.x; k < len; k += BLK_NT)
                push_far(a.F, a.Fw, hot_acc, a.nhot, sp[k], v, a.nslots != 0, node, pol);
            __syncthreads();  // slot s is free for the next bulk load
        }
        seq += nch;
    }
    __syncthreads();
    hot_flush(a.Fw, hot_acc, a.nhot, BLK_NT);
}

// ------------------------------------------------------------------ F: finalize
template <typename FT>
__device__ bool finalize_sweep(const SweepArgs<FT> &a, double mass, double ab, double mx, u64 steps, u64 nsel,
                               u64 hsteps);

template <typename FT>
__global__ void __launch_bounds__(FIN_NT) k_finalize(SweepArgs<FT> a, int nparts) {
    __shared__ double sm[FIN_NT / 32];
    __shared__ u64 sm64[FIN_NT / 32];
    double mass = 0.0, ab = 0.0, mx = 0.0;
    u64 steps = 0, nsel = 0, hsteps = 0;
    for (int p = threadIdx.x; p < nparts; p += FIN_NT) {
        mass += a.part_mass[p];
        ab += a.part_abs[p];
        mx = fmax(mx, a.part_max[p]);
        steps += a.part_steps[p];
        nsel += a.part_sel[p];
        if (fused_like(a.path)) hsteps += a.part_hsteps[p];
    }
    mass = block_sum<FIN_NT>(mass, sm);
    ab = block_sum<FIN_NT>(ab, sm);
    mx = block_max<FIN_NT>(mx, sm);
    steps = block_sum_u64<FIN_NT>(steps, sm64);
    nsel = block_sum_u64<FIN_NT>(nsel, sm64);
    hsteps = block_sum_u64<FIN_NT>(hsteps, sm64);
    if (threadIdx.x != 0) return;
    const bool done = finalize_sweep(a, mass, ab, mx, steps, nsel, hsteps);
    if (a.in_graph) cudaGraphSetConditional(a.cond, done ? 0u : 1u);
}

// The bookkeeping after a sweep (one thread): residual, counters, trace row,
// theta schedule, loop condition.  Returns whether the loop stops (the fused
// paths may instead ask for an exact check, c->need_check).
template <typename FT>
__device__ bool finalize_sweep(const SweepArgs<FT> &a, double mass, double ab, double mx, u64 steps, u64 nsel,
                               u64 hsteps) {
    SolveCtl *c = a.ctl;
    // binned path: the select pass saw F before any push of this sweep, so its
    // mass is exact; fused path: pushes race with the scan, so the residual is
    // carried incrementally like the reference's R (engine.py:322-325) and
    // re-derived exactly by k_mass_check before the loop may stop.
    const double residual = fused_like(a.path) ? c->residual - ab : (nsel ? mass - ab : mass);
    const double theta_used = c->theta;
    c->residual = residual;
    c->diffusions += nsel;
    c->steps += steps;
    c->hub_steps += hsteps;
    c->sweeps += 1;
    c->last_max = mx;
    if (a.trace && c->trace_len < (u64)a.trace_cap) {
        fr_trace_row &r = a.trace[c->trace_len];
        r.elementary_steps = (int64_t)c->steps;
        r.diffusions = (int64_t)c->diffusions;
        r.sweeps = (int64_t)c->sweeps;
        r.residual = residual;
        r.theta = theta_used;
        u64 tns;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tns));
        r.t_ns = (int64_t)tns;
    }
    c->trace_len += 1;
    // theta schedule
    double th = theta_used;
    if (a.select == FR_SELECT_MAX) {
        th = a.decay * mx;
    } else if (a.policy == FR_THETA_GEOMETRIC) {
        th *= a.decay;
    } else if (a.policy == FR_THETA_ADAPTIVE) {
        // steer the edges pushed per sweep toward edge_frac * m (the measured
        // optimum of scan cost vs. edge work is ~0.2 m at d = 0.85 and 0.99):
        // nominal decay when on target, slower when the sweep pushed more,
        // faster when it pushed less; theta may rise after an overshoot
        const double target = a.edge_frac * (double)a.m;
        const double ratio = target > 0.0 ? (double)steps / target : 1.0;
        th *= fmin(fmax(a.decay * sqrt(fmax(ratio, 1e-6)), 0.25), 1.5);
    }
    // a sweep that found nothing: decay until the largest fluid qualifies, as
    // repeated empty passes of the reference sweep scheduler would (sched.py:101-108)
    if (nsel == 0 && mx > 0.0)
        while (th > mx) th *= a.decay;
    c->theta = th;
    c->qcount[0] = c->qcount[1] = c->qcount[2] = 0;
    // deferred hub rows: the queue the sweep just consumed (its blocks exited only
    // once it was empty) is free for the next sweep's rows
    c->hub_cnt[c->sweeps & 1] = 0;
    c->hub_next[c->sweeps & 1] = 0;
    for (int q = 0; q < SW_MAX_SEGS; q++) c->seg_next[q * SEG_PAD] = 0;
    const bool budget = (long long)c->sweeps >= a.max_sweeps ||
                        (a.max_diffusions > 0 && (long long)c->diffusions >= a.max_diffusions);
    bool done;
    if (fused_like(a.path)) {
        // converged (by the estimate) or drained: verify with an exact sum first
        // signed fluid: positive and negative pushes cancel, so the true |F|_1
        // falls faster than the incremental estimate; re-derive it every n
        // diffusions as the reference does (engine.py:331-333)
        const bool refresh = c->is_signed && c->diffusions >= c->next_refresh;
        if (refresh) c->next_refresh = c->diffusions + (u64)a.n;
        const bool maybe = residual <= a.thr || (nsel == 0 && mx == 0.0) || refresh;
        c->need_check = maybe ? 1u : 0u;
        done = budget;
    } else {
        done = budget || residual <= a.thr || mass == 0.0;
    }
    c->stop = done ? 1u : 0u;
    return done;
}

// ------------------------------------------------------------------ small graphs: one block, one launch
// For n <= SMALL_N the per-sweep launches of the graph (six kernel nodes,
// ~40 us per sweep) cost more than the sweep itself, so a single block of
// 1024 threads runs the whole loop: prologue, sweeps (thread per node, the
// same selection, take and push as k_sweep, F and H resident in L2), the
// bookkeeping of k_finalize (finalize_sweep) and the exact checks, separated
// by block barriers.  F is read with ld.global.cg: other threads' pushes land
// in L2, and a line a thread cached in L1 would go stale.
static constexpr int SMALL_NT = 1024;
static constexpr long long SMALL_N = 1 << 17;

template <typename FT>
__device__ __forceinline__ FT ld_cg(const FT *p) { return __ldcg(p); }

template <typename FT>
__global__ void __launch_bounds__(SMALL_NT, 1) k_solve_small(SweepArgs<FT> a) {
    __shared__ double sm[SMALL_NT / 32];
    __shared__ double dsc_sm[DSC_TAB];
    __shared__ double s_red[SMALL_NT / 32][2];
    __shared__ u64 s_red64[SMALL_NT / 32][2];
    __shared__ double s_theta, s_theta_h1;
    __shared__ u64 s_sweep;
    __shared__ u32 s_stop, s_check, s_sample;
    __shared__ u64 s_row;
    SolveCtl *c = a.ctl;
    const long long n = a.n;
    FT *__restrict__ F = a.F;
    const u64 *__restrict__ off = a.off;
    const u32 *__restrict__ tgt = a.tgt;
    const double keep_frac = 1.0 - a.d;
    for (int q = threadIdx.x; q < DSC_TAB; q += SMALL_NT) dsc_sm[q] = q ? a.d / (double)q : 0.0;
    auto score_of = [&](long long i, double af) -> double {
        double sc = a.weight ? af * a.weight[i] : af;
        if (a.beta != 0.0f) sc = af * deg_weight(a.beta, off[i + 1] - off[i]);
        return sc;
    };
    // prologue (k_mass_partials + k_prologue): exact mass, threshold = max score
    {
        double mass = 0.0, mx = 0.0, neg = 0.0;
        for (long long i = threadIdx.x; i < n; i += SMALL_NT) {
            const double f = (double)ld_cg(F + i);
            const double af = fabs(f);
            mass += af;
            neg = fmin(neg, f);
            mx = fmax(mx, score_of(i, af));
        }
        mass = block_sum<SMALL_NT>(mass, sm);
        mx = block_max<SMALL_NT>(mx, sm);
        neg = -block_max<SMALL_NT>(-neg, sm);
        if (threadIdx.x == 0) {
            c->theta = mx;  // sched.py:89-90
            c->last_max = mx;
            c->residual = mass;
            c->mass0 = mass;
            c->is_signed = neg < 0.0 ? 1u : 0u;
            c->next_refresh = c->diffusions + (u64)n;
            c->next_trace = c->diffusions + (u64)a.trace_every;
            c->stop = (mass <= a.thr || mass == 0.0) ? 1u : 0u;
            s_theta = mx;
            s_sweep = c->sweeps;
            s_stop = c->stop;
        }
        __syncthreads();
    }
    while (!s_stop) {
        const double theta = s_theta;
        const u64 sweep = s_sweep;
        double absorbed = 0.0, mx = 0.0;
        u64 steps = 0, nsel = 0;
        for (long long i = threadIdx.x; i < n; i += SMALL_NT) {
            const FT f = ld_cg(F + i);
            const double af = fabs((double)f);
            const double score = score_of(i, af);
            mx = fmax(mx, score);
            bool sel;
            if (a.select == FR_SELECT_PER) sel = true;
            else if (a.select == FR_SELECT_RAND)
                sel = (double)(hmix(((u64)a.seed << 40) ^ (sweep << 32) ^ hmix((u64)i)) >> 11) * 0x1.0p-53 < a.rand_frac;
            else sel = score >= theta;
            if (!sel || f == (FT)0) continue;
            red_add(F + i, -f);  // take exactly the loaded fluid (as k_sweep)
            red_add(a.H + i, (double)f);
            nsel++;
            const u64 lo = off[i], hi = off[i + 1];
            const u64 deg = hi - lo;
            if (deg == 0) {
                absorbed += af;  // dangling: all of it leaves (PAPER sec. 3.3)
                continue;
            }
            absorbed += af * keep_frac;
            steps += deg;
            const FT v = (FT)((double)f * (deg < DSC_TAB ? dsc_sm[deg] : a.d / (double)deg));  // engine.py:321
            for (u64 k = lo; k < hi; k++) red_add(F + __ldg(tgt + k), v);
        }
        // the four sweep totals in one exchange through shared memory
        absorbed = warp_sum(absorbed);
        mx = warp_max(mx);
        steps = warp_sum_u64(steps);
        nsel = warp_sum_u64(nsel);
        if ((threadIdx.x & 31) == 0) {
            const int w = threadIdx.x >> 5;
            s_red[w][0] = absorbed;
            s_red[w][1] = mx;
            s_red64[w][0] = steps;
            s_red64[w][1] = nsel;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            absorbed = 0.0;
            mx = 0.0;
            steps = nsel = 0;
            for (int w = 0; w < SMALL_NT / 32; w++) {
                absorbed += s_red[w][0];
                mx = fmax(mx, s_red[w][1]);
                steps += s_red64[w][0];
                nsel += s_red64[w][1];
            }
            __threadfence();  // the sweep's reds are visible to the exact check below
            s_stop = finalize_sweep(a, 0.0, absorbed, mx, steps, nsel, 0ull) ? 1u : 0u;
            s_check = c->need_check;
            s_theta = c->theta;
            s_sweep = c->sweeps;
            s_sample = 0;
            if (a.ref && c->diffusions >= c->next_trace) {  // engine.py:334-336
                s_sample = 1;
                s_row = c->trace_len - 1;
                c->next_trace = c->diffusions + (u64)a.trace_every;
            }
        }
        __syncthreads();
        if (s_sample) {  // true error of the normalized history (engine.py:269-277)
            double h1 = 0.0;
            for (long long i = threadIdx.x; i < n; i += SMALL_NT) h1 += fabs(ld_cg(a.H + i));
            h1 = block_sum<SMALL_NT>(h1, sm);
            if (threadIdx.x == 0) s_theta_h1 = h1;
            __syncthreads();
            const double t = s_theta_h1;
            double e = 0.0;
            if (t > 0.0)
                for (long long i = threadIdx.x; i < n; i += SMALL_NT) e += fabs(ld_cg(a.H + i) / t - a.ref[i]);
            e = block_sum<SMALL_NT>(e, sm);
            if (threadIdx.x == 0 && t > 0.0 && (long long)s_row < a.trace_cap) a.true_err[s_row] = e;
            __syncthreads();
        }
        if (s_check) {  // k_mass_partials + k_mass_check
            double mass = 0.0;
            for (long long i = threadIdx.x; i < n; i += SMALL_NT) mass += fabs((double)ld_cg(F + i));
            mass = block_sum<SMALL_NT>(mass, sm);
            if (threadIdx.x == 0) {
                c->residual = mass;
                c->need_check = 0;
                const bool done = mass <= a.thr || mass == 0.0 || c->stop;
                c->stop = done ? 1u : 0u;
                s_stop = c->stop;
            }
            __syncthreads();
        }
    }
}

// ------------------------------------------------------------------ hot-set preparation
// The slot classes are a performance device only (results do not depend on
// them), so they are chosen from an in-degree ESTIMATE: the columns of one
// 128 B line in every 2^shift lines are counted (exact for shift = 0).
__global__ void k_sample_indeg(const u32 *__restrict__ tgt, long long m, int shift, u32 *__restrict__ cnt) {
    const long long lines = (m + 31) >> 5;
    const long long nsamp = (lines + (1ll << shift) - 1) >> shift;
    const int lane = threadIdx.x & 31;
    for (long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; w < nsamp;
         w += ((long long)gridDim.x * blockDim.x) >> 5) {
        const long long e = ((w << shift) << 5) + lane;
        if (e < m) atomicAdd(cnt + tgt[e], 1u);  // compiled to RED (result unused)
    }
}

static constexpr int IND_BINS = 1 << 16;  // histogram of the estimate, clipped at IND_BINS - 1
__global__ void k_indeg_hist(const u32 *__restrict__ cnt, long long n, u32 *__restrict__ hist) {
    // low bins (almost every node) are counted in shared memory first
    __shared__ u32 lo[1024];
    for (int q = threadIdx.x; q < 1024; q += blockDim.x) lo[q] = 0;
    __syncthreads();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const u32 c = min(cnt[i], (u32)(IND_BINS - 1));
        if (c < 1024) atomicAdd(&lo[c], 1u);
        else atomicAdd(hist + c, 1u);
    }
    __syncthreads();
    for (int q = threadIdx.x; q < 1024; q += blockDim.x)
        if (lo[q]) atomicAdd(hist + q, lo[q]);
}

// Nodes with tau_lo <= estimate < tau_hi get slots base, base+1, ... (< base+cap).
__global__ void k_collect_class(const u32 *__restrict__ cnt, long long n, u32 tau_lo, u32 tau_hi, u32 base, u32 cap,
                                u32 *__restrict__ slot_node, u32 *__restrict__ node_slot, u32 *count) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const u32 d = min(cnt[i], (u32)(IND_BINS - 1));
        if (d >= tau_lo && d < tau_hi) {
            const u32 k = atomicAdd(count, 1u);
            if (k < cap) {
                slot_node[base + k] = (u32)i;
                node_slot[i] = base + k;
            }
        }
    }
}

__global__ void k_encode_targets(const u32 *__restrict__ tgt, long long m, const u32 *__restrict__ node_slot,
                                 u32 *__restrict__ out) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < m; k += (long long)gridDim.x * blockDim.x) {
        const u32 t = tgt[k];
        const u32 s = node_slot[t];
        out[k] = s == 0xFFFFFFFFu ? t : (HOT_FLAG | s);
    }
}

int abs_sum_async(long long n, const void *x, int fp32, double *d_out, cudaStream_t st);  // fr_util.cu
int l1_error_async(long long n, const double *x, const double *ref, double *d_out, cudaStream_t st);  // fr_util.cu

}  // namespace fr

using namespace fr;

// ====================================================================== host side
template <typename FT>
static void *sweep_kernel(const SweepArgs<FT> &a) {
    if (a.path == PATH_OWNED) return a.off32 ? (void *)k_sweep_own<FT, false> : (void *)k_sweep_own<FT, true>;
    return a.off32 ? (void *)k_sweep<FT, false> : (void *)k_sweep<FT, true>;
}
template <typename FT>
static int sweep_threads(const SweepArgs<FT> &a) { return a.path == PATH_OWNED ? OWN_NT : SW_NT; }
// dynamic shared memory of the sweep kernel: the owned path's chunk fluid and hot slots
template <typename FT>
static size_t sweep_smem(const SweepArgs<FT> &a) {
    return a.path == PATH_OWNED ? sizeof(FT) * ((size_t)a.own_ch + (size_t)a.nhot) : 0;
}
template <typename FT>
static void launch_sweep(const SweepArgs<FT> &a, int grid, cudaStream_t st) {
    if (a.path == PATH_OWNED) {
        const size_t sm = sweep_smem(a);
        if (a.off32) k_sweep_own<FT, false><<<grid, OWN_NT, sm, st>>>(a);
        else k_sweep_own<FT, true><<<grid, OWN_NT, sm, st>>>(a);
        return;
    }
    if (a.off32) k_sweep<FT, false><<<grid, SW_NT, 0, st>>>(a);
    else k_sweep<FT, true><<<grid, SW_NT, 0, st>>>(a);
}

// Host-buffer entry point (fr_pagerank_host): the column indices arrive in
// pieces on a copy stream; the slot classes are estimated from the first
// pieces and every piece is encoded as soon as it has landed, so the setup
// overlaps the host-to-device copy instead of following it.
struct TargetPieces {
    int count;                    // pieces; edge range of piece k: [edge_end[k-1], edge_end[k])
    const long long *edge_end;    // ascending, edge_end[count-1] = m
    const cudaEvent_t *ready;     // recorded on the copy stream after piece k
    int sample_pieces;            // pieces whose columns decide the slot classes
    bool in_place;                // encode into the caller's column array (the caller owns it)
};

struct fr_solver {
    long long n, m;
    int fp32;
    int sel_grid, sweep_grid, thread_grid, warp_grid, block_grid, fold_grid;
    u32 nhot, nslots;
    cudaStream_t stream;  // creation stream (allocations and frees are ordered on it)
    SolveCtl *ctl;
    fr_trace_row *trace;
    long long trace_cap;
    void *qnode_buf, *qval_buf;
    double *parts;
    u64 *parts64;
    u32 *tgt_enc;      // fused path: column indices with slotted targets encoded
    u32 *off32;        // fused path: narrow row offsets (m < 2^32, n < 2^31), else null
    u32 *slot_node;
    void *fw_buf;
    double *true_err;  // sampled runs: true L1 error per trace row (NaN where not sampled)
    fr_solver_config cfg;
    const TargetPieces *pieces;  // setup only (fr_pagerank_host); null: targets resident
    int small;                   // n <= SMALL_N: the whole solve is one k_solve_small launch
    cudaGraph_t graph;
    cudaGraphExec_t exec;
    // both instantiations are kept; only one is used per solver
    SweepArgs<double> ad;
    SweepArgs<float> af;
};

template <typename FT>
static int add_kernel(cudaGraph_t g, cudaGraphNode_t *node, const cudaGraphNode_t *deps, size_t ndeps, void *func,
                      int grid, int block, void **args, size_t smem = 0) {
    cudaKernelNodeParams p = {};
    p.func = func;
    p.gridDim = dim3((unsigned)grid);
    p.blockDim = dim3((unsigned)block);
    p.sharedMemBytes = (unsigned)smem;
    p.kernelParams = args;
    FR_CUDA(cudaGraphAddKernelNode(node, g, deps, ndeps, &p));
    return FR_OK;
}

template <typename FT>
static int build_graph(fr_solver *s, SweepArgs<FT> &a) {
    FR_CUDA(cudaGraphCreate(&s->graph, 0));
    FR_CUDA(cudaGraphConditionalHandleCreate(&a.cond, s->graph, 0, 0));
    a.in_graph = 1;
    const char *ed = getenv("FR_HUB_DEFER");
    a.hub_defer = a.path == PATH_OWNED && a.hub_stride != 0 && (ed ? atoi(ed) != 0 : true) ? 1 : 0;
    int nparts = s->sel_grid;
    int nparts_sw = s->sweep_grid;
    int unguarded = 0, guarded = 1;
    // prologue
    void *args_a[] = {&a};
    void *args_an[] = {&a, &nparts};
    void *args_ans[] = {&a, &nparts_sw};
    void *args_m0[] = {&a, &unguarded};
    void *args_m1[] = {&a, &guarded};
    cudaGraphNode_t n_mass, n_pro, n_while;
    FR_TRY(add_kernel<FT>(s->graph, &n_mass, nullptr, 0, (void *)k_mass_partials<FT>, s->sel_grid, SEL_NT, args_m0));
    FR_TRY(add_kernel<FT>(s->graph, &n_pro, &n_mass, 1, (void *)k_prologue<FT>, 1, FIN_NT, args_an));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = a.cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    FR_CUDA(cudaGraphAddNode(&n_while, s->graph, &n_pro, 1, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    if (fused_like(a.path)) {
        // sweep -> hub pushes -> finalize -> (guarded) exact mass -> (guarded) check
        // owned path: the hub rows queued by a sweep are pushed by the next sweep's
        // blocks between their chunks (no hub node in the loop), the last sweep's by a
        // drain after the loop
        cudaGraphNode_t n_sw, n_hub, n_fold, n_fin, n_m, n_chk;
        FR_TRY(add_kernel<FT>(body, &n_sw, nullptr, 0, sweep_kernel(a), s->sweep_grid, sweep_threads(a), args_a,
                              sweep_smem(a)));
        if (a.hub_defer) {
            n_hub = n_sw;
        } else {
            FR_TRY(add_kernel<FT>(body, &n_hub, &n_sw, 1, (void *)k_push_block<FT>, s->block_grid, BLK_NT, args_a));
        }
        FR_TRY(add_kernel<FT>(body, &n_fold, &n_hub, 1, (void *)k_fold<FT>, s->fold_grid, 256, args_a));
        FR_TRY(add_kernel<FT>(body, &n_fin, &n_fold, 1, (void *)k_finalize<FT>, 1, FIN_NT, args_ans));
        FR_TRY(add_kernel<FT>(body, &n_m, &n_fin, 1, (void *)k_mass_partials<FT>, s->sel_grid, SEL_NT, args_m1));
        FR_TRY(add_kernel<FT>(body, &n_chk, &n_m, 1, (void *)k_mass_check<FT>, 1, FIN_NT, args_an));
    } else {
        // select -> three push bins (concurrent) -> fold of the warm slots -> finalize
        cudaGraphNode_t n_sel, n_p[3], n_fold, n_fin;
        FR_TRY(add_kernel<FT>(body, &n_sel, nullptr, 0, (void *)k_select<FT>, s->sel_grid, SEL_NT, args_a));
        FR_TRY(add_kernel<FT>(body, &n_p[0], &n_sel, 1, (void *)k_push_thread<FT>, s->thread_grid, 256, args_a));
        FR_TRY(add_kernel<FT>(body, &n_p[1], &n_sel, 1, (void *)k_push_warp<FT>, s->warp_grid, 256, args_a));
        FR_TRY(add_kernel<FT>(body, &n_p[2], &n_sel, 1, (void *)k_push_block<FT>, s->block_grid, BLK_NT, args_a));
        FR_TRY(add_kernel<FT>(body, &n_fold, n_p, 3, (void *)k_fold<FT>, s->fold_grid, 256, args_a));
        FR_TRY(add_kernel<FT>(body, &n_fin, &n_fold, 1, (void *)k_finalize<FT>, 1, FIN_NT, args_an));
    }
    if (a.hub_defer) {  // the rows the last sweep queued, then the warm slots they filled
        cudaGraphNode_t n_drain, n_dfold;
        FR_TRY(add_kernel<FT>(s->graph, &n_drain, &n_while, 1, (void *)k_push_block<FT>, s->block_grid, BLK_NT,
                              args_a));
        FR_TRY(add_kernel<FT>(s->graph, &n_dfold, &n_drain, 1, (void *)k_fold<FT>, s->fold_grid, 256, args_a));
    }
    FR_CUDA(cudaGraphInstantiate(&s->exec, s->graph, 0));
    return FR_OK;
}

__global__ void k_narrow_offsets(const u64 *__restrict__ off, long long n1, u32 *__restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n1; i += (long long)gridDim.x * blockDim.x)
        out[i] = (u32)off[i];
}

template <typename FT>
static int occupancy_grid(void *func, int threads, int sms) {
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, func, threads, 0) != cudaSuccess || per < 1) per = 1;
    return per * sms;
}

// Slot classes by in-degree: "hot" = up to `want_hot` highest in-degree nodes
// (pushes summed in shared memory), "warm" = the next up to `want_warm` (pushes
// into the compact array Fw).  A class is the largest threshold set that fits:
// {indeg >= tau} with the smallest tau whose count does not exceed the budget,
// read off one histogram of the in-degree estimate (k_sample_indeg: exact for
// m < 2^26, else 1 column line in 8 -- ~1 ms on config 5 instead of 32 ms for
// exact counting plus a synchronized threshold search).
// Writes the solver-private encoded column indices.
template <typename FT>
static int prepare_slots(fr_solver *s, SweepArgs<FT> &a, int want_hot, long long want_warm, cudaStream_t st) {
    if (want_hot > HOT_SLOTS) want_hot = HOT_SLOTS;
    if (want_hot < 0) want_hot = 0;
    if (want_warm < 0) want_warm = 0;
    if (want_warm > (long long)WARM_SLOTS * 8) want_warm = (long long)WARM_SLOTS * 8;
    const long long n = s->n, m = s->m;
    // a slotted column carries HOT_FLAG | slot, so node ids must stay below 2^31
    if (n > (1ll << 31)) return FR_OK;
    DeviceInfo di;
    FR_TRY(device_info(&di));
    Scratch scratch(st);
    // in-degree estimate from 1 line in 8 (exact below 2^26 edges)
    const int shift = m >= (1ll << 26) ? 3 : 0;
    u32 *cnt, *hist;
    FR_TRY(scratch.alloc(&cnt, (size_t)n));
    FR_TRY(scratch.alloc(&hist, (size_t)IND_BINS));
    FR_CUDA(cudaMemsetAsync(cnt, 0, sizeof(u32) * (size_t)n, st));
    FR_CUDA(cudaMemsetAsync(hist, 0, sizeof(u32) * (size_t)IND_BINS, st));
    const int g = di.sms * 8;
    const TargetPieces *tp = s->pieces;
    auto piece_begin = [&](int k) -> long long { return k ? tp->edge_end[k - 1] : 0; };
    double sampled = (double)m;  // edges whose columns were sampled
    if (tp) {
        for (int k = 0; k < tp->sample_pieces; k++) {
            FR_CUDA(cudaStreamWaitEvent(st, tp->ready[k], 0));
            k_sample_indeg<<<g, 256, 0, st>>>(a.tgt + piece_begin(k), tp->edge_end[k] - piece_begin(k), shift, cnt);
        }
        sampled = (double)tp->edge_end[tp->sample_pieces - 1];
    } else {
        k_sample_indeg<<<g, 256, 0, st>>>(a.tgt, m, shift, cnt);
    }
    // the estimate counts ~1 in `scale` of a node's in-edges
    const double scale = (double)(1ll << shift) * (sampled > 0.0 ? (double)m / sampled : 1.0);
    k_indeg_hist<<<g, 256, 0, st>>>(cnt, n, hist);
    std::vector<u32> h(IND_BINS);
    FR_CUDA(cudaMemcpyAsync(h.data(), hist, sizeof(u32) * IND_BINS, cudaMemcpyDeviceToHost, st));
    FR_CUDA(cudaStreamSynchronize(st));
    // ge[t] = #nodes whose estimate >= t
    std::vector<unsigned long long> ge(IND_BINS + 1, 0ull);
    for (int t = IND_BINS - 1; t >= 0; t--) ge[t] = ge[t + 1] + h[t];
    // smallest threshold >= floor (in-degree units) whose class fits the budget; IND_BINS if none
    auto threshold = [&](long long floor, unsigned long long budget) -> u32 {
        long long t0 = (long long)ceil((double)floor / scale);
        if (t0 < 1) t0 = 1;
        if (budget == 0 || t0 >= IND_BINS) return (u32)IND_BINS;
        for (long long t = t0; t < IND_BINS; t++)
            if (ge[t] <= budget) return (u32)t;
        return (u32)(IND_BINS - 1);  // clipped bin: take a capped subset of it
    };
    // a target needs many pushes per sweep before an L2 slot or shared memory pays
    const u32 tau_hot = threshold(64, (unsigned long long)want_hot);
    u32 tau_warm = threshold(8, (unsigned long long)(want_hot + want_warm));
    if (tau_warm > tau_hot) tau_warm = tau_hot;
    u32 *node_slot, *d_count;
    FR_TRY(scratch.alloc(&node_slot, (size_t)n));
    FR_TRY(scratch.alloc(&d_count, 1));
    FR_CUDA(cudaMemsetAsync(node_slot, 0xFF, sizeof(u32) * (size_t)n, st));
    const size_t cap = (size_t)want_hot + (size_t)want_warm;
    if (cap == 0) return FR_OK;
    FR_TRY(pool_alloc((void **)&s->slot_node, sizeof(u32) * cap, st));
    u32 nhot = 0, nwarm = 0;
    FR_CUDA(cudaMemsetAsync(d_count, 0, sizeof(u32), st));
    k_collect_class<<<g, 256, 0, st>>>(cnt, n, tau_hot, 0xFFFFFFFFu, 0, (u32)want_hot, s->slot_node, node_slot, d_count);
    FR_CUDA(cudaMemcpyAsync(&nhot, d_count, sizeof(u32), cudaMemcpyDeviceToHost, st));
    FR_CUDA(cudaStreamSynchronize(st));
    if (nhot > (u32)want_hot) nhot = (u32)want_hot;
    FR_CUDA(cudaMemsetAsync(d_count, 0, sizeof(u32), st));
    k_collect_class<<<g, 256, 0, st>>>(cnt, n, tau_warm, tau_hot, nhot, (u32)want_warm, s->slot_node, node_slot,
                                       d_count);
    FR_CUDA(cudaMemcpyAsync(&nwarm, d_count, sizeof(u32), cudaMemcpyDeviceToHost, st));
    FR_CUDA(cudaStreamSynchronize(st));
    if (nwarm > (u32)want_warm) nwarm = (u32)want_warm;
    const u32 nslots = nhot + nwarm;
    if (nslots == 0) return FR_OK;
    u32 *enc;
    if (tp && tp->in_place) {
        enc = const_cast<u32 *>(a.tgt);
    } else {
        FR_TRY(pool_alloc((void **)&s->tgt_enc, sizeof(u32) * (size_t)m, st));
        enc = s->tgt_enc;
    }
    FR_TRY(pool_alloc(&s->fw_buf, sizeof(FT) * (size_t)nslots, st));
    FR_CUDA(cudaMemsetAsync(s->fw_buf, 0, sizeof(FT) * (size_t)nslots, st));
    if (tp) {
        for (int k = 0; k < tp->count; k++) {  // later pieces: the stream waits for them to land
            if (k >= tp->sample_pieces) FR_CUDA(cudaStreamWaitEvent(st, tp->ready[k], 0));
            const long long b = piece_begin(k);
            k_encode_targets<<<g, 256, 0, st>>>(a.tgt + b, tp->edge_end[k] - b, node_slot, enc + b);
        }
    } else {
        k_encode_targets<<<g, 256, 0, st>>>(a.tgt, m, node_slot, enc);
    }
    FR_CUDA(cudaGetLastError());
    if (!tp) FR_CUDA(cudaStreamSynchronize(st));  // (the scratch frees below are stream-ordered either way)
    a.tgt = enc;
    a.slot_node = s->slot_node;
    a.Fw = reinterpret_cast<FT *>(s->fw_buf);
    a.nhot = nhot;
    a.nslots = nslots;
    s->nhot = nhot;
    s->nslots = nslots;
    return FR_OK;
}

template <typename FT>
static int setup(fr_solver *s, SweepArgs<FT> &a, const int64_t *d_offsets, const uint32_t *d_targets,
                 const double *d_w, void *d_fluid, double *d_history, cudaStream_t st) {
    DeviceInfo di;
    FR_TRY(device_info(&di));
    const fr_solver_config &c = s->cfg;
    a = SweepArgs<FT>{};
    a.F = reinterpret_cast<FT *>(d_fluid);
    a.H = d_history;
    a.off = reinterpret_cast<const u64 *>(d_offsets);
    a.tgt = d_targets;
    a.weight = d_w;
    a.ctl = s->ctl;
    a.n = s->n;
    a.m = s->m;
    a.trace = s->trace;
    a.trace_cap = s->trace_cap;
    a.max_sweeps = c.max_sweeps > 0 ? c.max_sweeps : 1000000;
    a.max_diffusions = c.max_diffusions;
    a.d = c.damping;
    a.thr = c.target_error * (1.0 - c.damping);
    a.decay = c.decay;
    a.rand_frac = c.rand_frac;
    a.edge_frac = c.edge_frac > 0.0 ? c.edge_frac : 0.2;
    a.t0 = c.thread_max_degree > 0 ? (u32)c.thread_max_degree : 8u;
    a.t2 = c.block_min_degree > 0 ? (u32)c.block_min_degree : 2048u;
    if (a.t2 <= a.t0) a.t2 = a.t0 + 1;
    a.select = c.select;
    a.policy = c.policy;
    a.seed = c.seed;
    a.path = c.kernel_path == 1 ? PATH_BINNED : (c.kernel_path == 2 ? PATH_OWNED : PATH_FUSED);
    a.beta = (float)c.degree_exponent;
    // op2 (1/(out+1), sched.py:131-138) is the exponent 1: no weight array needed
    if (c.select == FR_SELECT_OP2 && a.weight == nullptr) a.beta = 1.0f;
    {
        // tuning knobs for experiments (tools/prof_solver.py); defaults measured on config 5
        const char *e1 = getenv("FR_SEGS"), *e2 = getenv("FR_CHUNK");
        a.segs = e1 ? atoi(e1) : 32;
        a.chunk = e2 ? (u32)atoi(e2) : 8u;
        if (a.segs < 1) a.segs = 1;
        if (a.segs > SW_MAX_SEGS) a.segs = SW_MAX_SEGS;
        if (a.chunk < 1) a.chunk = 1;
        const char *e3 = getenv("FR_OWN_CHUNK");
        long long ch = e3 ? atoll(e3) : 2048;
        u32 p2 = 256;
        while ((long long)p2 < ch && p2 < (1u << 16)) p2 <<= 1;
        // default: 2048-node chunks, halved (down to 1024) while there are fewer
        // chunks than resident blocks (graphs below ~2.7M nodes), so every SM
        // gets work (config 2, N=1M: 5.8 -> 5.1 ms)
        if (!e3)
            while (p2 > 1024 && (long long)(s->n / p2) < (long long)di.sms * FR_OWN_MINB) p2 >>= 1;
        a.own_ch = p2;
        const char *e4 = getenv("FR_OWN_REV");
        a.own_rev = e4 ? (u32)(atoi(e4) != 0) : 1u;
    }
    // queues: a selected node lands in exactly one bin
    const long long n = s->n, m = s->m;
    // the fused path only queues hub rows; the binned path needs all three bins
    const bool binned = c.kernel_path == 1;
    const long long cap0 = binned ? n : 0;
    const long long cap1 = binned ? std::min<long long>(n, m / ((long long)a.t0 + 1) + 1) : 0;
    const long long cap2 = std::min<long long>(n, m / (long long)a.t2 + 1);
    // the owned path's deferred hub rows use two queues (sweep parity) of cap2 + 1
    const long long cap2x = c.kernel_path == 2 ? 2 * (cap2 + 1) : cap2;
    a.hub_stride = c.kernel_path == 2 && cap2 + 1 < (1ll << 31) ? (u32)(cap2 + 1) : 0u;
    FR_TRY(pool_alloc(&s->qnode_buf, sizeof(u32) * (size_t)(cap0 + cap1 + cap2x + 3), st));
    FR_TRY(pool_alloc(&s->qval_buf, sizeof(FT) * (size_t)(cap0 + cap1 + cap2x + 3), st));
    u32 *qn = (u32 *)s->qnode_buf;
    FT *qv = (FT *)s->qval_buf;
    a.qnode[0] = qn;
    a.qnode[1] = qn + cap0 + 1;
    a.qnode[2] = qn + cap0 + cap1 + 2;
    a.qval[0] = qv;
    a.qval[1] = qv + cap0 + 1;
    a.qval[2] = qv + cap0 + cap1 + 2;
    s->sel_grid = occupancy_grid<FT>((void *)k_select<FT>, SEL_NT, di.sms);
    const long long tiles = (n + SEL_TILE - 1) / SEL_TILE;
    if (s->sel_grid > tiles) s->sel_grid = (int)std::max<long long>(1, tiles);
    s->thread_grid = occupancy_grid<FT>((void *)k_push_thread<FT>, 256, di.sms);
    s->warp_grid = occupancy_grid<FT>((void *)k_push_warp<FT>, 256, di.sms);
    s->block_grid = occupancy_grid<FT>((void *)k_push_block<FT>, BLK_NT, di.sms);
    {
        const char *e = getenv("FR_SMALL");
        s->small = fused_like(a.path) && n <= SMALL_N && !(e && e[0] == '0');
    }
    a.off32 = nullptr;
    // FR_FORCE_WIDE=1 keeps the 64-bit kernel on small graphs (tests of the
    // m >= 2^32 / n >= 2^31 path, which no test-sized graph would take)
    const char *fw = getenv("FR_FORCE_WIDE");
    const bool force_wide = fw && fw[0] == '1';
    if (fused_like(a.path) && !s->small && !force_wide && m < (1ll << 32) && n < (1ll << 31)) {
        FR_TRY(pool_alloc((void **)&s->off32, sizeof(u32) * (size_t)(n + 1), st));
        k_narrow_offsets<<<di.sms * 8, 256, 0, st>>>(a.off, n + 1, s->off32);
        FR_CUDA(cudaGetLastError());
        a.off32 = s->off32;
    }

    // upper bound of the sweep grid (the partial arrays are sized by it); the
    // owned path's grid depends on its shared memory, known after the slots
    s->sweep_grid = occupancy_grid<FT>(sweep_kernel(a), sweep_threads(a), di.sms);
    const long long wtiles = ((n + 31) / 32 + SW_NT / 32 - 1) / (SW_NT / 32);
    if (s->sweep_grid > wtiles) s->sweep_grid = (int)std::max<long long>(1, wtiles);
    if (a.path == PATH_OWNED) s->sweep_grid = di.sms * 32;
    const int P = std::max(s->sel_grid, s->sweep_grid);
    FR_TRY(pool_alloc((void **)&s->parts, sizeof(double) * 3 * (size_t)P, st));
    FR_TRY(pool_alloc((void **)&s->parts64, sizeof(u64) * 3 * (size_t)P, st));
    a.part_mass = s->parts;
    a.part_abs = s->parts + P;
    a.part_max = s->parts + 2 * P;
    a.part_steps = s->parts64;
    a.part_sel = s->parts64 + P;
    a.part_hsteps = s->parts64 + 2 * P;
    a.slot_node = nullptr;
    a.Fw = nullptr;
    a.nhot = 0;
    a.nslots = 0;
    if (m > 0 && !s->small) {
        // owned path: 512 hot slots, so nine 128-thread blocks (chunk fluid + hot
        // table, 20 KB each) fit one SM's shared memory
        const int hot_default = a.path == PATH_OWNED ? HOT_SLOTS / 4 : HOT_SLOTS;
        const int want_hot = c.hot_slots < 0 ? 0 : (c.hot_slots ? c.hot_slots : hot_default);
        const long long want_warm = c.warm_slots < 0 ? 0 : (c.warm_slots ? c.warm_slots : (long long)WARM_DEFAULT);
        FR_TRY(prepare_slots(s, a, want_hot, want_warm, st));
    }
    s->fold_grid = (int)std::max<long long>(1, std::min<long long>((long long)di.sms * 8, ((long long)a.nslots + 255) / 256));
    if (s->small) return FR_OK;  // no graph: one launch per solve
    if (a.path == PATH_OWNED) {
        const size_t sm = sweep_smem(a);
        FR_CUDA(cudaFuncSetAttribute(sweep_kernel(a), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        int per = 0;
        FR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, sweep_kernel(a), OWN_NT, sm));
        if (per < 1) {
            set_error("owned sweep: %zu bytes of shared memory per block do not fit", sm);
            return FR_ERR_ARG;
        }
        const long long chunks = (n + a.own_ch - 1) / a.own_ch;
        s->sweep_grid = (int)std::max<long long>(1, std::min<long long>((long long)per * di.sms, chunks));
    }
    return build_graph<FT>(s, a);
}

static int solver_create(int64_t n, int64_t m, const int64_t *d_offsets, const uint32_t *d_targets,
                         const double *d_score_weight, void *d_fluid, double *d_history, const fr_solver_config *cfg,
                         int64_t trace_cap, void *stream, const TargetPieces *pieces, fr_solver **out);

extern "C" int fr_solver_create(int64_t n, int64_t m, const int64_t *d_offsets, const uint32_t *d_targets,
                                const double *d_score_weight, void *d_fluid, double *d_history,
                                const fr_solver_config *cfg, int64_t trace_cap, void *stream, fr_solver **out) {
    return solver_create(n, m, d_offsets, d_targets, d_score_weight, d_fluid, d_history, cfg, trace_cap, stream,
                         nullptr, out);
}

// fr_pagerank_host's variant (fr_capi.cu): targets arriving in pieces, encoded in place.
int solver_create_pieces(int64_t n, int64_t m, const int64_t *d_offsets, uint32_t *d_targets, void *d_fluid,
                         double *d_history, const fr_solver_config *cfg, void *stream, int count,
                         const long long *edge_end, const cudaEvent_t *ready, fr_solver **out) {
    TargetPieces tp{count, edge_end, ready, count > 1 ? count - 1 : count, true};
    return solver_create(n, m, d_offsets, d_targets, nullptr, d_fluid, d_history, cfg, 0, stream,
                         count > 0 ? &tp : nullptr, out);
}

static int solver_create(int64_t n, int64_t m, const int64_t *d_offsets, const uint32_t *d_targets,
                         const double *d_score_weight, void *d_fluid, double *d_history, const fr_solver_config *cfg,
                         int64_t trace_cap, void *stream, const TargetPieces *pieces, fr_solver **out) {
    if (!out || !cfg || n < 1 || n > 0xFFFFFFFFll || m < 0 || !d_offsets || !d_fluid || !d_history ||
        (m > 0 && !d_targets)) {
        set_error("fr_solver_create: bad arguments");
        return FR_ERR_ARG;
    }
    if (!(cfg->damping > 0.0 && cfg->damping <= 1.0) || !(cfg->target_error > 0.0) ||
        !(cfg->decay > 0.0 && cfg->decay < 1.0)) {
        set_error("fr_solver_create: need 0 < damping <= 1, target_error > 0, 0 < decay < 1");
        return FR_ERR_ARG;
    }
    if (cfg->damping >= 1.0 && cfg->max_diffusions <= 0 && cfg->max_sweeps <= 0) {
        set_error("undamped diagnostic mode requires max_diffusions");
        return FR_ERR_ARG;
    }
    if (cfg->select < FR_SELECT_SWEEP || cfg->select > FR_SELECT_OP2 || cfg->policy < FR_THETA_EXHAUST ||
        cfg->policy > FR_THETA_ADAPTIVE) {
        set_error("fr_solver_create: unknown select rule or theta policy");
        return FR_ERR_ARG;
    }
    if (cfg->select == FR_SELECT_OP && !d_score_weight) {
        set_error("fr_solver_create: op needs per-node score weights 1/((in+1)(out+1))");
        return FR_ERR_ARG;
    }
    fr_solver *s = new fr_solver();
    s->n = n;
    s->m = m;
    s->cfg = *cfg;
    s->fp32 = cfg->fluid_fp32 ? 1 : 0;
    s->trace_cap = trace_cap > 0 ? trace_cap : 0;
    s->stream = (cudaStream_t)stream;
    s->pieces = pieces;
    int rc = FR_OK;
    do {
        if ((rc = pool_alloc((void **)&s->ctl, sizeof(SolveCtl), (cudaStream_t)stream)) != FR_OK) break;
        if (s->trace_cap &&
            (rc = pool_alloc((void **)&s->trace, sizeof(fr_trace_row) * (size_t)s->trace_cap, (cudaStream_t)stream)) !=
                FR_OK)
            break;
        // all setup work is ordered on the caller's stream (its inputs may still be in flight there)
        rc = s->fp32 ? setup<float>(s, s->af, d_offsets, d_targets, d_score_weight, d_fluid, d_history,
                                    (cudaStream_t)stream)
                     : setup<double>(s, s->ad, d_offsets, d_targets, d_score_weight, d_fluid, d_history,
                                     (cudaStream_t)stream);
    } while (0);
    s->pieces = nullptr;
    if (rc != FR_OK) {
        fr_solver_destroy(s);
        return rc;
    }
    *out = s;
    return FR_OK;
}

static int reset_ctl(fr_solver *s, cudaStream_t st) {
    FR_CUDA(cudaMemsetAsync(s->ctl, 0, sizeof(SolveCtl), st));
    return FR_OK;
}

static int read_stats(fr_solver *s, cudaStream_t st, fr_solve_stats *h, double *exact = nullptr) {
    static thread_local SolveCtl c;
    FR_CUDA(cudaMemcpyAsync(&c, s->ctl, offsetof(SolveCtl, seg_next), cudaMemcpyDeviceToHost, st));
    FR_CUDA(cudaStreamSynchronize(st));
    if (exact) *exact = c.exact;
    if (h) {
        h->diffusions = (int64_t)c.diffusions;
        h->elementary_steps = (int64_t)c.steps;
        h->sweeps = (int64_t)c.sweeps;
        h->residual = c.residual;
        h->theta = c.theta;
        h->trace_len = (int64_t)c.trace_len;
        h->hub_edges = (int64_t)c.hub_steps;
    }
    return FR_OK;
}

extern "C" int fr_solver_run(fr_solver *s, void *stream, fr_solve_stats *h_stats) {
    if (!s) { set_error("fr_solver_run: null solver"); return FR_ERR_ARG; }
    cudaStream_t st = (cudaStream_t)stream;
    FR_TRY(reset_ctl(s, st));
    if (s->small) {
        if (s->fp32) k_solve_small<float><<<1, SMALL_NT, 0, st>>>(s->af);
        else k_solve_small<double><<<1, SMALL_NT, 0, st>>>(s->ad);
    } else {
        FR_CUDA(cudaGraphLaunch(s->exec, st));
    }
    FR_CUDA(cudaGetLastError());
    // exact sum |F| after the loop (the stopping rule of engine.py:290-293),
    // stream-ordered into the control block; one host sync for all stats
    FR_TRY(abs_sum_async(s->n, s->fp32 ? (void *)s->af.F : (void *)s->ad.F, s->fp32, &s->ctl->exact, st));
    fr_solve_stats hs;
    double exact = 0.0;
    FR_TRY(read_stats(s, st, &hs, &exact));
    hs.residual = exact;
    if (h_stats) *h_stats = hs;
    const double thr = s->cfg.target_error * (1.0 - s->cfg.damping);
    const long long cap = s->cfg.max_sweeps > 0 ? s->cfg.max_sweeps : 1000000;
    // an explicit budget (max_sweeps / max_diffusions) is a normal stop, like the
    // reference's max_diffusions (engine.py:294-295); only the implicit cap is an error
    const bool explicit_budget = s->cfg.max_sweeps > 0 || s->cfg.max_diffusions > 0;
    if (exact > thr && hs.sweeps >= cap && !explicit_budget) {
        set_error("no convergence within %lld sweeps (bound %.3g > target %.3g)", cap,
                  exact / (1.0 - s->cfg.damping), s->cfg.target_error);
        return FR_ERR_NO_CONVERGENCE;
    }
    return FR_OK;
}

template <typename FT>
static int run_profiled(fr_solver *s, SweepArgs<FT> a, cudaStream_t st, fr_solve_stats *h_stats, double *ms,
                        int64_t *launches) {
    a.in_graph = 0;
    a.hub_defer = 0;  // host-launched sweeps push the hub rows after each sweep (k_push_block)
    int nparts = s->sel_grid, nparts_sw = s->sweep_grid;
    FR_TRY(reset_ctl(s, st));
    if (s->small) {  // one launch: all of it is class 0
        for (int k = 0; k < 5; k++) { ms[k] = 0.0; launches[k] = 0; }
        cudaEvent_t e0, e1;
        FR_CUDA(cudaEventCreate(&e0));
        FR_CUDA(cudaEventCreate(&e1));
        FR_CUDA(cudaEventRecord(e0, st));
        k_solve_small<FT><<<1, SMALL_NT, 0, st>>>(a);
        FR_CUDA(cudaEventRecord(e1, st));
        FR_CUDA(cudaGetLastError());
        FR_CUDA(cudaEventSynchronize(e1));
        float t = 0.f;
        FR_CUDA(cudaEventElapsedTime(&t, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        ms[0] = t;
        launches[0] = 1;
        fr_solve_stats hs;
        FR_TRY(read_stats(s, st, &hs));
        double exact = 0.0;
        FR_TRY(fr_abs_sum(s->n, (void *)a.F, s->fp32, &exact, (void *)st));
        hs.residual = exact;
        if (h_stats) *h_stats = hs;
        return FR_OK;
    }
    k_mass_partials<FT><<<s->sel_grid, SEL_NT, 0, st>>>(a, 0);
    k_prologue<FT><<<1, FIN_NT, 0, st>>>(a, nparts);
    FR_CUDA(cudaGetLastError());
    cudaEvent_t ev[6];
    for (int i = 0; i < 6; i++) FR_CUDA(cudaEventCreate(&ev[i]));
    for (int k = 0; k < 5; k++) { ms[k] = 0.0; launches[k] = 0; }
    u32 stop = 0;
    FR_CUDA(cudaMemcpyAsync(&stop, &s->ctl->stop, sizeof(u32), cudaMemcpyDeviceToHost, st));
    FR_CUDA(cudaStreamSynchronize(st));
    const bool fused = fused_like(a.path);
    while (!stop) {
        // kernel classes: 0 select/sweep, 1 thread-bin push, 2 warp-bin push, 3 block-bin push, 4 finalize
        FR_CUDA(cudaEventRecord(ev[0], st));
        if (fused) launch_sweep<FT>(a, s->sweep_grid, st);
        else k_select<FT><<<s->sel_grid, SEL_NT, 0, st>>>(a);
        FR_CUDA(cudaEventRecord(ev[1], st));
        if (!fused) k_push_thread<FT><<<s->thread_grid, 256, 0, st>>>(a);
        FR_CUDA(cudaEventRecord(ev[2], st));
        if (!fused) k_push_warp<FT><<<s->warp_grid, 256, 0, st>>>(a);
        FR_CUDA(cudaEventRecord(ev[3], st));
        k_push_block<FT><<<s->block_grid, BLK_NT, 0, st>>>(a);
        FR_CUDA(cudaEventRecord(ev[4], st));
        k_fold<FT><<<s->fold_grid, 256, 0, st>>>(a);
        k_finalize<FT><<<1, FIN_NT, 0, st>>>(a, fused ? nparts_sw : nparts);
        if (fused) {
            k_mass_partials<FT><<<s->sel_grid, SEL_NT, 0, st>>>(a, 1);
            k_mass_check<FT><<<1, FIN_NT, 0, st>>>(a, nparts);
        }
        FR_CUDA(cudaEventRecord(ev[5], st));
        FR_CUDA(cudaGetLastError());
        FR_CUDA(cudaMemcpyAsync(&stop, &s->ctl->stop, sizeof(u32), cudaMemcpyDeviceToHost, st));
        FR_CUDA(cudaStreamSynchronize(st));
        for (int k = 0; k < 5; k++) {
            float t = 0.f;
            FR_CUDA(cudaEventElapsedTime(&t, ev[k], ev[k + 1]));
            ms[k] += t;
            if (fused ? (k == 0 || k >= 3) : true) launches[k] += 1;
        }
    }
    for (int i = 0; i < 6; i++) cudaEventDestroy(ev[i]);
    fr_solve_stats hs;
    FR_TRY(read_stats(s, st, &hs));
    double exact = 0.0;
    FR_TRY(fr_abs_sum(s->n, (void *)a.F, s->fp32, &exact, (void *)st));
    hs.residual = exact;
    if (h_stats) *h_stats = hs;
    return FR_OK;
}

extern "C" int fr_solver_run_profiled(fr_solver *s, void *stream, fr_solve_stats *h_stats, double *h_ms,
                                      int64_t *h_launches) {
    if (!s || !h_ms || !h_launches) { set_error("fr_solver_run_profiled: bad arguments"); return FR_ERR_ARG; }
    cudaStream_t st = (cudaStream_t)stream;
    return s->fp32 ? run_profiled<float>(s, s->af, st, h_stats, h_ms, h_launches)
                   : run_profiled<double>(s, s->ad, st, h_stats, h_ms, h_launches);
}

// Sampled run (engine.py:240-341 with reference=...): the same sweeps as
// fr_solver_run, launched one by one from the host (the single-block path
// samples inside its launch); after every sweep that brings the diffusion
// count to the next multiple of trace_every, the true L1 error of the
// normalized history against d_reference goes into the trace row's slot.
template <typename FT>
static int run_sampled(fr_solver *s, SweepArgs<FT> a, cudaStream_t st, const double *ref, long long every,
                       fr_solve_stats *h_stats) {
    FR_TRY(reset_ctl(s, st));
    a.hub_defer = 0;
    a.ref = ref;
    a.trace_every = every;
    a.true_err = s->true_err;
    a.in_graph = 0;
    if (s->small) {
        k_solve_small<FT><<<1, SMALL_NT, 0, st>>>(a);
        FR_CUDA(cudaGetLastError());
    } else {
        const int nparts = s->sel_grid, nparts_sw = s->sweep_grid;
        k_mass_partials<FT><<<s->sel_grid, SEL_NT, 0, st>>>(a, 0);
        k_prologue<FT><<<1, FIN_NT, 0, st>>>(a, nparts);
        FR_CUDA(cudaGetLastError());
        const bool fused = fused_like(a.path);
        struct { u32 stop; u64 diffusions, trace_len; } h;
        u64 next = (u64)every;
        for (;;) {
            FR_CUDA(cudaMemcpyAsync(&h.stop, &s->ctl->stop, sizeof(u32), cudaMemcpyDeviceToHost, st));
            FR_CUDA(cudaMemcpyAsync(&h.diffusions, &s->ctl->diffusions, sizeof(u64), cudaMemcpyDeviceToHost, st));
            FR_CUDA(cudaMemcpyAsync(&h.trace_len, &s->ctl->trace_len, sizeof(u64), cudaMemcpyDeviceToHost, st));
            FR_CUDA(cudaStreamSynchronize(st));
            if (h.trace_len > 0 && h.diffusions >= next) {
                next = h.diffusions + (u64)every;
                if ((long long)h.trace_len - 1 < s->trace_cap)
                    FR_TRY(l1_error_async(s->n, a.H, ref, s->true_err + (h.trace_len - 1), st));
            }
            if (h.stop) break;
            if (fused) launch_sweep<FT>(a, s->sweep_grid, st);
            else k_select<FT><<<s->sel_grid, SEL_NT, 0, st>>>(a);
            if (!fused) {
                k_push_thread<FT><<<s->thread_grid, 256, 0, st>>>(a);
                k_push_warp<FT><<<s->warp_grid, 256, 0, st>>>(a);
            }
            k_push_block<FT><<<s->block_grid, BLK_NT, 0, st>>>(a);
            k_fold<FT><<<s->fold_grid, 256, 0, st>>>(a);
            k_finalize<FT><<<1, FIN_NT, 0, st>>>(a, fused ? nparts_sw : nparts);
            if (fused) {
                k_mass_partials<FT><<<s->sel_grid, SEL_NT, 0, st>>>(a, 1);
                k_mass_check<FT><<<1, FIN_NT, 0, st>>>(a, nparts);
            }
            FR_CUDA(cudaGetLastError());
        }
    }
    FR_TRY(abs_sum_async(s->n, (const void *)a.F, s->fp32, &s->ctl->exact, st));
    fr_solve_stats hs;
    double exact = 0.0;
    FR_TRY(read_stats(s, st, &hs, &exact));
    hs.residual = exact;
    if (h_stats) *h_stats = hs;
    return FR_OK;
}

extern "C" int fr_solver_run_sampled(fr_solver *s, void *stream, const double *d_reference, int64_t trace_every,
                                     fr_solve_stats *h_stats) {
    if (!s || !d_reference || trace_every < 1) { set_error("fr_solver_run_sampled: bad arguments"); return FR_ERR_ARG; }
    if (s->trace_cap < 1) { set_error("fr_solver_run_sampled: the solver keeps no trace (trace_cap 0)"); return FR_ERR_ARG; }
    cudaStream_t st = (cudaStream_t)stream;
    if (!s->true_err) FR_TRY(pool_alloc((void **)&s->true_err, sizeof(double) * (size_t)s->trace_cap, st));
    FR_CUDA(cudaMemsetAsync(s->true_err, 0xFF, sizeof(double) * (size_t)s->trace_cap, st));  // all-ones = NaN
    return s->fp32 ? run_sampled<float>(s, s->af, st, d_reference, trace_every, h_stats)
                   : run_sampled<double>(s, s->ad, st, d_reference, trace_every, h_stats);
}

// True errors of the last sampled run, one per trace row (NaN: not sampled).
extern "C" int fr_solver_trace_errors(fr_solver *s, double *h_err, int64_t cap, void *stream) {
    if (!s || !h_err) { set_error("fr_solver_trace_errors: bad arguments"); return FR_ERR_ARG; }
    cudaStream_t st = (cudaStream_t)stream;
    const long long k = std::min<long long>(cap, s->trace_cap);
    if (!s->true_err) {
        for (long long i = 0; i < cap; i++) h_err[i] = NAN;
        return FR_OK;
    }
    if (k > 0) {
        FR_CUDA(cudaMemcpyAsync(h_err, s->true_err, sizeof(double) * (size_t)k, cudaMemcpyDeviceToHost, st));
        FR_CUDA(cudaStreamSynchronize(st));
    }
    for (long long i = k; i < cap; i++) h_err[i] = NAN;
    return FR_OK;
}

extern "C" int fr_solver_trace(fr_solver *s, fr_trace_row *h_rows, int64_t cap, int64_t *h_len, void *stream) {
    if (!s) { set_error("fr_solver_trace: null solver"); return FR_ERR_ARG; }
    cudaStream_t st = (cudaStream_t)stream;
    SolveCtl c;
    FR_CUDA(cudaMemcpyAsync(&c, s->ctl, sizeof(c), cudaMemcpyDeviceToHost, st));
    FR_CUDA(cudaStreamSynchronize(st));
    long long len = (long long)std::min<u64>(c.trace_len, (u64)s->trace_cap);
    if (h_len) *h_len = (int64_t)c.trace_len;
    long long k = std::min<long long>(len, cap);
    if (k > 0 && h_rows) {
        FR_CUDA(cudaMemcpyAsync(h_rows, s->trace, sizeof(fr_trace_row) * (size_t)k, cudaMemcpyDeviceToHost, st));
        FR_CUDA(cudaStreamSynchronize(st));
    }
    return FR_OK;
}

extern "C" int fr_solver_destroy(fr_solver *s) {
    if (!s) return FR_OK;
    if (s->exec) cudaGraphExecDestroy(s->exec);
    if (s->graph) cudaGraphDestroy(s->graph);
    // stream-ordered frees on the creation stream (callers destroy a solver
    // only after the work that uses it has completed)
    cudaStream_t st = s->stream;
    pool_free(s->ctl, st);
    pool_free(s->trace, st);
    pool_free(s->qnode_buf, st);
    pool_free(s->qval_buf, st);
    pool_free(s->parts, st);
    pool_free(s->parts64, st);
    pool_free(s->tgt_enc, st);
    pool_free(s->off32, st);
    pool_free(s->slot_node, st);
    pool_free(s->fw_buf, st);
    pool_free(s->true_err, st);
    delete s;
    return FR_OK;
}
