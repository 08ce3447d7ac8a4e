// fr_diffuse.cu -- data-parallel threshold-sweep D-iteration on the device.
//
// Reference semantics: engine.py:240-341 run() driving the ALGO-REF diffusion
// step (engine.py:315-329; PAPER sec. 2.2 / 3.3) under a node-selection rule
// (sched.py).  Because H_n + F_n = F_0 + dP H_n holds for ANY selection order
// (PAPER Theorem 3.1), a whole frontier of nodes can diffuse at once.  One
// sweep is:
//
//   S  k_select      read F once (coalesced), fused exact L1 mass of F, max
//                    score, and for every node with |f| (x weight) >= theta:
//                    F[i] = 0, H[i] += f (swap done in registers), absorbed
//                    mass, and a degree-binned enqueue (ballot/popc-free:
//                    one packed block scan per tile, 3 atomics per tile)
//   P  k_push_thread thread per node    (deg <= thread_max_degree)
//      k_push_warp   warp per node      (128-bit coalesced column loads)
//      k_push_block  block per hub node (adjacency staged into shared memory
//                    by cp.async.bulk, 4-stage mbarrier pipeline)
//                    all three: red.global.add of f*d/deg into F
//   F  k_finalize    fixed-order reduction of the block partials (bit-
//                    reproducible residual), counters, trace row, theta
//                    schedule, and the loop condition for the graph.
//
// The sweep loop is a CUDA-graph while-node: the host launches one graph per
// solve and waits once; there is no per-sweep host round trip.
#include <math.h>

#include <algorithm>
#include <vector>

#include "fr_common.cuh"

namespace fr {

static constexpr int SEL_NT = 256;
static constexpr int SEL_IT = 4;
static constexpr long long SEL_TILE = SEL_NT * SEL_IT;
static constexpr int FIN_NT = 256;
static constexpr int BLK_NT = 512;
static constexpr int BLK_CHUNK = 2048;  // uint32 column indices per stage (8 KB)
static constexpr int BLK_STAGES = 4;

struct SolveCtl {
    double theta;       // threshold of the next sweep
    double residual;    // mass - absorbed after the last sweep
    double last_max;    // max score seen by the last select pass
    double mass0;       // exact mass at the start of the solve
    u64 diffusions, steps, sweeps;
    u64 trace_len;
    u32 qcount[3];
    u32 stop;
};

template <typename FT>
struct SweepArgs {
    FT *F;
    double *H;
    const u64 *off;
    const u32 *tgt;
    const double *weight;  // score multiplier (op/op2) or null
    SolveCtl *ctl;
    u32 *qnode[3];
    FT *qval[3];
    double *part_mass, *part_abs, *part_max;
    u64 *part_steps, *part_sel;
    fr_trace_row *trace;
    long long n;
    long long trace_cap;
    long long max_sweeps;
    long long max_diffusions;
    double d, thr, decay, rand_frac;
    u32 t0, t2;  // deg <= t0 -> thread bin; deg >= t2 -> block bin
    int select, policy;
    u32 seed;
    int in_graph;
    cudaGraphConditionalHandle cond;
};

__device__ __forceinline__ u64 hmix(u64 z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// ------------------------------------------------------------------ prologue
template <typename FT>
__global__ void __launch_bounds__(SEL_NT) k_mass_partials(SweepArgs<FT> a) {
    __shared__ double sm[SEL_NT / 32];
    double mass = 0.0, mx = 0.0;
    for (long long i = blockIdx.x * (long long)SEL_NT + threadIdx.x; i < a.n; i += (long long)gridDim.x * SEL_NT) {
        const double af = fabs((double)a.F[i]);
        mass += af;
        mx = fmax(mx, a.weight ? af * a.weight[i] : af);
    }
    const double bm = block_sum<SEL_NT>(mass, sm);
    const double bx = block_max<SEL_NT>(mx, sm);
    if (threadIdx.x == 0) {
        a.part_mass[blockIdx.x] = bm;
        a.part_max[blockIdx.x] = bx;
    }
}

template <typename FT>
__global__ void __launch_bounds__(FIN_NT) k_prologue(SweepArgs<FT> a, int nparts) {
    __shared__ double sm[FIN_NT / 32];
    double mass = 0.0, mx = 0.0;
    for (int p = threadIdx.x; p < nparts; p += FIN_NT) {
        mass += a.part_mass[p];
        mx = fmax(mx, a.part_max[p]);
    }
    mass = block_sum<FIN_NT>(mass, sm);
    mx = block_max<FIN_NT>(mx, sm);
    if (threadIdx.x == 0) {
        SolveCtl *c = a.ctl;
        c->theta = mx;  // sched.py:89-90: threshold starts at the max fluid
        c->last_max = mx;
        c->residual = mass;
        c->mass0 = mass;
        c->qcount[0] = c->qcount[1] = c->qcount[2] = 0;
        c->stop = (mass <= a.thr || mass == 0.0) ? 1u : 0u;
        if (a.in_graph) cudaGraphSetConditional(a.cond, c->stop ? 0u : 1u);
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
                const double score = a.weight ? af * a.weight[i] : af;
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
    const u32 cnt = a.ctl->qcount[0];
    const u32 *__restrict__ qn = a.qnode[0];
    const FT *__restrict__ qv = a.qval[0];
    for (u32 e = blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += gridDim.x * blockDim.x) {
        const u32 node = qn[e];
        const FT v = qv[e];
        const u64 lo = a.off[node], hi = a.off[node + 1];
        for (u64 k = lo; k < hi; k++) red_add(a.F + __ldg(a.tgt + k), v);
    }
}

template <typename FT>
__global__ void __launch_bounds__(256) k_push_warp(SweepArgs<FT> a) {
    const u32 cnt = a.ctl->qcount[1];
    const int lane = threadIdx.x & 31;
    const u32 nwarps = gridDim.x * (blockDim.x >> 5);
    const uint4 *tgt4 = reinterpret_cast<const uint4 *>(a.tgt);
    for (u32 e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); e < cnt; e += nwarps) {
        const u32 node = a.qnode[1][e];
        const FT v = a.qval[1][e];
        const u64 lo = a.off[node], hi = a.off[node + 1];
        const u64 a0 = min(hi, (lo + 3) & ~3ull);
        const u64 a1 = max(a0, hi & ~3ull);
        if (lo + lane < a0) red_add(a.F + __ldg(a.tgt + lo + lane), v);
        if (a1 + lane < hi) red_add(a.F + __ldg(a.tgt + a1 + lane), v);
        for (u64 q = (a0 >> 2) + lane; q < (a1 >> 2); q += 32) {
            const uint4 t = ld_stream_u4(tgt4 + q);
            red_add(a.F + t.x, v);
            red_add(a.F + t.y, v);
            red_add(a.F + t.z, v);
            red_add(a.F + t.w, v);
        }
    }
}

__device__ __forceinline__ u32 smem_u32(const void *p) { return (u32)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(u64 *bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u64 *bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64 *bar, u32 parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "FR_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra FR_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, u32 bytes, u64 *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Block per hub node.  The 16-byte-aligned body of the adjacency row streams
// through a BLK_STAGES-deep ring of shared-memory chunks filled by the bulk
// copy engine (cp.async.bulk -> UBLKCP), so column-index loads overlap the
// red.global.add scatter of the previous chunks.
template <typename FT>
__global__ void __launch_bounds__(BLK_NT) k_push_block(SweepArgs<FT> a) {
    __shared__ __align__(128) u32 stage[BLK_STAGES][BLK_CHUNK];
    __shared__ __align__(8) u64 bar[BLK_STAGES];
    const u32 cnt = a.ctl->qcount[2];
    if (blockIdx.x >= cnt) return;
    if (threadIdx.x == 0) {
        for (int s = 0; s < BLK_STAGES; s++) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    u32 seq = 0;  // chunks consumed by this block so far (slot = seq % STAGES, parity = (seq / STAGES) & 1)
    for (u32 e = blockIdx.x; e < cnt; e += gridDim.x) {
        const u32 node = a.qnode[2][e];
        const FT v = a.qval[2][e];
        const u64 lo = a.off[node], hi = a.off[node + 1];
        const u64 a0 = min(hi, (lo + 3) & ~3ull);
        const u64 a1 = max(a0, hi & ~3ull);
        if (lo + threadIdx.x < a0) red_add(a.F + __ldg(a.tgt + lo + threadIdx.x), v);
        if (a1 + threadIdx.x < hi) red_add(a.F + __ldg(a.tgt + a1 + threadIdx.x), v);
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
            for (u32 k = threadIdx.x; k < len; k += BLK_NT) red_add(a.F + sp[k], v);
            __syncthreads();  // slot s is free for the next bulk load
        }
        seq += nch;
    }
}

// ------------------------------------------------------------------ F: finalize
template <typename FT>
__global__ void __launch_bounds__(FIN_NT) k_finalize(SweepArgs<FT> a, int nparts) {
    __shared__ double sm[FIN_NT / 32];
    __shared__ u64 sm64[FIN_NT / 32];
    double mass = 0.0, ab = 0.0, mx = 0.0;
    u64 steps = 0, nsel = 0;
    for (int p = threadIdx.x; p < nparts; p += FIN_NT) {
        mass += a.part_mass[p];
        ab += a.part_abs[p];
        mx = fmax(mx, a.part_max[p]);
        steps += a.part_steps[p];
        nsel += a.part_sel[p];
    }
    mass = block_sum<FIN_NT>(mass, sm);
    ab = block_sum<FIN_NT>(ab, sm);
    mx = block_max<FIN_NT>(mx, sm);
    steps = block_sum_u64<FIN_NT>(steps, sm64);
    nsel = block_sum_u64<FIN_NT>(nsel, sm64);
    if (threadIdx.x != 0) return;
    SolveCtl *c = a.ctl;
    const double residual = nsel ? mass - ab : mass;
    const double theta_used = c->theta;
    c->residual = residual;
    c->diffusions += nsel;
    c->steps += steps;
    c->sweeps += 1;
    c->last_max = mx;
    if (a.trace && c->trace_len < (u64)a.trace_cap) {
        fr_trace_row &r = a.trace[c->trace_len];
        r.elementary_steps = (int64_t)c->steps;
        r.diffusions = (int64_t)c->diffusions;
        r.sweeps = (int64_t)c->sweeps;
        r.residual = residual;
        r.theta = theta_used;
    }
    c->trace_len += 1;
    // theta schedule
    double th = theta_used;
    if (a.select == FR_SELECT_MAX) {
        th = a.decay * mx;
    } else if (a.policy == FR_THETA_GEOMETRIC) {
        th *= a.decay;
    }
    // a sweep that found nothing: decay until the largest fluid qualifies, as
    // repeated empty passes of the reference sweep scheduler would (sched.py:101-108)
    if (nsel == 0 && mx > 0.0)
        while (th > mx) th *= a.decay;
    c->theta = th;
    c->qcount[0] = c->qcount[1] = c->qcount[2] = 0;
    const bool done = residual <= a.thr || mass == 0.0 || (long long)c->sweeps >= a.max_sweeps ||
                      (a.max_diffusions > 0 && (long long)c->diffusions >= a.max_diffusions);
    c->stop = done ? 1u : 0u;
    if (a.in_graph) cudaGraphSetConditional(a.cond, done ? 0u : 1u);
}

}  // namespace fr

using namespace fr;

// ====================================================================== host side
struct fr_solver {
    long long n, m;
    int fp32;
    int sel_grid, thread_grid, warp_grid, block_grid;
    SolveCtl *ctl;
    fr_trace_row *trace;
    long long trace_cap;
    void *qnode_buf, *qval_buf;
    double *parts;
    u64 *parts64;
    fr_solver_config cfg;
    cudaGraph_t graph;
    cudaGraphExec_t exec;
    // both instantiations are kept; only one is used per solver
    SweepArgs<double> ad;
    SweepArgs<float> af;
};

template <typename FT>
static int add_kernel(cudaGraph_t g, cudaGraphNode_t *node, const cudaGraphNode_t *deps, size_t ndeps, void *func,
                      int grid, int block, void **args) {
    cudaKernelNodeParams p = {};
    p.func = func;
    p.gridDim = dim3((unsigned)grid);
    p.blockDim = dim3((unsigned)block);
    p.sharedMemBytes = 0;
    p.kernelParams = args;
    FR_CUDA(cudaGraphAddKernelNode(node, g, deps, ndeps, &p));
    return FR_OK;
}

template <typename FT>
static int build_graph(fr_solver *s, SweepArgs<FT> &a) {
    FR_CUDA(cudaGraphCreate(&s->graph, 0));
    FR_CUDA(cudaGraphConditionalHandleCreate(&a.cond, s->graph, 0, 0));
    a.in_graph = 1;
    int nparts = s->sel_grid;
    static void *dummy;
    (void)dummy;
    // prologue
    void *args_a[] = {&a};
    void *args_an[] = {&a, &nparts};
    cudaGraphNode_t n_mass, n_pro, n_while;
    FR_TRY(add_kernel<FT>(s->graph, &n_mass, nullptr, 0, (void *)k_mass_partials<FT>, s->sel_grid, SEL_NT, args_a));
    FR_TRY(add_kernel<FT>(s->graph, &n_pro, &n_mass, 1, (void *)k_prologue<FT>, 1, FIN_NT, args_an));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = a.cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    FR_CUDA(cudaGraphAddNode(&n_while, s->graph, &n_pro, 1, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    cudaGraphNode_t n_sel, n_p[3], n_fin;
    FR_TRY(add_kernel<FT>(body, &n_sel, nullptr, 0, (void *)k_select<FT>, s->sel_grid, SEL_NT, args_a));
    FR_TRY(add_kernel<FT>(body, &n_p[0], &n_sel, 1, (void *)k_push_thread<FT>, s->thread_grid, 256, args_a));
    FR_TRY(add_kernel<FT>(body, &n_p[1], &n_sel, 1, (void *)k_push_warp<FT>, s->warp_grid, 256, args_a));
    FR_TRY(add_kernel<FT>(body, &n_p[2], &n_sel, 1, (void *)k_push_block<FT>, s->block_grid, BLK_NT, args_a));
    FR_TRY(add_kernel<FT>(body, &n_fin, n_p, 3, (void *)k_finalize<FT>, 1, FIN_NT, args_an));
    FR_CUDA(cudaGraphInstantiate(&s->exec, s->graph, 0));
    return FR_OK;
}

template <typename FT>
static int occupancy_grid(void *func, int threads, int sms) {
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, func, threads, 0) != cudaSuccess || per < 1) per = 1;
    return per * sms;
}

template <typename FT>
static int setup(fr_solver *s, SweepArgs<FT> &a, const int64_t *d_offsets, const uint32_t *d_targets,
                 const double *d_w, void *d_fluid, double *d_history) {
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
    a.trace = s->trace;
    a.trace_cap = s->trace_cap;
    a.max_sweeps = c.max_sweeps > 0 ? c.max_sweeps : 1000000;
    a.max_diffusions = c.max_diffusions;
    a.d = c.damping;
    a.thr = c.target_error * (1.0 - c.damping);
    a.decay = c.decay;
    a.rand_frac = c.rand_frac;
    a.t0 = c.thread_max_degree > 0 ? (u32)c.thread_max_degree : 8u;
    a.t2 = c.block_min_degree > 0 ? (u32)c.block_min_degree : 2048u;
    if (a.t2 <= a.t0) a.t2 = a.t0 + 1;
    a.select = c.select;
    a.policy = c.policy;
    a.seed = c.seed;
    // queues: a selected node lands in exactly one bin
    const long long n = s->n, m = s->m;
    const long long cap0 = n;
    const long long cap1 = std::min<long long>(n, m / ((long long)a.t0 + 1) + 1);
    const long long cap2 = std::min<long long>(n, m / (long long)a.t2 + 1);
    FR_CUDA(cudaMalloc(&s->qnode_buf, sizeof(u32) * (size_t)(cap0 + cap1 + cap2 + 3)));
    FR_CUDA(cudaMalloc(&s->qval_buf, sizeof(FT) * (size_t)(cap0 + cap1 + cap2 + 3)));
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
    const int P = s->sel_grid;
    FR_CUDA(cudaMalloc(&s->parts, sizeof(double) * 3 * (size_t)P));
    FR_CUDA(cudaMalloc(&s->parts64, sizeof(u64) * 2 * (size_t)P));
    a.part_mass = s->parts;
    a.part_abs = s->parts + P;
    a.part_max = s->parts + 2 * P;
    a.part_steps = s->parts64;
    a.part_sel = s->parts64 + P;
    return build_graph<FT>(s, a);
}

extern "C" int fr_solver_create(int64_t n, int64_t m, const int64_t *d_offsets, const uint32_t *d_targets,
                                const double *d_score_weight, void *d_fluid, double *d_history,
                                const fr_solver_config *cfg, int64_t trace_cap, void *stream, fr_solver **out) {
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
        cfg->policy > FR_THETA_MASS) {
        set_error("fr_solver_create: unknown select rule or theta policy");
        return FR_ERR_ARG;
    }
    if ((cfg->select == FR_SELECT_OP || cfg->select == FR_SELECT_OP2) && !d_score_weight) {
        set_error("fr_solver_create: op/op2 need per-node score weights");
        return FR_ERR_ARG;
    }
    (void)stream;
    fr_solver *s = new fr_solver();
    s->n = n;
    s->m = m;
    s->cfg = *cfg;
    s->fp32 = cfg->fluid_fp32 ? 1 : 0;
    s->trace_cap = trace_cap > 0 ? trace_cap : 0;
    int rc = FR_OK;
    do {
        if (cudaMalloc(&s->ctl, sizeof(SolveCtl)) != cudaSuccess) { rc = cuda_fail(cudaGetLastError(), "cudaMalloc(ctl)", __FILE__, __LINE__); break; }
        if (s->trace_cap &&
            cudaMalloc(&s->trace, sizeof(fr_trace_row) * (size_t)s->trace_cap) != cudaSuccess) {
            rc = cuda_fail(cudaGetLastError(), "cudaMalloc(trace)", __FILE__, __LINE__);
            break;
        }
        rc = s->fp32 ? setup<float>(s, s->af, d_offsets, d_targets, d_score_weight, d_fluid, d_history)
                     : setup<double>(s, s->ad, d_offsets, d_targets, d_score_weight, d_fluid, d_history);
    } while (0);
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

static int read_stats(fr_solver *s, cudaStream_t st, fr_solve_stats *h) {
    SolveCtl c;
    FR_CUDA(cudaMemcpyAsync(&c, s->ctl, sizeof(c), cudaMemcpyDeviceToHost, st));
    FR_CUDA(cudaStreamSynchronize(st));
    if (h) {
        h->diffusions = (int64_t)c.diffusions;
        h->elementary_steps = (int64_t)c.steps;
        h->sweeps = (int64_t)c.sweeps;
        h->residual = c.residual;
        h->theta = c.theta;
        h->trace_len = (int64_t)c.trace_len;
    }
    return FR_OK;
}

extern "C" int fr_solver_run(fr_solver *s, void *stream, fr_solve_stats *h_stats) {
    if (!s) { set_error("fr_solver_run: null solver"); return FR_ERR_ARG; }
    cudaStream_t st = (cudaStream_t)stream;
    FR_TRY(reset_ctl(s, st));
    FR_CUDA(cudaGraphLaunch(s->exec, st));
    FR_CUDA(cudaGetLastError());
    fr_solve_stats hs;
    FR_TRY(read_stats(s, st, &hs));
    // exact check of the stopping rule (engine.py:290-293)
    double exact = 0.0;
    FR_TRY(fr_abs_sum(s->n, s->fp32 ? (void *)s->af.F : (void *)s->ad.F, s->fp32, &exact, stream));
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
    int nparts = s->sel_grid;
    FR_TRY(reset_ctl(s, st));
    k_mass_partials<FT><<<s->sel_grid, SEL_NT, 0, st>>>(a);
    k_prologue<FT><<<1, FIN_NT, 0, st>>>(a, nparts);
    FR_CUDA(cudaGetLastError());
    cudaEvent_t ev[6];
    for (int i = 0; i < 6; i++) FR_CUDA(cudaEventCreate(&ev[i]));
    for (int k = 0; k < 5; k++) { ms[k] = 0.0; launches[k] = 0; }
    u32 stop = 0;
    FR_CUDA(cudaMemcpyAsync(&stop, &s->ctl->stop, sizeof(u32), cudaMemcpyDeviceToHost, st));
    FR_CUDA(cudaStreamSynchronize(st));
    while (!stop) {
        FR_CUDA(cudaEventRecord(ev[0], st));
        k_select<FT><<<s->sel_grid, SEL_NT, 0, st>>>(a);
        FR_CUDA(cudaEventRecord(ev[1], st));
        k_push_thread<FT><<<s->thread_grid, 256, 0, st>>>(a);
        FR_CUDA(cudaEventRecord(ev[2], st));
        k_push_warp<FT><<<s->warp_grid, 256, 0, st>>>(a);
        FR_CUDA(cudaEventRecord(ev[3], st));
        k_push_block<FT><<<s->block_grid, BLK_NT, 0, st>>>(a);
        FR_CUDA(cudaEventRecord(ev[4], st));
        k_finalize<FT><<<1, FIN_NT, 0, st>>>(a, nparts);
        FR_CUDA(cudaEventRecord(ev[5], st));
        FR_CUDA(cudaGetLastError());
        FR_CUDA(cudaMemcpyAsync(&stop, &s->ctl->stop, sizeof(u32), cudaMemcpyDeviceToHost, st));
        FR_CUDA(cudaStreamSynchronize(st));
        for (int k = 0; k < 5; k++) {
            float t = 0.f;
            FR_CUDA(cudaEventElapsedTime(&t, ev[k], ev[k + 1]));
            ms[k] += t;
            launches[k] += 1;
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
    cudaFree(s->ctl);
    cudaFree(s->trace);
    cudaFree(s->qnode_buf);
    cudaFree(s->qval_buf);
    cudaFree(s->parts);
    cudaFree(s->parts64);
    delete s;
    return FR_OK;
}
