// fr_spmv.cu -- power iteration (MAT-ITER), the in-repo comparison solver.
//
// baseline.py:20-56: x <- v; repeat y = d*P*x + (1-d)*v; y += (1 - sum y)*v;
// diff = |y - x|_1; x = y; until diff*d/(1-d) <= target.  P*x is a pull SpMV
// over the transposed CSR (rows = targets, columns = sources ascending, the
// reference's graph.to_matrix(), graph.py:158-165):
//   s_i = sum_{j in in(i)} z_j,   z_j = x_j / outdeg_j (0 for dangling j)
// Short rows: warp per tile of 32 rows over the tile's compacted edge space
// (k_pi_rows<false>).  Hub rows (in-degree > LONG_ROW: the Zipf in-degree hubs,
// whose parents are spread over all ids) are regrouped by SOURCE BLOCK: hub row
// h's sources are ascending, so its parents in block b (2^PI_SB ids, 2 MB of z)
// are one contiguous slice of in_src, "row (b, h)".  The (b, h) rows are
// processed block-major (k_pi_rows<true> and, for slices longer than LONG_ROW,
// k_pi_segs), so the warps in flight gather from a few blocks' worth of z that
// stays in L2 -- instead of one random 64 B DRAM burst per 8 B gathered -- and
// add their sums into the hub's s (25k hubs on config 5: L2-resident).
// The iteration loop is a CUDA-graph while-node (no host round trip).
#include <math.h>

#include <algorithm>
#include <vector>

#include "fr_common.cuh"

namespace fr {

static constexpr int PI_NT = 256;
static constexpr u64 LONG_ROW = 1024;
static constexpr u64 SEG = 256;  // long-slice segment: the segments in flight span a few source blocks of z (L2)
#ifndef FR_PI_SB
#define FR_PI_SB 18
#endif
static constexpr int PI_SB = FR_PI_SB;  // source block: 2^18 ids = 2 MB of z

#ifndef FR_PI_SEGS
#define FR_PI_SEGS 16
#endif
static constexpr int PI_SEGS = FR_PI_SEGS;  // in-order fronts of the row kernels
static constexpr int PI_PAD = 16;           // u64 per counter: one 128 B line each
static constexpr u32 PI_CHUNK = 4;          // tiles per claim

struct PiCtl {
    double c;       // teleport re-injection 1 - sum(y) of the coming iteration
    double diff;
    double sum_v;
    u64 iters;
    u32 stop;
    u32 pad;
    u64 seg_next[2][PI_SEGS * PI_PAD];  // row kernels (short, hub): next tile of each front
};

// zero the tile counters of both row kernels (one block)
__device__ __forceinline__ void reset_fronts(PiCtl *c) {
    for (int q = threadIdx.x; q < 2 * PI_SEGS; q += blockDim.x) c->seg_next[q / PI_SEGS][(q % PI_SEGS) * PI_PAD] = 0;
}

struct PiArgs {
    long long n;
    const u64 *in_off;
    const u32 *in_src;
    const double *inv;  // 1/outdeg or 0
    const double *v;    // teleport (null: uniform v_const)
    double v_const;
    double *x;
    double *zb[2];      // z = x/outdeg, double-buffered: iteration k gathers zb[k & 1], writes zb[(k + 1) & 1]
    double *s_hub;      // [nhub] in-sums of the hub rows, added by the slice kernels
    // hub rows regrouped by source block: row (b, h) = b * nhub + h is the slice
    // hub_src[h_lo[r], h_lo[r] + h_cnt[r]) of hub row hub_node[h] -- a private copy of
    // the hub rows' in-edges stored block-major, so the slices of consecutive (b, h)
    // rows are contiguous (slices longer than LONG_ROW sit after them as segments)
    const u32 *hub_src;
    const u64 *h_lo;
    const u32 *h_cnt, *hub_node;
    long long h_rows;
    u32 nhub;
    const u64 *seg_row, *seg_lo, *seg_hi;  // (b, h) slices longer than LONG_ROW, seg_row = hub index h
    long long nseg;
    double *part_d, *part_nd;  // per-block |y - x|_1 and sum of y over non-dangling nodes
    int nparts;                // partial slots of the row kernel; the hub update's blocks follow
    int row_grid;              // blocks of the short-row kernel in use (<= nparts)
    int hub_grid;
    PiCtl *ctl;
    double d, target;
    long long max_iter;
    int in_graph;
    cudaGraphConditionalHandle cond;
};

__device__ __forceinline__ const double *z_rd(const PiArgs &a, u64 it) { return a.zb[it & 1]; }
__device__ __forceinline__ double *z_wr(const PiArgs &a, u64 it) { return a.zb[(it + 1) & 1]; }

// baseline.py:41-43 for row i, with the re-injection c = 1 - sum(y) known before the
// product: sum(P x) = sum of x over the non-dangling nodes (every column of P sums
// to 1), so c follows from the previous update (k_pi_check) and the update is
// fused into the row kernels (no separate pass over s, x, v, 1/deg)
// (xi, w, vi: the row's x, 1/outdeg and teleport, loaded by the caller ahead of time)
__device__ __forceinline__ void pi_update_row(const PiArgs &a, long long i, double s, double c, double *zw,
                                              double xi, double w, double vi, double &diff, double &nd) {
    double y = a.d * s + (1.0 - a.d) * vi;
    y += c * vi;
    diff += fabs(y - xi);
    a.x[i] = y;
    zw[i] = y * w;
    if (w != 0.0) nd += y;
}

__global__ void __launch_bounds__(PI_NT) k_pi_init(PiArgs a) {
    __shared__ double sm[PI_NT / 32];
    double nd = 0.0;
    for (long long i = blockIdx.x * (long long)PI_NT + threadIdx.x; i < a.n; i += (long long)gridDim.x * PI_NT) {
        const double xi = a.v ? a.v[i] : a.v_const;
        const double w = a.inv[i];
        a.x[i] = xi;
        a.zb[0][i] = xi * w;
        if (w != 0.0) nd += xi;
    }
    for (long long h = blockIdx.x * (long long)PI_NT + threadIdx.x; h < a.nhub; h += (long long)gridDim.x * PI_NT)
        a.s_hub[h] = 0.0;
    nd = block_sum<PI_NT>(nd, sm);
    if (threadIdx.x == 0) {
        a.part_nd[blockIdx.x] = nd;
        a.part_d[blockIdx.x] = 0.0;
    }
}

// c of the first iteration from the partials of k_pi_init (one block)
__global__ void __launch_bounds__(PI_NT) k_pi_start(PiArgs a) {
    __shared__ double sm[PI_NT / 32];
    double t = 0.0;
    for (int p = threadIdx.x; p < a.nparts; p += PI_NT) t += a.part_nd[p];
    t = block_sum<PI_NT>(t, sm);
    reset_fronts(a.ctl);
    if (threadIdx.x == 0) {
        a.ctl->c = 1.0 - (a.d * t + (1.0 - a.d) * a.ctl->sum_v);
        a.ctl->iters = 0;
        a.ctl->stop = 0;
        if (a.in_graph) cudaGraphSetConditional(a.cond, 1u);
    }
}

// Warp per tile of 32 consecutive rows; rows longer than LONG_ROW are skipped
// here (their slices add into s_hub, k_pi_hub_update finishes them).  The tile's
// short rows are contiguous ranges of in_src, so their concatenation (the tile's
// compacted edge space, E edges) is split into 32 equal contiguous chunks, one
// per lane: every lane streams its column indices in order with PI_UNROLL
// independent loads and gathers in flight, and adds its partial sum of a row to
// the row's shared-memory accumulator when it walks past the row's end.  Per-lane
// work is E/32 edges whatever the degree mix.  HUB = false: the row's update
// follows in the same pass; HUB = true: rows are (b, h) slices of hub_src and the
// sums go to s_hub[h].
#ifndef FR_PI_UNROLL
#define FR_PI_UNROLL 4
#endif
static constexpr int PI_UNROLL = FR_PI_UNROLL;
#ifndef FR_PI_MINB
#define FR_PI_MINB 4  // 4 blocks x 8 warps per SM: <= 64 registers
#endif
template <bool HUB, typename G>
__device__ __forceinline__ void pi_tile(const PiArgs &a, long long t, long long nrows, u32 *s_pre, u64 *s_lo,
                                        double *s_acc, G gather, double *zw, double c, double &diff, double &nd) {
    constexpr u32 FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const long long r = t * 32 + lane;
    const u32 *__restrict__ src = HUB ? a.hub_src : a.in_src;
    u64 lo = 0, deg = 0;
    bool hub_row = false;
    if (r < nrows) {
        if (HUB) {
            lo = a.h_lo[r];
            deg = a.h_cnt[r];
        } else {
            lo = a.in_off[r];
            deg = a.in_off[r + 1] - lo;
        }
        if (deg > LONG_ROW) {  // hub rows (short kernel) / long slices (k_pi_segs)
            deg = 0;
            hub_row = true;
        }
    }
    // the update's operands are loaded now, in flight with the gathers
    double xo = 0.0, wo = 0.0, vo = a.v_const;
    if (!HUB && r < nrows && !hub_row) {
        xo = a.x[r];
        wo = a.inv[r];
        if (a.v) vo = a.v[r];
    }
    u32 inc = (u32)deg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += y;
    }
    const u32 E = __shfl_sync(FULL, inc, 31);
    __syncwarp();
    s_pre[lane + 1] = inc;
    if (lane == 0) s_pre[0] = 0;
    s_lo[lane] = lo;
    s_acc[lane] = 0.0;
    __syncwarp();
    const u32 chunk = (E + 31) >> 5;
    u32 q = lane * chunk;
    const u32 qe = min(E, q + chunk);
    if (q < qe) {
        // the row holding edge q: the largest k with pre[k] <= q
        int k = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1)
            if (s_pre[k + step] <= q) k += step;
        u32 rend = s_pre[k + 1];
        u64 base = s_lo[k] - s_pre[k];  // src position of edge q' of row k: base + q'
        double acc = 0.0;
        // software pipeline: the column indices of the next batch are loaded
        // while the current batch's gathers are in flight (the load walk has
        // its own row cursor lk / lre / lbs, ahead of the accumulate cursor)
        int lk = k;
        u32 lre = rend;
        u64 lbs = base;
        u32 lq = q;  // next edge whose index is loaded
        auto load_batch = [&](u32 (&sv)[PI_UNROLL]) {
#pragma unroll
            for (int j = 0; j < PI_UNROLL; j++) {
                sv[j] = 0;
                if (lq < qe) {
                    while (lq >= lre) {
                        lk++;
                        lre = s_pre[lk + 1];
                        lbs = s_lo[lk] - s_pre[lk];
                    }
                    sv[j] = __ldg(src + lbs + lq);
                    lq++;
                }
            }
        };
        u32 srcA[PI_UNROLL], srcB[PI_UNROLL];
        load_batch(srcA);
        while (q < qe) {
            double zv[PI_UNROLL];
#pragma unroll
            for (int j = 0; j < PI_UNROLL; j++) zv[j] = q + j < qe ? gather(srcA[j]) : 0.0;
            load_batch(srcB);
#pragma unroll
            for (int j = 0; j < PI_UNROLL; j++) {
                if (q < qe) {
                    while (q >= rend) {  // left row k: hand its partial sum over
                        if (acc != 0.0) atomicAdd(&s_acc[k], acc);
                        acc = 0.0;
                        k++;
                        rend = s_pre[k + 1];
                    }
                    acc += zv[j];
                    q++;
                }
            }
#pragma unroll
            for (int j = 0; j < PI_UNROLL; j++) srcA[j] = srcB[j];
        }
        if (acc != 0.0) atomicAdd(&s_acc[k], acc);
    }
    __syncwarp();
    if (r < nrows) {
        const double v = s_acc[lane];
        if (HUB) {
            if (v != 0.0) atomicAdd(a.s_hub + (u64)r % a.nhub, v);
        } else if (!hub_row) {
            pi_update_row(a, r, v, c, zw, xo, wo, vo, diff, nd);
        }
    }
}

// Short rows (HUB = false) and hub slices (HUB = true), warp per 32-row tile:
// tiles are claimed in order from PI_SEGS contiguous fronts (PI_CHUNK per
// claim), so the rows in flight -- and the z lines they gather -- stay within a
// few narrow windows (a grid-stride walk lets the warps drift apart).
template <bool HUB>
__global__ void __launch_bounds__(PI_NT, FR_PI_MINB) k_pi_rows(PiArgs a) {
    constexpr u32 FULL = 0xffffffffu;
    constexpr int NW = PI_NT / 32;
    __shared__ u32 s_pre[NW][33];
    __shared__ u64 s_lo[NW][32];
    __shared__ double s_acc[NW][32];
    __shared__ double sm[NW];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long nrows = HUB ? a.h_rows : a.n;
    const long long ntiles = (nrows + 31) / 32;
    const long long seg_len = (ntiles + PI_SEGS - 1) / PI_SEGS;
    u64 *next = a.ctl->seg_next[HUB ? 1 : 0];
    int seg = (int)(((long long)blockIdx.x * NW + w) % PI_SEGS), misses = 0;
    long long t = 0, t_end = 0;
    const u64 it = a.ctl->iters;
    const double c = a.ctl->c;
    const double *__restrict__ z = z_rd(a, it);
    double *zw = z_wr(a, it);
    double diff = 0.0, nd = 0.0;
    for (;;) {
        if (t >= t_end) {
            bool got = false;
            while (misses < PI_SEGS) {
                u64 k = 0;
                if (lane == 0) k = atomicAdd(next + seg * PI_PAD, (u64)PI_CHUNK);
                k = __shfl_sync(FULL, k, 0);
                const long long s0 = seg * seg_len, s1 = min(ntiles, s0 + seg_len);
                if (s0 + (long long)k < s1) {
                    t = s0 + (long long)k;
                    t_end = min(s1, t + (long long)PI_CHUNK);
                    got = true;
                    break;
                }
                seg = (seg + 1) % PI_SEGS;
                misses++;
            }
            if (!got) break;
        }
        pi_tile<HUB>(a, t, nrows, s_pre[w], s_lo[w], s_acc[w], [&](u32 j) { return z[j]; }, zw, c, diff, nd);
        t++;
    }
    if (!HUB) {
        diff = block_sum<PI_NT>(diff, sm);
        nd = block_sum<PI_NT>(nd, sm);
        if (threadIdx.x == 0) {
            a.part_d[blockIdx.x] = diff;
            a.part_nd[blockIdx.x] = nd;
        }
    }
}

// Warp per segment of a long (b, h) slice.
__global__ void __launch_bounds__(PI_NT) k_pi_segs(PiArgs a) {
    const int lane = threadIdx.x & 31;
    const double *__restrict__ z = z_rd(a, a.ctl->iters);
    const long long nw = (long long)gridDim.x * (PI_NT / 32);
    for (long long q = blockIdx.x * (long long)(PI_NT / 32) + (threadIdx.x >> 5); q < a.nseg; q += nw) {
        const u64 lo = a.seg_lo[q], hi = a.seg_hi[q];
        double acc = 0.0;
        for (u64 k = lo + lane; k < hi; k += 32) acc += z[__ldg(a.hub_src + k)];
        acc = warp_sum(acc);
        if (lane == 0) atomicAdd(a.s_hub + a.seg_row[q], acc);
    }
}

// The hub rows' update once every slice has been added (and s_hub cleared for
// the next iteration).
__global__ void __launch_bounds__(PI_NT) k_pi_hub_update(PiArgs a) {
    __shared__ double sm[PI_NT / 32];
    const u64 it = a.ctl->iters;
    const double c = a.ctl->c;
    double *zw = z_wr(a, it);
    double diff = 0.0, nd = 0.0;
    for (long long h = blockIdx.x * (long long)PI_NT + threadIdx.x; h < a.nhub; h += (long long)gridDim.x * PI_NT) {
        const double s = a.s_hub[h];
        a.s_hub[h] = 0.0;
        const u32 i = a.hub_node[h];
        pi_update_row(a, i, s, c, zw, a.x[i], a.inv[i], a.v ? a.v[i] : a.v_const, diff, nd);
    }
    diff = block_sum<PI_NT>(diff, sm);
    nd = block_sum<PI_NT>(nd, sm);
    if (threadIdx.x == 0) {
        a.part_d[a.nparts + blockIdx.x] = diff;
        a.part_nd[a.nparts + blockIdx.x] = nd;
    }
}

__global__ void __launch_bounds__(PI_NT) k_pi_check(PiArgs a) {
    __shared__ double sm[PI_NT / 32];
    double t = 0.0, nd = 0.0;
    for (int p = threadIdx.x; p < a.row_grid + a.hub_grid; p += PI_NT) {
        const int q = p < a.row_grid ? p : a.nparts + (p - a.row_grid);
        t += a.part_d[q];
        nd += a.part_nd[q];
    }
    t = block_sum<PI_NT>(t, sm);
    nd = block_sum<PI_NT>(nd, sm);
    reset_fronts(a.ctl);
    if (threadIdx.x == 0) {
        PiCtl *c = a.ctl;
        c->diff = t;
        c->c = 1.0 - (a.d * nd + (1.0 - a.d) * c->sum_v);  // baseline.py:42 for the next iteration
        c->iters += 1;
        const bool done = t * (a.d / (1.0 - a.d)) <= a.target || (long long)c->iters >= a.max_iter;
        c->stop = done ? 1u : 0u;
        if (a.in_graph) cudaGraphSetConditional(a.cond, done ? 0u : 1u);
    }
}

__global__ void k_pi_inv(long long n, const u64 *__restrict__ off, double *__restrict__ inv) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const u64 d = off[i + 1] - off[i];
        inv[i] = d ? 1.0 / (double)d : 0.0;
    }
}
__global__ void k_long_rows(long long n, const u64 *__restrict__ off, u32 *list, u32 *count) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        if (off[i + 1] - off[i] > LONG_ROW) list[atomicAdd(count, 1u)] = (u32)i;
}

// Parents of hub row h per source block: h_cnt[(j >> PI_SB) * H + h] (warp per
// hub row; the sources are ascending, so a warp's keys come in runs)
__global__ void k_hub_count(const u32 *__restrict__ hub, u32 H, const u64 *__restrict__ in_off,
                            const u32 *__restrict__ in_src, u32 *__restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const u32 nw = gridDim.x * (blockDim.x >> 5);
    for (u32 h = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); h < H; h += nw) {
        const u64 lo = in_off[hub[h]], hi = in_off[hub[h] + 1];
        for (u64 k0 = lo; k0 < hi; k0 += 32) {
            const bool v = k0 + lane < hi;
            const u64 key = v ? (u64)(in_src[k0 + lane] >> PI_SB) * H + h : ~0ull;
            const u32 same = __match_any_sync(0xffffffffu, key);
            if (v && lane == __ffs(same) - 1) atomicAdd(cnt + key, (u32)__popc(same));
        }
    }
}
// Start of slice (b, h) in in_src: hub row start + parents in blocks before b.
__global__ void k_hub_lo(const u32 *__restrict__ hub, u32 H, long long nb, const u64 *__restrict__ in_off,
                         const u32 *__restrict__ cnt, u64 *__restrict__ lo) {
    for (u32 h = blockIdx.x * blockDim.x + threadIdx.x; h < H; h += gridDim.x * blockDim.x) {
        u64 pos = in_off[hub[h]];
        for (long long b = 0; b < nb; b++) {
            lo[(u64)b * H + h] = pos;
            pos += cnt[(u64)b * H + h];
        }
    }
}
// Block-major private copy of the hub rows' in-edges: slice r moves from
// in_src[from[r], +cnt[r]) to hub_src[to[r], +cnt[r]) (warp per slice).
__global__ void k_hub_copy(long long R, const u32 *__restrict__ in_src, const u64 *__restrict__ from,
                           const u64 *__restrict__ to, const u32 *__restrict__ cnt, u32 *__restrict__ hub_src) {
    const int lane = threadIdx.x & 31;
    const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long r = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); r < R; r += nw) {
        const u64 f = from[r], t = to[r];
        const u32 c = cnt[r];
        for (u32 k = lane; k < c; k += 32) hub_src[t + k] = in_src[f + k];
    }
}

}  // namespace fr

using namespace fr;

struct fr_power {
    long long n, m;
    PiArgs a;
    double *buf;
    u64 *segbuf;
    void *hubbuf;
    PiCtl *ctl;
    cudaGraph_t graph;
    cudaGraphExec_t exec;
    double target;
    long long max_iter;
    int grid;
};

static int add_node(cudaGraph_t g, cudaGraphNode_t *node, const cudaGraphNode_t *dep, void *func, int grid, void **args) {
    cudaKernelNodeParams p = {};
    p.func = func;
    p.gridDim = dim3((unsigned)grid);
    p.blockDim = dim3(PI_NT);
    p.kernelParams = args;
    FR_CUDA(cudaGraphAddKernelNode(node, g, dep, dep ? 1 : 0, &p));
    return FR_OK;
}

// One iteration: short rows with their update, hub slices, long hub segments,
// the hub rows' update, the stopping rule (and c of the next iteration).
static int power_build_graph(fr_power *p) {
    if (p->exec) { cudaGraphExecDestroy(p->exec); p->exec = nullptr; }
    if (p->graph) { cudaGraphDestroy(p->graph); p->graph = nullptr; }
    FR_CUDA(cudaGraphCreate(&p->graph, 0));
    FR_CUDA(cudaGraphConditionalHandleCreate(&p->a.cond, p->graph, 0, 0));
    p->a.in_graph = 1;
    p->a.target = p->target;
    p->a.max_iter = p->max_iter;
    void *args[] = {&p->a};
    cudaGraphNode_t n_init, n_start, n_while;
    FR_TRY(add_node(p->graph, &n_init, nullptr, (void *)k_pi_init, p->grid, args));
    FR_TRY(add_node(p->graph, &n_start, &n_init, (void *)k_pi_start, 1, args));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = p->a.cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    FR_CUDA(cudaGraphAddNode(&n_while, p->graph, &n_start, 1, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    cudaGraphNode_t n1, n1h, n2, n3, n4;
    FR_TRY(add_node(body, &n1, nullptr, (void *)k_pi_rows<false>, p->grid, args));
    FR_TRY(add_node(body, &n1h, &n1, (void *)k_pi_rows<true>, p->grid, args));
    FR_TRY(add_node(body, &n2, &n1h, (void *)k_pi_segs, p->grid, args));
    FR_TRY(add_node(body, &n3, &n2, (void *)k_pi_hub_update, p->a.hub_grid, args));
    FR_TRY(add_node(body, &n4, &n3, (void *)k_pi_check, 1, args));
    FR_CUDA(cudaGraphInstantiate(&p->exec, p->graph, 0));
    return FR_OK;
}

extern "C" int fr_power_destroy(fr_power *p) {
    if (!p) return FR_OK;
    if (p->exec) cudaGraphExecDestroy(p->exec);
    if (p->graph) cudaGraphDestroy(p->graph);
    cudaFree(p->buf);
    cudaFree(p->segbuf);
    cudaFree(p->hubbuf);
    cudaFree(p->ctl);
    delete p;
    return FR_OK;
}

extern "C" int fr_power_create(int64_t n, int64_t m, const int64_t *d_out_offsets, const int64_t *d_in_offsets,
                               const uint32_t *d_in_sources, double damping, const double *d_teleport, void *stream,
                               fr_power **out) {
    if (!out || n < 1 || m < 0 || !d_out_offsets || !d_in_offsets || (m > 0 && !d_in_sources) ||
        !(damping > 0.0 && damping < 1.0)) {
        set_error("power iteration requires damping < 1 and a valid graph");
        return FR_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    DeviceInfo di;
    FR_TRY(device_info(&di));
    fr_power *p = new fr_power();
    p->n = n;
    p->m = m;
    int rc = FR_OK;
    do {
        PiArgs &a = p->a;
        a.n = n;
        a.in_off = reinterpret_cast<const u64 *>(d_in_offsets);
        a.in_src = d_in_sources;
        a.d = damping;
        p->grid = di.sms * 8;
        a.nparts = p->grid;
        a.row_grid = p->grid;
        cudaError_t e;
        // hub rows: in-degree > LONG_ROW
        Scratch scratch(st);
        u32 *d_list, *d_cnt;
        if ((rc = scratch.alloc(&d_list, (size_t)std::min<long long>(n, m / (long long)LONG_ROW + 1))) != FR_OK) break;
        if ((rc = scratch.alloc(&d_cnt, 1)) != FR_OK) break;
        cudaMemsetAsync(d_cnt, 0, sizeof(u32), st);
        k_long_rows<<<p->grid, PI_NT, 0, st>>>(n, a.in_off, d_list, d_cnt);
        u32 nlong = 0;
        cudaMemcpyAsync(&nlong, d_cnt, sizeof(u32), cudaMemcpyDeviceToHost, st);
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) { rc = cuda_fail(e, "long rows", __FILE__, __LINE__); break; }
        a.nhub = nlong;
        a.hub_grid = (int)std::max<long long>(1, std::min<long long>(p->grid, ((long long)nlong + PI_NT - 1) / PI_NT));
        // inv, x, z (two buffers), s_hub [, v] + partials (|y - x| and non-dangling sums)
        const size_t nv = d_teleport ? (size_t)n : 0;
        const size_t parts = (size_t)(p->grid + a.hub_grid);
        const size_t nz = ((size_t)n + 31) & ~(size_t)31;
        if ((e = cudaMalloc(&p->buf, sizeof(double) * (2 * nz + 2 * (size_t)n + nlong + nv + 2 * parts))) != cudaSuccess ||
            (e = cudaMalloc(&p->ctl, sizeof(PiCtl))) != cudaSuccess) {
            rc = cuda_fail(e, "cudaMalloc(power)", __FILE__, __LINE__);
            break;
        }
        a.zb[0] = p->buf;
        a.zb[1] = a.zb[0] + nz;
        double *inv = a.zb[1] + nz;
        a.inv = inv;
        a.x = inv + n;
        a.s_hub = a.x + n;
        double *v = a.s_hub + nlong;
        a.part_d = v + nv;
        a.part_nd = a.part_d + parts;
        a.ctl = p->ctl;
        k_pi_inv<<<p->grid, PI_NT, 0, st>>>(n, reinterpret_cast<const u64 *>(d_out_offsets), inv);
        double sum_v = 1.0;
        if (d_teleport) {
            if ((e = cudaMemcpyAsync(v, d_teleport, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, st)) !=
                cudaSuccess) {
                rc = cuda_fail(e, "copy teleport", __FILE__, __LINE__);
                break;
            }
            a.v = v;
            if ((rc = fr_abs_sum(n, v, 0, &sum_v, st)) != FR_OK) break;
        } else {
            // uniform teleport: v_i = 1/n is not stored (one 8 B read less per row)
            a.v = nullptr;
            a.v_const = 1.0 / (double)n;
            sum_v = (double)n * a.v_const;
        }
        PiCtl hc = {};
        hc.sum_v = sum_v;
        if ((e = cudaMemcpyAsync(p->ctl, &hc, sizeof(hc), cudaMemcpyHostToDevice, st)) != cudaSuccess) {
            rc = cuda_fail(e, "ctl", __FILE__, __LINE__);
            break;
        }
        // hub rows regrouped by source block into a private block-major copy
        std::vector<u64> seg_row, seg_lo, seg_hi;
        const long long nb = (n + (1ll << PI_SB) - 1) >> PI_SB;
        a.h_rows = nlong ? nb * (long long)nlong : 0;
        if (nlong) {
            const size_t R = (size_t)a.h_rows;
            u64 *d_from, *d_to;
            if ((rc = scratch.alloc(&d_from, R)) != FR_OK) break;
            if ((rc = scratch.alloc(&d_to, R)) != FR_OK) break;
            std::vector<u32> cnt(R), hubs(nlong);
            u64 *h_lo;
            u32 *h_cnt, *hub;
            {
                // counts first (they size the copy)
                u32 *d_hub, *d_hcnt;
                if ((rc = scratch.alloc(&d_hub, nlong)) != FR_OK) break;
                if ((rc = scratch.alloc(&d_hcnt, R)) != FR_OK) break;
                cudaMemcpyAsync(d_hub, d_list, sizeof(u32) * nlong, cudaMemcpyDeviceToDevice, st);
                cudaMemsetAsync(d_hcnt, 0, sizeof(u32) * R, st);
                k_hub_count<<<p->grid, PI_NT, 0, st>>>(d_hub, nlong, a.in_off, a.in_src, d_hcnt);
                k_hub_lo<<<(nlong + 255) / 256, 256, 0, st>>>(d_hub, nlong, nb, a.in_off, d_hcnt, d_from);
                cudaMemcpyAsync(cnt.data(), d_hcnt, sizeof(u32) * R, cudaMemcpyDeviceToHost, st);
                cudaMemcpyAsync(hubs.data(), d_hub, sizeof(u32) * nlong, cudaMemcpyDeviceToHost, st);
                if ((e = cudaStreamSynchronize(st)) != cudaSuccess) { rc = cuda_fail(e, "hub slices", __FILE__, __LINE__); break; }
                // hub_src layout: the short slices in (b, h) order, then the long ones
                std::vector<u64> to(R);
                u64 pos = 0;
                for (size_t r = 0; r < R; r++)
                    if (cnt[r] <= LONG_ROW) { to[r] = pos; pos += cnt[r]; }
                const u64 es = pos;
                for (size_t r = 0; r < R; r++)
                    if (cnt[r] > LONG_ROW) {
                        to[r] = pos;
                        for (u64 b = pos; b < pos + cnt[r]; b += SEG) {
                            seg_row.push_back(r % nlong);
                            seg_lo.push_back(b);
                            seg_hi.push_back(std::min<u64>(pos + cnt[r], b + SEG));
                        }
                        pos += cnt[r];
                    }
                (void)es;
                if ((e = cudaMalloc(&p->hubbuf, sizeof(u64) * R + sizeof(u32) * (R + nlong + pos) + 16)) !=
                    cudaSuccess) {
                    rc = cuda_fail(e, "cudaMalloc(hub slices)", __FILE__, __LINE__);
                    break;
                }
                h_lo = (u64 *)p->hubbuf;
                h_cnt = (u32 *)(h_lo + R);
                hub = h_cnt + R;
                u32 *hub_src = hub + nlong;
                cudaMemcpyAsync(d_to, to.data(), sizeof(u64) * R, cudaMemcpyHostToDevice, st);
                k_hub_copy<<<p->grid, PI_NT, 0, st>>>((long long)R, a.in_src, d_from, d_to, d_hcnt, hub_src);
                cudaMemcpyAsync(h_lo, d_to, sizeof(u64) * R, cudaMemcpyDeviceToDevice, st);
                cudaMemcpyAsync(h_cnt, d_hcnt, sizeof(u32) * R, cudaMemcpyDeviceToDevice, st);
                cudaMemcpyAsync(hub, d_hub, sizeof(u32) * nlong, cudaMemcpyDeviceToDevice, st);
                if ((e = cudaStreamSynchronize(st)) != cudaSuccess) { rc = cuda_fail(e, "hub copy", __FILE__, __LINE__); break; }
                a.hub_src = hub_src;
            }
            if (rc != FR_OK) break;
            a.h_lo = h_lo;
            a.h_cnt = h_cnt;
            a.hub_node = hub;
        }
        a.nseg = (long long)seg_row.size();
        if ((e = cudaMalloc(&p->segbuf, sizeof(u64) * (3 * seg_row.size() + 3))) != cudaSuccess) {
            rc = cuda_fail(e, "segments", __FILE__, __LINE__);
            break;
        }
        a.seg_row = p->segbuf;
        a.seg_lo = p->segbuf + seg_row.size() + 1;
        a.seg_hi = p->segbuf + 2 * seg_row.size() + 2;
        if (a.nseg) {
            cudaMemcpy((void *)a.seg_row, seg_row.data(), sizeof(u64) * seg_row.size(), cudaMemcpyHostToDevice);
            cudaMemcpy((void *)a.seg_lo, seg_lo.data(), sizeof(u64) * seg_row.size(), cudaMemcpyHostToDevice);
            cudaMemcpy((void *)a.seg_hi, seg_hi.data(), sizeof(u64) * seg_row.size(), cudaMemcpyHostToDevice);
        }
        if ((e = cudaGetLastError()) != cudaSuccess) { rc = cuda_fail(e, "power setup", __FILE__, __LINE__); break; }
    } while (0);
    if (rc != FR_OK) {
        fr_power_destroy(p);
        return rc;
    }
    *out = p;
    return FR_OK;
}

// The same iterations launched one by one from the host with CUDA events around
// each kernel class: the roofline report of bench.py, not the timed path.
// h_ms[0] = short rows with their update (k_pi_rows<false>), h_ms[1] = hub slices
// by source block (k_pi_rows<true>), h_ms[2] = long hub slices (k_pi_segs), h_ms[3]
// = the rest (hub rows' update, check), summed over the iterations.
extern "C" int fr_power_run_profiled(fr_power *p, double target_error, int64_t max_iterations, double *d_x,
                                     int64_t *h_iterations, double *h_ms, void *stream) {
    if (!p || !(target_error > 0.0) || !d_x || !h_ms) {
        set_error("fr_power_run_profiled: bad arguments");
        return FR_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    PiArgs a = p->a;
    a.in_graph = 0;
    a.target = target_error;
    a.max_iter = max_iterations > 0 ? max_iterations : 1000000;
    cudaEvent_t ev[5];
    for (int i = 0; i < 5; i++) FR_CUDA(cudaEventCreate(&ev[i]));
    h_ms[0] = h_ms[1] = h_ms[2] = h_ms[3] = 0.0;
    k_pi_init<<<p->grid, PI_NT, 0, st>>>(a);
    k_pi_start<<<1, PI_NT, 0, st>>>(a);
    PiCtl hc = {};
    for (;;) {
        FR_CUDA(cudaEventRecord(ev[0], st));
        k_pi_rows<false><<<p->grid, PI_NT, 0, st>>>(a);
        FR_CUDA(cudaEventRecord(ev[1], st));
        k_pi_rows<true><<<p->grid, PI_NT, 0, st>>>(a);
        FR_CUDA(cudaEventRecord(ev[2], st));
        k_pi_segs<<<p->grid, PI_NT, 0, st>>>(a);
        FR_CUDA(cudaEventRecord(ev[3], st));
        k_pi_hub_update<<<a.hub_grid, PI_NT, 0, st>>>(a);
        k_pi_check<<<1, PI_NT, 0, st>>>(a);
        FR_CUDA(cudaEventRecord(ev[4], st));
        FR_CUDA(cudaGetLastError());
        FR_CUDA(cudaMemcpyAsync(&hc, p->ctl, sizeof(hc), cudaMemcpyDeviceToHost, st));
        FR_CUDA(cudaStreamSynchronize(st));
        for (int k = 0; k < 4; k++) {
            float t = 0.f;
            FR_CUDA(cudaEventElapsedTime(&t, ev[k], ev[k + 1]));
            h_ms[k] += t;
        }
        if (hc.stop) break;
    }
    for (int i = 0; i < 5; i++) cudaEventDestroy(ev[i]);
    FR_CUDA(cudaMemcpyAsync(d_x, p->a.x, sizeof(double) * (size_t)p->n, cudaMemcpyDeviceToDevice, st));
    FR_CUDA(cudaStreamSynchronize(st));
    if (h_iterations) *h_iterations = (int64_t)hc.iters;
    return FR_OK;
}

extern "C" int fr_power_run(fr_power *p, double target_error, int64_t max_iterations, double *d_x,
                            int64_t *h_iterations, double *h_diff, void *stream) {
    if (!p || !(target_error > 0.0) || !d_x) { set_error("fr_power_run: bad arguments"); return FR_ERR_ARG; }
    cudaStream_t st = (cudaStream_t)stream;
    const long long mi = max_iterations > 0 ? max_iterations : 1000000;
    if (!p->exec || p->target != target_error || p->max_iter != mi) {
        p->target = target_error;
        p->max_iter = mi;
        FR_TRY(power_build_graph(p));
    }
    FR_CUDA(cudaGraphLaunch(p->exec, st));
    PiCtl hc;
    FR_CUDA(cudaMemcpyAsync(&hc, p->ctl, sizeof(hc), cudaMemcpyDeviceToHost, st));
    FR_CUDA(cudaMemcpyAsync(d_x, p->a.x, sizeof(double) * (size_t)p->n, cudaMemcpyDeviceToDevice, st));
    FR_CUDA(cudaStreamSynchronize(st));
    if (h_iterations) *h_iterations = (int64_t)hc.iters;
    if (h_diff) *h_diff = hc.diff;
    if (hc.diff * (p->a.d / (1.0 - p->a.d)) > target_error) {
        set_error("no convergence within %lld iterations", mi);
        return FR_ERR_NO_CONVERGENCE;
    }
    return FR_OK;
}
