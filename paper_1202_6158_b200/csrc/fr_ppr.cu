// fr_ppr.cu -- batched personalized PageRank by D-iteration (BASELINE config 4).
//
// B <= 64 personalization vectors V_c diffuse together: fluid F and history H
// are n x B row-major fp64 arrays, so one visit of an edge scatters a B-wide
// vector (each lane of a warp owns columns lane and lane + 32).  Every column
// is an independent instance of engine.py:240-341 (teleport = V_c); the sweep
// rule is the scalar solver's threshold sweep applied to the row maximum over
// the columns that are still active, and column c stops (freezes: no more
// pushes) once its residual R_c <= target*(1-d) is confirmed by an exact sum.
//
// Two formulations of a sweep (the same fixed point; parity is checked per column):
//   push (k_ppr_sweep): a selected row scatters its B-wide push into each child
//     with red.global.add -- every edge visit is B fp64 reductions in L2;
//   pull (fr_ppr_set_pull; k_ppr_take + k_ppr_pull): the selected rows are taken
//     and their pushes d*f/deg written once to a row buffer (sent) with a
//     selection bitmap; then every node sums the sent rows of its selected
//     parents over the transposed CSR into its own fluid row (plain loads and
//     stores, no atomics: the 64-wide scatter was bound by the L2 reduction
//     units, ~2e11 fp64 adds/s), and keeps its exact row maximum (rmax), so the
//     next take reads 8 B per row instead of the row.  The pull is Jacobi within
//     a sweep (a push reaches its child in the next sweep).
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "fr_common.cuh"

namespace fr {

static constexpr int PP_NT = 256;
#ifndef FR_PP_SEGS
#define FR_PP_SEGS 16
#endif
#ifndef FR_PP_CHUNK
#define FR_PP_CHUNK 32  // scanned 8-128 with the hot-row kernel: 32 -> 68.5 ms, 64 -> 71.4, 128 -> 76.6
#endif
static constexpr int PP_SEGS = FR_PP_SEGS;
static constexpr int PP_CHUNK = FR_PP_CHUNK;  // consecutive nodes per reservation (one warp per node)
static constexpr u64 PULL_LONG = 1024;  // pull: rows with more parents are split into segments
static constexpr u64 PULL_SEG = 2048;   // parents per segment
static constexpr u32 PP_HOT_FLAG = 0x80000000u;
static constexpr int PP_HOT_MAX = 32;   // hot rows per block: 32 x 64 fp64 = 16 KB of shared memory

struct PprCtl {
    double theta;
    double resid[64];      // incremental residual per column
    double exact[64];      // exact residual per column (after a check)
    u64 active;            // bit c: column c still diffusing
    u64 need_check;        // columns whose incremental residual crossed the target
    u64 diffusions, steps, sweeps;
    u64 pushes;            // column values scattered (one red.add each)
    u64 seg_next[PP_SEGS * 16];  // one 128 B line per front counter
    u32 stop;
    u32 pad;
};

struct PprArgs {
    double *F, *H;
    const u64 *off;
    const u32 *tgt;
    PprCtl *ctl;
    // pull formulation (null in_off: push)
    const u64 *in_off;
    const u32 *in_src;
    double *sent;        // [n][B] push values d*f/deg of the rows taken this sweep
    u32 *selbits;        // [ceil(n/32)] rows taken this sweep that have children
    double *rmax;        // [n] exact max_c |F[i][c]| over all columns
    double *part_max2;   // [2 grid] max of the rows updated by the pull (short rows, hub rows)
    // rows with more than PULL_LONG parents: summed by 2048-parent segments into
    // per-segment partial rows, then added per hub in a fixed order
    const u32 *hub_node;  // [nhub]
    const u32 *hub_seg;   // [nhub + 1] first segment of each hub
    const u64 *seg_lo, *seg_hi;  // [nseg] in_src range of each segment
    // push: the rows of the nhot highest in-degree nodes (Zipf hubs) are summed
    // per block in shared memory and flushed once per block; tgt_enc is the
    // column copy in which such targets carry PP_HOT_FLAG | slot
    const u32 *tgt_enc;
    const u32 *hot_node;  // [nhot]
    int nhot;
    double *seg_acc;      // [nseg][B]
    u32 nhub, nseg;
    double *part_abs;    // [grid][64]
    double *part_max;    // [grid]
    u64 *part_sel, *part_steps, *part_push;
    double *part_mass;   // [grid][64] for exact checks
    long long n;
    int B;
    int nparts;
    double d, thr, decay;
    long long max_sweeps;
    int in_graph;
    cudaGraphConditionalHandle cond;
};

__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Warp per node, nodes taken in order from PP_SEGS segments (as the scalar sweep).
__global__ void __launch_bounds__(PP_NT, 4) k_ppr_sweep(PprArgs a) {
    extern __shared__ __align__(16) double hot_acc[];  // [nhot][B]
    __shared__ double s_abs[PP_NT / 32][64];
    __shared__ double s_red[PP_NT / 32];
    __shared__ u64 s_red64[PP_NT / 32];
    constexpr u32 FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    PprCtl *c = a.ctl;
    const double theta = c->theta;
    const u64 active = c->active;
    const int B = a.B;
    const bool own0 = lane < B && ((active >> lane) & 1ull);
    const bool own1 = lane + 32 < B && ((active >> (lane + 32)) & 1ull);
    double ab0 = 0.0, ab1 = 0.0, mx = 0.0;
    u64 nsel = 0, steps = 0, npush = 0;
    const int nhot = a.nhot;
    for (int q = threadIdx.x; q < nhot * B; q += PP_NT) hot_acc[q] = 0.0;
    __syncthreads();
    const u32 *__restrict__ tgt = nhot ? a.tgt_enc : a.tgt;
    const long long seg_len = (a.n + PP_SEGS - 1) / PP_SEGS;
    int seg = (int)((blockIdx.x * (PP_NT / 32) + wid) % PP_SEGS), misses = 0;
    long long node = 0, chunk_end = 0;
    auto grab = [&]() -> bool {
        while (misses < PP_SEGS) {
            unsigned long long k = 0;
            if (lane == 0) k = atomicAdd(&c->seg_next[seg * 16], (unsigned long long)PP_CHUNK);
            k = __shfl_sync(FULL, k, 0);
            const long long s0 = (long long)seg * seg_len;
            const long long s1 = s0 + seg_len < a.n ? s0 + seg_len : a.n;
            if (s0 + (long long)k < s1) {
                node = s0 + (long long)k;
                chunk_end = node + PP_CHUNK < s1 ? node + PP_CHUNK : s1;
                misses = 0;
                return true;
            }
            seg = (seg + 1) % PP_SEGS;
            misses++;
        }
        return false;
    };
    bool have = grab();
    while (have) {
        const long long i = node;
        double *Fi = a.F + (size_t)i * B;
        const double f0 = own0 ? Fi[lane] : 0.0;
        const double f1 = own1 ? Fi[lane + 32] : 0.0;
        const double rowmax = warp_max_d(fmax(fabs(f0), fabs(f1)));
        mx = fmax(mx, rowmax);
        if (rowmax >= theta && rowmax > 0.0) {
            const u64 lo = a.off[i], hi = a.off[i + 1];
            const u32 deg = (u32)(hi - lo);
            double s0 = 0.0, s1 = 0.0;
            double *Hi = a.H + (size_t)i * B;
            if (own0) s0 = __longlong_as_double((long long)atomicExch((unsigned long long *)(Fi + lane), 0ull));
            if (own1) s1 = __longlong_as_double((long long)atomicExch((unsigned long long *)(Fi + lane + 32), 0ull));
            if (own0) Hi[lane] += s0;
            if (own1) Hi[lane + 32] += s1;
            // one row visit per warp: only lane 0 counts it (the block sums add every lane)
            if (lane == 0) nsel++;
            if (deg == 0) {
                ab0 += fabs(s0);
                ab1 += fabs(s1);
            } else {
                ab0 += fabs(s0) * (1.0 - a.d);
                ab1 += fabs(s1) * (1.0 - a.d);
                if (lane == 0) steps += deg;
                const double w = a.d / (double)deg;
                const double p0 = s0 * w, p1 = s1 * w;  // sent*(d/deg), engine.py:321
                npush += (u64)deg * ((own0 && p0 != 0.0) + (own1 && p1 != 0.0));
                for (u32 k0 = 0; k0 < deg; k0 += 32) {
                    const u32 cnt = deg - k0 < 32u ? deg - k0 : 32u;
                    const u32 tv = lane < cnt ? __ldg(tgt + lo + k0 + lane) : 0u;
                    // the encoded copy keeps each row's hot targets at its end, so the
                    // batch's hot targets (if any) are lanes [cold, cnt)
                    const u32 hm = nhot ? __ballot_sync(FULL, lane < cnt && (tv & PP_HOT_FLAG)) : 0u;
                    const u32 cold = hm ? (u32)(__ffs(hm) - 1) : cnt;
                    for (u32 j = 0; j < cold; j++) {
                        const u32 t = __shfl_sync(FULL, tv, j);
                        double *Ft = a.F + (size_t)t * B;
                        if (own0 && p0 != 0.0) red_add(Ft + lane, p0);
                        if (own1 && p1 != 0.0) red_add(Ft + lane + 32, p1);
                    }
                    for (u32 j = cold; j < cnt; j++) {  // one row of the block's table each
                        const u32 t = __shfl_sync(FULL, tv, j);
                        double *Ht = hot_acc + (size_t)(t & ~PP_HOT_FLAG) * B;
                        if (own0 && p0 != 0.0) atomicAdd(Ht + lane, p0);
                        if (own1 && p1 != 0.0) atomicAdd(Ht + lane + 32, p1);
                    }
                }
            }
        }
        node++;
        have = node < chunk_end ? true : grab();
    }
    __syncthreads();  // every push into the hot table is done
    for (int q = threadIdx.x; q < nhot * B; q += PP_NT) {
        const double v = hot_acc[q];
        if (v != 0.0) red_add(a.F + (size_t)a.hot_node[q / B] * B + q % B, v);
    }
    // per-column absorbed mass: lanes own columns, reduce over the block's warps
    s_abs[wid][lane] = ab0;
    s_abs[wid][lane + 32] = ab1;
    __syncthreads();
    if (threadIdx.x < 64) {
        double t = 0.0;
        for (int w = 0; w < PP_NT / 32; w++) t += s_abs[w][threadIdx.x];
        a.part_abs[(size_t)blockIdx.x * 64 + threadIdx.x] = t;
    }
    const double bmx = block_max<PP_NT>(mx, s_red);
    const u64 bsel = block_sum_u64<PP_NT>(nsel, s_red64);
    const u64 bst = block_sum_u64<PP_NT>(steps, s_red64);
    const u64 bpu = block_sum_u64<PP_NT>(npush, s_red64);
    if (threadIdx.x == 0) {
        a.part_max[blockIdx.x] = bmx;
        a.part_sel[blockIdx.x] = bsel;
        a.part_steps[blockIdx.x] = bst;
        a.part_push[blockIdx.x] = bpu;
    }
}

// Pull formulation, take: warp per tile of 32 rows (grid-stride).  A row whose
// exact maximum (rmax) reaches theta is read; it diffuses when its maximum over
// the active columns does: F row -> 0, H += f, sent row = f*d/deg (0 in frozen
// columns), its bit set; the tile's bitmap word is written whole every sweep.
__global__ void __launch_bounds__(PP_NT) k_ppr_take(PprArgs a) {
    __shared__ double s_abs[PP_NT / 32][64];
    __shared__ double s_red[PP_NT / 32];
    __shared__ u64 s_red64[PP_NT / 32];
    constexpr u32 FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    PprCtl *c = a.ctl;
    const double theta = c->theta;
    const u64 active = c->active;
    const int B = a.B;
    const bool own0 = lane < B && ((active >> lane) & 1ull);
    const bool own1 = lane + 32 < B && ((active >> (lane + 32)) & 1ull);
    const bool col0 = lane < B, col1 = lane + 32 < B;
    double ab0 = 0.0, ab1 = 0.0, mx = 0.0;
    u64 nsel = 0, steps = 0, npush = 0;
    const long long ntiles = (a.n + 31) / 32;
    for (long long tl = blockIdx.x * (long long)(PP_NT / 32) + wid; tl < ntiles;
         tl += (long long)gridDim.x * (PP_NT / 32)) {
        const long long i0 = tl * 32, ti = i0 + lane;
        const bool v = ti < a.n;
        const double r = v ? a.rmax[ti] : 0.0;
        const bool cand = r >= theta && r > 0.0;
        if (!cand) mx = fmax(mx, r);
        u32 cm = __ballot_sync(FULL, cand);
        u32 bits = 0;
        while (cm) {
            const int j = __ffs(cm) - 1;
            cm &= cm - 1;
            const long long i = i0 + j;
            double *Fi = a.F + (size_t)i * B;
            const double f0 = own0 ? Fi[lane] : 0.0;
            const double f1 = own1 ? Fi[lane + 32] : 0.0;
            const double rowmax = warp_max_d(fmax(fabs(f0), fabs(f1)));  // active columns
            if (!(rowmax >= theta && rowmax > 0.0)) {
                // frozen columns hold the rest of rmax: keep the active maximum
                mx = fmax(mx, rowmax);
                if (lane == 0) a.rmax[i] = rowmax;
                continue;
            }
            const u64 lo = a.off[i], hi = a.off[i + 1];
            const u32 deg = (u32)(hi - lo);
            double *Hi = a.H + (size_t)i * B;
            if (own0) {
                Fi[lane] = 0.0;
                Hi[lane] += f0;
            }
            if (own1) {
                Fi[lane + 32] = 0.0;
                Hi[lane + 32] += f1;
            }
            if (lane == 0) {
                a.rmax[i] = 0.0;  // the frozen columns are not searched again (their fluid stays)
                nsel++;
            }
            if (deg == 0) {
                ab0 += fabs(f0);
                ab1 += fabs(f1);
                continue;
            }
            ab0 += fabs(f0) * (1.0 - a.d);
            ab1 += fabs(f1) * (1.0 - a.d);
            if (lane == 0) steps += deg;
            const double w = a.d / (double)deg;
            const double p0 = f0 * w, p1 = f1 * w;  // sent*(d/deg), engine.py:321
            npush += (u64)deg * ((own0 && p0 != 0.0) + (own1 && p1 != 0.0));
            double *Si = a.sent + (size_t)i * B;
            if (col0) Si[lane] = p0;
            if (col1) Si[lane + 32] = p1;
            bits |= 1u << j;
        }
        if (lane == 0 && i0 < a.n) a.selbits[tl] = bits;
    }
    s_abs[wid][lane] = ab0;
    s_abs[wid][lane + 32] = ab1;
    __syncthreads();
    if (threadIdx.x < 64) {
        double t = 0.0;
        for (int w = 0; w < PP_NT / 32; w++) t += s_abs[w][threadIdx.x];
        a.part_abs[(size_t)blockIdx.x * 64 + threadIdx.x] = t;
    }
    const double bmx = block_max<PP_NT>(mx, s_red);
    const u64 bsel = block_sum_u64<PP_NT>(nsel, s_red64);
    const u64 bst = block_sum_u64<PP_NT>(steps, s_red64);
    const u64 bpu = block_sum_u64<PP_NT>(npush, s_red64);
    if (threadIdx.x == 0) {
        a.part_max[blockIdx.x] = bmx;
        a.part_sel[blockIdx.x] = bsel;
        a.part_steps[blockIdx.x] = bst;
        a.part_push[blockIdx.x] = bpu;
    }
}

// Sum of the sent rows of the selected parents in in_src[lo, hi) (warp; lanes
// hold columns lane and lane + 32); returns whether any parent was selected.
__device__ __forceinline__ bool pull_range(const PprArgs &a, u64 lo, u64 hi, bool col0, bool col1, double &acc0,
                                           double &acc1) {
    constexpr u32 FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int B = a.B;
    bool any = false;
    for (u64 k0 = lo; k0 < hi; k0 += 32) {
        const bool v = k0 + lane < hi;
        const u32 j = v ? __ldg(a.in_src + k0 + lane) : 0u;
        const bool sel = v && ((__ldg(a.selbits + (j >> 5)) >> (j & 31)) & 1u);
        u32 sm = __ballot_sync(FULL, sel);
        any |= sm != 0;
        // two parents per step: their four 256 B loads in flight together
        while (sm) {
            const int b0 = __ffs(sm) - 1;
            sm &= sm - 1;
            const u32 j0 = __shfl_sync(FULL, j, b0);
            int b1 = -1;
            if (sm) {
                b1 = __ffs(sm) - 1;
                sm &= sm - 1;
            }
            const u32 j1 = __shfl_sync(FULL, j, b1 < 0 ? b0 : b1);
            const double *S0 = a.sent + (size_t)j0 * B;
            const double *S1 = a.sent + (size_t)j1 * B;
            const double x0 = col0 ? S0[lane] : 0.0, x1 = col1 ? S0[lane + 32] : 0.0;
            const double y0 = (col0 && b1 >= 0) ? S1[lane] : 0.0, y1 = (col1 && b1 >= 0) ? S1[lane + 32] : 0.0;
            acc0 += x0;
            acc1 += x1;
            acc0 += y0;
            acc1 += y1;
        }
    }
    return any;
}

// F row i += (acc0, acc1); its new exact maximum over the active columns
__device__ __forceinline__ double pull_apply(const PprArgs &a, long long i, bool col0, bool col1, bool own0, bool own1,
                                             double acc0, double acc1) {
    const int lane = threadIdx.x & 31;
    double *Fi = a.F + (size_t)i * a.B;
    double f0 = 0.0, f1 = 0.0;
    if (col0) {
        f0 = Fi[lane] + acc0;
        Fi[lane] = f0;
    }
    if (col1) {
        f1 = Fi[lane + 32] + acc1;
        Fi[lane + 32] = f1;
    }
    const double rm = warp_max_d(fmax(own0 ? fabs(f0) : 0.0, own1 ? fabs(f1) : 0.0));
    if (lane == 0 && a.rmax) a.rmax[i] = rm;
    return rm;
}

// Pull: warp per node, nodes in order (grid-stride: the warps in flight cover a
// narrow id window, so the sent rows of the local parents stay in L2).  The
// node's parents are tested against the bitmap 32 at a time; each selected
// parent's sent row is added (two coalesced 256 B loads); the node's own fluid
// row is then updated in place with its new exact maximum.  Rows with more than
// PULL_LONG parents (the Zipf in-degree hubs) are left to k_ppr_pull_segs.
__global__ void __launch_bounds__(PP_NT) k_ppr_pull(PprArgs a) {
    __shared__ double s_red[PP_NT / 32];
    const int lane = threadIdx.x & 31;
    const int B = a.B;
    const bool col0 = lane < B, col1 = lane + 32 < B;
    const u64 active = a.ctl->active;
    const bool own0 = col0 && ((active >> lane) & 1ull);
    const bool own1 = col1 && ((active >> (lane + 32)) & 1ull);
    double mx = 0.0;
    const long long nw = (long long)gridDim.x * (PP_NT / 32);
    for (long long i = blockIdx.x * (long long)(PP_NT / 32) + (threadIdx.x >> 5); i < a.n; i += nw) {
        const u64 lo = a.in_off[i], hi = a.in_off[i + 1];
        if (hi - lo > PULL_LONG) continue;
        double acc0 = 0.0, acc1 = 0.0;
        if (!pull_range(a, lo, hi, col0, col1, acc0, acc1)) continue;
        mx = fmax(mx, pull_apply(a, i, col0, col1, own0, own1, acc0, acc1));
    }
    mx = block_max<PP_NT>(mx, s_red);
    if (threadIdx.x == 0) a.part_max2[blockIdx.x] = mx;
}

// Hub rows, warp per segment of PULL_SEG parents: the partial row into seg_acc.
__global__ void __launch_bounds__(PP_NT) k_ppr_pull_segs(PprArgs a) {
    const int lane = threadIdx.x & 31;
    const int B = a.B;
    const bool col0 = lane < B, col1 = lane + 32 < B;
    const long long nw = (long long)gridDim.x * (PP_NT / 32);
    for (long long q = blockIdx.x * (long long)(PP_NT / 32) + (threadIdx.x >> 5); q < a.nseg; q += nw) {
        double acc0 = 0.0, acc1 = 0.0;
        const u64 lo = a.seg_lo[q], hi = a.seg_hi[q];
        pull_range(a, lo, hi, col0, col1, acc0, acc1);
        double *P = a.seg_acc + (size_t)q * B;
        if (col0) P[lane] = acc0;
        if (col1) P[lane + 32] = acc1;
    }
}

// Hub rows, warp per hub: its segments' partial rows added in segment order.
__global__ void __launch_bounds__(PP_NT) k_ppr_pull_hubs(PprArgs a) {
    __shared__ double s_red[PP_NT / 32];
    const int lane = threadIdx.x & 31;
    const int B = a.B;
    const bool col0 = lane < B, col1 = lane + 32 < B;
    const u64 active = a.ctl->active;
    const bool own0 = col0 && ((active >> lane) & 1ull);
    const bool own1 = col1 && ((active >> (lane + 32)) & 1ull);
    double mx = 0.0;
    const long long nw = (long long)gridDim.x * (PP_NT / 32);
    for (long long h = blockIdx.x * (long long)(PP_NT / 32) + (threadIdx.x >> 5); h < a.nhub; h += nw) {
        double acc0 = 0.0, acc1 = 0.0;
        for (u32 q = a.hub_seg[h]; q < a.hub_seg[h + 1]; q++) {
            const double *P = a.seg_acc + (size_t)q * B;
            if (col0) acc0 += P[lane];
            if (col1) acc1 += P[lane + 32];
        }
        mx = fmax(mx, pull_apply(a, a.hub_node[h], col0, col1, own0, own1, acc0, acc1));
    }
    mx = block_max<PP_NT>(mx, s_red);
    if (threadIdx.x == 0) a.part_max2[a.nparts + blockIdx.x] = mx;
}

// Column masses |F_c|_1 (all columns, or only when a check is pending).
__global__ void __launch_bounds__(PP_NT) k_ppr_mass(PprArgs a, int guarded) {
    __shared__ double s[PP_NT / 32][64];
    if (guarded && !a.ctl->need_check) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __shared__ double s_red[PP_NT / 32];
    const int B = a.B;
    double m0 = 0.0, m1 = 0.0, mx = 0.0;
    for (long long i = blockIdx.x * (long long)(PP_NT / 32) + wid; i < a.n; i += (long long)gridDim.x * (PP_NT / 32)) {
        const double *Fi = a.F + (size_t)i * B;
        const double x0 = lane < B ? fabs(Fi[lane]) : 0.0;
        const double x1 = lane + 32 < B ? fabs(Fi[lane + 32]) : 0.0;
        m0 += x0;
        m1 += x1;
        mx = fmax(mx, fmax(x0, x1));
        if (!guarded && a.rmax) {  // prologue of the pull formulation: exact row maxima
            const double rm = warp_max_d(fmax(x0, x1));
            if (lane == 0) a.rmax[i] = rm;
        }
    }
    s[wid][lane] = m0;
    s[wid][lane + 32] = m1;
    __syncthreads();
    if (threadIdx.x < 64) {
        double t = 0.0;
        for (int w = 0; w < PP_NT / 32; w++) t += s[w][threadIdx.x];
        a.part_mass[(size_t)blockIdx.x * 64 + threadIdx.x] = t;
    }
    mx = block_max<PP_NT>(mx, s_red);
    if (threadIdx.x == 0) a.part_max[blockIdx.x] = mx;
}

// Prologue (check = 0) and exact check (check = 1): one block of 64 threads.
__global__ void k_ppr_settle(PprArgs a, int check) {
    PprCtl *c = a.ctl;
    const int col = threadIdx.x;
    if (check && !c->need_check) return;
    double t = 0.0;
    for (int p = 0; p < a.nparts; p++) t += a.part_mass[(size_t)p * 64 + col];
    __shared__ u64 s_done;
    if (col == 0) s_done = 0;
    __syncthreads();
    if (col < a.B) {
        const bool pending = !check || ((c->need_check >> col) & 1ull);
        if (pending) {
            c->exact[col] = t;
            c->resid[col] = t;
            if (t <= a.thr) atomicOr(&s_done, 1ull << col);
        }
    }
    __syncthreads();
    if (col == 0) {
        if (!check) {  // prologue: the threshold starts at the largest fluid (sched.py:89-90)
            double mx = 0.0;
            for (int p = 0; p < a.nparts; p++) mx = fmax(mx, a.part_max[p]);
            c->theta = mx;
        }
        c->active &= ~s_done;
        c->need_check = 0;
        const bool stop = c->active == 0 || (long long)c->sweeps >= a.max_sweeps;
        c->stop = stop ? 1u : 0u;
        if (a.in_graph) cudaGraphSetConditional(a.cond, stop ? 0u : 1u);
    }
}

// The bookkeeping after a sweep.  PP_NT threads reduce the per-block partials
// (nparts = the sweep grid, ~600): a single thread walking them serially took
// ~110 us per sweep, 10% of the config-4 solve.
__global__ void __launch_bounds__(PP_NT) k_ppr_finalize(PprArgs a) {
    PprCtl *c = a.ctl;
    const int t = threadIdx.x, col = t & 63, q = t >> 6;
    __shared__ double s_ab[PP_NT / 64][64];
    __shared__ double s_red[PP_NT / 32];
    __shared__ u64 s_red64[PP_NT / 32];
    __shared__ u64 s_need;
    __shared__ double s_max;
    double abq = 0.0;  // column col over the parts q, q + 4, ...
    for (int p = q; p < a.nparts; p += PP_NT / 64) abq += a.part_abs[(size_t)p * 64 + col];
    s_ab[q][col] = abq;
    double mx = 0.0;
    u64 sel = 0, st = 0, pu = 0;
    for (int p = t; p < a.nparts; p += PP_NT) {
        mx = fmax(mx, a.part_max[p]);
        if (a.in_off) mx = fmax(mx, fmax(a.part_max2[p], a.part_max2[a.nparts + p]));
        sel += a.part_sel[p];
        st += a.part_steps[p];
        pu += a.part_push[p];
    }
    mx = block_max<PP_NT>(mx, s_red);
    sel = block_sum_u64<PP_NT>(sel, s_red64);
    st = block_sum_u64<PP_NT>(st, s_red64);
    pu = block_sum_u64<PP_NT>(pu, s_red64);
    if (t == 0) {
        s_need = 0;
        c->pushes += pu;
        s_max = mx;
        c->diffusions += sel;
        c->steps += st;
        c->sweeps += 1;
        for (int k = 0; k < PP_SEGS; k++) c->seg_next[k * 16] = 0;
    }
    __syncthreads();
    double ab = 0.0;
    if (t < 64)
        for (int k = 0; k < PP_NT / 64; k++) ab += s_ab[k][col];
    __syncthreads();
    if (t < 64 && col < a.B && ((c->active >> col) & 1ull)) {
        const double r = c->resid[col] - ab;
        c->resid[col] = r;
        if (r <= a.thr) atomicOr(&s_need, 1ull << col);
    }
    __syncthreads();
    if (t == 0) {
        double th = c->theta * a.decay;
        const double mx = s_max;
        if (mx > 0.0)
            while (th > mx) th *= a.decay;
        c->theta = th;
        // a column drained to zero everywhere also needs its exact check
        c->need_check = s_need | (mx == 0.0 ? c->active : 0ull);
        const bool stop = (long long)c->sweeps >= a.max_sweeps;
        c->stop = stop ? 1u : 0u;
        if (a.in_graph) cudaGraphSetConditional(a.cond, stop ? 0u : 1u);
    }
}

__global__ void k_ppr_init(long long n, int B, int k, const u32 *__restrict__ seeds, double damping, double *F,
                           double *H) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * (long long)B;
         e += (long long)gridDim.x * blockDim.x) {
        F[e] = 0.0;
        H[e] = 0.0;
    }
}
__global__ void k_ppr_seed(int B, int k, const u32 *__restrict__ seeds, double damping, double *F) {
    // V_c uniform over the k seeds of column c: F = (1-d) * V_c (repeated seeds accumulate)
    const int c = blockIdx.x;
    for (int j = threadIdx.x; j < k; j += blockDim.x)
        atomicAdd(F + (size_t)seeds[(size_t)c * k + j] * B + c, (1.0 - damping) * (1.0 / (double)k));
}

__global__ void k_ppr_colsum(long long n, int B, const double *__restrict__ H, double *out) {
    __shared__ double s[PP_NT / 32][64];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double m0 = 0.0, m1 = 0.0;
    for (long long i = blockIdx.x * (long long)(PP_NT / 32) + wid; i < n; i += (long long)gridDim.x * (PP_NT / 32)) {
        if (lane < B) m0 += fabs(H[(size_t)i * B + lane]);
        if (lane + 32 < B) m1 += fabs(H[(size_t)i * B + lane + 32]);
    }
    s[wid][lane] = m0;
    s[wid][lane + 32] = m1;
    __syncthreads();
    if (threadIdx.x < 64 && threadIdx.x < B) {
        double t = 0.0;
        for (int w = 0; w < PP_NT / 32; w++) t += s[w][threadIdx.x];
        atomicAdd(out + threadIdx.x, t);
    }
}
__global__ void k_ppr_scale(long long n, int B, const double *__restrict__ H, const double *__restrict__ tot,
                            double *R) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * (long long)B;
         e += (long long)gridDim.x * blockDim.x) {
        const double t = tot[e % B];
        R[e] = t > 0.0 ? H[e] / t : H[e];
    }
}

// hot rows (push formulation): in-degree count and the encoded column copy
__global__ void k_ppr_indeg(const u32 *__restrict__ tgt, long long m, u32 *__restrict__ cnt) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m; e += (long long)gridDim.x * blockDim.x)
        atomicAdd(cnt + tgt[e], 1u);
}
// warp per row: the row's targets with the hot ones (PP_HOT_FLAG | slot) moved to
// its end (order within a row does not matter to the pushes)
__global__ void k_ppr_encode(const u64 *__restrict__ off, long long n, const u32 *__restrict__ tgt,
                             const int *__restrict__ slot_of, u32 *__restrict__ enc) {
    const int lane = threadIdx.x & 31;
    const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long i = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nw) {
        const u64 lo = off[i], hi = off[i + 1];
        u32 nhot_row = 0;
        for (u64 k0 = lo; k0 < hi; k0 += 32) {
            const bool v = k0 + lane < hi;
            const u32 t = v ? tgt[k0 + lane] : 0u;
            nhot_row += __popc(__ballot_sync(0xffffffffu, v && slot_of[t] >= 0));
        }
        const u64 hot0 = hi - nhot_row;  // first position of the hot block
        u32 seen_cold = 0, seen_hot = 0;
        for (u64 k0 = lo; k0 < hi; k0 += 32) {
            const bool v = k0 + lane < hi;
            const u32 t = v ? tgt[k0 + lane] : 0u;
            const int sl = v ? slot_of[t] : -1;
            const u32 hm = __ballot_sync(0xffffffffu, v && sl >= 0);
            const u32 cm = __ballot_sync(0xffffffffu, v && sl < 0);
            const u32 below = (1u << lane) - 1u;
            if (v) {
                if (sl >= 0) enc[hot0 + seen_hot + __popc(hm & below)] = PP_HOT_FLAG | (u32)sl;
                else enc[lo + seen_cold + __popc(cm & below)] = t;
            }
            seen_hot += __popc(hm);
            seen_cold += __popc(cm);
        }
    }
}

}  // namespace fr

using namespace fr;

struct fr_ppr {
    long long n, m;
    int B, grid;
    PprArgs a;
    PprCtl *ctl;
    double *parts;
    u64 *parts64;
    double *pull_buf;  // sent [n][B], rmax [n], part_max2 [2 grid], selection bitmap
    void *hub_buf;     // hub rows of the pull: nodes, segment starts, segment ranges and partial rows
    u32 *hot_buf;      // push: encoded column copy [m] + hot row ids [nhot]
    cudaGraph_t graph;
    cudaGraphExec_t exec;
    fr_solver_config cfg;
};

static int ppr_add(cudaGraph_t g, cudaGraphNode_t *node, const cudaGraphNode_t *dep, void *func, int grid, int block,
                   void **args, unsigned smem = 0) {
    cudaKernelNodeParams p = {};
    p.sharedMemBytes = smem;
    p.func = func;
    p.gridDim = dim3((unsigned)grid);
    p.blockDim = dim3((unsigned)block);
    p.kernelParams = args;
    FR_CUDA(cudaGraphAddKernelNode(node, g, dep, dep ? 1 : 0, &p));
    return FR_OK;
}

// prologue (theta0, masses, settle) then while { sweep (push, or take + pull),
// finalize, mass?, check? }
static int ppr_build_graph(fr_ppr *p) {
    if (p->exec) { cudaGraphExecDestroy(p->exec); p->exec = nullptr; }
    if (p->graph) { cudaGraphDestroy(p->graph); p->graph = nullptr; }
    PprArgs &a = p->a;
    FR_CUDA(cudaGraphCreate(&p->graph, 0));
    FR_CUDA(cudaGraphConditionalHandleCreate(&a.cond, p->graph, 0, 0));
    a.in_graph = 1;
    static int zero = 0, one = 1;
    void *args[] = {&a};
    void *args0[] = {&a, &zero};
    void *args1[] = {&a, &one};
    cudaGraphNode_t n1, n2, nw;
    FR_TRY(ppr_add(p->graph, &n1, nullptr, (void *)k_ppr_mass, p->grid, PP_NT, args0));
    FR_TRY(ppr_add(p->graph, &n2, &n1, (void *)k_ppr_settle, 1, 64, args0));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = a.cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    FR_CUDA(cudaGraphAddNode(&nw, p->graph, &n2, 1, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    cudaGraphNode_t b0, bp, b1, b2, b3;
    if (a.in_off) {
        cudaGraphNode_t bs, bh;
        FR_TRY(ppr_add(body, &b0, nullptr, (void *)k_ppr_take, p->grid, PP_NT, args));
        FR_TRY(ppr_add(body, &bs, &b0, (void *)k_ppr_pull, p->grid, PP_NT, args));
        FR_TRY(ppr_add(body, &bh, &bs, (void *)k_ppr_pull_segs, p->grid, PP_NT, args));
        FR_TRY(ppr_add(body, &bp, &bh, (void *)k_ppr_pull_hubs, p->grid, PP_NT, args));
    } else {
        FR_TRY(ppr_add(body, &bp, nullptr, (void *)k_ppr_sweep, p->grid, PP_NT, args,
                       (unsigned)(sizeof(double) * (size_t)a.nhot * (size_t)a.B)));
    }
    FR_TRY(ppr_add(body, &b1, &bp, (void *)k_ppr_finalize, 1, PP_NT, args));
    FR_TRY(ppr_add(body, &b2, &b1, (void *)k_ppr_mass, p->grid, PP_NT, args1));
    FR_TRY(ppr_add(body, &b3, &b2, (void *)k_ppr_settle, 1, 64, args1));
    FR_CUDA(cudaGraphInstantiate(&p->exec, p->graph, 0));
    return FR_OK;
}

static int ppr_host_loop(fr_ppr *p, cudaStream_t st) {
    PprArgs a = p->a;
    a.in_graph = 0;
    const unsigned smem = (unsigned)(sizeof(double) * (size_t)a.nhot * (size_t)a.B);
    k_ppr_mass<<<p->grid, PP_NT, 0, st>>>(a, 0);
    k_ppr_settle<<<1, 64, 0, st>>>(a, 0);
    for (;;) {
        if (a.in_off) {
            k_ppr_take<<<p->grid, PP_NT, 0, st>>>(a);
            k_ppr_pull<<<p->grid, PP_NT, 0, st>>>(a);
            k_ppr_pull_segs<<<p->grid, PP_NT, 0, st>>>(a);
            k_ppr_pull_hubs<<<p->grid, PP_NT, 0, st>>>(a);
        } else {
            k_ppr_sweep<<<p->grid, PP_NT, smem, st>>>(a);
        }
        k_ppr_finalize<<<1, PP_NT, 0, st>>>(a);
        k_ppr_mass<<<p->grid, PP_NT, 0, st>>>(a, 1);
        k_ppr_settle<<<1, 64, 0, st>>>(a, 1);
        FR_CUDA(cudaGetLastError());
        u32 stop = 0;
        FR_CUDA(cudaMemcpyAsync(&stop, &p->ctl->stop, sizeof(stop), cudaMemcpyDeviceToHost, st));
        FR_CUDA(cudaStreamSynchronize(st));
        if (stop) return FR_OK;
    }
}

extern "C" int fr_ppr_destroy(fr_ppr *p) {
    if (!p) return FR_OK;
    if (p->exec) cudaGraphExecDestroy(p->exec);
    if (p->graph) cudaGraphDestroy(p->graph);
    cudaFree(p->ctl);
    cudaFree(p->parts);
    cudaFree(p->parts64);
    cudaFree(p->pull_buf);
    cudaFree(p->hub_buf);
    cudaFree(p->hot_buf);
    delete p;
    return FR_OK;
}

extern "C" int fr_ppr_init(int64_t n, int32_t B, const uint32_t *d_seeds, int32_t k, double damping, double *d_fluid,
                           double *d_history, void *stream) {
    if (n < 1 || B < 1 || B > 64 || k < 1 || !d_seeds || !d_fluid || !d_history) {
        set_error("fr_ppr_init: need n >= 1, 1 <= B <= 64, k >= 1 and buffers");
        return FR_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    DeviceInfo di;
    FR_TRY(device_info(&di));
    k_ppr_init<<<di.sms * 8, 256, 0, st>>>(n, B, k, d_seeds, damping, d_fluid, d_history);
    k_ppr_seed<<<B, 128, 0, st>>>(B, k, d_seeds, damping, d_fluid);
    FR_CUDA(cudaGetLastError());
    return FR_OK;
}

extern "C" int fr_ppr_create(int64_t n, int64_t m, const int64_t *d_offsets, const uint32_t *d_targets, int32_t B,
                             double *d_fluid, double *d_history, const fr_solver_config *cfg, void *stream,
                             fr_ppr **out) {
    if (!out || !cfg || n < 1 || n > 0xFFFFFFFFll || m < 0 || B < 1 || B > 64 || !d_offsets || !d_fluid ||
        !d_history || (m > 0 && !d_targets)) {
        set_error("fr_ppr_create: bad arguments (1 <= B <= 64)");
        return FR_ERR_ARG;
    }
    if (!(cfg->damping > 0.0 && cfg->damping < 1.0) || !(cfg->target_error > 0.0) ||
        !(cfg->decay > 0.0 && cfg->decay < 1.0)) {
        set_error("fr_ppr_create: need 0 < damping < 1, target_error > 0, 0 < decay < 1");
        return FR_ERR_ARG;
    }
    (void)stream;
    DeviceInfo di;
    FR_TRY(device_info(&di));
    fr_ppr *p = new fr_ppr();
    p->n = n;
    p->m = m;
    p->B = B;
    p->cfg = *cfg;
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_ppr_sweep, PP_NT, 0);
    p->grid = std::max(1, per) * di.sms;
    int rc = FR_OK;
    do {
        cudaError_t e;
        if ((e = cudaMalloc(&p->ctl, sizeof(PprCtl))) != cudaSuccess ||
            (e = cudaMalloc(&p->parts, sizeof(double) * (size_t)p->grid * (64 + 1 + 64))) != cudaSuccess ||
            (e = cudaMalloc(&p->parts64, sizeof(u64) * (size_t)p->grid * 3)) != cudaSuccess) {
            rc = cuda_fail(e, "cudaMalloc(ppr)", __FILE__, __LINE__);
            break;
        }
        PprArgs &a = p->a;
        a.F = d_fluid;
        a.H = d_history;
        a.off = reinterpret_cast<const u64 *>(d_offsets);
        a.tgt = d_targets;
        a.ctl = p->ctl;
        a.part_abs = p->parts;
        a.part_max = p->parts + (size_t)p->grid * 64;
        a.part_mass = p->parts + (size_t)p->grid * 65;
        a.part_sel = p->parts64;
        a.part_steps = p->parts64 + p->grid;
        a.part_push = p->parts64 + 2 * (size_t)p->grid;
        a.n = n;
        a.B = B;
        a.nparts = p->grid;
        a.d = cfg->damping;
        a.thr = cfg->target_error * (1.0 - cfg->damping);
        a.decay = cfg->decay;
        a.max_sweeps = cfg->max_sweeps > 0 ? cfg->max_sweeps : 1000000;
        // hot rows: the nhot highest in-degree nodes (FR_PP_HOT, default 16; 0 = off)
        a.nhot = 0;
        {
            const char *env = getenv("FR_PP_HOT");
            int want = env ? atoi(env) : 16;
            want = std::max(0, std::min(want, PP_HOT_MAX));
            if (want > n) want = (int)n;
            if (want > 0 && m > 0 && n < (1ll << 31)) {
                Scratch scratch((cudaStream_t)stream);
                u32 *cnt;
                int *slot_of;
                if ((rc = scratch.alloc(&cnt, (size_t)n)) != FR_OK) break;
                if ((rc = scratch.alloc(&slot_of, (size_t)n)) != FR_OK) break;
                cudaStream_t st = (cudaStream_t)stream;
                cudaMemsetAsync(cnt, 0, sizeof(u32) * (size_t)n, st);
                k_ppr_indeg<<<di.sms * 8, 256, 0, st>>>(d_targets, m, cnt);
                std::vector<u32> hc((size_t)n);
                cudaMemcpyAsync(hc.data(), cnt, sizeof(u32) * (size_t)n, cudaMemcpyDeviceToHost, st);
                if ((e = cudaStreamSynchronize(st)) != cudaSuccess) { rc = cuda_fail(e, "ppr in-degree", __FILE__, __LINE__); break; }
                std::vector<u32> idx((size_t)n);
                for (long long i = 0; i < n; i++) idx[i] = (u32)i;
                std::partial_sort(idx.begin(), idx.begin() + want, idx.end(),
                                  [&](u32 x, u32 y) { return hc[x] != hc[y] ? hc[x] > hc[y] : x < y; });
                std::vector<int> so((size_t)n, -1);
                for (int k = 0; k < want; k++) so[idx[k]] = k;
                if ((e = cudaMalloc(&p->hot_buf, sizeof(u32) * ((size_t)m + want))) != cudaSuccess) {
                    rc = cuda_fail(e, "cudaMalloc(ppr hot rows)", __FILE__, __LINE__);
                    break;
                }
                cudaMemcpyAsync(slot_of, so.data(), sizeof(int) * (size_t)n, cudaMemcpyHostToDevice, st);
                k_ppr_encode<<<di.sms * 8, 256, 0, st>>>(reinterpret_cast<const u64 *>(d_offsets), n, d_targets,
                                                         slot_of, p->hot_buf);
                cudaMemcpyAsync(p->hot_buf + m, idx.data(), sizeof(u32) * want, cudaMemcpyHostToDevice, st);
                if ((e = cudaStreamSynchronize(st)) != cudaSuccess) { rc = cuda_fail(e, "ppr encode", __FILE__, __LINE__); break; }
                a.tgt_enc = p->hot_buf;
                a.hot_node = p->hot_buf + m;
                a.nhot = want;
            }
        }
        rc = ppr_build_graph(p);
    } while (0);
    if (rc != FR_OK) {
        fr_ppr_destroy(p);
        return rc;
    }
    *out = p;
    return FR_OK;
}

// Switches a handle to the pull formulation over the transposed CSR (the
// graph's in-edges: in_offsets int64[n+1], in_sources uint32[m], sources of
// each row ascending, as graph.py to_matrix()).
extern "C" int fr_ppr_set_pull(fr_ppr *p, const int64_t *d_in_offsets, const uint32_t *d_in_sources) {
    if (!p || !d_in_offsets || (p->m > 0 && !d_in_sources)) {
        set_error("fr_ppr_set_pull: need a handle and the transposed CSR");
        return FR_ERR_ARG;
    }
    PprArgs &a = p->a;
    if (!p->pull_buf) {
        const size_t nb = (size_t)p->n * p->B + (size_t)p->n + 2 * (size_t)p->grid + ((size_t)p->n + 63) / 64 + 1;
        cudaError_t e = cudaMalloc(&p->pull_buf, sizeof(double) * nb);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(ppr pull)", __FILE__, __LINE__);
        a.sent = p->pull_buf;
        a.rmax = a.sent + (size_t)p->n * p->B;
        a.part_max2 = a.rmax + p->n;
        a.selbits = reinterpret_cast<u32 *>(a.part_max2 + 2 * (size_t)p->grid);
    }
    // hub rows (more than PULL_LONG parents) and their PULL_SEG segments, from a
    // host copy of the in-offsets (once per handle)
    std::vector<int64_t> ioff((size_t)p->n + 1);
    FR_CUDA(cudaMemcpy(ioff.data(), d_in_offsets, sizeof(int64_t) * ioff.size(), cudaMemcpyDeviceToHost));
    std::vector<u32> hubs, hseg(1, 0);
    std::vector<u64> slo;
    for (long long i = 0; i < p->n; i++) {
        const u64 lo = (u64)ioff[i], hi = (u64)ioff[i + 1];
        if (hi - lo <= PULL_LONG) continue;
        hubs.push_back((u32)i);
        for (u64 b = lo; b < hi; b += PULL_SEG) slo.push_back(b);
        hseg.push_back((u32)slo.size());
    }
    std::vector<u64> srange;  // segment ends
    {
        size_t q = 0;
        for (size_t h = 0; h < hubs.size(); h++) {
            const u64 hi = (u64)ioff[hubs[h] + 1];
            for (; q < hseg[h + 1]; q++) srange.push_back(q + 1 < hseg[h + 1] ? slo[q + 1] : hi);
        }
    }
    cudaFree(p->hub_buf);
    p->hub_buf = nullptr;
    const size_t nh = hubs.size(), ns = slo.size();
    const size_t bytes = sizeof(u32) * (nh + nh + 1) + 16 + sizeof(u64) * 2 * ns + sizeof(double) * ns * p->B + 16;
    cudaError_t e = cudaMalloc(&p->hub_buf, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(ppr hubs)", __FILE__, __LINE__);
    char *b = (char *)p->hub_buf;
    u64 *d_lo = (u64 *)b;
    u64 *d_hi = d_lo + ns;
    double *d_acc = (double *)(d_hi + ns);
    u32 *d_hub = (u32 *)(d_acc + ns * p->B);
    u32 *d_hseg = d_hub + nh;
    if (ns) {
        FR_CUDA(cudaMemcpy(d_lo, slo.data(), sizeof(u64) * ns, cudaMemcpyHostToDevice));
        FR_CUDA(cudaMemcpy(d_hi, srange.data(), sizeof(u64) * ns, cudaMemcpyHostToDevice));
    }
    if (nh) FR_CUDA(cudaMemcpy(d_hub, hubs.data(), sizeof(u32) * nh, cudaMemcpyHostToDevice));
    FR_CUDA(cudaMemcpy(d_hseg, hseg.data(), sizeof(u32) * (nh + 1), cudaMemcpyHostToDevice));
    a.hub_node = d_hub;
    a.hub_seg = d_hseg;
    a.seg_lo = d_lo;
    a.seg_hi = d_hi;
    a.seg_acc = d_acc;
    a.nhub = (u32)nh;
    a.nseg = (u32)ns;
    p->a.in_off = reinterpret_cast<const u64 *>(d_in_offsets);
    p->a.in_src = d_in_sources;
    return ppr_build_graph(p);
}

extern "C" int fr_ppr_run(fr_ppr *p, void *stream, fr_solve_stats *h_stats, double *h_col_residual) {
    if (!p) { set_error("fr_ppr_run: null handle"); return FR_ERR_ARG; }
    cudaStream_t st = (cudaStream_t)stream;
    PprCtl init = {};
    init.active = p->B == 64 ? ~0ull : ((1ull << p->B) - 1ull);
    FR_CUDA(cudaMemcpyAsync(p->ctl, &init, sizeof(init), cudaMemcpyHostToDevice, st));
    if (getenv("FR_PPR_HOSTLOOP")) {
        // diagnostic (profilers): the graph's kernels launched from the host, one sweep
        // per stop-flag read-back, so ncu can select and time them one by one
        FR_TRY(ppr_host_loop(p, st));
    } else {
        FR_CUDA(cudaGraphLaunch(p->exec, st));
    }
    PprCtl c;
    FR_CUDA(cudaMemcpyAsync(&c, p->ctl, sizeof(c), cudaMemcpyDeviceToHost, st));
    FR_CUDA(cudaStreamSynchronize(st));
    if (h_stats) {
        h_stats->diffusions = (int64_t)c.diffusions;
        h_stats->elementary_steps = (int64_t)c.steps;
        h_stats->sweeps = (int64_t)c.sweeps;
        double mx = 0.0;
        for (int col = 0; col < p->B; col++) mx = std::max(mx, c.exact[col]);
        h_stats->residual = mx;
        h_stats->theta = c.theta;
        h_stats->trace_len = 0;
        h_stats->hub_edges = (int64_t)c.pushes;  // batched PPR: column values scattered
    }
    if (h_col_residual)
        for (int col = 0; col < p->B; col++) h_col_residual[col] = c.exact[col];
    // an explicit sweep budget is a normal stop (as fr_solver_run); only the implicit cap is an error
    if (c.active && p->cfg.max_sweeps <= 0) {
        set_error("batched PPR: %d columns did not converge within the sweep budget", __builtin_popcountll(c.active));
        return FR_ERR_NO_CONVERGENCE;
    }
    return FR_OK;
}

extern "C" int fr_ppr_normalize(int64_t n, int32_t B, const double *d_history, double *d_rank, void *stream) {
    if (n < 1 || B < 1 || B > 64 || !d_history || !d_rank) { set_error("fr_ppr_normalize: bad arguments"); return FR_ERR_ARG; }
    cudaStream_t st = (cudaStream_t)stream;
    DeviceInfo di;
    FR_TRY(device_info(&di));
    Scratch scratch(st);
    double *tot;
    FR_TRY(scratch.alloc(&tot, 64));
    FR_CUDA(cudaMemsetAsync(tot, 0, sizeof(double) * 64, st));
    k_ppr_colsum<<<di.sms * 4, PP_NT, 0, st>>>(n, B, d_history, tot);
    k_ppr_scale<<<di.sms * 8, 256, 0, st>>>(n, B, d_history, tot, d_rank);
    FR_CUDA(cudaGetLastError());
    FR_CUDA(cudaStreamSynchronize(st));
    return FR_OK;
}
