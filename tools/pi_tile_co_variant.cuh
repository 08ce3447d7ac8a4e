// Rejected variant of pi_tile (fr_spmv.cu), kept for the record: round 2, session 6.
// Measured on config 5 (profiles/r02_s6_spmv_coalesced.log): short rows 8.23 ms per
// iteration with 4 windows in flight (9.22 ms with 2) against 7.25 ms for the per-lane
// streams of pi_tile; parity tests pass.  To try it: paste above k_pi_rows in
// fr_spmv.cu and call pi_tile_co<HUB>(a, t, nrows, s_acc[w], gather, zw, c, diff, nd).
// Coalesced variant of pi_tile (FR_PI_COALESCED): the tile's compacted edge space is
// walked 32 consecutive edges at a time, one edge per lane, so a window's column indices
// are one coalesced load (one L1 wavefront instead of one per lane and index), and the
// gathered values are summed per row by a segmented shuffle scan over the lanes; the
// row of an edge position follows from a REDUX.OR head mask over the lane-compacted
// rows as in k_sweep_own (fr_diffuse.cu).  PI_CO_U windows are in flight per group.
#ifndef FR_PI_COALESCED
#define FR_PI_COALESCED 0
#endif
#ifndef FR_PI_CO_U
#define FR_PI_CO_U 4
#endif
template <bool HUB, typename G>
__device__ __forceinline__ void pi_tile_co(const PiArgs &a, long long t, long long nrows, double *s_acc, G gather,
                                           double *zw, double c, double &diff, double &nd) {
    constexpr u32 FULL = 0xffffffffu;
    constexpr int U = FR_PI_CO_U;
    const int lane = threadIdx.x & 31;
    const long long r = t * 32 + lane;
    const u32 *__restrict__ src = HUB ? a.hub_src : a.in_src;
    u64 lo = 0;
    u32 deg = 0;
    bool hub_row = false;
    if (r < nrows) {
        u64 dg;
        if (HUB) {
            lo = a.h_lo[r];
            dg = a.h_cnt[r];
        } else {
            lo = a.in_off[r];
            dg = a.in_off[r + 1] - lo;
        }
        if (dg > LONG_ROW) hub_row = true;  // hub rows (short kernel) / long slices (k_pi_segs)
        else deg = (u32)dg;
    }
    // the update's operands are loaded now, in flight with the gathers
    double xo = 0.0, wo = 0.0, vo = a.v_const;
    if (!HUB && r < nrows && !hub_row) {
        xo = a.x[r];
        wo = a.inv[r];
        if (a.v) vo = a.v[r];
    }
    u32 inc = deg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += y;
    }
    const u32 E = __shfl_sync(FULL, inc, 31);
    const u32 start = inc - deg;
    // the active rows of a tile lie in increasing order within a 2^32-edge span of src
    // (long slices, stored after the short ones, are not active here): 32-bit offsets
    // from the first active row's start
    const bool act = deg > 0;
    const u32 amask = __ballot_sync(FULL, act);
    const u64 lo0 = __shfl_sync(FULL, lo, amask ? __ffs((int)amask) - 1 : 0);
    const u32 na = (u32)__popc(amask);
    const u32 arank = (u32)__popc(amask & ((1u << lane) - 1u));
    int csrc = 0;  // lane of the (lane + 1)-th active row
#pragma unroll
    for (int s2 = 16; s2 > 0; s2 >>= 1) {
        const int x = csrc + s2;
        if ((u32)__popc(amask & ((1u << x) - 1u)) <= (u32)lane) csrc = x;
    }
    const u32 cst0 = __shfl_sync(FULL, start, csrc);
    const u32 cstart = (u32)lane < na ? cst0 : 0xffffffffu;
    const u32 cbase = __shfl_sync(FULL, (u32)(lo - lo0) - start, csrc);
    __syncwarp();
    s_acc[lane] = 0.0;
    __syncwarp();
    const u32 *__restrict__ src0 = src + lo0;
    for (u32 g0 = 0; g0 < E; g0 += 32u * U) {
        u32 idx[U], rr[U], hm[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const u32 w0 = g0 + 32u * u;
            idx[u] = 0;
            rr[u] = 0;
            hm[u] = 1u;
            if (w0 < E) {  // warp-uniform
                const u32 tt = cstart - w0;  // 1..31: this row's head lies inside the window
                const u32 heads = __reduce_or_sync(FULL, (tt - 1u < 31u) ? (1u << tt) : 0u);
                const u32 nb = (u32)__popc(__ballot_sync(FULL, cstart <= w0));  // >= 1
                const u32 p = w0 + (u32)lane;
                const u32 rk = nb + (u32)__popc(heads & ((2u << lane) - 1u)) - 1u;
                const u32 cb = __shfl_sync(FULL, cbase, (int)rk);
                if (p < E) idx[u] = __ldg(src0 + (u32)(cb + p));
                rr[u] = rk;
                hm[u] = heads | 1u;
            }
        }
        double zv[U];
#pragma unroll
        for (int u = 0; u < U; u++) zv[u] = g0 + 32u * u + (u32)lane < E ? gather(idx[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < U; u++) {
            const u32 w0 = g0 + 32u * u;
            if (w0 < E) {  // warp-uniform
                double x = zv[u];
                // segment head at or below this lane (bit 0: the row continuing from the last window)
                const int hp = 31 - __clz((int)(hm[u] & ((2u << lane) - 1u)));
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const double y = __shfl_up_sync(FULL, x, o);
                    if (lane - o >= hp) x += y;
                }
                const u32 p = w0 + (u32)lane;
                const bool tail = p < E && (lane == 31 || p == E - 1u || ((hm[u] >> ((lane + 1) & 31)) & 1u));
                if (tail) s_acc[rr[u]] += x;  // one lane per row and window
                __syncwarp();
            }
        }
    }
    if (r < nrows) {
        const double v = act ? s_acc[arank] : 0.0;
        if (HUB) {
            if (v != 0.0) atomicAdd(a.s_hub + (u64)r % a.nhub, v);
        } else if (!hub_row) {
            pi_update_row(a, r, v, c, zw, xo, wo, vo, diff, nd);
        }
    }
}

