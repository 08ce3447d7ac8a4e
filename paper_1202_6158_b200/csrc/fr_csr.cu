// fr_csr.cu -- CSR construction on the device from an edge list.
//
// Replaces the reference's SparseGraph.from_edges (graph.py:74-97) and the
// cleaning pass build_clean_edges (graph.py:183-200):
//   1. out-degree histogram      (warp-aggregated atomics via match.any)
//   2. exclusive scan            (fr_scan.cu, uint32 counts -> int64 offsets)
//   3. counting-sort scatter     (warp-aggregated cursor atomics)
//   4. per-row sort + dedup, degree-binned:
//        deg <= 16        thread per row, insertion sort in registers/L1
//        17 .. 1024       warp per row, bitonic network in shared memory
//        1025 .. 49152    block per row, bitonic network in shared memory
//        > 49152          segmented bitonic network in global memory
//                         (one launch per stage over all huge rows)
//   5. scan of unique counts -> final offsets, squeeze of the unique prefixes
// Output is bit-identical to the reference: offsets = cumsum(bincount(src)),
// children of each row ascending (the reference's lexsort((dst, src))).
#include <algorithm>
#include <vector>

#include "fr_common.cuh"

namespace fr {

int exclusive_scan_u32_to_u64(const u32 *in, u64 *out, long long n, cudaStream_t st);

enum { FLAG_RANGE = 1, FLAG_LOOP = 2, FLAG_DUP = 4 };
static constexpr u32 NO_KEY = 0xFFFFFFFFu;
static constexpr int SMALL_MAX = 16;
static constexpr int WARP_MAX = 1024;
static constexpr int BLOCK_MAX = 49152;

struct CsrCounters {
    u64 loops;
    u64 dups;
    u32 flags;
    u32 n_warp, n_block, n_huge;
};

__device__ __forceinline__ u32 lanemask_lt() {
    u32 m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ------------------------------------------------------------------ 1. histogram
// Each warp walks 32 consecutive edges per step (coalesced 128 B loads of src
// and dst); lanes holding the same source merge their increments first.
__global__ void __launch_bounds__(256) k_csr_hist(const u32 *__restrict__ src, const u32 *__restrict__ dst, long long m,
                                                  long long n, int clean, u32 *__restrict__ cnt, CsrCounters *ctr) {
    const int lane = threadIdx.x & 31;
    const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
    long long loops = 0;
    u32 flags = 0;
    for (long long base = ((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; base < m;
         base += nwarps * 32) {
        const long long e = base + lane;
        u32 key = NO_KEY;
        if (e < m) {
            const u32 s = ld_stream_u32(src + e), t = ld_stream_u32(dst + e);
            if ((long long)s >= n || (long long)t >= n) flags |= FLAG_RANGE;
            else if (s == t) { loops++; if (!clean) flags |= FLAG_LOOP; }
            else key = s;
        }
        const u32 grp = __match_any_sync(0xffffffffu, key);
        if (key != NO_KEY && lane == __ffs(grp) - 1) atomicAdd(cnt + key, (u32)__popc(grp));
    }
    loops = (long long)warp_sum_u64((u64)loops);
    flags = __reduce_or_sync(0xffffffffu, flags);
    if (lane == 0) {
        if (loops) atomicAdd(&ctr->loops, (u64)loops);
        if (flags) atomicOr(&ctr->flags, flags);
    }
}

// ------------------------------------------------------------------ 3. scatter
__global__ void __launch_bounds__(256) k_csr_scatter(const u32 *__restrict__ src, const u32 *__restrict__ dst, long long m,
                                                     const u64 *__restrict__ raw_off, u32 *__restrict__ cursor,
                                                     u32 *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long base = ((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; base < m;
         base += nwarps * 32) {
        const long long e = base + lane;
        u32 key = NO_KEY, t = 0;
        if (e < m) {
            const u32 s = ld_stream_u32(src + e);
            t = ld_stream_u32(dst + e);
            if (s != t) key = s;  // range already validated
        }
        const u32 grp = __match_any_sync(0xffffffffu, key);
        const int leader = __ffs(grp) - 1;
        u32 slot = 0;
        if (key != NO_KEY && lane == leader) slot = atomicAdd(cursor + key, (u32)__popc(grp));
        slot = __shfl_sync(0xffffffffu, slot, leader);
        if (key != NO_KEY) out[raw_off[key] + slot + __popc(grp & lanemask_lt())] = t;
    }
}

// ------------------------------------------------------------------ 4a. small rows, thread per row
// Also routes larger rows to the warp / block / huge work lists.
__global__ void __launch_bounds__(256) k_csr_sort_small(long long n, const u64 *__restrict__ raw_off, u32 *__restrict__ tmp,
                                                        u32 *__restrict__ ucnt, u32 *__restrict__ list_warp,
                                                        u32 *__restrict__ list_block, u32 *__restrict__ list_huge,
                                                        CsrCounters *ctr) {
    const int lane = threadIdx.x & 31;
    u64 dups = 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    // uniform trip count across the warp so the ballots below are converged
    const long long start = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long trips = (n + stride - 1) / stride;
    for (long long tr = 0; tr < trips; tr++) {
        const long long i = start + tr * stride;
        int bin = -1;
        if (i < n) {
            const u64 b = raw_off[i], e = raw_off[i + 1];
            const u32 deg = (u32)(e - b);
            if (deg <= SMALL_MAX) {
                u32 v[SMALL_MAX];
                for (u32 k = 0; k < deg; k++) {
                    u32 x = tmp[b + k];
                    int p = (int)k - 1;
                    while (p >= 0 && v[p] > x) { v[p + 1] = v[p]; p--; }
                    v[p + 1] = x;
                }
                u32 w = 0;
                for (u32 k = 0; k < deg; k++) {
                    if (k > 0 && v[k] == v[k - 1]) continue;
                    tmp[b + w++] = v[k];
                }
                ucnt[i] = w;
                dups += deg - w;
            } else {
                bin = deg <= WARP_MAX ? 0 : (deg <= BLOCK_MAX ? 1 : 2);
            }
        }
#pragma unroll
        for (int q = 0; q < 3; q++) {
            const u32 mask = __ballot_sync(0xffffffffu, bin == q);
            if (mask) {
                u32 base = 0;
                const int leader = __ffs(mask) - 1;
                u32 *counter = q == 0 ? &ctr->n_warp : (q == 1 ? &ctr->n_block : &ctr->n_huge);
                u32 *list = q == 0 ? list_warp : (q == 1 ? list_block : list_huge);
                if (lane == leader) base = atomicAdd(counter, (u32)__popc(mask));
                base = __shfl_sync(0xffffffffu, base, leader);
                if (bin == q) list[base + __popc(mask & lanemask_lt())] = (u32)i;
            }
        }
    }
    dups = warp_sum_u64(dups);
    if (lane == 0 && dups) atomicAdd(&ctr->dups, dups);
}

// Comparator slot t of a flip-bitonic stage -> (lo, hi) positions.
__device__ __forceinline__ void bitonic_pair(u32 t, u32 k, u32 j, bool flip, u32 &lo, u32 &hi) {
    if (flip) {
        const u32 half = k >> 1, blk = t / half, off = t % half;
        lo = blk * k + off;
        hi = blk * k + (k - 1 - off);
    } else {
        lo = (t / j) * 2 * j + (t % j);
        hi = lo + j;
    }
}

// ------------------------------------------------------------------ 4b. warp per row (17..1024)
__global__ void __launch_bounds__(256) k_csr_sort_warp(const u32 *__restrict__ list, CsrCounters *ctr,
                                                       const u64 *__restrict__ raw_off, u32 *__restrict__ tmp,
                                                       u32 *__restrict__ ucnt) {
    __shared__ u32 sm_all[8][WARP_MAX];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    u32 *s = sm_all[wid];
    const u32 count = ctr->n_warp;
    u64 dups = 0;
    for (u32 r = blockIdx.x * 8 + wid; r < count; r += gridDim.x * 8) {
        const u32 row = list[r];
        const u64 b = raw_off[row];
        const u32 len = (u32)(raw_off[row + 1] - b);
        for (u32 k = lane; k < len; k += 32) s[k] = tmp[b + k];
        u32 P = 1;
        while (P < len) P <<= 1;
        __syncwarp();
        for (u32 k = 2; k <= P; k <<= 1) {
            for (u32 j = k >> 1; j > 0; j >>= 1) {
                const bool flip = (j == (k >> 1));
                for (u32 t = lane; t < P / 2; t += 32) {
                    u32 lo, hi;
                    bitonic_pair(t, k, j, flip, lo, hi);
                    if (hi < len) {
                        const u32 a = s[lo], c = s[hi];
                        if (a > c) { s[lo] = c; s[hi] = a; }
                    }
                }
                __syncwarp();
            }
        }
        u32 w = 0;
        for (u32 k0 = 0; k0 < len; k0 += 32) {
            const u32 k = k0 + lane;
            const bool keep = k < len && (k == 0 || s[k] != s[k - 1]);
            const u32 mask = __ballot_sync(0xffffffffu, keep);
            if (keep) tmp[b + w + __popc(mask & lanemask_lt())] = s[k];
            w += __popc(mask);
        }
        if (lane == 0) ucnt[row] = w;
        dups += len - w;
        __syncwarp();
    }
    if (lane == 0 && dups) atomicAdd(&ctr->dups, dups);
}

// ------------------------------------------------------------------ 4c. block per row (1025..49152)
__global__ void __launch_bounds__(1024) k_csr_sort_block(const u32 *__restrict__ list, CsrCounters *ctr,
                                                         const u64 *__restrict__ raw_off, u32 *__restrict__ tmp,
                                                         u32 *__restrict__ ucnt) {
    extern __shared__ u32 s[];
    __shared__ u64 scan_sm[1024 / 32 + 1];
    const u32 count = ctr->n_block;
    for (u32 r = blockIdx.x; r < count; r += gridDim.x) {
        const u32 row = list[r];
        const u64 b = raw_off[row];
        const u32 len = (u32)(raw_off[row + 1] - b);
        for (u32 k = threadIdx.x; k < len; k += blockDim.x) s[k] = tmp[b + k];
        u32 P = 1;
        while (P < len) P <<= 1;
        __syncthreads();
        for (u32 k = 2; k <= P; k <<= 1) {
            for (u32 j = k >> 1; j > 0; j >>= 1) {
                const bool flip = (j == (k >> 1));
                for (u32 t = threadIdx.x; t < P / 2; t += blockDim.x) {
                    u32 lo, hi;
                    bitonic_pair(t, k, j, flip, lo, hi);
                    if (hi < len) {
                        const u32 a = s[lo], c = s[hi];
                        if (a > c) { s[lo] = c; s[hi] = a; }
                    }
                }
                __syncthreads();
            }
        }
        u64 w = 0;
        for (u32 k0 = 0; k0 < len; k0 += blockDim.x) {
            const u32 k = k0 + threadIdx.x;
            const bool keep = k < len && (k == 0 || s[k] != s[k - 1]);
            u64 tot;
            const u64 pos = block_excl_scan<1024>(keep ? 1ull : 0ull, scan_sm, &tot);
            if (keep) tmp[b + w + pos] = s[k];
            w += tot;
        }
        if (threadIdx.x == 0) {
            ucnt[row] = (u32)w;
            if (len - w) atomicAdd(&ctr->dups, (u64)(len - w));
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ 4d. huge rows (> 49152)
// One launch per bitonic stage; blockIdx.y = huge row, x strides comparator slots.
__global__ void __launch_bounds__(256) k_csr_bitonic_stage(const u32 *__restrict__ list, u32 nhuge,
                                                           const u64 *__restrict__ raw_off, u32 *__restrict__ tmp,
                                                           u32 k, u32 j) {
    const bool flip = (j == (k >> 1));
    for (u32 h = blockIdx.y; h < nhuge; h += gridDim.y) {
        const u32 row = list[h];
        const u64 b = raw_off[row];
        const u32 len = (u32)(raw_off[row + 1] - b);
        u32 P = 1;
        while (P < len) P <<= 1;
        if (k > P) continue;  // this row already finished sorting
        u32 *a = tmp + b;
        for (u32 t = blockIdx.x * blockDim.x + threadIdx.x; t < P / 2; t += gridDim.x * blockDim.x) {
            u32 lo, hi;
            bitonic_pair(t, k, j, flip, lo, hi);
            if (hi < len) {
                const u32 x = a[lo], y = a[hi];
                if (x > y) { a[lo] = y; a[hi] = x; }
            }
        }
    }
}

// In-place forward compaction of a sorted huge row, chunk by chunk (one block
// per row).  A chunk only writes positions below its own end, and position
// k0-1 is either untouched or rewritten with its own value, so reading the
// left neighbour from global memory stays exact.
__global__ void __launch_bounds__(1024) k_csr_dedup_huge(const u32 *__restrict__ list, u32 nhuge,
                                                         const u64 *__restrict__ raw_off, u32 *__restrict__ tmp,
                                                         u32 *__restrict__ ucnt, CsrCounters *ctr) {
    __shared__ u64 scan_sm[1024 / 32 + 1];
    for (u32 h = blockIdx.x; h < nhuge; h += gridDim.x) {
        const u32 row = list[h];
        const u64 b = raw_off[row];
        const u32 len = (u32)(raw_off[row + 1] - b);
        u32 *a = tmp + b;
        u64 w = 0;
        for (u32 k0 = 0; k0 < len; k0 += blockDim.x) {
            const u32 k = k0 + threadIdx.x;
            const u32 x = k < len ? a[k] : 0u;
            const u32 left = (k > 0 && k < len) ? a[k - 1] : 0u;
            const bool keep = k < len && (k == 0 || x != left);
            u64 tot;
            const u64 pos = block_excl_scan<1024>(keep ? 1ull : 0ull, scan_sm, &tot);
            __syncthreads();  // every read of this chunk precedes any write of it
            if (keep) a[w + pos] = x;
            w += tot;
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            ucnt[row] = (u32)w;
            if (len - w) atomicAdd(&ctr->dups, (u64)(len - w));
        }
    }
}

__global__ void k_huge_maxlen(const u32 *__restrict__ list, u32 nhuge, const u64 *__restrict__ raw_off, u64 *out) {
    u64 mx = 0;
    for (u32 h = threadIdx.x; h < nhuge; h += blockDim.x) {
        const u32 row = list[h];
        const u64 len = raw_off[row + 1] - raw_off[row];
        mx = len > mx ? len : mx;
    }
    atomicMax(out, mx);
}

// ------------------------------------------------------------------ 5. squeeze
// Warp per row: copy the unique prefix of each row to its final place.
__global__ void __launch_bounds__(256) k_csr_squeeze(long long n, const u64 *__restrict__ raw_off,
                                                     const u64 *__restrict__ off, const u32 *__restrict__ tmp,
                                                     u32 *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long i = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nwarps) {
        const u64 src0 = raw_off[i], dst0 = off[i];
        const u64 len = off[i + 1] - dst0;
        for (u64 k = lane; k < len; k += 32) out[dst0 + k] = tmp[src0 + k];
    }
}

// In-degree counting.  Zipf in-degree hubs receive a large share of all
// increments and one address serialises in its L2 slice, so every counter is
// spread over INDEG_COPIES copies in separate regions (copy = warp % copies),
// summed afterwards.
static constexpr int INDEG_COPIES = 8;

__global__ void k_count_in_degree(const u32 *__restrict__ tgt, long long m, long long n, u32 *__restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
    u32 *__restrict__ copy = cnt + (size_t)(gw % INDEG_COPIES) * (size_t)n;
    for (long long base = gw * 32; base < m; base += nwarps * 32) {
        const long long e = base + lane;
        const u32 key = e < m ? ld_stream_u32(tgt + e) : NO_KEY;
        const u32 grp = __match_any_sync(0xffffffffu, key);
        if (key != NO_KEY && lane == __ffs(grp) - 1) atomicAdd(copy + key, (u32)__popc(grp));
    }
}

__global__ void k_sum_copies(const u32 *__restrict__ cnt, long long n, u64 *__restrict__ indeg) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        u64 s = 0;
#pragma unroll
        for (int c = 0; c < INDEG_COPIES; c++) s += cnt[(size_t)c * (size_t)n + i];
        indeg[i] = s;
    }
}

}  // namespace fr

using namespace fr;

extern "C" int fr_csr_build(int64_t n, int64_t m, const uint32_t *d_src, const uint32_t *d_dst, int32_t clean,
                            int64_t *d_offsets, uint32_t *d_targets, int64_t *h_stats, void *stream) {
    if (n < 0 || n > 0xFFFFFFFFll || m < 0 || !d_offsets || (m > 0 && (!d_src || !d_dst || !d_targets))) {
        set_error("fr_csr_build: bad arguments (n=%lld m=%lld)", (long long)n, (long long)m);
        return FR_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    DeviceInfo di;
    FR_TRY(device_info(&di));
    Scratch scratch(st);
    u64 *off = reinterpret_cast<u64 *>(d_offsets);
    if (n == 0) {
        FR_CUDA(cudaMemsetAsync(off, 0, sizeof(u64), st));
        if (h_stats) h_stats[0] = h_stats[1] = h_stats[2] = 0;
        if (m > 0) { set_error("edge endpoint out of range"); return FR_ERR_RANGE; }
        return FR_OK;
    }
    CsrCounters *ctr;
    u32 *cnt, *ucnt;
    u64 *raw_off;
    FR_TRY(scratch.alloc(&ctr, 1));
    FR_TRY(scratch.alloc(&cnt, (size_t)n));
    FR_TRY(scratch.alloc(&ucnt, (size_t)n));
    FR_TRY(scratch.alloc(&raw_off, (size_t)n + 1));
    FR_CUDA(cudaMemsetAsync(ctr, 0, sizeof(CsrCounters), st));
    FR_CUDA(cudaMemsetAsync(cnt, 0, sizeof(u32) * (size_t)n, st));
    const int g = di.sms * 8;

    // 1. histogram + validation
    if (m > 0) k_csr_hist<<<g, 256, 0, st>>>(d_src, d_dst, m, n, clean, cnt, ctr);
    FR_CUDA(cudaGetLastError());
    CsrCounters hc;
    FR_CUDA(cudaMemcpyAsync(&hc, ctr, sizeof(hc), cudaMemcpyDeviceToHost, st));
    FR_CUDA(cudaStreamSynchronize(st));
    if (hc.flags & FLAG_RANGE) { set_error("edge endpoint out of range"); return FR_ERR_RANGE; }
    if (hc.flags & FLAG_LOOP) { set_error("self-loop in edge arrays"); return FR_ERR_SELF_LOOP; }

    // 2. scan
    FR_TRY(exclusive_scan_u32_to_u64(cnt, raw_off, n, st));
    // 3. scatter (strict mode writes straight into the output)
    u32 *tmp = d_targets;
    if (clean) FR_TRY(scratch.alloc(&tmp, (size_t)m));
    FR_CUDA(cudaMemsetAsync(cnt, 0, sizeof(u32) * (size_t)n, st));
    if (m > 0) k_csr_scatter<<<g, 256, 0, st>>>(d_src, d_dst, m, raw_off, cnt, tmp);
    FR_CUDA(cudaGetLastError());

    // 4. per-row sort + dedup
    u32 *list_warp, *list_block, *list_huge;
    const size_t cap_warp = (size_t)std::min<long long>(n, m / (SMALL_MAX + 1) + 1);
    const size_t cap_block = (size_t)std::min<long long>(n, m / (WARP_MAX + 1) + 1);
    const size_t cap_huge = (size_t)std::min<long long>(n, m / (BLOCK_MAX + 1) + 1);
    FR_TRY(scratch.alloc(&list_warp, cap_warp));
    FR_TRY(scratch.alloc(&list_block, cap_block));
    FR_TRY(scratch.alloc(&list_huge, cap_huge));
    k_csr_sort_small<<<g, 256, 0, st>>>(n, raw_off, tmp, ucnt, list_warp, list_block, list_huge, ctr);
    k_csr_sort_warp<<<g, 256, 0, st>>>(list_warp, ctr, raw_off, tmp, ucnt);
    const size_t block_smem = BLOCK_MAX * sizeof(u32);
    FR_CUDA(cudaFuncSetAttribute(k_csr_sort_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)block_smem));
    k_csr_sort_block<<<di.sms, 1024, block_smem, st>>>(list_block, ctr, raw_off, tmp, ucnt);
    FR_CUDA(cudaGetLastError());
    FR_CUDA(cudaMemcpyAsync(&hc, ctr, sizeof(hc), cudaMemcpyDeviceToHost, st));
    FR_CUDA(cudaStreamSynchronize(st));
    if (hc.n_huge > 0) {
        // the largest huge row fixes the stage schedule
        u64 *d_maxlen;
        FR_TRY(scratch.alloc(&d_maxlen, 1));
        FR_CUDA(cudaMemsetAsync(d_maxlen, 0, sizeof(u64), st));
        k_huge_maxlen<<<1, 256, 0, st>>>(list_huge, hc.n_huge, raw_off, d_maxlen);
        u64 maxlen = 0;
        FR_CUDA(cudaMemcpyAsync(&maxlen, d_maxlen, sizeof(u64), cudaMemcpyDeviceToHost, st));
        FR_CUDA(cudaStreamSynchronize(st));
        u32 P = 1;
        while (P < maxlen) P <<= 1;
        const unsigned gy = std::min<u32>(hc.n_huge, 65535u);
        const unsigned gx = (unsigned)std::max<u64>(1, std::min<u64>((P / 2 + 255) / 256, (u64)di.sms * 8 / gy + 1));
        for (u32 k = 2; k <= P; k <<= 1)
            for (u32 j = k >> 1; j > 0; j >>= 1)
                k_csr_bitonic_stage<<<dim3(gx, gy), 256, 0, st>>>(list_huge, hc.n_huge, raw_off, tmp, k, j);
        k_csr_dedup_huge<<<std::min<u32>(hc.n_huge, (u32)di.sms), 1024, 0, st>>>(list_huge, hc.n_huge, raw_off, tmp,
                                                                               ucnt, ctr);
        FR_CUDA(cudaGetLastError());
        FR_CUDA(cudaMemcpyAsync(&hc, ctr, sizeof(hc), cudaMemcpyDeviceToHost, st));
        FR_CUDA(cudaStreamSynchronize(st));
    }
    if (!clean && hc.dups) { set_error("duplicate edge in edge arrays"); return FR_ERR_DUPLICATE; }

    // 5. final offsets and squeeze
    if (hc.dups == 0) {
        FR_CUDA(cudaMemcpyAsync(off, raw_off, sizeof(u64) * ((size_t)n + 1), cudaMemcpyDeviceToDevice, st));
        if (tmp != d_targets && m - (long long)hc.loops > 0)
            FR_CUDA(cudaMemcpyAsync(d_targets, tmp, sizeof(u32) * (size_t)(m - (long long)hc.loops),
                                    cudaMemcpyDeviceToDevice, st));
    } else {
        FR_TRY(exclusive_scan_u32_to_u64(ucnt, off, n, st));
        k_csr_squeeze<<<g, 256, 0, st>>>(n, raw_off, off, tmp, d_targets);
        FR_CUDA(cudaGetLastError());
    }
    FR_CUDA(cudaStreamSynchronize(st));
    if (h_stats) {
        h_stats[0] = (int64_t)(m - (long long)hc.loops - (long long)hc.dups);
        h_stats[1] = (int64_t)hc.dups;
        h_stats[2] = (int64_t)hc.loops;
    }
    return FR_OK;
}

extern "C" int fr_in_degree(int64_t n, int64_t m, const uint32_t *d_targets, int64_t *d_in_degree, void *stream) {
    if (n < 0 || m < 0 || (n > 0 && !d_in_degree)) { set_error("fr_in_degree: bad arguments"); return FR_ERR_ARG; }
    cudaStream_t st = (cudaStream_t)stream;
    DeviceInfo di;
    FR_TRY(device_info(&di));
    if (n == 0) return FR_OK;
    Scratch scratch(st);
    u32 *cnt;
    FR_TRY(scratch.alloc(&cnt, (size_t)n * INDEG_COPIES));
    FR_CUDA(cudaMemsetAsync(cnt, 0, sizeof(u32) * (size_t)n * INDEG_COPIES, st));
    if (m > 0) k_count_in_degree<<<di.sms * 8, 256, 0, st>>>(d_targets, m, n, cnt);
    k_sum_copies<<<di.sms * 8, 256, 0, st>>>(cnt, n, reinterpret_cast<u64 *>(d_in_degree));
    FR_CUDA(cudaGetLastError());
    return FR_OK;
}
