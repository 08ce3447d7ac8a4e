// fr_scan.cu -- exclusive prefix sum of uint32 counts into uint64 offsets
// (out has n+1 entries, out[n] = total): the "exclusive scan" stage of the
// device CSR construction and of the generator's edge offsets.
// Reduce-then-scan: tile sums -> single-block scan of tile sums -> tile rescan.
#include "fr_common.cuh"

namespace fr {

static constexpr int SCAN_NT = 256;
static constexpr int SCAN_IT = 16;
static constexpr long long SCAN_TILE = SCAN_NT * SCAN_IT;

// Loads the thread's SCAN_IT consecutive items (blocked arrangement).
__device__ __forceinline__ void load_blocked(const u32 *__restrict__ in, long long n, long long base, u32 v[SCAN_IT]) {
    const long long i0 = base + (long long)threadIdx.x * SCAN_IT;
    if (i0 + SCAN_IT <= n) {
        const uint4 *p = reinterpret_cast<const uint4 *>(in + i0);
#pragma unroll
        for (int q = 0; q < SCAN_IT / 4; q++) {
            uint4 x = ld_stream_u4(p + q);
            v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < SCAN_IT; q++) v[q] = (i0 + q < n) ? in[i0 + q] : 0u;
    }
}

__global__ void __launch_bounds__(SCAN_NT) k_scan_tiles(const u32 *__restrict__ in, long long n, u64 *__restrict__ tsum) {
    __shared__ u64 sm[SCAN_NT / 32];
    const long long base = (long long)blockIdx.x * SCAN_TILE;
    u32 v[SCAN_IT];
    load_blocked(in, n, base, v);
    u64 s = 0;
#pragma unroll
    for (int q = 0; q < SCAN_IT; q++) s += v[q];
    u64 t = block_sum_u64<SCAN_NT>(s, sm);
    if (threadIdx.x == 0) tsum[blockIdx.x] = t;
}

// Single block: in-place exclusive scan of tile sums; writes the grand total.
__global__ void __launch_bounds__(1024) k_scan_tsum(u64 *__restrict__ tsum, long long ntiles, u64 *__restrict__ total_out) {
    __shared__ u64 sm[1024 / 32 + 1];
    const long long per = (ntiles + 1023) / 1024;
    const long long b = threadIdx.x * per;
    const long long e = b + per < ntiles ? b + per : ntiles;
    u64 s = 0;
    for (long long i = b; i < e; i++) s += tsum[i];
    u64 tot;
    u64 run = block_excl_scan<1024>(s, sm, &tot);
    for (long long i = b; i < e; i++) {
        u64 x = tsum[i];
        tsum[i] = run;
        run += x;
    }
    if (threadIdx.x == 0) *total_out = tot;
}

__global__ void __launch_bounds__(SCAN_NT) k_scan_apply(const u32 *__restrict__ in, long long n, const u64 *__restrict__ tsum,
                                                        u64 *__restrict__ out) {
    __shared__ u64 sm[SCAN_NT / 32 + 1];
    const long long base = (long long)blockIdx.x * SCAN_TILE;
    u32 v[SCAN_IT];
    load_blocked(in, n, base, v);
    u64 s = 0;
#pragma unroll
    for (int q = 0; q < SCAN_IT; q++) s += v[q];
    u64 tot;
    u64 run = block_excl_scan<SCAN_NT>(s, sm, &tot) + tsum[blockIdx.x];
    const long long i0 = base + (long long)threadIdx.x * SCAN_IT;
#pragma unroll
    for (int q = 0; q < SCAN_IT; q++) {
        if (i0 + q < n) out[i0 + q] = run;
        run += v[q];
    }
}

int exclusive_scan_u32_to_u64(const u32 *in, u64 *out, long long n, cudaStream_t st) {
    if (n <= 0) {
        FR_CUDA(cudaMemsetAsync(out, 0, sizeof(u64), st));
        return FR_OK;
    }
    const long long ntiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    Scratch scratch(st);
    u64 *tsum;
    FR_TRY(scratch.alloc(&tsum, (size_t)ntiles));
    k_scan_tiles<<<(unsigned)ntiles, SCAN_NT, 0, st>>>(in, n, tsum);
    k_scan_tsum<<<1, 1024, 0, st>>>(tsum, ntiles, out + n);
    k_scan_apply<<<(unsigned)ntiles, SCAN_NT, 0, st>>>(in, n, tsum, out);
    FR_CUDA(cudaGetLastError());
    return FR_OK;
}

}  // namespace fr
