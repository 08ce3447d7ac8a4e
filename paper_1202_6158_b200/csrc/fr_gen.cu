// fr_gen.cu -- seeded synthetic graph generator on the device (BASELINE.json
// configs 1-5).  Bit-identical to the specification in oracle/fr_oracle.c
// (fro_gen_degrees / fro_gen_edges): every value is a pure function of
// (seed, node, slot) through a counter-based hash, and the two lookup tables
// (power-law out-degree CDF, Zipf CDF) are built on the host by the same
// sequential double-precision loops, then uploaded.
#include <math.h>

#include <vector>

#include "fr_common.cuh"

namespace fr {

#define FR_GOLD 0x9E3779B97F4A7C15ull

__host__ __device__ __forceinline__ u64 mix64(u64 z) {
    z += FR_GOLD;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ u64 stream_key(u64 seed, u64 stream) { return mix64(seed + stream * FR_GOLD); }
__host__ __device__ __forceinline__ u64 frand(u64 key, u64 a, u64 b) { return mix64(mix64(key ^ a) + b); }
__device__ __forceinline__ double u53(u64 r) { return __dmul_rn((double)(r >> 11), 0x1.0p-53); }

enum { STREAM_DEG = 1, STREAM_EDGE = 3, STREAM_ZIPF = 4, STREAM_FEISTEL = 5 };

static uint32_t frac_to_u32(double f) {
    double x = floor(f * 4294967296.0);
    if (x < 0) x = 0;
    if (x > 4294967295.0) x = 4294967295.0;
    return (uint32_t)x;
}

__device__ __forceinline__ long long search_right(const double *__restrict__ cdf, long long len, double x) {
    long long lo = 0, hi = len - 1;
    while (lo < hi) {
        long long mid = lo + (hi - lo) / 2;
        if (__ldg(cdf + mid) > x) hi = mid; else lo = mid + 1;
    }
    return lo;
}

struct FeistelKeys {
    u64 k[4];
    int half;
};

__device__ __forceinline__ u64 feistel(u64 x, u64 n, const FeistelKeys &fk) {
    const u64 mask = (1ull << fk.half) - 1;
    do {
        u64 L = x >> fk.half, R = x & mask;
#pragma unroll
        for (int r = 0; r < 4; r++) {
            u64 t = R;
            R = L ^ (mix64(R ^ fk.k[r]) & mask);
            L = t;
        }
        x = (L << fk.half) | R;
    } while (x >= n);
    return x;
}

// ------------------------------------------------------------------ host tables
// Same loops, same order, as fro_gen_powerlaw_table / fro_gen_zipf_table.
static int powerlaw_table(const fr_gen_config *c, std::vector<double> &cdf, u64 *scale_q32) {
    int64_t kmax = c->max_degree;
    if (kmax < 1) return -1;
    cdf.resize((size_t)kmax);
    double cum = 0.0, wsum = 0.0, kwsum = 0.0;
    for (int64_t k = 1; k <= kmax; k++) {
        double w = pow((double)k, -c->alpha);
        cum += w;
        cdf[k - 1] = cum;
    }
    for (int64_t k = 1; k <= kmax; k++) {
        double w = pow((double)k, -c->alpha);
        wsum += w;
        kwsum += (double)k * w;
    }
    for (int64_t k = 0; k < kmax; k++) cdf[k] = cdf[k] / cum;
    cdf[kmax - 1] = 1.0;
    double p_live = 1.0 - (double)frac_to_u32(c->dangling_frac) / 4294967296.0;
    double mean_k = kwsum / wsum;
    double scale = c->mean_degree / (p_live * mean_k);
    *scale_q32 = (u64)llround(scale * 4294967296.0);
    return 0;
}

static void zipf_table(int64_t n, double s, double *cdf) {
    double cum = 0.0;
    for (int64_t k = 0; k < n; k++) {
        double w = (s == 1.0) ? 1.0 / (double)(k + 1) : pow((double)(k + 1), -s);
        cum += w;
        cdf[k] = cum;
    }
    for (int64_t k = 0; k < n; k++) cdf[k] = cdf[k] / cum;
    cdf[n - 1] = 1.0;
}

// ------------------------------------------------------------------ kernels
__global__ void k_gen_deg_uniform(long long n, u64 kd, int max_out, u32 *__restrict__ deg) {
    for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < n;
         u += (long long)gridDim.x * blockDim.x) {
        u64 g = frand(kd, (u64)u, 0) % (u64)(max_out + 1);
        if (n < 2) g = 0;
        else if (g > (u64)(n - 1)) g = (u64)(n - 1);
        deg[u] = (u32)g;
    }
}

__global__ void k_gen_deg_web(long long n, u64 kd, u32 dthr, const double *__restrict__ plcdf, int kmax,
                              u64 scale_q32, u32 *__restrict__ deg) {
    for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < n;
         u += (long long)gridDim.x * blockDim.x) {
        u64 g = 0;
        if (n >= 2 && (u32)(frand(kd, (u64)u, 0) >> 32) >= dthr) {
            u64 k = (u64)search_right(plcdf, kmax, u53(frand(kd, (u64)u, 1))) + 1;
            g = (k * scale_q32 + (frand(kd, (u64)u, 2) & 0xffffffffull)) >> 32;
            if (g < 1) g = 1;
            if (g > (u64)(n - 1)) g = (u64)(n - 1);
        }
        deg[u] = (u32)g;
    }
}

struct EdgeGenArgs {
    long long n;
    int kind;
    int window;
    u32 lthr;
    u64 ke, kz;
    FeistelKeys fk;
    const double *zcdf;
};

__device__ __forceinline__ u32 gen_target(const EdgeGenArgs &a, long long u, long long j, bool zipf_only) {
    u64 r = frand(a.ke, (u64)u, (u64)j);
    if (a.kind == 0) {
        u64 t = r % (u64)(a.n - 1);
        if (t >= (u64)u) t++;
        return (u32)t;
    }
    if (!zipf_only && (u32)(r >> 32) < a.lthr) {
        u32 w2 = 2u * (u32)a.window;
        long long o = (long long)((u32)r % w2);
        long long off = o < a.window ? o - a.window : o - a.window + 1;
        long long v = (u + off) % a.n;
        if (v < 0) v += a.n;
        return (u32)v;
    }
    long long rank = search_right(a.zcdf, a.n, u53(frand(a.kz, (u64)u, (u64)j)));
    return (u32)feistel((u64)rank, (u64)a.n, a.fk);
}

// first position in t[lo, hi) holding a value >= x
__device__ __forceinline__ long long lower_u32(const u32 *__restrict__ t, long long lo, long long hi, u64 x) {
    while (lo < hi) {
        const long long mid = lo + (hi - lo) / 2;
        if ((u64)t[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Ids of u's local window (u +- w, wrapped, u excluded) present in its sorted row.
__device__ long long window_count(const u32 *__restrict__ t, long long lo, long long hi, long long u, long long w,
                                  long long n) {
    auto range = [&](long long x, long long y) { return lower_u32(t, lo, hi, (u64)y + 1) - lower_u32(t, lo, hi, (u64)x); };
    if (2 * w + 1 >= n) return hi - lo;
    const long long x = u - w, y = u + w;
    if (x >= 0 && y < n) return range(x, y);
    if (x < 0) return range(0, y) + range(x + n, n - 1);
    return range(x, n - 1) + range(0, y - n);
}

// One warp per source node; lanes cover its slots.  Fill rounds pass the clean
// graph so far (off, tgt): a node whose local window it already completes
// draws from the Zipf class only.
__global__ void __launch_bounds__(256) k_gen_edges(EdgeGenArgs a, const u32 *__restrict__ deg,
                                                   const u64 *__restrict__ eoff, const u64 *__restrict__ off,
                                                   const u32 *__restrict__ tgt, u32 *__restrict__ src,
                                                   u32 *__restrict__ dst) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    const long long wfull = 2ll * a.window < a.n - 1 ? 2ll * a.window : a.n - 1;
    for (long long u = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); u < a.n; u += warps) {
        const long long g = deg[u];
        if (g == 0) continue;
        const u64 base = eoff[u];
        bool zonly = false;
        if (a.kind == 1 && off) {
            int full = 0;
            if (lane == 0) full = window_count(tgt, (long long)off[u], (long long)off[u + 1], u, a.window, a.n) >= wfull;
            zonly = __shfl_sync(0xffffffffu, full, 0) != 0;
        }
        for (long long j = lane; j < g; j += 32) {
            src[base + j] = (u32)u;
            dst[base + j] = gen_target(a, u, j, zonly);
        }
    }
}

int exclusive_scan_u32_to_u64(const u32 *in, u64 *out, long long n, cudaStream_t st);  // fr_scan.cu

}  // namespace fr

using namespace fr;

static int grid_for(long long work, int threads) {
    DeviceInfo di;
    if (device_info(&di) != FR_OK) return 0;
    long long g = (work + threads - 1) / threads;
    long long cap = (long long)di.sms * 16;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

static int check_gen_config(const fr_gen_config *c, int64_t n) {
    if (!c || n < 1 || n > 0xFFFFFFFFll) {
        set_error("generator: need 1 <= n < 2^32 and a config");
        return FR_ERR_ARG;
    }
    if (c->kind == 0) {
        if (c->max_out < 0) { set_error("generator: max_out must be >= 0"); return FR_ERR_ARG; }
    } else if (c->kind == 1) {
        if (c->max_degree < 1 || c->window < 1 || !(c->mean_degree > 0) || !(c->alpha > 0)) {
            set_error("generator: web config needs max_degree, window >= 1 and mean_degree, alpha > 0");
            return FR_ERR_ARG;
        }
    } else {
        set_error("generator: unknown kind %d", c->kind);
        return FR_ERR_ARG;
    }
    return FR_OK;
}

extern "C" int fr_gen_degrees(const fr_gen_config *c, int64_t n, uint64_t seed, uint32_t *d_deg,
                              int64_t *h_total, void *stream) {
    FR_TRY(check_gen_config(c, n));
    cudaStream_t st = (cudaStream_t)stream;
    Scratch scratch(st);
    const u64 kd = stream_key(seed, STREAM_DEG);
    const int threads = 256;
    if (c->kind == 0) {
        k_gen_deg_uniform<<<grid_for(n, threads), threads, 0, st>>>(n, kd, c->max_out, d_deg);
    } else {
        std::vector<double> cdf;
        u64 scale_q32;
        if (powerlaw_table(c, cdf, &scale_q32)) { set_error("generator: bad power-law table"); return FR_ERR_ARG; }
        double *d_cdf;
        FR_TRY(scratch.alloc(&d_cdf, cdf.size()));
        FR_CUDA(cudaMemcpyAsync(d_cdf, cdf.data(), cdf.size() * sizeof(double), cudaMemcpyHostToDevice, st));
        k_gen_deg_web<<<grid_for(n, threads), threads, 0, st>>>(n, kd, frac_to_u32(c->dangling_frac), d_cdf,
                                                                c->max_degree, scale_q32, d_deg);
        FR_CUDA(cudaGetLastError());
        // keep the table alive until the kernel has consumed it
        FR_CUDA(cudaStreamSynchronize(st));
    }
    FR_CUDA(cudaGetLastError());
    if (h_total) {
        u64 *d_off;
        FR_TRY(scratch.alloc(&d_off, (size_t)n + 1));
        FR_TRY(exclusive_scan_u32_to_u64(d_deg, d_off, n, st));
        u64 tot = 0;
        FR_CUDA(cudaMemcpyAsync(&tot, d_off + n, sizeof(u64), cudaMemcpyDeviceToHost, st));
        FR_CUDA(cudaStreamSynchronize(st));
        *h_total = (int64_t)tot;
    }
    return FR_OK;
}

extern "C" int fr_gen_edges(const fr_gen_config *c, int64_t n, uint64_t seed, const uint32_t *d_deg,
                            uint32_t *d_src, uint32_t *d_dst, void *stream) {
    return fr_gen_edges_round(c, n, seed, 0, d_deg, nullptr, nullptr, d_src, d_dst, stream);
}

// Fill round r > 0 redraws the slots that cleaning dropped (d_deg = per-node
// deficit) from fresh edge / Zipf streams; the Feistel permutation, a property
// of the graph, is the same in every round (oracle: fro_gen_edges_round).
static constexpr u64 FILL_GOLD = 0xD1B54A32D192ED03ull;

extern "C" int fr_gen_edges_round(const fr_gen_config *c, int64_t n, uint64_t seed, uint32_t round,
                                  const uint32_t *d_deg, const int64_t *d_offsets, const uint32_t *d_targets,
                                  uint32_t *d_src, uint32_t *d_dst, void *stream) {
    FR_TRY(check_gen_config(c, n));
    cudaStream_t st = (cudaStream_t)stream;
    Scratch scratch(st);
    EdgeGenArgs a;
    a.n = n;
    a.kind = c->kind;
    a.window = c->window;
    a.lthr = frac_to_u32(c->local_frac);
    a.ke = stream_key(seed, STREAM_EDGE);
    a.kz = stream_key(seed, STREAM_ZIPF);
    if (round) {
        a.ke = mix64(a.ke ^ ((u64)round * FILL_GOLD));
        a.kz = mix64(a.kz ^ ((u64)round * FILL_GOLD));
    }
    for (int r = 0; r < 4; r++) a.fk.k[r] = stream_key(seed, STREAM_FEISTEL + r);
    {
        int bits = 2;
        while ((1ull << bits) < (u64)n) bits++;
        if (bits & 1) bits++;
        a.fk.half = bits / 2;
    }
    a.zcdf = nullptr;
    std::vector<double> z;
    if (c->kind == 1) {
        z.resize((size_t)n);
        zipf_table(n, c->zipf_s, z.data());
        double *d_z;
        FR_TRY(scratch.alloc(&d_z, (size_t)n));
        FR_CUDA(cudaMemcpyAsync(d_z, z.data(), (size_t)n * sizeof(double), cudaMemcpyHostToDevice, st));
        a.zcdf = d_z;
    }
    u64 *d_eoff;
    FR_TRY(scratch.alloc(&d_eoff, (size_t)n + 1));
    FR_TRY(exclusive_scan_u32_to_u64(d_deg, d_eoff, n, st));
    DeviceInfo di;
    FR_TRY(device_info(&di));
    k_gen_edges<<<di.sms * 8, 256, 0, st>>>(a, d_deg, d_eoff, reinterpret_cast<const u64 *>(d_offsets), d_targets,
                                            d_src, d_dst);
    FR_CUDA(cudaGetLastError());
    FR_CUDA(cudaStreamSynchronize(st));  // host table z must outlive the upload
    return FR_OK;
}
