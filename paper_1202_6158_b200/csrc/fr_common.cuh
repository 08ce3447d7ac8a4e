// fr_common.cuh -- shared device/host helpers for the fluidrank B200 kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/fluidrank_b200.h"

namespace fr {

typedef unsigned long long u64;
typedef unsigned int u32;

// ---------------------------------------------------------------- errors
void set_error(const char *fmt, ...);
int cuda_fail(cudaError_t e, const char *what, const char *file, int line);

#define FR_CUDA(x)                                                              \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) return ::fr::cuda_fail(e_, #x, __FILE__, __LINE__); \
    } while (0)

#define FR_TRY(x)                   \
    do {                            \
        int rc_ = (x);              \
        if (rc_ != FR_OK) return rc_; \
    } while (0)

// Device facts cached per process (148 SMs on B200).
struct DeviceInfo {
    int device = -1;
    int sms = 0;
    int max_smem_optin = 0;
};
int device_info(DeviceInfo *out);

// Stream-ordered allocations from the device's default pool.  The pool keeps
// freed memory reserved (release threshold = max), so the multi-GB solver
// buffers of repeated create/destroy cycles (the host-buffer entry point)
// are recycled instead of being re-mapped by cudaMalloc/cudaFree each call.
int pool_alloc(void **p, size_t bytes, cudaStream_t st);
void pool_free(void *p, cudaStream_t st);

// Stream-ordered scratch allocation; freed in the destructor on the same stream.
struct Scratch {
    cudaStream_t stream;
    void *ptrs[16];
    int count = 0;
    explicit Scratch(cudaStream_t s) : stream(s) {}
    ~Scratch() {
        for (int i = count - 1; i >= 0; i--) pool_free(ptrs[i], stream);
    }
    template <typename T>
    int alloc(T **p, size_t elems) {
        size_t bytes = elems * sizeof(T);
        if (bytes == 0) bytes = 16;
        int rc = pool_alloc((void **)p, bytes, stream);
        if (rc != FR_OK) return rc;
        ptrs[count++] = *p;
        return FR_OK;
    }
};

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ u64 warp_sum_u64(u64 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Fixed-shape block reduction (deterministic for a fixed blockDim).
template <int NT>
__device__ __forceinline__ double block_sum(double v, double *smem /* NT/32 */) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) smem[w] = v;
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = l < NT / 32 ? smem[l] : 0.0;
        r = warp_sum(r);
    }
    return r;  // valid in thread 0
}
template <int NT>
__device__ __forceinline__ double block_max(double v, double *smem) {
    v = warp_max(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) smem[w] = v;
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = l < NT / 32 ? smem[l] : 0.0;
        r = warp_max(r);
    }
    return r;
}
template <int NT>
__device__ __forceinline__ u64 block_sum_u64(u64 v, u64 *smem) {
    v = warp_sum_u64(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) smem[w] = v;
    __syncthreads();
    u64 r = 0;
    if (w == 0) {
        r = l < NT / 32 ? smem[l] : 0ull;
        r = warp_sum_u64(r);
    }
    return r;
}

// Inclusive warp scan (u64).
__device__ __forceinline__ u64 warp_incl_scan(u64 v) {
    const int l = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u64 t = __shfl_up_sync(0xffffffffu, v, o);
        if (l >= o) v += t;
    }
    return v;
}

// Exclusive block scan (u64); returns the block total through *total.
template <int NT>
__device__ __forceinline__ u64 block_excl_scan(u64 v, u64 *smem /* NT/32 + 1 */, u64 *total) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    u64 inc = warp_incl_scan(v);
    __syncthreads();
    if (l == 31) smem[w] = inc;
    __syncthreads();
    if (w == 0) {
        u64 s = l < NT / 32 ? smem[l] : 0ull;
        u64 si = warp_incl_scan(s);
        if (l < NT / 32) smem[l] = si - s;
        if (l == NT / 32 - 1) smem[NT / 32] = si;
    }
    __syncthreads();
    *total = smem[NT / 32];
    return smem[w] + inc - v;
}

// Fire-and-forget global adds (REDG).
__device__ __forceinline__ void red_add(double *p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void red_add(float *p, float v) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// Fire-and-forget shared-memory add at a 32-bit shared-window address (ptxas expands it to
// the LDS + ATOMS.CAST.SPIN loop of atomicAdd, addressed from the caller's register instead
// of a shared base it re-derives at every site).
__device__ __forceinline__ void shared_red_add(u32 saddr, double v) {
    asm volatile("red.shared.add.f64 [%0], %1;" ::"r"(saddr), "d"(v) : "memory");
}
__device__ __forceinline__ void shared_red_add(u32 saddr, float v) {
    asm volatile("red.shared.add.f32 [%0], %1;" ::"r"(saddr), "f"(v) : "memory");
}

// Two predicated fire-and-forget global adds in one block (no branches): plain when `plain`,
// with the L2 cache-policy hint when `hinted`; neither flag set: nothing is issued.
__device__ __forceinline__ void red_add_pred2(double *p, double v, u64 pol, bool plain, bool hinted) {
    asm volatile(
        "{\n\t.reg .pred pn, pc;\n\t"
        "setp.ne.u32 pn, %3, 0;\n\t"
        "setp.ne.u32 pc, %4, 0;\n\t"
        "@pn red.global.add.f64 [%0], %1;\n\t"
        "@pc red.global.add.L2::cache_hint.f64 [%0], %1, %2;\n\t}"
        ::"l"(p), "d"(v), "l"(pol), "r"((u32)plain), "r"((u32)hinted)
        : "memory");
}
__device__ __forceinline__ void red_add_pred2(float *p, float v, u64 pol, bool plain, bool hinted) {
    asm volatile(
        "{\n\t.reg .pred pn, pc;\n\t"
        "setp.ne.u32 pn, %3, 0;\n\t"
        "setp.ne.u32 pc, %4, 0;\n\t"
        "@pn red.global.add.f32 [%0], %1;\n\t"
        "@pc red.global.add.L2::cache_hint.f32 [%0], %1, %2;\n\t}"
        ::"l"(p), "f"(v), "l"(pol), "r"((u32)plain), "r"((u32)hinted)
        : "memory");
}

// Fire-and-forget global add with an L2 cache-policy hint (createpolicy).
__device__ __forceinline__ void red_add_hint(double *p, double v, u64 pol) {
    asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void red_add_hint(float *p, float v, u64 pol) {
    asm volatile("red.global.add.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ u64 policy_evict_first() {
    u64 pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// Streaming (read-once) loads that do not allocate in L1.
__device__ __forceinline__ uint4 ld_stream_u4(const uint4 *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ u32 ld_stream_u32(const u32 *p) {
    u32 r;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

// mbarrier + bulk-copy (TMA engine, UBLKCP) helpers
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

}  // namespace fr
