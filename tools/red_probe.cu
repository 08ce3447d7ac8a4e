// red_probe.cu -- calibrate red.global.add.f64 throughput on B200 against the
// footprint and locality of the targets (tools/, not part of the product).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_probe red_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ void red_add(double *p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// mode 0: uniform random over [0, window) ; mode 1: i + (+-1000) local, i streamed in order
// mode 2: like 1 but plain load + store (non-atomic, racy) to compare ; mode 3: atomicAdd (returning)
// mode 11: local pattern, warps take 128-node chunks in order from a global counter
__global__ void probe_dyn(double *F, long long n, long long total, unsigned long long *ctr) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned long long k = 0;
        if (lane == 0) k = atomicAdd(ctr, 1ull);
        k = __shfl_sync(0xffffffffu, k, 0);
        const long long base = (long long)k * 128;
        if (base >= total) break;
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const long long i = base + u * 32 + lane;
            uint64_t h = mix((uint64_t)i * 0x9E37ull + 17);
            long long off = (long long)(h % 2001) - 1000;
            long long t = ((i % n) + off + n) % n;
            red_add(F + t, 1.0);
        }
    }
}

__global__ void probe(double *F, long long n, long long window, long long per_thread, int mode, double *sink) {
    const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long nt = (long long)gridDim.x * blockDim.x;
    double acc = 0;
    for (long long k = 0; k < per_thread; k++) {
        const long long i = k * nt + tid;  // streamed index
        uint64_t h = mix((uint64_t)i * 0x9E37ull + 17);
        long long t;
        if (mode == 0) t = (long long)(h % (uint64_t)window);
        else if (mode == 4) t = 0;
        else if (mode == 5 || mode == 6 || mode == 9 || mode == 10) {
            // approx Zipf(1) rank over [0, n): t = floor(n^u) - 1
            const double u = (double)(h >> 11) * 0x1.0p-53;
            t = (long long)exp(u * log((double)n)) - 1;
            if (t < 0) t = 0;
            if (t >= n) t = n - 1;
            if (mode == 9 || mode == 10) {
                if (t < 2048) continue;  // aggregated in shared memory instead
                if (mode == 10 && t < 2000000) { red_add(F + t, 1.0); continue; }  // compact L2-resident hub array
            }
            if (mode != 5) t = (long long)(((uint64_t)t * 0x9E3779B97F4A7C15ull) % (uint64_t)n);
        } else {
            long long off = (long long)(h % 2001) - 1000;
            t = ((i % n) + off + n) % n;
        }
        if (mode == 7 || mode == 8) {
            // prefetch the line 4096 nodes ahead of the streamed front into L2
            const long long pf = (i % n) + (mode == 7 ? 4096 : 16384);
            if (pf < n) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(F + pf));
        }
        if (mode == 2) { F[t] = F[t] + 1.0; }
        else if (mode == 3) acc += atomicAdd(F + t, 1.0);
        else red_add(F + t, 1.0);
    }
    if (acc == 12345.0) *sink = acc;
}

// element-type comparison: the same target streams with f64, f32 and u64 reds
__device__ __forceinline__ void red_t(double *p) { asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(1.0) : "memory"); }
__device__ __forceinline__ void red_t(float *p) { asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(1.0f) : "memory"); }
__device__ __forceinline__ void red_t(unsigned long long *p) {
    asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(1ull) : "memory");
}
template <typename T>
__global__ void probe_type(T *F, long long n, long long window, long long per_thread, int local) {
    const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long nt = (long long)gridDim.x * blockDim.x;
    for (long long k = 0; k < per_thread; k++) {
        const long long i = k * nt + tid;
        uint64_t h = mix((uint64_t)i * 0x9E37ull + 17);
        long long t;
        if (local) {
            long long off = (long long)(h % 2001) - 1000;
            t = ((i % n) + off + n) % n;
        } else {
            t = (long long)(h % (uint64_t)window);
        }
        red_t(F + t);
    }
}
template <typename T>
void run_type(const char *name, T *F, long long n, int blocks, int threads, long long per) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const long long nt = (long long)blocks * threads;
    for (int local = 0; local < 2; local++) {
        for (long long w : {1ll << 23, n}) {
            if (local && w != n) continue;
            probe_type<T><<<blocks, threads>>>(F, n, w, per, local);
            cudaEventRecord(a);
            probe_type<T><<<blocks, threads>>>(F, n, w, per, local);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("%-4s %-30s %8.3f ms  %7.1f G ops/s\n", name,
                   local ? "local +-1000, streamed" : (w == n ? "uniform, all n" : "uniform, 8M elements"), ms,
                   per * nt / (ms * 1e6));
        }
    }
}

int main() {
    const long long n = 100000000;  // 800 MB of doubles
    double *F, *sink;
    cudaMalloc(&F, n * sizeof(double));
    cudaMalloc(&sink, 8);
    cudaMemset(F, 0, n * sizeof(double));
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256;
    const long long nt = (long long)blocks * threads;
    const long long total = 400000000;  // reds per launch
    const long long per = total / nt;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    struct { int mode; long long window; const char *name; } cases[] = {
        {0, 1 << 17, "uniform 1 MB"},   {0, 1 << 21, "uniform 16 MB"}, {0, 1 << 23, "uniform 64 MB"},
        {0, 1 << 24, "uniform 128 MB"}, {0, 1 << 25, "uniform 256 MB"}, {0, n, "uniform 800 MB"},
        {1, n, "local +-1000, streamed"}, {2, n, "local, plain ld+st"}, {3, n, "local, atomicAdd returning"},
        {3, 1 << 21, "uniform 16 MB atomicAdd returning"}, {4, n, "single address"},
        {5, n, "zipf(1) ranks contiguous (hub-first)"}, {6, n, "zipf(1) ranks scattered"},
        {9, n, "zipf scattered, top-2048 ranks removed"}, {10, n, "zipf: top-2048 removed, ranks<2M compact"}};
    for (auto &c : cases) {
        probe<<<blocks, threads>>>(F, n, c.window, per, c.mode, sink);  // warm
        cudaEventRecord(a);
        probe<<<blocks, threads>>>(F, n, c.window, per, c.mode, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-36s %8.3f ms  %7.1f G ops/s\n", c.name, ms, per * nt / (ms * 1e6));
    }
    {
        unsigned long long *ctr;
        cudaMalloc(&ctr, 8);
        for (int rep = 0; rep < 2; rep++) {
            cudaMemset(ctr, 0, 8);
            cudaEventRecord(a);
            probe_dyn<<<blocks, threads>>>(F, n, per * nt, ctr);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("%-36s %8.3f ms  %7.1f G ops/s\n", "local, in-order dynamic chunks", ms, per * nt / (ms * 1e6));
        }
    }
    run_type<double>("f64", F, n, blocks, threads, per);
    run_type<float>("f32", reinterpret_cast<float *>(F), n, blocks, threads, per);
    run_type<unsigned long long>("u64", reinterpret_cast<unsigned long long *>(F), n, blocks, threads, per);
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
