// fr_util.cu -- state initialisation, L1 reductions, normalisation and the
// single-node diffusion step.
#include <math.h>

#include <map>
#include <mutex>
#include <utility>

#include "fr_common.cuh"

namespace fr {

static constexpr int RED_NT = 256;

template <typename FT>
__global__ void k_init_state(long long n, double damping, const double *__restrict__ tel, FT *__restrict__ F,
                             double *__restrict__ H) {
    const double inv_n = 1.0 / (double)n;
    const double scale = 1.0 - damping;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double v = tel ? tel[i] : inv_n;  // np.full(n, 1.0/n)
        F[i] = (FT)(damping >= 1.0 ? v : scale * v);
        if (H) H[i] = 0.0;
    }
}

template <typename FT>
__global__ void __launch_bounds__(RED_NT) k_abs_partials(long long n, const FT *__restrict__ x, double *__restrict__ part) {
    __shared__ double sm[RED_NT / 32];
    double s = 0.0;
    for (long long i = blockIdx.x * (long long)RED_NT + threadIdx.x; i < n; i += (long long)gridDim.x * RED_NT)
        s += fabs((double)x[i]);
    s = block_sum<RED_NT>(s, sm);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(RED_NT) k_sum_parts(const double *__restrict__ part, int nparts, double *out) {
    __shared__ double sm[RED_NT / 32];
    double s = 0.0;
    for (int p = threadIdx.x; p < nparts; p += RED_NT) s += part[p];
    s = block_sum<RED_NT>(s, sm);
    if (threadIdx.x == 0) *out = s;
}

// sum |x_i / total - ref_i| (engine.py:271-274: the trace's true L1 error of the
// normalized history); total = *d_total, 0 means "x is not normalized" (x used as is)
__global__ void __launch_bounds__(RED_NT) k_err_partials(long long n, const double *__restrict__ x,
                                                         const double *__restrict__ ref, const double *d_total,
                                                         double *__restrict__ part) {
    __shared__ double sm[RED_NT / 32];
    const double t = *d_total;
    const double inv = t > 0.0 ? 1.0 / t : 1.0;
    double s = 0.0;
    for (long long i = blockIdx.x * (long long)RED_NT + threadIdx.x; i < n; i += (long long)gridDim.x * RED_NT)
        s += fabs(x[i] * inv - ref[i]);
    s = block_sum<RED_NT>(s, sm);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_scale(long long n, const double *__restrict__ x, const double *total, double *__restrict__ y) {
    const double t = *total;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] = t > 0.0 ? x[i] / t : x[i];
}

// engine.py:175-199: one node, one warp.
__global__ void k_diffuse_node(const u64 *__restrict__ off, const u32 *__restrict__ tgt, double *F, double *H,
                               long long node, double d, double *sent_out) {
    const double sent = F[node];
    if (threadIdx.x == 0) *sent_out = sent;
    if (sent == 0.0) return;
    const u64 lo = off[node], hi = off[node + 1];
    __syncwarp();
    if (threadIdx.x == 0) {
        F[node] = 0.0;
        H[node] += sent;
    }
    __syncwarp();
    const double push = sent * (d / (double)(hi - lo));
    for (u64 k = lo + threadIdx.x; k < hi; k += 32) atomicAdd(F + tgt[k], push);
}

int reduce_grid(long long n) {
    DeviceInfo di;
    if (device_info(&di) != FR_OK) return 1;
    long long g = (n + RED_NT - 1) / RED_NT;
    long long cap = (long long)di.sms * 8;
    return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

// Persistent reduction scratch, one buffer per (device, stream): the L1 sums
// run every solve, and a stream-ordered malloc/free per call showed up as
// tens-of-milliseconds stalls in the solve timeline.  Never freed (a few KB).
static std::mutex g_scratch_mu;
static std::map<std::pair<int, cudaStream_t>, double *> g_scratch;
static constexpr size_t SCRATCH_DOUBLES = 8192;

int reduce_scratch(cudaStream_t st, double **out) {
    int dev = 0;
    FR_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_scratch_mu);
    auto key = std::make_pair(dev, st);
    auto it = g_scratch.find(key);
    if (it == g_scratch.end()) {
        double *p = nullptr;
        FR_CUDA(cudaMalloc(&p, sizeof(double) * SCRATCH_DOUBLES));
        it = g_scratch.emplace(key, p).first;
    }
    *out = it->second;
    return FR_OK;
}

// sum |x| into the device double *d_out, stream-ordered, no host sync.
int abs_sum_async(long long n, const void *x, int fp32, double *d_out, cudaStream_t st) {
    double *part;
    FR_TRY(reduce_scratch(st, &part));
    const int g = reduce_grid(n);
    if ((size_t)g + 1 > SCRATCH_DOUBLES) { set_error("reduction scratch too small"); return FR_ERR_ARG; }
    if (fp32) k_abs_partials<float><<<g, RED_NT, 0, st>>>(n, (const float *)x, part);
    else k_abs_partials<double><<<g, RED_NT, 0, st>>>(n, (const double *)x, part);
    k_sum_parts<<<1, RED_NT, 0, st>>>(part, g, d_out);
    FR_CUDA(cudaGetLastError());
    return FR_OK;
}

// |x/|x|_1 - ref|_1 into the device double *d_out, stream-ordered.
int l1_error_async(long long n, const double *x, const double *ref, double *d_out, cudaStream_t st) {
    double *part;
    FR_TRY(reduce_scratch(st, &part));
    const int g = reduce_grid(n);
    if ((size_t)g + 2 > SCRATCH_DOUBLES) { set_error("reduction scratch too small"); return FR_ERR_ARG; }
    double *d_total = part + SCRATCH_DOUBLES - 2;
    FR_TRY(abs_sum_async(n, x, 0, d_total, st));
    k_err_partials<<<g, RED_NT, 0, st>>>(n, x, ref, d_total, part);
    k_sum_parts<<<1, RED_NT, 0, st>>>(part, g, d_out);
    FR_CUDA(cudaGetLastError());
    return FR_OK;
}

}  // namespace fr

using namespace fr;

extern "C" int fr_l1_error(int64_t n, const double *d_history, const double *d_reference, double *h_err,
                           void *stream) {
    if (n < 1 || !d_history || !d_reference || !h_err) { set_error("fr_l1_error: bad arguments"); return FR_ERR_ARG; }
    cudaStream_t st = (cudaStream_t)stream;
    double *part;
    FR_TRY(reduce_scratch(st, &part));
    double *d_out = part + SCRATCH_DOUBLES - 1;
    FR_TRY(l1_error_async(n, d_history, d_reference, d_out, st));
    FR_CUDA(cudaMemcpyAsync(h_err, d_out, sizeof(double), cudaMemcpyDeviceToHost, st));
    FR_CUDA(cudaStreamSynchronize(st));
    return FR_OK;
}

extern "C" int fr_init_state(int64_t n, double damping, const double *d_teleport, void *d_fluid, int32_t fluid_fp32,
                             double *d_history, void *stream) {
    if (n < 1 || !d_fluid) { set_error("fr_init_state: bad arguments"); return FR_ERR_ARG; }
    cudaStream_t st = (cudaStream_t)stream;
    const int g = reduce_grid(n);
    if (fluid_fp32) k_init_state<float><<<g, RED_NT, 0, st>>>(n, damping, d_teleport, (float *)d_fluid, d_history);
    else k_init_state<double><<<g, RED_NT, 0, st>>>(n, damping, d_teleport, (double *)d_fluid, d_history);
    FR_CUDA(cudaGetLastError());
    return FR_OK;
}

extern "C" int fr_abs_sum(int64_t n, const void *d_x, int32_t x_fp32, double *h_sum, void *stream) {
    if (n < 0 || (n > 0 && !d_x) || !h_sum) { set_error("fr_abs_sum: bad arguments"); return FR_ERR_ARG; }
    if (n == 0) { *h_sum = 0.0; return FR_OK; }
    cudaStream_t st = (cudaStream_t)stream;
    double *part;
    FR_TRY(reduce_scratch(st, &part));
    double *d_out = part + SCRATCH_DOUBLES - 1;
    FR_TRY(abs_sum_async(n, d_x, x_fp32, d_out, st));
    FR_CUDA(cudaMemcpyAsync(h_sum, d_out, sizeof(double), cudaMemcpyDeviceToHost, st));
    FR_CUDA(cudaStreamSynchronize(st));
    return FR_OK;
}

extern "C" int fr_normalize(int64_t n, const double *d_history, double *d_rank, double *h_total, void *stream) {
    if (n < 1 || !d_history || !d_rank) { set_error("fr_normalize: bad arguments"); return FR_ERR_ARG; }
    cudaStream_t st = (cudaStream_t)stream;
    double *part;
    FR_TRY(reduce_scratch(st, &part));
    double *d_total = part + SCRATCH_DOUBLES - 1;
    FR_TRY(abs_sum_async(n, d_history, 0, d_total, st));
    k_scale<<<reduce_grid(n), RED_NT, 0, st>>>(n, d_history, d_total, d_rank);
    FR_CUDA(cudaGetLastError());
    if (h_total) {
        FR_CUDA(cudaMemcpyAsync(h_total, d_total, sizeof(double), cudaMemcpyDeviceToHost, st));
        FR_CUDA(cudaStreamSynchronize(st));
    }
    return FR_OK;
}

extern "C" int fr_diffuse_node(int64_t n, const int64_t *d_offsets, const uint32_t *d_targets, double *d_fluid,
                               double *d_history, int64_t node, double damping, double *h_sent, void *stream) {
    if (node < 0 || node >= n) { set_error("node %lld out of range", (long long)node); return FR_ERR_ARG; }
    cudaStream_t st = (cudaStream_t)stream;
    Scratch scratch(st);
    double *d_sent;
    FR_TRY(scratch.alloc(&d_sent, 1));
    k_diffuse_node<<<1, 32, 0, st>>>(reinterpret_cast<const u64 *>(d_offsets), d_targets, d_fluid, d_history, node,
                                     damping, d_sent);
    FR_CUDA(cudaGetLastError());
    double sent = 0.0;
    FR_CUDA(cudaMemcpyAsync(&sent, d_sent, sizeof(double), cudaMemcpyDeviceToHost, st));
    FR_CUDA(cudaStreamSynchronize(st));
    if (h_sent) *h_sent = sent;
    return FR_OK;
}
