// fr_capi.cu -- error state, device facts and the host-buffer end-to-end entry.
#include <stdarg.h>
#include <stdio.h>

#include <mutex>

#include "fr_common.cuh"

namespace fr {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int cuda_fail(cudaError_t e, const char *what, const char *file, int line) {
    set_error("CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e), cudaGetErrorString(e), file, line, what);
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return FR_ERR_NO_DEVICE;
    return FR_ERR_CUDA;
}

int device_info(DeviceInfo *out) {
    static thread_local DeviceInfo cache;
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice", __FILE__, __LINE__);
    if (cache.device != dev) {
        DeviceInfo d;
        d.device = dev;
        e = cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute", __FILE__, __LINE__);
        cudaDeviceGetAttribute(&d.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cache = d;
    }
    *out = cache;
    return FR_OK;
}

int pool_alloc(void **p, size_t bytes, cudaStream_t st) {
    static std::mutex mu;
    static bool configured[64] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice", __FILE__, __LINE__);
    {
        std::lock_guard<std::mutex> lock(mu);
        if (dev < 64 && !configured[dev]) {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                unsigned long long thr = ~0ull;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
            configured[dev] = true;
        }
    }
    if (bytes == 0) bytes = 16;
    e = cudaMallocAsync(p, bytes, st);
    if (e != cudaSuccess) {
        *p = nullptr;
        return cuda_fail(e, "cudaMallocAsync", __FILE__, __LINE__);
    }
    return FR_OK;
}

void pool_free(void *p, cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
}

}  // namespace fr

using namespace fr;

extern "C" const char *fr_last_error(void) { return g_err; }
extern "C" int fr_abi_version(void) { return FR_ABI_VERSION; }

extern "C" int fr_device_sms(void) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count < 1) {
        cudaGetLastError();
        return 0;
    }
    DeviceInfo di;
    return device_info(&di) == FR_OK ? di.sms : 0;
}

// fr_diffuse.cu: solver setup on column indices that arrive in pieces (encoded in place)
int solver_create_pieces(int64_t n, int64_t m, const int64_t *d_offsets, uint32_t *d_targets, void *d_fluid,
                         double *d_history, const fr_solver_config *cfg, void *stream, int count,
                         const long long *edge_end, const cudaEvent_t *ready, fr_solver **out);

static constexpr int HOST_PIECES = 8;  // column-index pieces of a large host-buffer solve

extern "C" int fr_pagerank_host(int64_t n, int64_t m, const int64_t *h_offsets, const uint32_t *h_targets,
                                const double *h_teleport, const fr_solver_config *cfg, double *h_rank,
                                fr_solve_stats *h_stats) {
    if (n < 1 || m < 0 || !h_offsets || (m > 0 && !h_targets) || !cfg || !h_rank) {
        set_error("fr_pagerank_host: bad arguments");
        return FR_ERR_ARG;
    }
    if (h_teleport) {
        // DiffusionParams.validate (engine.py:47-54): non-negative, sums to 1 within 1e-12
        double sum = 0.0, comp = 0.0;
        for (int64_t i = 0; i < n; i++) {
            const double v = h_teleport[i];
            if (!(v >= 0.0)) {
                set_error("teleport vector has negative entries");
                return FR_ERR_ARG;
            }
            const double y = v - comp, t = sum + y;  // compensated sum
            comp = (t - sum) - y;
            sum = t;
        }
        if (fabs(sum - 1.0) > 1e-12) {
            set_error("teleport vector sums to %.17g, expected 1", sum);
            return FR_ERR_ARG;
        }
    }
    // compute on st; the CSR travels on cs: offsets first, then the column
    // indices in pieces, so the solver setup (slot classes from the first
    // pieces, encoding of each piece as it lands) overlaps the copy
    cudaStream_t st, cs;
    FR_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    FR_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    const int pieces = m >= (1ll << 26) ? HOST_PIECES : 1;
    cudaEvent_t ev_alloc = nullptr, ev_off = nullptr, ev_tel = nullptr, ev_piece[HOST_PIECES] = {};
    long long edge_end[HOST_PIECES];
    int rc = FR_OK;
    fr_solver *s = nullptr;
    int64_t *d_off = nullptr;
    uint32_t *d_tgt = nullptr;
    double *d_h = nullptr;
    void *d_f = nullptr;
    const size_t fsz = cfg->fluid_fp32 ? sizeof(float) : sizeof(double);
    do {
        cudaError_t e;
        if ((rc = pool_alloc((void **)&d_off, sizeof(int64_t) * (size_t)(n + 1), st)) != FR_OK ||
            (rc = pool_alloc((void **)&d_tgt, sizeof(uint32_t) * (size_t)(m > 0 ? m : 1), st)) != FR_OK ||
            (rc = pool_alloc((void **)&d_h, sizeof(double) * (size_t)n, st)) != FR_OK ||
            (rc = pool_alloc(&d_f, fsz * (size_t)n, st)) != FR_OK)
            break;
        if ((e = cudaEventCreateWithFlags(&ev_alloc, cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&ev_off, cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&ev_tel, cudaEventDisableTiming)) != cudaSuccess) {
            rc = cuda_fail(e, "cudaEventCreate", __FILE__, __LINE__);
            break;
        }
        for (int k = 0; k < pieces && rc == FR_OK; k++)
            if ((e = cudaEventCreateWithFlags(&ev_piece[k], cudaEventDisableTiming)) != cudaSuccess)
                rc = cuda_fail(e, "cudaEventCreate", __FILE__, __LINE__);
        if (rc != FR_OK) break;
        // the copies may only start once the stream-ordered allocations exist
        if ((e = cudaEventRecord(ev_alloc, st)) != cudaSuccess || (e = cudaStreamWaitEvent(cs, ev_alloc, 0)) != cudaSuccess ||
            (e = cudaMemcpyAsync(d_off, h_offsets, sizeof(int64_t) * (size_t)(n + 1), cudaMemcpyHostToDevice, cs)) !=
                cudaSuccess ||
            (e = cudaEventRecord(ev_off, cs)) != cudaSuccess) {
            rc = cuda_fail(e, "cudaMemcpyAsync(H2D offsets)", __FILE__, __LINE__);
            break;
        }
        // the teleport vector lands in the history buffer: k_init_state reads tel[i]
        // before the same thread zeroes H[i], so no separate device copy is needed
        if (h_teleport &&
            ((e = cudaMemcpyAsync(d_h, h_teleport, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, cs)) !=
                 cudaSuccess ||
             (e = cudaEventRecord(ev_tel, cs)) != cudaSuccess)) {
            rc = cuda_fail(e, "cudaMemcpyAsync(H2D teleport)", __FILE__, __LINE__);
            break;
        }
        for (int k = 0; k < pieces; k++) {
            const long long b = k ? edge_end[k - 1] : 0;
            edge_end[k] = k + 1 == pieces ? (long long)m : ((long long)m * (k + 1) / pieces) & ~31ll;
            if (edge_end[k] > b &&
                (e = cudaMemcpyAsync(d_tgt + b, h_targets + b, sizeof(uint32_t) * (size_t)(edge_end[k] - b),
                                     cudaMemcpyHostToDevice, cs)) != cudaSuccess) {
                rc = cuda_fail(e, "cudaMemcpyAsync(H2D targets)", __FILE__, __LINE__);
                break;
            }
            if ((e = cudaEventRecord(ev_piece[k], cs)) != cudaSuccess) {
                rc = cuda_fail(e, "cudaEventRecord", __FILE__, __LINE__);
                break;
            }
        }
        if (rc != FR_OK) break;
        if (h_teleport && (e = cudaStreamWaitEvent(st, ev_tel, 0)) != cudaSuccess) {
            rc = cuda_fail(e, "cudaStreamWaitEvent", __FILE__, __LINE__);
            break;
        }
        if ((rc = fr_init_state(n, cfg->damping, h_teleport ? d_h : nullptr, d_f, cfg->fluid_fp32, d_h, st)) != FR_OK)
            break;
        if ((e = cudaStreamWaitEvent(st, ev_off, 0)) != cudaSuccess) {
            rc = cuda_fail(e, "cudaStreamWaitEvent", __FILE__, __LINE__);
            break;
        }
        if (pieces > 1) {
            rc = solver_create_pieces(n, m, d_off, d_tgt, d_f, d_h, cfg, st, pieces, edge_end, ev_piece, &s);
        } else {
            if ((e = cudaStreamWaitEvent(st, ev_piece[0], 0)) != cudaSuccess) {
                rc = cuda_fail(e, "cudaStreamWaitEvent", __FILE__, __LINE__);
                break;
            }
            rc = fr_solver_create(n, m, d_off, d_tgt, nullptr, d_f, d_h, cfg, 0, st, &s);
        }
        if (rc != FR_OK) break;
        // every piece has landed before the solve (setup may not have waited for all of them)
        if ((e = cudaStreamWaitEvent(st, ev_piece[pieces - 1], 0)) != cudaSuccess) {
            rc = cuda_fail(e, "cudaStreamWaitEvent", __FILE__, __LINE__);
            break;
        }
        if ((rc = fr_solver_run(s, st, h_stats)) != FR_OK) break;
        // rank = history / |history|_1, computed in place, then one D2H copy
        if ((rc = fr_normalize(n, d_h, d_h, nullptr, st)) != FR_OK) break;
        if ((e = cudaMemcpyAsync(h_rank, d_h, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, st)) != cudaSuccess) {
            rc = cuda_fail(e, "cudaMemcpyAsync(D2H)", __FILE__, __LINE__);
            break;
        }
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) rc = cuda_fail(e, "sync", __FILE__, __LINE__);
    } while (0);
    // the copy stream may still run after an error: let it drain before the frees
    cudaStreamSynchronize(cs);
    if (s) fr_solver_destroy(s);
    pool_free(d_off, st);
    pool_free(d_tgt, st);
    pool_free(d_h, st);
    pool_free(d_f, st);
    cudaStreamSynchronize(st);
    if (ev_alloc) cudaEventDestroy(ev_alloc);
    if (ev_off) cudaEventDestroy(ev_off);
    if (ev_tel) cudaEventDestroy(ev_tel);
    for (int k = 0; k < HOST_PIECES; k++)
        if (ev_piece[k]) cudaEventDestroy(ev_piece[k]);
    cudaStreamDestroy(cs);
    cudaStreamDestroy(st);
    return rc;
}
