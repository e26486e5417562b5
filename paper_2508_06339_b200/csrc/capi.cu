// capi.cu -- C ABI of libbsvd (include/bsvd.h): validation, workspace
// planning and the stream-ordered stage pipeline.  Mirrors
// secondstage.py:510-542 svdvals:  validate -> pad -> stage 1 -> stage 2 ->
// stage 3 -> first orig_n values, descending, compute dtype.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

#include <atomic>

static thread_local char g_err[512] = "";
static std::atomic<unsigned long long> g_launches{0};

namespace bsvd_host {
void count_launch(unsigned n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
bsvd_status set_error(bsvd_status st, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return st;
}
bsvd_status cuda_error(cudaError_t e, const char *where) {
    if (e == cudaErrorMemoryAllocation)
        return set_error(BSVD_E_OOM, "CUDA out of memory in %s", where);
    return set_error(BSVD_E_CUDA, "CUDA error %s (%s) in %s", cudaGetErrorName(e),
                     cudaGetErrorString(e), where);
}
}  // namespace bsvd_host

using namespace bsvd;
using bsvd_host::cuda_error;
using bsvd_host::set_error;

namespace {

size_t elem_size(bsvd_dtype d) { return d == BSVD_FP64 ? 8 : (d == BSVD_FP32 ? 4 : 2); }
size_t compute_size(bsvd_dtype d) { return d == BSVD_FP64 ? 8 : 4; }
bool dtype_ok(int d) { return d == BSVD_FP64 || d == BSVD_FP32 || d == BSVD_FP16; }
size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

bsvd_config resolve_cfg(const bsvd_config *cfg, int64_t n) {
    bsvd_config c;
    if (cfg) {
        c = *cfg;
    } else {
        c.tilesize = bsvd_default_tilesize(n);
        c.colperblock = 0;
        c.splitk = 1;
        c.fused = 1;
    }
    if (c.colperblock <= 0) c.colperblock = c.tilesize;
    return c;
}

bool use_flat(bsvd_dtype dt, int ts) { return flat_supported(ts, dt == BSVD_FP64 ? 8 : 4); }

struct Plan {
    int64_t n, N, np, batch;
    int ts;
    size_t off_flag, off_scale, off_work, off_d, off_e, off_scratch, total;
    size_t stage1_bytes, chase_bytes, bisect_bytes;
};

Plan make_plan(bsvd_dtype dt, int64_t n, int64_t batch, const bsvd_config &c, int algo) {
    Plan p{};
    p.n = n;
    p.ts = c.tilesize;
    p.N = std::max<int64_t>(1, (n + p.ts - 1) / p.ts);
    p.np = p.N * p.ts;
    p.batch = batch;
    const size_t es = elem_size(dt), cs = compute_size(dt);
    size_t s1;
    if (algo == BSVD_STAGE1_FAITHFUL) {
        s1 = (size_t)p.ts * 2 * p.N * p.N * cs;   // TauStore, matrix.py:184-215
    } else {
        switch (dt) {
        case BSVD_FP64: s1 = tree_workspace_bytes<double, double>(p.np, p.ts); break;
        case BSVD_FP32: s1 = tree_workspace_bytes<float, float>(p.np, p.ts); break;
        default: s1 = tree_workspace_bytes<__half, float>(p.np, p.ts); break;
        }
        s1 *= (size_t)batch;
        if (use_flat(dt, p.ts)) s1 = std::max(s1, flat_workspace_bytes(p.np, p.ts, batch));
    }
    p.stage1_bytes = align_up(s1);
    p.chase_bytes = align_up(chase_workspace_bytes(p.np, p.ts, batch));
    p.bisect_bytes = align_up(bisect_workspace_bytes(p.np, batch));
    size_t off = 0;
    p.off_flag = off;  off += 256;
    p.off_scale = off; off += align_up((size_t)batch * 16);   // amax bits | unscale
    p.off_work = off;  off += align_up((size_t)batch * p.np * p.np * es);
    p.off_d = off;     off += align_up((size_t)batch * p.np * 8);
    p.off_e = off;     off += align_up((size_t)batch * p.np * 8);
    p.off_scratch = off;
    off += std::max(p.stage1_bytes, std::max(p.chase_bytes, p.bisect_bytes));
    p.total = off;
    return p;
}

bsvd_status check_common(bsvd_dtype dtype, int64_t n, int64_t lda, const bsvd_config &c) {
    if (!dtype_ok(dtype)) return set_error(BSVD_E_CONFIG, "unsupported dtype code %d", (int)dtype);
    if (n < 1) return set_error(BSVD_E_SHAPE, "matrix must have size >= 1");
    if (lda < n) return set_error(BSVD_E_SHAPE, "lda %lld < n %lld", (long long)lda, (long long)n);
    return bsvd_validate_config(&c);
}

template <typename S, typename C>
bsvd_status stage1(S *work, const Plan &p, const bsvd_config &c, int algo, char *scratch,
                   cudaStream_t st, bsvd_timers *timers) {
    cudaError_t e = cudaSuccess;
    if (algo == BSVD_STAGE1_FAITHFUL) {
        C *tau = (C *)scratch;
        for (int64_t b = 0; b < p.batch; ++b) {
            BSVD_CUDA_TRY(cudaMemsetAsync(tau, 0, (size_t)p.ts * 2 * p.N * p.N * sizeof(C), st));
            e = banddiag_faithful<S, C>(work + b * p.np * p.np, p.np, p.ts, c.colperblock, tau, st, c.splitk);
            if (e != cudaSuccess) return cuda_error(e, "stage 1 (faithful)");
        }
        return BSVD_OK;
    }
    double pms = 0, tms = 0;
    if (sizeof(C) == 4 && flat_supported(p.ts, 4)) {
        e = banddiag_flat<S>(work, p.np, p.ts, p.batch, p.np * p.np, scratch, st, timers ? &pms : nullptr,
                             timers ? &tms : nullptr);
        if (timers) {
            timers->panel_s += pms * 1e-3;
            timers->trailing_s += tms * 1e-3;
        }
        if (e != cudaSuccess) return cuda_error(e, "stage 1 (flat)");
        return BSVD_OK;
    }
    cudaEvent_t evp[2], evt[2];
    if (timers) {
        for (int i = 0; i < 2; ++i) {
            cudaEventCreate(&evp[i]);
            cudaEventCreate(&evt[i]);
        }
    }
    e = banddiag_tree<S, C>(work, p.np, p.ts, p.batch, p.np * p.np, scratch, st,
                            timers ? evp : nullptr, timers ? evt : nullptr, &pms, &tms);
    if (timers) {
        timers->panel_s += pms * 1e-3;
        timers->trailing_s += tms * 1e-3;
        for (int i = 0; i < 2; ++i) {
            cudaEventDestroy(evp[i]);
            cudaEventDestroy(evt[i]);
        }
    }
    if (e != cudaSuccess) return cuda_error(e, "stage 1 (tree)");
    return BSVD_OK;
}

template <typename S, typename C>
bsvd_status pipeline(const S *a, const Plan &p, int64_t lda, int64_t stride,
                     const bsvd_config &c, const bsvd_options &opt, C *values, char *ws,
                     cudaStream_t st, bsvd_timers *timers) {
    int *flag = (int *)(ws + p.off_flag);
    S *work = (S *)(ws + p.off_work);
    double *d = (double *)(ws + p.off_d);
    double *e = (double *)(ws + p.off_e);
    char *scratch = ws + p.off_scratch;
    BSVD_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int), st));
    // fast path: power-of-two normalisation (util.cu); the faithful path keeps
    // the reference's scale-dependent arithmetic
    const bool norm = opt.stage1_algo != BSVD_STAGE1_FAITHFUL;
    unsigned long long *amax = norm ? (unsigned long long *)(ws + p.off_scale) : nullptr;
    double *unscale = norm ? (double *)(ws + p.off_scale) + p.batch : nullptr;
    cudaError_t err = copy_in_pad<S>(a, p.n, lda, stride, work, p.np, p.batch, flag, st, amax, unscale);
    if (err != cudaSuccess) return cuda_error(err, "copy-in");
    if (opt.check_finite) {
        int h = 0;
        BSVD_CUDA_TRY(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
        BSVD_CUDA_TRY(cudaStreamSynchronize(st));
        if (h) return set_error(BSVD_E_VALIDATION, "input contains NaN or Inf entries");
    }
    bsvd_status s = stage1<S, C>(work, p, c, opt.stage1_algo, scratch, st, timers);
    if (s != BSVD_OK) return s;
    cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr;
    if (timers) {
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventCreate(&e2);
        cudaEventRecord(e0, st);
    }
    err = band_to_bidiagonal<S>(work, p.np, p.np, p.ts, p.batch, p.np * p.np, d, e, scratch, st);
    if (err != cudaSuccess) return cuda_error(err, "stage 2 (bulge chase)");
    if (timers) cudaEventRecord(e1, st);
    err = bidiagonal_values<C>(d, e, p.np, p.batch, values, p.n, p.n, scratch, st);
    if (err != cudaSuccess) return cuda_error(err, "stage 3 (bisection)");
    if (norm && (err = unscale_values<C>(values, p.n, p.n, p.batch, unscale, st)) != cudaSuccess)
        return cuda_error(err, "unscale");
    if (timers) {
        cudaEventRecord(e2, st);
        cudaEventSynchronize(e2);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        timers->bidiagonal_s += ms * 1e-3;
        cudaEventElapsedTime(&ms, e1, e2);
        timers->diagonal_s += ms * 1e-3;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaEventDestroy(e2);
    }
    return BSVD_OK;
}

bsvd_status run(const void *a, bsvd_dtype dtype, int64_t n, int64_t lda, int64_t stride,
                int64_t batch, const bsvd_config *cfg, const bsvd_options *opt_in, void *values,
                void *workspace, size_t ws_bytes, void *stream, bsvd_timers *timers) {
    bsvd_config c = resolve_cfg(cfg, n);
    bsvd_status s = check_common(dtype, n, lda, c);
    if (s != BSVD_OK) return s;
    if (batch < 1) return set_error(BSVD_E_SHAPE, "batch must be >= 1");
    if (batch > 1 && stride < lda * n)
        return set_error(BSVD_E_SHAPE, "batch stride %lld < lda*n", (long long)stride);
    bsvd_options opt;
    bsvd_default_options(&opt);
    if (opt_in) opt = *opt_in;
    if (opt.stage1_algo != BSVD_STAGE1_TREE && opt.stage1_algo != BSVD_STAGE1_FAITHFUL)
        return set_error(BSVD_E_CONFIG, "unknown stage1_algo %d", opt.stage1_algo);
    if (!a || !values) return set_error(BSVD_E_SHAPE, "null matrix or values pointer");
    if (c.tilesize & (c.tilesize - 1)) opt.stage1_algo = BSVD_STAGE1_FAITHFUL;  // tree: 2^k edges
    Plan p = make_plan(dtype, n, batch, c, opt.stage1_algo);
    cudaStream_t st = (cudaStream_t)stream;
    char *ws = (char *)workspace;
    bool owned = false;
    if (!ws) {
        cudaError_t e = cudaMallocAsync((void **)&ws, p.total, st);
        if (e != cudaSuccess) return cuda_error(e, "workspace allocation");
        owned = true;
    } else if (ws_bytes < p.total) {
        return set_error(BSVD_E_OOM, "workspace of %zu bytes < required %zu", ws_bytes, p.total);
    }
    if (timers) memset(timers, 0, sizeof(*timers));
    switch (dtype) {
    case BSVD_FP64:
        s = pipeline<double, double>((const double *)a, p, lda, stride, c, opt, (double *)values, ws, st, timers);
        break;
    case BSVD_FP32:
        s = pipeline<float, float>((const float *)a, p, lda, stride, c, opt, (float *)values, ws, st, timers);
        break;
    default:
        s = pipeline<__half, float>((const __half *)a, p, lda, stride, c, opt, (float *)values, ws, st, timers);
        break;
    }
    if (owned) cudaFreeAsync(ws, st);
    return s;
}

}  // namespace

extern "C" {

const char *bsvd_last_error(void) { return g_err; }
uint64_t bsvd_launch_counter(void) { return g_launches.load(std::memory_order_relaxed); }
const char *bsvd_version(void) { return "bsvd-b200 0.1.0 (sm_100a)"; }

bsvd_status bsvd_validate_config(const bsvd_config *cfg) {
    if (!cfg) return set_error(BSVD_E_CONFIG, "null config");
    const int ts = cfg->tilesize;
    if (ts < 4 || ts > 128)
        return set_error(BSVD_E_CONFIG, "tilesize must be an integer in [4, 128], got %d", ts);
    const int cpb = cfg->colperblock <= 0 ? ts : cfg->colperblock;
    if (cpb < 1 || cpb > ts || ts % cpb)
        return set_error(BSVD_E_CONFIG, "colperblock must divide tilesize and lie in [1, %d], got %d", ts, cpb);
    const int kmax = std::min(ts, 1024 / ts);
    if (cfg->splitk < 1 || cfg->splitk > kmax)
        return set_error(BSVD_E_CONFIG,
                         "splitk must lie in [1, min(TILESIZE, 1024/TILESIZE)] = [1, %d], got %d",
                         kmax, cfg->splitk);
    // The fast path is specialised for power-of-two tile edges (every
    // KernelConfig.for_size value); other edges run the faithful path.
    return BSVD_OK;
}

int32_t bsvd_default_tilesize(int64_t n) {
    int32_t ts = 4;
    while (ts < 128 && (int64_t)ts * 8 < n) ts *= 2;
    return ts;
}

void bsvd_default_options(bsvd_options *opt) {
    memset(opt, 0, sizeof(*opt));
    opt->stage1_algo = BSVD_STAGE1_TREE;
    opt->check_finite = 1;
}

size_t bsvd_workspace_bytes(bsvd_dtype dtype, int64_t n, int64_t batch, const bsvd_config *cfg) {
    if (!dtype_ok(dtype) || n < 1 || batch < 1) return 0;
    bsvd_config c = resolve_cfg(cfg, n);
    const Plan a = make_plan(dtype, n, batch, c, BSVD_STAGE1_TREE);
    const Plan b = make_plan(dtype, n, batch, c, BSVD_STAGE1_FAITHFUL);
    return std::max(a.total, b.total);
}

bsvd_status bsvd_svdvals(const void *a, bsvd_dtype dtype, int64_t n, int64_t lda,
                         const bsvd_config *cfg, void *values, void *workspace, size_t ws_bytes,
                         void *stream, bsvd_timers *timers) {
    return run(a, dtype, n, lda, lda * n, 1, cfg, nullptr, values, workspace, ws_bytes, stream, timers);
}

bsvd_status bsvd_svdvals_ex(const void *a, bsvd_dtype dtype, int64_t n, int64_t lda,
                            const bsvd_config *cfg, const bsvd_options *opt, void *values,
                            void *workspace, size_t ws_bytes, void *stream, bsvd_timers *timers) {
    return run(a, dtype, n, lda, lda * n, 1, cfg, opt, values, workspace, ws_bytes, stream, timers);
}

bsvd_status bsvd_svdvals_batched(const void *a, bsvd_dtype dtype, int64_t n, int64_t lda,
                                 int64_t stride, int64_t batch, const bsvd_config *cfg,
                                 void *values, void *workspace, size_t ws_bytes, void *stream,
                                 bsvd_timers *timers) {
    return run(a, dtype, n, lda, stride, batch, cfg, nullptr, values, workspace, ws_bytes, stream, timers);
}

bsvd_status bsvd_banddiag(void *a, bsvd_dtype dtype, int64_t n, const bsvd_config *cfg,
                          const bsvd_options *opt_in, void *workspace, size_t ws_bytes,
                          void *stream) {
    bsvd_config c = resolve_cfg(cfg, n);
    bsvd_status s = check_common(dtype, n, n, c);
    if (s != BSVD_OK) return s;
    if (n % c.tilesize)
        return set_error(BSVD_E_SHAPE, "matrix is %lldx%lld, not a multiple of tilesize %d",
                         (long long)n, (long long)n, c.tilesize);
    bsvd_options opt;
    bsvd_default_options(&opt);
    if (opt_in) opt = *opt_in;
    if (c.tilesize & (c.tilesize - 1)) opt.stage1_algo = BSVD_STAGE1_FAITHFUL;
    Plan p = make_plan(dtype, n, 1, c, opt.stage1_algo);
    if (ws_bytes < p.stage1_bytes)
        return set_error(BSVD_E_OOM, "workspace of %zu bytes < required %zu", ws_bytes, p.stage1_bytes);
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e;
    switch (dtype) {
    case BSVD_FP64:
        s = stage1<double, double>((double *)a, p, c, opt.stage1_algo, (char *)workspace, st, nullptr);
        e = clear_outside_band<double>((double *)a, n, c.tilesize, 1, st);
        break;
    case BSVD_FP32:
        s = stage1<float, float>((float *)a, p, c, opt.stage1_algo, (char *)workspace, st, nullptr);
        e = clear_outside_band<float>((float *)a, n, c.tilesize, 1, st);
        break;
    default:
        s = stage1<__half, float>((__half *)a, p, c, opt.stage1_algo, (char *)workspace, st, nullptr);
        e = clear_outside_band<__half>((__half *)a, n, c.tilesize, 1, st);
        break;
    }
    if (s != BSVD_OK) return s;
    if (e != cudaSuccess) return cuda_error(e, "clear_outside_band");
    return BSVD_OK;
}

size_t bsvd_band_workspace_bytes(int64_t n, int32_t bw) {
    if (n < 1 || bw < 1 || bw > 128) return 0;
    return chase_workspace_bytes(n, bw, 1);
}

bsvd_status bsvd_band_to_bidiagonal(const void *band, bsvd_dtype dtype, int64_t n, int32_t bw,
                                    double *d, double *e, void *workspace, size_t ws_bytes,
                                    void *stream) {
    if (!dtype_ok(dtype)) return set_error(BSVD_E_CONFIG, "unsupported dtype code %d", (int)dtype);
    if (n < 1) return set_error(BSVD_E_SHAPE, "matrix must have size >= 1");
    if (bw < 1 || bw > 128) return set_error(BSVD_E_CONFIG, "band width must lie in [1, 128], got %d", bw);
    const size_t need = chase_workspace_bytes(n, bw, 1);
    if (ws_bytes < need) return set_error(BSVD_E_OOM, "workspace of %zu bytes < required %zu", ws_bytes, need);
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t err;
    switch (dtype) {
    case BSVD_FP64: err = band_to_bidiagonal<double>((const double *)band, n, n, bw, 1, 0, d, e, workspace, st); break;
    case BSVD_FP32: err = band_to_bidiagonal<float>((const float *)band, n, n, bw, 1, 0, d, e, workspace, st); break;
    default: err = band_to_bidiagonal<__half>((const __half *)band, n, n, bw, 1, 0, d, e, workspace, st); break;
    }
    if (err != cudaSuccess) return cuda_error(err, "band_to_bidiagonal");
    return BSVD_OK;
}

bsvd_status bsvd_bidiagonal_values(const double *d, const double *e, int64_t n, double *values,
                                   void *stream) {
    if (n < 1) return set_error(BSVD_E_SHAPE, "bidiagonal matrix must have size >= 1");
    cudaStream_t st = (cudaStream_t)stream;
    void *ws = nullptr;
    BSVD_CUDA_TRY(cudaMallocAsync(&ws, bisect_workspace_bytes(n, 1), st));
    cudaError_t err = bidiagonal_values<double>(d, e, n, 1, values, n, n, ws, st);
    cudaFreeAsync(ws, st);
    if (err != cudaSuccess) return cuda_error(err, "bidiagonal_values");
    return BSVD_OK;
}

// ---- reference tile kernels ------------------------------------------------

#define DISPATCH3(dtype, CALL64, CALL32, CALL16) \
    switch (dtype) {                             \
    case BSVD_FP64: err = CALL64; break;         \
    case BSVD_FP32: err = CALL32; break;         \
    case BSVD_FP16: err = CALL16; break;         \
    default: return set_error(BSVD_E_CONFIG, "unsupported dtype code %d", (int)dtype); \
    }

bsvd_status bsvd_geqrt(void *tile, int64_t rs, int64_t cs, bsvd_dtype dtype, int32_t ts, void *tau,
                       void *stream) {
    if (ts < 4 || ts > 128) return set_error(BSVD_E_CONFIG, "tilesize must be an integer in [4, 128], got %d", ts);
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t err;
    DISPATCH3(dtype,
              (launch_geqrt_faithful<double, double>((double *)tile, rs, cs, ts, (double *)tau, 1, 0, 0, st)),
              (launch_geqrt_faithful<float, float>((float *)tile, rs, cs, ts, (float *)tau, 1, 0, 0, st)),
              (launch_geqrt_faithful<__half, float>((__half *)tile, rs, cs, ts, (float *)tau, 1, 0, 0, st)));
    if (err != cudaSuccess) return cuda_error(err, "geqrt");
    return BSVD_OK;
}

bsvd_status bsvd_tsqrt_chain(void *r, int64_t rs, int64_t cs, void *const *b_tiles,
                             void *const *taus, int32_t nb, bsvd_dtype dtype, int32_t ts,
                             void *stream) {
    if (ts < 4 || ts > 128) return set_error(BSVD_E_CONFIG, "tilesize must be an integer in [4, 128], got %d", ts);
    cudaStream_t st = (cudaStream_t)stream;
    TileArr bs{b_tiles}, ta{taus};
    cudaError_t err;
    DISPATCH3(dtype,
              (launch_tsqrt_faithful<double, double>((double *)r, rs, cs, bs, ta, nb, ts, st)),
              (launch_tsqrt_faithful<float, float>((float *)r, rs, cs, bs, ta, nb, ts, st)),
              (launch_tsqrt_faithful<__half, float>((__half *)r, rs, cs, bs, ta, nb, ts, st)));
    if (err != cudaSuccess) return cuda_error(err, "tsqrt_chain");
    return BSVD_OK;
}

static bsvd_status check_splitk(int32_t ts, int32_t nsplit) {
    const int kmax = std::min((int)ts, 1024 / (int)ts);
    if (nsplit < 1 || nsplit > kmax)
        return set_error(BSVD_E_CONFIG,
                         "splitk must lie in [1, min(TILESIZE, 1024/TILESIZE)] = [1, %d], got %d", kmax, nsplit);
    return BSVD_OK;
}

bsvd_status bsvd_geqrt_splitk(void *tile, int64_t rs, int64_t cs, bsvd_dtype dtype, int32_t ts, int32_t splitk,
                              void *tau, void *stream) {
    if (ts < 4 || ts > 128) return set_error(BSVD_E_CONFIG, "tilesize must be an integer in [4, 128], got %d", ts);
    if (bsvd_status s = check_splitk(ts, splitk)) return s;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t err;
    DISPATCH3(dtype,
              (launch_geqrt_faithful<double, double>((double *)tile, rs, cs, ts, (double *)tau, 1, 0, 0, st, splitk)),
              (launch_geqrt_faithful<float, float>((float *)tile, rs, cs, ts, (float *)tau, 1, 0, 0, st, splitk)),
              (launch_geqrt_faithful<__half, float>((__half *)tile, rs, cs, ts, (float *)tau, 1, 0, 0, st, splitk)));
    if (err != cudaSuccess) return cuda_error(err, "geqrt_splitk");
    return BSVD_OK;
}

bsvd_status bsvd_tsqrt_chain_splitk(void *r, int64_t rs, int64_t cs, void *const *b_tiles, void *const *taus,
                                    int32_t nb, bsvd_dtype dtype, int32_t ts, int32_t splitk, void *stream) {
    if (ts < 4 || ts > 128) return set_error(BSVD_E_CONFIG, "tilesize must be an integer in [4, 128], got %d", ts);
    if (bsvd_status s = check_splitk(ts, splitk)) return s;
    cudaStream_t st = (cudaStream_t)stream;
    TileArr bs{b_tiles}, ta{taus};
    cudaError_t err;
    DISPATCH3(dtype,
              (launch_tsqrt_faithful<double, double>((double *)r, rs, cs, bs, ta, nb, ts, st, splitk)),
              (launch_tsqrt_faithful<float, float>((float *)r, rs, cs, bs, ta, nb, ts, st, splitk)),
              (launch_tsqrt_faithful<__half, float>((__half *)r, rs, cs, bs, ta, nb, ts, st, splitk)));
    if (err != cudaSuccess) return cuda_error(err, "tsqrt_chain_splitk");
    return BSVD_OK;
}

bsvd_status bsvd_unmqr(const void *panel, int64_t rs, int64_t cs, const void *tau, void *x,
                       int64_t xrs, int64_t xcs, int64_t ncols, bsvd_dtype dtype, int32_t ts,
                       int32_t colperblock, void *stream) {
    const int cpb = colperblock <= 0 ? ts : colperblock;
    if (ts < 4 || ts > 128 || ts % cpb) return set_error(BSVD_E_CONFIG, "bad tilesize/colperblock %d/%d", ts, cpb);
    if (ncols <= 0 || ncols % cpb)
        return set_error(BSVD_E_SHAPE, "unmqr column count %lld is not a positive multiple of %d", (long long)ncols, cpb);
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t err;
    DISPATCH3(dtype,
              (launch_unmqr_faithful<double, double>((const double *)panel, rs, cs, (const double *)tau, (double *)x, xrs, xcs, ncols, ts, cpb, st)),
              (launch_unmqr_faithful<float, float>((const float *)panel, rs, cs, (const float *)tau, (float *)x, xrs, xcs, ncols, ts, cpb, st)),
              (launch_unmqr_faithful<__half, float>((const __half *)panel, rs, cs, (const float *)tau, (__half *)x, xrs, xcs, ncols, ts, cpb, st)));
    if (err != cudaSuccess) return cuda_error(err, "unmqr");
    return BSVD_OK;
}

bsvd_status bsvd_tsmqr_fused(void *y, int64_t rs, int64_t cs, void *const *x_rows,
                             void *const *v_tiles, void *const *taus, int32_t nb, int64_t ncols,
                             bsvd_dtype dtype, int32_t ts, int32_t colperblock, void *stream) {
    const int cpb = colperblock <= 0 ? ts : colperblock;
    if (ts < 4 || ts > 128 || ts % cpb) return set_error(BSVD_E_CONFIG, "bad tilesize/colperblock %d/%d", ts, cpb);
    if (ncols <= 0 || ncols % cpb)
        return set_error(BSVD_E_SHAPE, "tsmqr column count %lld is not a positive multiple of %d", (long long)ncols, cpb);
    cudaStream_t st = (cudaStream_t)stream;
    TileArr xs{x_rows}, vs{v_tiles}, ta{taus};
    cudaError_t err;
    DISPATCH3(dtype,
              (launch_tsmqr_faithful<double, double>((double *)y, rs, cs, xs, vs, ta, nb, ncols, ts, cpb, st)),
              (launch_tsmqr_faithful<float, float>((float *)y, rs, cs, xs, vs, ta, nb, ncols, ts, cpb, st)),
              (launch_tsmqr_faithful<__half, float>((__half *)y, rs, cs, xs, vs, ta, nb, ncols, ts, cpb, st)));
    if (err != cudaSuccess) return cuda_error(err, "tsmqr_fused");
    return BSVD_OK;
}

}  // extern "C"
