/*
 * bsvd.h -- C ABI of the B200-native singular-value engine (libbsvd.so).
 *
 * Drop-in boundary for the reference `bandsvd` hot path (arXiv 2508.06339
 * reference package).  Every entry point below names the reference
 * interface it replaces (file:line under the reference's pkg/src/bandsvd/).
 * All matrix / vector pointers are DEVICE pointers unless stated otherwise;
 * every call is stream-ordered and asynchronous on `stream` (a cudaStream_t
 * passed as void*, NULL = legacy default stream) unless stated otherwise.
 * The caller owns all memory; the library never frees caller pointers.
 * Inputs are never modified.  No torch types cross this boundary.
 *
 * Errors: every call returns a bsvd_status; bsvd_last_error() returns a
 * thread-local message naming the offending field, mirroring the Python
 * exception text (errors.py:4-41).
 */
#ifndef BSVD_H_
#define BSVD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* errors.py:4-41 -> status codes (the Python shim maps them back to the
 * reference's exception classes). */
typedef enum {
    BSVD_OK = 0,
    BSVD_E_SHAPE = 2,        /* ShapeError: non-square, n < 1, tile multiples   */
    BSVD_E_CONFIG = 3,       /* ConfigError: KernelConfig validation            */
    BSVD_E_VALIDATION = 4,   /* ValidationError: NaN / Inf input                */
    BSVD_E_CONVERGENCE = 5,  /* ConvergenceError (kept for ABI parity; bisection */
                             /* always terminates)                              */
    BSVD_E_CUDA = 6,         /* CUDA runtime / launch failure                   */
    BSVD_E_OOM = 7,          /* workspace too small / allocation failure        */
    BSVD_E_NOTIMPL = 8       /* unsupported combination                         */
} bsvd_status;

/* precision.py:35-37 (FP64 / FP32 / FP16-storage), codes = BSVD file dtype
 * codes (matrix.py:18). FP16 is storage-only: fp32 compute, RNE on store. */
typedef enum { BSVD_FP64 = 1, BSVD_FP32 = 2, BSVD_FP16 = 3 } bsvd_dtype;

/* kernels.py:32-55 KernelConfig(tilesize, colperblock, splitk, fused).
 * colperblock <= 0 means "None" (defaults to tilesize).  Validated exactly
 * like KernelConfig.__post_init__. tilesize is also the band width. */
typedef struct {
    int32_t tilesize;
    int32_t colperblock;
    int32_t splitk;
    int32_t fused;
} bsvd_config;

/* Stage-1 algorithm.  TREE (default): tiled QR/LQ with a binary reduction
 * tree per panel and WY trailing updates (same tile operators, shorter
 * critical path).  FAITHFUL: the reference's flat TSQRT chain with its exact
 * per-item arithmetic (bit-identical band to bandreduce.py:91-110). */
typedef enum { BSVD_STAGE1_TREE = 0, BSVD_STAGE1_FAITHFUL = 1 } bsvd_stage1_algo;

typedef struct {
    int32_t stage1_algo;     /* bsvd_stage1_algo                                */
    int32_t check_finite;    /* 1: reject NaN/Inf before any compute (default)  */
    int32_t reserved[6];
} bsvd_options;

/* bench.py:25 PHASE_KEYS; filled with device-event times (seconds) when a
 * non-NULL pointer is passed (adds per-phase event records + one sync). */
typedef struct {
    double panel_s, trailing_s, bidiagonal_s, diagonal_s;
} bsvd_timers;

/* ---- configuration ----------------------------------------------------- */

/* kernels.py:42-55 KernelConfig.__post_init__ */
bsvd_status bsvd_validate_config(const bsvd_config *cfg);
/* kernels.py:57-64 KernelConfig.for_size: ts=4, doubled while ts<128 && 8ts<n */
int32_t bsvd_default_tilesize(int64_t n);
void bsvd_default_options(bsvd_options *opt);
const char *bsvd_last_error(void);
const char *bsvd_version(void);
/* Number of CUDA kernels this library has launched in this process (all
 * streams, all calls) -- the benchmark's launch-count evidence. */
uint64_t bsvd_launch_counter(void);

/* ---- whole path: secondstage.py:510-542 svdvals ------------------------ */

/* Device workspace needed by bsvd_svdvals / _batched for this shape. */
size_t bsvd_workspace_bytes(bsvd_dtype dtype, int64_t n, int64_t batch, const bsvd_config *cfg);

/* All n singular values of the column-major n x n matrix `a` (leading
 * dimension lda >= n, storage precision `dtype`), descending, written to
 * `values` in the COMPUTE precision (double for FP64, float for FP32 and
 * FP16).  A row-major tensor may be passed as its transpose (sigma(A) =
 * sigma(A^T)).  cfg == NULL -> KernelConfig.for_size(n).  Synchronous with
 * respect to the host only for the finite check (one 4-byte D2H read). */
bsvd_status bsvd_svdvals(const void *a, bsvd_dtype dtype, int64_t n, int64_t lda,
                         const bsvd_config *cfg, void *values,
                         void *workspace, size_t ws_bytes, void *stream,
                         bsvd_timers *timers);

bsvd_status bsvd_svdvals_ex(const void *a, bsvd_dtype dtype, int64_t n, int64_t lda,
                            const bsvd_config *cfg, const bsvd_options *opt, void *values,
                            void *workspace, size_t ws_bytes, void *stream,
                            bsvd_timers *timers);

/* `batch` independent matrices a + i*stride (elements), values + i*n.
 * The reference farms matrices over processes (bench.py:161-189); here
 * every launch covers the whole batch. */
bsvd_status bsvd_svdvals_batched(const void *a, bsvd_dtype dtype, int64_t n, int64_t lda,
                                 int64_t stride, int64_t batch, const bsvd_config *cfg,
                                 void *values, void *workspace, size_t ws_bytes,
                                 void *stream, bsvd_timers *timers);

/* ---- stage entry points (secondstage.py / bandreduce.py) --------------- */

/* bandreduce.py:91-120 banddiag: in place on the PADDED column-major
 * n x n matrix (n a multiple of tilesize, lda = n), upper band of width
 * tilesize left in `a`, entries outside the band zeroed. */
bsvd_status bsvd_banddiag(void *a, bsvd_dtype dtype, int64_t n, const bsvd_config *cfg,
                          const bsvd_options *opt, void *workspace, size_t ws_bytes,
                          void *stream);

/* secondstage.py:452-470 band_to_bidiagonal: upper band (column-major n x n,
 * band width bw, storage precision) -> float64 d[n], e[n-1]. */
/* Device workspace bsvd_band_to_bidiagonal needs for an order-n band of width bw. */
size_t bsvd_band_workspace_bytes(int64_t n, int32_t bw);

bsvd_status bsvd_band_to_bidiagonal(const void *band, bsvd_dtype dtype, int64_t n, int32_t bw,
                                    double *d, double *e, void *workspace, size_t ws_bytes,
                                    void *stream);

/* secondstage.py:473-507 bidiagonal_values: float64 d[n], e[n-1] -> values
 * (descending, float64) by Sturm-count bisection on the Golub-Kahan
 * tridiagonal. */
bsvd_status bsvd_bidiagonal_values(const double *d, const double *e, int64_t n, double *values,
                                   void *stream);

/* ---- reference tile kernels, bit-faithful (kernels.py:442-559) ----------
 * Views are (pointer, row stride, column stride) in elements, so the lazy
 * transpose of matrix.py:93-154 is a stride swap.  tau vectors are in the
 * compute precision.  These reproduce the reference's per-work-item
 * arithmetic exactly (serial sums, no FMA contraction). */

/* kernels.py:442-456 geqrt (splitk == 1 path) */
bsvd_status bsvd_geqrt(void *tile, int64_t rs, int64_t cs, bsvd_dtype dtype, int32_t ts,
                       void *tau, void *stream);
/* kernels.py:484-500 tsqrt_chain: R tile + nb B tiles at b_tiles[l] (device
 * array of nb device pointers), taus[l] likewise. */
bsvd_status bsvd_tsqrt_chain(void *r, int64_t rs, int64_t cs, void *const *b_tiles,
                             void *const *taus, int32_t nb, bsvd_dtype dtype, int32_t ts,
                             void *stream);
/* kernels.py:459-470 geqrt_splitk (geqrt_splitk_kernel :233-283): the tile
 * QR with each column's norm and dot products split over `splitk` row
 * segments and combined by _pairwise_sum (:191-199); splitk in
 * [1, min(ts, 1024/ts)], bitwise equal to bsvd_geqrt at splitk == 1. */
bsvd_status bsvd_geqrt_splitk(void *tile, int64_t rs, int64_t cs, bsvd_dtype dtype, int32_t ts, int32_t splitk,
                              void *tau, void *stream);
/* kernels.py:479-481 tsqrt_splitk / :503-515 _tsqrt_chain_splitk
 * (tsqrt_splitk_kernel :316-361), same segment / pairwise sums. */
bsvd_status bsvd_tsqrt_chain_splitk(void *r, int64_t rs, int64_t cs, void *const *b_tiles, void *const *taus,
                                    int32_t nb, bsvd_dtype dtype, int32_t ts, int32_t splitk, void *stream);
/* kernels.py:518-532 unmqr */
bsvd_status bsvd_unmqr(const void *panel, int64_t rs, int64_t cs, const void *tau, void *x,
                       int64_t xrs, int64_t xcs, int64_t ncols, bsvd_dtype dtype, int32_t ts,
                       int32_t colperblock, void *stream);
/* kernels.py:535-559 tsmqr_fused */
bsvd_status bsvd_tsmqr_fused(void *y, int64_t rs, int64_t cs, void *const *x_rows,
                             void *const *v_tiles, void *const *taus, int32_t nb, int64_t ncols,
                             bsvd_dtype dtype, int32_t ts, int32_t colperblock, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* BSVD_H_ */
