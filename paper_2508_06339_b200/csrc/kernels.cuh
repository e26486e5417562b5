// kernels.cuh -- launcher declarations shared by the .cu translation units.
#pragma once
#include "common.cuh"

namespace bsvd {

// Sequences of tiles: regular stride (driver) or explicit pointer arrays (ABI).
struct TileSeq {
    char *base;
    int64_t step;  // bytes
    __host__ __device__ void *get(int l) const { return base + (int64_t)l * step; }
};
struct TileArr {
    void *const *ptrs;
    __host__ __device__ void *get(int l) const { return ptrs[l]; }
};

// ---- faithful.cu (bit-exact reference kernels) ---------------------------
template <typename S, typename C>
cudaError_t launch_geqrt_faithful(S *a, int64_t rs, int64_t cs, int ts, C *tau, int64_t batch,
                                  int64_t a_bstride, int64_t tau_bstride, cudaStream_t st, int nsplit = 1);
template <typename S, typename C, typename TS_, typename TA_>
cudaError_t launch_tsqrt_faithful(S *r, int64_t rs, int64_t cs, TS_ bs, TA_ taus, int nb, int ts,
                                  cudaStream_t st, int nsplit = 1);
template <typename S, typename C>
cudaError_t launch_unmqr_faithful(const S *panel, int64_t prs, int64_t pcs, const C *tau, S *x,
                                  int64_t xrs, int64_t xcs, int64_t ncols, int ts, int cpb,
                                  cudaStream_t st);
template <typename S, typename C, typename TS_, typename TA_>
cudaError_t launch_tsmqr_faithful(S *y, int64_t rs, int64_t cs, TS_ xs, TS_ vs, TA_ taus, int nb,
                                  int64_t ncols, int ts, int cpb, cudaStream_t st);
template <typename S, typename C>
cudaError_t banddiag_faithful(S *a, int64_t n, int ts, int cpb, C *tau, cudaStream_t st, int splitk = 1);

// ---- stage1_tree.cu (fast stage 1) ---------------------------------------
// Workspace bytes for one matrix of padded order n with tile ts.
template <typename S, typename C>
size_t tree_workspace_bytes(int64_t n, int ts);
// Stage 1 in place on the padded matrix a (n = N*ts, column-major), batch
// matrices at a + b*a_bstride; ws from tree_workspace_bytes * batch.
template <typename S, typename C>
cudaError_t banddiag_tree(S *a, int64_t n, int ts, int64_t batch, int64_t a_bstride, void *ws,
                          cudaStream_t st, cudaEvent_t *ev_panel, cudaEvent_t *ev_trail,
                          double *panel_ms, double *trail_ms);

// ---- stage1_flat.cu (flat cluster panel + one compact-WY update per side) --
// fp32 compute (FP32 / FP16 storage), ts in {64, 128}.
bool flat_supported(int ts, int elem_bytes);
size_t flat_workspace_bytes(int64_t n, int ts, int64_t batch);
template <typename S>
cudaError_t banddiag_flat(S *a, int64_t n, int ts, int64_t batch, int64_t a_bstride, void *ws,
                          cudaStream_t st, double *panel_ms, double *trail_ms);

// ---- stage1_flat_tc.cu (tcgen05 3xTF32 trailing-update products, TMA-fed;
// ts = 128, FP32 / FP16 storage)
bool flat_tc_supported(int ts, int elem_bytes);
struct FlatTcPlan;
FlatTcPlan *flat_tc_plan(void *a, int elem_bytes, int64_t n, int64_t batch, int64_t a_bstride, const float *vcm0,
                         const float *vcm1, const float *vrm0, const float *vrm1, const float *w2t,
                         int64_t ws_bstride);
void flat_tc_plan_free(FlatTcPlan *p);
cudaError_t launch_flat_tc(const FlatTcPlan *plan, int par, int mode, bool lq, int M, int C, int row_base,
                           int col_base, float *Wp, float *Gp, int64_t ws_bstride, int ns, int rps, void *a,
                           int64_t n, int64_t a_bstride, int64_t batch, cudaStream_t st);

// ---- stage1_apply.cu (per-level WY trailing updates, ts >= 16) ----------
template <typename S, typename C, int TS>
cudaError_t launch_apply_levels(S *a, int64_t n, int64_t batch, int64_t a_bstride, bool lq,
                                int64_t top, int64_t k, int64_t m, const C *nodes,
                                int64_t ws_bstride, cudaStream_t st);
// ext != nullptr: two-tile leaves (m counts them; mtiles = the panel's tile
// rows), leaf-level update from the leaf2 region, TT tile rows strided by 2.
template <typename S, typename C, int TS>
cudaError_t launch_apply_level(S *a, int64_t n, int64_t batch, int64_t a_bstride, bool lq,
                               int64_t top, int64_t k, int64_t m, const C *nodes,
                               int64_t ws_bstride, int j, cudaStream_t st, const C *ext = nullptr,
                               int64_t mtiles = 0);
// Tensor-core (tcgen05 3xTF32) variant for fp32 compute at ts = 128.
template <typename S>
cudaError_t launch_apply_level_tc(S *a, int64_t n, int64_t batch, int64_t a_bstride, bool lq, int64_t top,
                                  int64_t k, int64_t m, const float *img, int64_t img_bstride, int j,
                                  cudaStream_t st);

// ---- stage2_chase.cu -------------------------------------------------------
size_t chase_workspace_bytes(int64_t n, int bw, int64_t batch);
// Upper band (column-major padded n x n in S, band width bw) -> d, e (fp64).
template <typename S>
cudaError_t band_to_bidiagonal(const S *a, int64_t n, int64_t lda, int bw, int64_t batch,
                               int64_t a_bstride, double *d, double *e, void *ws,
                               cudaStream_t st);

// ---- stage3_bisect.cu ------------------------------------------------------
// Singular values of (d, e) by Sturm bisection on the Golub-Kahan tridiagonal.
// out: first n_out values, descending, cast to OutT; batch matrices with
// d/e strides n / (n-1) and out stride out_stride.
template <typename OutT>
cudaError_t bidiagonal_values(const double *d, const double *e, int64_t n, int64_t batch,
                              OutT *out, int64_t n_out, int64_t out_stride, void *ws,
                              cudaStream_t st);
size_t bisect_workspace_bytes(int64_t n, int64_t batch);

// ---- util.cu ---------------------------------------------------------------
template <typename C>
cudaError_t unscale_values(C *v, int64_t n, int64_t stride, int64_t batch, const double *unscale, cudaStream_t st);
template <typename S>
cudaError_t copy_in_pad(const S *src, int64_t n, int64_t lda, int64_t src_bstride, S *dst,
                        int64_t np, int64_t batch, int *nonfinite_flag, cudaStream_t st,
                        unsigned long long *amax = nullptr, double *unscale = nullptr);
template <typename S>
cudaError_t clear_outside_band(S *a, int64_t n, int bw, int64_t batch, cudaStream_t st);

}  // namespace bsvd
