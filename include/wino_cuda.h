/*
 * wino_cuda.h — C-ABI of the B200-native Winograd layer (arXiv 1702.08597).
 *
 * Drop-in boundary for the reference's layer API.  Each entry
 * point names the reference interface it replaces (paths relative to
 * /root/reference/proj).  No C++ types, no exceptions, no CUDA headers: device
 * buffers are plain pointers, streams are `void*` (a cudaStream_t), and every
 * call returns a wino_status whose values map 1:1 onto the reference's
 * exception classes; wino_last_error() holds the message (thread-local).
 *
 * Device layouts (row-major, fp32):
 *   input  I  : N × C × H × W         (unpadded; `pad` is folded into φ)
 *   output O  : N × K × Ho × Wo       Ho = H + 2·pad − r + 1
 *   grad_in dI: N × C × H × W
 *   grad_w    : sparse plan — nnz-compact values in CSR order, slice-major
 *               ((i,j) row-major, then rows k, then the row's columns), i.e. the
 *               order of PointwiseCsr<float>::values (sparse.hpp:19-38);
 *               dense plan — K × C × p × q (the W_F layout, layer.hpp:36).
 */
#ifndef WINO_CUDA_H
#define WINO_CUDA_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define WINO_API __attribute__((visibility("default")))
#else
#define WINO_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum wino_status {
    WINO_OK = 0,
    WINO_SHAPE_ERROR = 1,        /* wino::ShapeError         tensor.hpp:12-15     */
    WINO_CONSISTENCY_ERROR = 2,  /* wino::ConsistencyError   layer.hpp:11-14      */
    WINO_CORRUPT_FORMAT = 3,     /* wino::CorruptFormatError sparse.hpp:12-15     */
    WINO_CAPABILITY_ERROR = 4,   /* wino::CapabilityError    transforms.hpp:10-13 */
    WINO_CUDA_ERROR = 5,         /* device / runtime failure (no reference analogue) */
    WINO_INVALID_ARGUMENT = 6    /* null pointer, bad enum (std::invalid_argument, bindings.cpp:140) */
} wino_status;

/* Mirrors wino::TileGeometry (transforms.hpp:39-53), square tiles only. */
typedef struct wino_geometry {
    int64_t c, h_i, w_i, h_o, w_o, h_op, w_op, h_ip, w_ip;
    int64_t m, r, p, tiles_y, tiles_x, t;
} wino_geometry;

/* make_geometry (transforms.cpp:147-172). WINO_SHAPE_ERROR if the image is smaller
 * than the kernel. */
WINO_API int wino_make_geometry(int64_t c, int64_t h_i, int64_t w_i, int m, int r, wino_geometry* out);
/* phi (transforms.cpp:179-187) / psi (transforms.cpp:189-194); WINO_SHAPE_ERROR when out of range. */
WINO_API int wino_phi(const wino_geometry* g, int64_t t, int64_t i, int64_t j, int64_t* y, int64_t* x);
WINO_API int wino_psi(const wino_geometry* g, int64_t y, int64_t x, int64_t* t, int64_t* i, int64_t* j);

/* Transform constants exactly as the reference builds them, row-major doubles:
 * a p×m (TransformSet::a1), b p×p (b1), g p×r (g1).  m=2,r=3 gives the fixed
 * f2x2_3x3_transforms (transforms.cpp:7-19, chosen by bindings.cpp:41-44), every
 * other (m,r) the Cook–Toom construction (transforms.cpp:71-145);
 * WINO_CAPABILITY_ERROR when m+r−1 > 8. */
WINO_API int wino_transforms(int m, int r, double* a, double* b, double* g);

/* ---------------------------------------------------------------------------- */
/* Layer plan (one Winograd layer; replaces the TransformSet/TileGeometry/weights */
/* triple passed to winograd_forward, layer.hpp:28-43, and sparse_forward,      */
/* sparse.hpp:78-82)                                                             */
/* ---------------------------------------------------------------------------- */

typedef struct wino_layer_desc {
    int c, k;          /* input / output channels                            */
    int h, w;          /* unpadded input extents                             */
    int pad;           /* zero padding folded into φ: geometry = make_geometry(c, h+2pad, w+2pad) */
    int m, r;          /* F(m×m, r×r); kernels are built for r=3, m ∈ {2,4,6} */
    const double* a;   /* p×m TransformSet::a1 entries, or NULL for wino_transforms(m,r) */
    const double* b;   /* p×p TransformSet::b1 entries, or NULL                          */
    int device;        /* CUDA device ordinal                                            */
} wino_layer_desc;

typedef struct wino_plan wino_plan;
typedef struct wino_cache wino_cache;

WINO_API int wino_plan_create(const wino_layer_desc* desc, wino_plan** out);
WINO_API int wino_plan_destroy(wino_plan* plan);
/* geometry of the (padded) layer; nnz_total (−1 before weights are set); is_dense */
WINO_API int wino_plan_info(const wino_plan* plan, wino_geometry* geom, int64_t* nnz_total, int* is_dense);

/* Weights, sparse form: a PointwiseCsr<float> (sparse.hpp:19-38) given as p·q host
 * slices in (i,j) row-major order: row_ptr[s] has K+1 entries, col_idx[s]/values[s]
 * have nnz[s].  Fully validated (the reference's spmdm only bounds-checks columns,
 * sparse.cpp:58, and reads row_ptr[K] unchecked): row_ptr[0]==0, monotone,
 * row_ptr[K]==nnz[s], col_idx < C and strictly increasing within a row — any
 * violation is WINO_CORRUPT_FORMAT.  Builds the device CSR and the CSC (W_Fᵀ)
 * used by the backward pass.  Synchronous. */
WINO_API int wino_set_weights_csr(wino_plan* plan, const uint64_t* const* row_ptr,
                         const uint64_t* const* col_idx, const float* const* values,
                         const uint64_t* nnz);
/* Weights from a dense host W_F (K×C×p×q f64, layer.hpp:36).
 *   dense = 0: compress<float> (sparse.cpp:9-36, keep |v| > zero_tol, or v != 0 when
 *              zero_tol == 0) then as above; dW is nnz-compact.
 *   dense = 1: every coordinate is a weight (zeros included, the dense layer's semantics);
 *              exact reference-order kernels; dW is K×C×p×q.
 *   dense = 2: as 1, but Z, dĨ_F and dW_F run as 3xTF32 tcgen05 GEMMs on the tensor cores with
 *              every 32-wide k-block accumulated in a fresh TMEM accumulator and folded into
 *              fp64 by the epilogue (error ~2e-7 of Σ|w·x|, the fp32 rounding level).
 *   dense = 3: as 2 but one TMEM accumulation chain per tile (faster; ~1e-6 of Σ|w·x| on O/dI,
 *              ~2e-5 normwise on dW_F from the fp32 chain over n·T).
 *   Layers whose C or K is not a multiple of 4 (TMA strides) use the dense=1 kernels. */
WINO_API int wino_set_weights(wino_plan* plan, const double* w_f, double zero_tol, int dense);
/* Structure of the device CSR (for parity checks): per-slice nnz[p·q]; if the other
 * pointers are non-null they receive row_ptr (p·q·(K+1), slice-local offsets),
 * col_idx and values (nnz_total, CSR order). */
WINO_API int wino_get_csr(const wino_plan* plan, uint64_t* nnz, uint64_t* row_ptr, uint64_t* col_idx,
                 float* values);
/* Device pointer to the live CSR values (nnz_total floats, CSR order) for in-place
 * optimizer updates; wino_values_updated() refreshes the CSC copy from it. */
WINO_API int wino_weight_values(wino_plan* plan, float** values_dev);
WINO_API int wino_values_updated(wino_plan* plan, void* stream);

/* ForwardCache (layer.hpp:19-25) on the device: Ĩ_F and dL/dZ for up to n_max images. */
WINO_API int wino_cache_create(wino_plan* plan, int n_max, wino_cache** out);
WINO_API int wino_cache_destroy(wino_cache* cache);

/* winograd_forward (layer.cpp:45-96) / sparse_forward (sparse.cpp:190-253), batched:
 * I (device, n×C×H×W) -> O (device, n×K×Ho×Wo).  cache may be NULL (inference);
 * otherwise it receives Ĩ_F and loses any previous dL/dZ (layer.cpp:88). flags:
 * WINO_FWD_RELU applies max(·,0) to O in the output-transform epilogue. */
#define WINO_FWD_RELU 1
WINO_API int wino_forward(wino_plan* plan, int n, const float* input, float* output, wino_cache* cache,
                 int flags, void* stream);
/* winograd_backward_weights (layer.cpp:98-132): dL/dO (device, n×K×Ho×Wo) ->
 * dW (device, see header), storing dL/dZ in the cache.  WINO_BWD_RELU_MASK: dL/dO is
 * first multiplied by [O > 0] with O = relu_out (the trainer's mask, train.cpp:193).
 * dW receives the sum over the n images (the trainer's Σ_n before its 1/B, train.cpp:200). */
#define WINO_BWD_RELU_MASK 1
WINO_API int wino_backward_weights(wino_plan* plan, const float* grad_output, const float* relu_out,
                          wino_cache* cache, float* grad_w, int flags, void* stream);
/* backward_weights + backward_input in one call: dZ first, then dW_F on an internal stream
 * concurrently with dĨ_F -> dI on `stream` (they share only the read-only dZ and Ĩ_F); `stream`
 * waits for both before the call's work is complete.  Same results as the two calls.
 * grad_input may be NULL (no dI: the first layer of a stack, train.cpp:201). */
WINO_API int wino_backward(wino_plan* plan, const float* grad_output, const float* relu_out,
                           wino_cache* cache, float* grad_w, float* grad_input, int flags, void* stream);
/* One training step of the layer: wino_forward followed by wino_backward with both gradients
 * (no ReLU flags), bit for bit, but scheduled by data dependence rather than call order: dZ
 * needs only grad_output, so the dO -> dZ -> dĨ_F -> dI chain starts beside the forward on a
 * side stream and dW_F starts as soon as Ĩ_F and dZ exist (a second side stream); both join
 * `stream` before return.  The caller (train.cpp:158-211 per sample; a batched trainer per
 * layer) owns the cache exactly as with the two calls. */
WINO_API int wino_forward_backward(wino_plan* plan, int n, const float* input, float* output, wino_cache* cache,
                                   const float* grad_output, float* grad_w, float* grad_input, void* stream);
/* The data-parallel exchange: sum grad_w (count floats; count < 0 = this plan's
 * dW_F length, nnz-compact or K×C×p×q) in place over an NCCL communicator (`nccl_comm` is an
 * ncclComm_t), on `stream`.  The scale 1/N_global of train.cpp:166,200 stays with the update.
 * NCCL is resolved at run time (already-loaded libnccl.so.2 first); WINO_CAPABILITY_ERROR if none. */
WINO_API int wino_allreduce_dw(wino_plan* plan, void* nccl_comm, float* grad_w, int64_t count, void* stream);
/* The same exchange inside the backward: with a communicator set (NULL clears it), every call
 * that produces dW_F (backward_weights, backward, forward_backward, backward_weights_cached) sums
 * grad_w over it right after the dW_F kernels, on the dW_F stream — so in backward and
 * forward_backward the exchange overlaps the dĨ_F -> dI chain (and the forward's tail) instead
 * of following the step.  grad_w holds the sum over ranks when the call's work completes on
 * `stream`.  Every rank must make the same calls in the same order (NCCL's rule). */
WINO_API int wino_set_dw_allreduce(wino_plan* plan, void* nccl_comm);
/* Image ranges of one batch of n_total images, for overlapping host transfers with compute
 * (the CSR kernels only).  forward_range computes images [n0, n1) into the batch's cache (input
 * and output point at image n0); backward_range computes their dL/dZ, dĨ_F and dI (grad_output,
 * relu_out, grad_input point at image n0); once every range has run, backward_weights_cached
 * computes dW_F over the whole batch.  n0·T must be a multiple of 4.  Results are bitwise those of
 * the whole-batch calls (every kernel is per column, and dW_F runs once over all columns). */
WINO_API int wino_forward_range(wino_plan* plan, int n_total, int n0, int n1, const float* input,
                                float* output, wino_cache* cache, int flags, void* stream);
WINO_API int wino_backward_range(wino_plan* plan, int n0, int n1, const float* grad_output,
                                 const float* relu_out, wino_cache* cache, float* grad_input, int flags,
                                 void* stream);
WINO_API int wino_backward_weights_cached(wino_plan* plan, wino_cache* cache, float* grad_w, void* stream);
/* winograd_backward_input (layer.cpp:134-171): dI (device, n×C×H×W).
 * WINO_CONSISTENCY_ERROR if backward_weights has not run on this cache. */
WINO_API int wino_backward_input(wino_plan* plan, const wino_cache* cache, float* grad_input, void* stream);

/* The weight update of train_step (train.cpp:210-290), on the live weights, in fp64 on the
 * fp32 values.  Per coordinate of the plan (a sparse plan holds only unmasked coordinates, so
 * frozen zeros are never touched — train.cpp:280):
 *   g = scale·grad;  reg = λ·sign(w) (norm 1) | λ·w/‖w‖₂ (norm 2, 0 when ‖w‖ = 0)
 *   v = w − lr·(g + reg);  prune && λ > 0: v = 0 when |v|·(|g| + β) < ε  (train.cpp:108-110)
 * grad is in the layout backward_weights wrote (nnz-compact, or K×C×p×q for a dense plan).
 * Non-finite results are counted on the device (wino_update_status).  Asynchronous on
 * `stream`, capturable in a CUDA graph; refreshes the CSC copy and tensor-core operands. */
typedef struct wino_update {
    double lr;     /* the layer's learning rate (lr · wino_lr_mult for Winograd layers) */
    double scale;  /* gradient scale: 1/B for a Σ over B images (train.cpp:166) */
    double lambda; /* regularisation factor; 0 = none */
    double eps;    /* gradient-threshold ε (PruneConfig::eps) */
    double beta;   /* gradient-threshold β (PruneConfig::beta) */
    int norm;      /* 1 or 2 (fine-tuning uses 2, train.cpp:262) */
    int prune;     /* apply the threshold (StepMode::prune) */
} wino_update;
WINO_API int wino_update_weights(wino_plan* plan, const float* grad_w, const wino_update* update,
                                 void* stream);
/* Masked SGD (the fine-tune step): wino_update_weights with norm 2, λ = l2, no threshold. */
WINO_API int wino_sgd_step(wino_plan* plan, const float* grad_w, float lr, float scale, float l2,
                  void* stream);
/* Synchronizes; *nonfinite = non-finite updated weights since the last call (then reset).
 * A nonzero count is the reference's TrainingError "divergence" (train.cpp:288). */
WINO_API int wino_update_status(wino_plan* plan, int64_t* nonfinite);
/* Re-derive the CSR from the plan's current weights on the device, exactly as compress
 * (sparse.cpp:9-36) of those weights would: a dense plan after pruning steps becomes the sparse
 * plan of its surviving coordinates (set_masks_from_zeros + fine-tune, train.cpp:322-338). */
WINO_API int wino_recompress(wino_plan* plan, double zero_tol);

/* Plan options.
 *   WINO_OPT_DW_MODE: how dW_F (layer.cpp:118-128, on the mask of train.cpp:281-283) is computed.
 *     0 (default, the only mode): exact — Ĩ_F and dZ recomputed in the reference's f64 by the
 *       fused K1/K4 kernels and written as 5 balanced base-256 int8 digits (one exponent per
 *       (segment, slice, row) from max|I| / max|dO|); the 15 high-weight digit pairs are
 *       multiplied exactly on tcgen05 kind::i8 into int32 TMEM, combined and chunk-summed in fp64,
 *       then gathered on the mask in CSR order.  Matches the reference's f64 layer within the
 *       strict per-element bound (~2^-35 of Σ|products|).  Other values: WINO_INVALID_ARGUMENT. */
#define WINO_OPT_DW_MODE 1
/*   WINO_OPT_CONTRACTION: how a sparse plan runs Z = W_F·Ĩ_F and dĨ_F = W_Fᵀ·dZ:
 *     0 (default) the CSR kernels — the reference's association order, forward bitwise equal
 *       to sparse_forward<float>;
 *     1 tensor cores — the 3xTF32 tcgen05 GEMM (per-k-block fp64 folding) over the zero-filled
 *       W_F slices; fp32-level accuracy (within the north_star tolerance, not bitwise).  Masked
 *       coordinates stay exactly zero (the operands are re-scattered from the CSR values on
 *       every update).  Requires C, K multiples of 4.
 *     2 auto — tensor cores when the plan's density reaches WINO_OPT_AUTO_DENSITY per mille
 *       (default: the measured crossover — 110 for 128 < C, K <= 256, where the hybrid CSR kernel
 *       runs, 80 otherwise), else the CSR kernels; re-decided whenever the weights change. */
#define WINO_OPT_CONTRACTION 2
#define WINO_OPT_AUTO_DENSITY 3
/*   WINO_OPT_SPMM_OPERANDS: where the CSR kernels keep their dense operand chunk (Ĩ_F / dZ):
 *     0 (default) auto — tensor memory (tcgen05.ld, operand rows spread over the lane quarters
 *       by stage, wino_spmm_tm.cuh) when 128 < rows <= 512, the density is >= 4% and the work
 *       units fill the GPU twice; shared memory otherwise;
 *     1 shared memory always; 2 tensor memory whenever 128 < rows <= 512; 3 hybrid whenever
 *     128 < rows <= 256: operand rows [0,128) in tensor memory and the rest in shared memory, one
 *     warp per output row and no stage handoffs (auto picks it when the slice's entry stream fits
 *     in shared memory next to the chunk).  All are bitwise the reference's order. */
#define WINO_OPT_SPMM_OPERANDS 4
WINO_API int wino_set_option(wino_plan* plan, int option, int value);

/* ---------------------------------------------------------------------------- */
/* Instrumentation                                                               */
/* ---------------------------------------------------------------------------- */
/* Number of kernels this plan has launched since creation (or the last reset). */
WINO_API int64_t wino_launch_count(const wino_plan* plan);
WINO_API void wino_reset_launch_count(wino_plan* plan);
/* Per-kernel CUDA-event timing on the launching stream. enable=1 starts recording
 * (events around every launch); wino_profile_read synchronises and returns, for up
 * to `cap` kernel kinds, the summed milliseconds and launch counts. Names are static. */
WINO_API int wino_profile_enable(wino_plan* plan, int enable);
WINO_API int wino_profile_read(wino_plan* plan, int cap, const char** names, double* ms, int64_t* launches,
                      int* n_kinds);

WINO_API const char* wino_last_error(void);
WINO_API const char* wino_version(void);

#ifdef __cplusplus
}
#endif
#endif /* WINO_CUDA_H */
