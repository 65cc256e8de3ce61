// The weight update of train_step (train.cpp:210-290) on the live CSR values, and the
// device-side weight snapshot that re-derives the CSR after pruning.
//
// Per coordinate (train.cpp:265-287), in fp64 on the fp32 stored values:
//   g   = scale · grad                       (the 1/B of train.cpp:166,200)
//   reg = λ·sign(w)            (norm 1)      reg_grad, train.cpp:213-218
//       = λ·w/‖w‖₂ (0 if ‖w‖=0) (norm 2)
//   v   = w − lr·(g + reg)
//   prune && λ > 0:  v = 0  if |v|·(|g| + β) < ε        threshold_value, train.cpp:108-110
//   non-finite v is counted (the reference throws TrainingError "divergence").
// Masked (frozen-zero) coordinates do not exist in a sparse plan's CSR, so they are never
// touched — the fine-tune rule of train.cpp:280.
#pragma once

#include <cstdint>

namespace wino {

struct UpdateParams {
    double lr, scale, lambda, eps, beta;
    int norm, prune;
};

// Deterministic Σ v² in fp64: fixed block → slice assignment, partials reduced in fixed order.
__global__ void sumsq_partial_kernel(const float* __restrict__ vals, int64_t n, double* __restrict__ partial) {
    __shared__ double red[32];
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = vals[i];
        s += v * v;
    }
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) partial[blockIdx.x] = s;
    }
}

__global__ void sumsq_final_kernel(const double* __restrict__ partial, int nparts, double* __restrict__ out) {
    __shared__ double red[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += partial[i];
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) *out = s;
    }
}

// vals: CSR order.  grad: the layout backward_weights produced — CSR order for a sparse plan,
// K×C×p×q for a dense plan (kcpq = 1; vals[(s·K + k)·C + c] ↔ grad[(k·C + c)·p² + s]).
// sumsq: Σ w² (read only for norm 2 with λ ≠ 0).
__global__ void update_kernel(float* __restrict__ vals, const float* __restrict__ grad, int64_t n, int kcpq,
                              int K, int C, int P2, UpdateParams u, const double* __restrict__ sumsq,
                              unsigned long long* __restrict__ nonfinite) {
    const double nrm = (u.norm == 2 && u.lambda != 0.0) ? sqrt(*sumsq) : 0.0;
    unsigned long long bad = 0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        int64_t gi = e;
        if (kcpq) {
            const int64_t s = e / ((int64_t)K * C), kc = e - s * K * C;
            gi = kc * P2 + s;
        }
        // the reference's f64 expression order, rounded at every step (no FMA contraction)
        const double w = vals[e];
        const double g = __dmul_rn(u.scale, (double)grad[gi]);
        double reg = 0.0;
        if (u.lambda != 0.0) {
            if (u.norm == 1)
                reg = w > 0.0 ? u.lambda : (w < 0.0 ? -u.lambda : 0.0);
            else
                reg = nrm > 0.0 ? __ddiv_rn(__dmul_rn(u.lambda, w), nrm) : 0.0;
        }
        double v = __dsub_rn(w, __dmul_rn(u.lr, __dadd_rn(g, reg)));
        if (u.prune && u.lambda > 0.0 && __dmul_rn(fabs(v), __dadd_rn(fabs(g), u.beta)) < u.eps) v = 0.0;
        const float f = (float)v;
        if (!isfinite(f)) ++bad;  // includes finite f64 results beyond the fp32 range
        vals[e] = f;
    }
    if (bad) atomicAdd(nonfinite, bad);
}

// Current CSR values -> dense K×C×p×q f64 (zeros off the CSR), the source compress re-reads.
// One thread per (row k, slice s).
__global__ void csr_to_kcpq_f64_kernel(const int* __restrict__ rowptr, const int* __restrict__ colidx,
                                       const float* __restrict__ vals, int K, int C, int P2,
                                       double* __restrict__ dst) {
    const int64_t total = (int64_t)K * P2;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(t % P2), k = (int)(t / P2);
        const int b = rowptr[(int64_t)s * (K + 1) + k], e = rowptr[(int64_t)s * (K + 1) + k + 1];
        for (int i = b; i < e; ++i) dst[((int64_t)k * C + colidx[i]) * P2 + s] = (double)vals[i];
    }
}

// CSR values -> zero-filled slice-major W[s][k][c] fp32 (the tensor-core operand source of a
// sparse plan).  One thread per (row k, slice s).
__global__ void csr_scatter_dense_kernel(const int* __restrict__ rowptr, const int* __restrict__ colidx,
                                         const float* __restrict__ vals, int K, int C, int P2,
                                         float* __restrict__ dst) {
    const int64_t total = (int64_t)K * P2;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(t % P2), k = (int)(t / P2);
        const int b = rowptr[(int64_t)s * (K + 1) + k], e = rowptr[(int64_t)s * (K + 1) + k + 1];
        float* row = dst + ((int64_t)s * K + k) * C;
        for (int i = b; i < e; ++i) row[colidx[i]] = vals[i];
    }
}

}  // namespace wino
