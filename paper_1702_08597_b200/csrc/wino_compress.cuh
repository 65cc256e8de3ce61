// On-device compress<float> (sparse.cpp:9-36): the per-slice CSR of W_F(:,:,i,j) and its CSC
// (for dĨ_F = W_Fᵀ·dZ) built straight from the K×C×p×p f64 weights in HBM.
//
// Keep rule (sparse.cpp:18-19): |w| > zero_tol, or w != 0 when zero_tol == 0 (NaN is kept), on
// the f64 value; the stored value is (float)w.  Slices s = i·p + j in order, rows k ascending,
// columns c ascending inside a row — identical arrays to the reference's compress, so nothing
// downstream can tell the two apart (tests/test_gpu_parity.py compares them element by element).
//
// One thread per (row, slice) walks its row sequentially (ascending c for free); threads are
// numbered with the slice fastest, so a warp's loads w[(k·C + c)·p² + s] for consecutive s are
// contiguous: every pass reads W_F once, coalesced.  Columns work the same way per (c, s).
#pragma once

#include <cstdint>

namespace wino {

__device__ __forceinline__ bool keep_weight(double v, double tol, int keep_all) {
    return keep_all || fabs(v) > tol || (tol == 0.0 && v != 0.0);
}

// cnt[s·R + r] = kept entries of line r of slice s (rows: line = k over c; cols: line = c over k)
template <bool COLS>
__global__ void compress_count_kernel(const double* __restrict__ w, int K, int C, int P2, double tol,
                                      int keep_all, int* __restrict__ cnt) {
    const int lines = COLS ? C : K, len = COLS ? K : C;
    const int64_t total = (int64_t)lines * P2;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(t % P2), l = (int)(t / P2);
        const int64_t base = COLS ? (int64_t)l * P2 + s : (int64_t)l * C * P2 + s;
        const int64_t step = COLS ? (int64_t)C * P2 : P2;
        int n = 0;
#pragma unroll 8
        for (int x = 0; x < len; ++x) n += keep_weight(w[base + x * step], tol, keep_all);
        cnt[(int64_t)s * lines + l] = n;
    }
}

// Exclusive scan of cnt[s][l] (slice-major) into ptr[s·(L+1) + l] with global offsets, plus the
// closing ptr[s·(L+1) + L].  One block; n = P2·L is at most a few hundred thousand.
__global__ void compress_scan_kernel(const int* __restrict__ cnt, int P2, int L, int* __restrict__ ptr) {
    __shared__ int warp_tot[32];
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int64_t n = (int64_t)P2 * L;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int64_t base = 0; base < n; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        const int v = i < n ? cnt[i] : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_tot[wid] = x;
        __syncthreads();
        if (wid == 0) {
            int t = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += y;
            }
            if (lane < nw) warp_tot[lane] = t;  // inclusive prefix of warp totals
        }
        __syncthreads();
        const int excl = carry + (wid ? warp_tot[wid - 1] : 0) + x - v;
        if (i < n) {
            const int64_t s = i / L, l = i % L;
            ptr[s * (L + 1) + l] = excl;
            if (l == L - 1) ptr[s * (L + 1) + L] = excl + v;
        }
        __syncthreads();
        if (threadIdx.x == 0) carry += warp_tot[nw - 1];
        __syncthreads();
    }
}

// CSR fill: column indices, values, row-of-entry, the interleaved (col, value bits) stream and
// the dense position map pos[(s·K + k)·C + c] the CSC pass reads its permutation from.
__global__ void compress_fill_rows_kernel(const double* __restrict__ w, int K, int C, int P2, double tol,
                                          int keep_all, const int* __restrict__ rowptr, int* __restrict__ colidx,
                                          float* __restrict__ vals, int* __restrict__ rowof, int2* __restrict__ cv,
                                          int* __restrict__ pos) {
    const int64_t total = (int64_t)K * P2;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(t % P2), k = (int)(t / P2);
        const int64_t base = (int64_t)k * C * P2 + s;
        int e = rowptr[(int64_t)s * (K + 1) + k];
        int* prow = pos + ((int64_t)s * K + k) * C;
        for (int c0 = 0; c0 < C; c0 += 8) {  // 8 loads in flight, then the ordered appends
            double vv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) vv[j] = c0 + j < C ? w[base + (int64_t)(c0 + j) * P2] : 0.0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int c = c0 + j;
                if (c < C && keep_weight(vv[j], tol, keep_all)) {
                    const float f = (float)vv[j];
                    colidx[e] = c;
                    vals[e] = f;
                    rowof[e] = k;
                    cv[e] = make_int2(c, __float_as_int(f));
                    prow[c] = e;
                    ++e;
                }
            }
        }
    }
}

// CSC fill: rows ascending within a column (sparse.cpp's transpose order), perm = CSR position.
__global__ void compress_fill_cols_kernel(const double* __restrict__ w, int K, int C, int P2, double tol,
                                          int keep_all, const int* __restrict__ colptr, const int* __restrict__ pos,
                                          int* __restrict__ rowidx, int* __restrict__ perm, int2* __restrict__ cvT) {
    const int64_t total = (int64_t)C * P2;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(t % P2), c = (int)(t / P2);
        int d = colptr[(int64_t)s * (C + 1) + c];
        for (int k0 = 0; k0 < K; k0 += 8) {
            double vv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) vv[j] = k0 + j < K ? w[((int64_t)(k0 + j) * C + c) * P2 + s] : 0.0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int k = k0 + j;
                if (k < K && keep_weight(vv[j], tol, keep_all)) {
                    rowidx[d] = k;
                    perm[d] = pos[((int64_t)s * K + k) * C + c];
                    cvT[d] = make_int2(k, __float_as_int((float)vv[j]));
                    ++d;
                }
            }
        }
    }
}

}  // namespace wino
