// Precise dW_F mode (WINO_OPT_DW_MODE = 2): the fp32 residuals of Ĩ_F and dZ.
//
// Ĩ_F and dZ are stored in fp32 (bitwise the reference's f32 path).  Their rounding alone keeps
// an fp32-storage dW_F = dZ·Ĩ_Fᵀ off the reference's f64 result by more than the strict
// tolerance on a few entries with heavy cancellation.  These kernels recompute
// both transforms in fp64 with the reference's f64 coefficients and store lo = fl(x64 − hi):
// hi + lo represents the f64 transform to ~2^-48 relative, and the LO variant of the SDDMM
// (wino_kernels.cuh) consumes both.  Same thread mapping as K1 / K4.
#pragma once

#include <cstdint>

namespace wino {

struct CoefsD {
    double a[kMaxP * kMaxP];  // a1: p×m row-major
    double b[kMaxP * kMaxP];  // b1: p×p row-major
};

template <int M, int P>
__global__ void __launch_bounds__(256)
input_transform_lo_kernel(const float* __restrict__ in, const float* __restrict__ V, float* __restrict__ Vlo,
                          const CoefsD cf, int C, int H, int W, int pad, int tiles_x, int T, int NT, int NTs) {
    const int64_t plane = (int64_t)C * NTs;
    for (int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < plane;
         gid += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(gid / NTs);
        const int nt = (int)(gid - (int64_t)c * NTs);
        if (nt >= NT) {
#pragma unroll
            for (int s = 0; s < P * P; ++s) Vlo[(int64_t)s * plane + gid] = 0.f;
            continue;
        }
        double d[P][P];
        const int n = nt / T, t = nt - n * T;
        const int ty = t / tiles_x, tx = t - ty * tiles_x;
        const int y0 = ty * M - pad, x0 = tx * M - pad;
        const float* src = in + ((int64_t)n * C + c) * H * W;
#pragma unroll
        for (int i = 0; i < P; ++i) {
            const int y = y0 + i;
            const bool yok = (unsigned)y < (unsigned)H;
#pragma unroll
            for (int j = 0; j < P; ++j) {
                const int x = x0 + j;
                d[i][j] = (yok && (unsigned)x < (unsigned)W) ? (double)__ldg(src + y * W + x) : 0.0;
            }
        }
        double tmp[P][P];
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
            for (int j = 0; j < P; ++j) {
                double acc = 0.0;
#pragma unroll
                for (int k = 0; k < P; ++k) acc = fma(cf.b[k * P + i], d[k][j], acc);
                tmp[i][j] = acc;
            }
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
            for (int j = 0; j < P; ++j) {
                double acc = 0.0;
#pragma unroll
                for (int k = 0; k < P; ++k) acc = fma(cf.b[k * P + j], tmp[i][k], acc);
                const int64_t o = (int64_t)(i * P + j) * plane + gid;
                Vlo[o] = (float)(acc - (double)V[o]);
            }
    }
}

template <int M, int P, bool MASK>
__global__ void __launch_bounds__(256)
grad_z_lo_kernel(const float* __restrict__ dO, const float* __restrict__ relu_out, const float* __restrict__ DZ,
                 float* __restrict__ DZlo, const CoefsD cf, int K, int Ho, int Wo, int tiles_x, int T, int NT,
                 int NTs) {
    const int64_t plane = (int64_t)K * NTs;
    for (int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < plane;
         gid += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(gid / NTs);
        const int nt = (int)(gid - (int64_t)k * NTs);
        if (nt >= NT) {
#pragma unroll
            for (int s = 0; s < P * P; ++s) DZlo[(int64_t)s * plane + gid] = 0.f;
            continue;
        }
        double d[M][M];
        const int n = nt / T, t = nt - n * T;
        const int ty = t / tiles_x, tx = t - ty * tiles_x;
        const int64_t base = ((int64_t)n * K + k) * Ho * Wo;
#pragma unroll
        for (int y = 0; y < M; ++y) {
            const int oy = ty * M + y;
#pragma unroll
            for (int x = 0; x < M; ++x) {
                const int ox = tx * M + x;
                double v = 0.0;
                if (oy < Ho && ox < Wo) {
                    const int64_t o = base + oy * Wo + ox;
                    v = (double)__ldg(dO + o);
                    if (MASK && !(__ldg(relu_out + o) > 0.f)) v = 0.0;
                }
                d[y][x] = v;
            }
        }
        double m1[P][M];
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
            for (int x = 0; x < M; ++x) {
                double acc = 0.0;
#pragma unroll
                for (int y = 0; y < M; ++y) acc = fma(cf.a[i * M + y], d[y][x], acc);
                m1[i][x] = acc;
            }
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
            for (int j = 0; j < P; ++j) {
                double acc = 0.0;
#pragma unroll
                for (int x = 0; x < M; ++x) acc = fma(cf.a[j * M + x], m1[i][x], acc);
                const int64_t o = (int64_t)(i * P + j) * plane + gid;
                DZlo[o] = (float)(acc - (double)DZ[o]);
            }
    }
}

}  // namespace wino
