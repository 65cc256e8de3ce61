// Hand-written sm_100a kernels of the Winograd layer hot path.
//
// Device layouts (fp32, NTs = round_up(n·T, 4) is the padded row stride):
//   V  = Ĩ_F   [p·q][C][NTs]   column nt = n·T + t (image-major, tile-minor)
//   Z          [p·q][K][NTs]
//   DZ = dL/dZ [p·q][K][NTs]
//   DV = dĨ_F  [p·q][C][NTs]
// The tile dimension is contiguous (sparse.hpp:59-69) so every
// kernel streams rows of NT floats with coalesced, vectorised accesses.
//
// Numerics: every transform and the CSR contractions use products rounded to fp32
// and left-to-right sums from +0 with no fused multiply-add (__fmul_rn/__fadd_rn),
// in the reference's own association order (sparse.cpp:103-116, 151-184 for the
// forward; layer.cpp:107-116, 145-169 for the backward).  The forward output is
// therefore bit-identical to the reference's f32 sparse_forward.  dW_F (K5) is a
// reduction over n·T terms and is accumulated in fp64 across t-chunks.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "builtin_coefs.h"

namespace wino {

constexpr int kMaxP = 8;
constexpr unsigned kFull = 0xffffffffu;

// Transform constants cast to fp32 exactly as the reference casts them
// (to_precision<float>, sparse.cpp:73-76).  Passed by value: the coefficients sit
// in the kernel-parameter constant bank and feed FMUL as constant operands.
struct Coefs {
    float a[kMaxP * kMaxP];  // a1: p×m row-major, a(i,y) = a[i*M + y]
    float b[kMaxP * kMaxP];  // b1: p×p row-major, b(i,k) = b[i*P + k]
};

__device__ __forceinline__ float madd(float acc, float c, float x) {
    return __fadd_rn(acc, __fmul_rn(c, x));
}

// Coefficient policies.  RuntimeCoef reads the plan's Coefs (any TransformSet the caller
// passes).  ConstCoef<M,P> uses the built-in sets as compile-time constants (builtin_coefs.h,
// the reference's doubles cast to float): after unrolling, a zero coefficient drops its term
// and ±1 drops the multiply — bit-identical for finite inputs (acc starts at +0 and never
// becomes -0, so acc + (±0) == acc; 1·x == x; -1·x == -x exactly).
struct RuntimeCoef {
    static constexpr bool kConst = false;
};
template <int M, int P>
struct ConstCoef {
    static constexpr bool kConst = true;
};

template <class CF, int M, int P>
__device__ __forceinline__ float coef_a(const Coefs& cf, int i) {
    if constexpr (CF::kConst) return BuiltinCoefs<M, P>::A(i);
    else return cf.a[i];
}
template <class CF, int M, int P>
__device__ __forceinline__ float coef_b(const Coefs& cf, int i) {
    if constexpr (CF::kConst) return BuiltinCoefs<M, P>::B(i);
    else return cf.b[i];
}
template <class CF>
__device__ __forceinline__ float cmadd(float acc, float c, float x) {
    if constexpr (CF::kConst) {
        if (c == 0.f) return acc;
        if (c == 1.f) return __fadd_rn(acc, x);
        if (c == -1.f) return __fsub_rn(acc, x);
    }
    return madd(acc, c, x);
}

// Packed fp32 pairs (FFMA2 / FADD2 on Blackwell): two lanes of the same rounded operations.
// mul2 forms the rounded product with a runtime -0 addend z (so ptxas cannot contract it with the
// following add2 into one rounding); every result is bitwise the scalar __fmul_rn / __fadd_rn.
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
    unsigned long long v;
    asm("mov.b64 %0, {%1,%2};" : "=l"(v) : "f"(a), "f"(b));
    return v;
}
__device__ __forceinline__ void upk2(unsigned long long v, float& a, float& b) {
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ unsigned long long mul2(unsigned long long x, unsigned long long w, unsigned long long z) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x), "l"(w), "l"(z));
    return d;
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long sub2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
// acc2 += c·x2 with a compile-time coefficient: zero skipped, ±1 without the multiply (as cmadd)
template <class CF>
__device__ __forceinline__ unsigned long long cmadd2(unsigned long long acc, float c, unsigned long long x,
                                                     unsigned long long z) {
    if (c == 0.f) return acc;
    if (c == 1.f) return add2(acc, x);
    if (c == -1.f) return sub2(acc, x);
    return add2(acc, mul2(x, pk2(c, c), z));
}

// The same transform in the reference's doubles (the exact dW_F digit kernels, wino_xdw.cuh).
struct CoefsD {
    double a[kMaxP * kMaxP];  // a1: p×m row-major
    double b[kMaxP * kMaxP];  // b1: p×p row-major
};

// ---------------------------------------------------------------------------------
// K1: φ gather (pad folded in) + Ĩ_F = B1ᵀ·d·B2   (transforms.cpp:196-210, sparse.cpp:94-120)
// One thread per (c, nt); consecutive threads = consecutive tiles -> coalesced stores.
// ---------------------------------------------------------------------------------
template <int M, int P, class CF>
__global__ void __launch_bounds__(256)
input_transform_kernel(const float* __restrict__ in, float* __restrict__ V, const Coefs cf, int C,
                       int H, int W, int pad, int tiles_x, int T, int NT, int NTs, int NTr) {
    // grid (column blocks, C): c = blockIdx.y, nt = blockIdx.x·256 + thread.  Columns [0, NTr) of
    // V rows with stride NTs; columns >= NT are the zero padding.  (Training steps run the same
    // product fused with the exact dW_F digits, wino_xdw.cuh.)
    const int c = blockIdx.y;
    const int nt = blockIdx.x * blockDim.x + threadIdx.x;
    if (nt >= NTr) return;
    const int64_t plane = (int64_t)C * NTs;
    float d[P][P];
    if (nt < NT) {
        const int n = nt / T, t = nt - n * T;
        const int ty = t / tiles_x, tx = t - ty * tiles_x;
        const int y0 = ty * M - pad, x0 = tx * M - pad;
        const float* src = in + ((int64_t)n * C + c) * H * W;
        if (M == 4 && P == 6 && pad == 1 && (W & 3) == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
            // patch row = 4tx-1 | 4tx .. 4tx+3 (one aligned 16-byte load, always inside the row) | 4tx+4
#pragma unroll
            for (int i = 0; i < P; ++i) {
                const int y = y0 + i;
                if ((unsigned)y < (unsigned)H) {
                    const float* row = src + y * W + (x0 + 1);
                    const float4 v = __ldg(reinterpret_cast<const float4*>(row));
                    d[i][0] = x0 >= 0 ? __ldg(row - 1) : 0.f;
                    d[i][1] = v.x;
                    d[i][2] = v.y;
                    d[i][3] = v.z;
                    d[i][4] = v.w;
                    d[i][5] = x0 + 5 < W ? __ldg(row + 4) : 0.f;
                } else {
#pragma unroll
                    for (int j = 0; j < P; ++j) d[i][j] = 0.f;
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < P; ++i) {
                const int y = y0 + i;
                const bool yok = (unsigned)y < (unsigned)H;
#pragma unroll
                for (int j = 0; j < P; ++j) {
                    const int x = x0 + j;
                    d[i][j] = (yok && (unsigned)x < (unsigned)W) ? __ldg(src + y * W + x) : 0.f;
                }
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
            for (int j = 0; j < P; ++j) d[i][j] = 0.f;
    }
    float tmp[P][P];
#pragma unroll
    for (int i = 0; i < P; ++i)
#pragma unroll
        for (int j = 0; j < P; ++j) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < P; ++k) acc = cmadd<CF>(acc, coef_b<CF, M, P>(cf, k * P + i), d[k][j]);
            tmp[i][j] = acc;
        }
    float* vp = V + (int64_t)c * NTs + nt;
#pragma unroll
    for (int i = 0; i < P; ++i)
#pragma unroll
        for (int j = 0; j < P; ++j, vp += plane) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < P; ++k) acc = cmadd<CF>(acc, coef_b<CF, M, P>(cf, k * P + j), tmp[i][k]);
            *vp = acc;
        }
}

// ---------------------------------------------------------------------------------
// K3: O = ψ(A1ᵀ·Z·A2), crop, optional ReLU   (sparse.cpp:151-184; layer.cpp:79-95)
// One thread per (k, nt): 36 coalesced loads, 16 outputs.
// ---------------------------------------------------------------------------------
template <int M, int P, bool RELU, class CF>
__global__ void __launch_bounds__(256)
output_transform_kernel(const float* __restrict__ Z, float* __restrict__ O, const Coefs cf, int K,
                        int Ho, int Wo, int tiles_x, int T, int NT, int NTs) {
    // grid (column blocks, K): k = blockIdx.y, nt = blockIdx.x·256 + thread — 32-bit index math,
    // the 36 slice loads by pointer steps, the output rows by row pointers
    const int k = blockIdx.y;
    const int nt = blockIdx.x * blockDim.x + threadIdx.x;
    if (nt >= NT) return;
    const int64_t plane = (int64_t)K * NTs;
    const float* zp = Z + (int64_t)k * NTs + nt;
    float z[P][P];
#pragma unroll
    for (int i = 0; i < P; ++i)
#pragma unroll
        for (int j = 0; j < P; ++j, zp += plane) z[i][j] = __ldg(zp);
    float tmp[M][P];
#pragma unroll
    for (int y = 0; y < M; ++y)
#pragma unroll
        for (int j = 0; j < P; ++j) {
            float acc = 0.f;
#pragma unroll
            for (int i = 0; i < P; ++i) acc = cmadd<CF>(acc, coef_a<CF, M, P>(cf, i * M + y), z[i][j]);
            tmp[y][j] = acc;
        }
    const int n = nt / T, t = nt - n * T;
    const int ty = t / tiles_x, tx = t - ty * tiles_x;
    const int oy0 = ty * M, ox0 = tx * M;
    float* orow = O + (((int64_t)n * K + k) * Ho + oy0) * Wo + ox0;
    // whole tile inside the image and 16-byte-aligned rows: one vector store per output row
    const bool vec = M == 4 && (Wo & 3) == 0 && oy0 + M <= Ho && (reinterpret_cast<uintptr_t>(O) & 15) == 0;
#pragma unroll
    for (int y = 0; y < M; ++y, orow += Wo) {
        float r[M];
#pragma unroll
        for (int x = 0; x < M; ++x) {
            float acc = 0.f;
#pragma unroll
            for (int j = 0; j < P; ++j) acc = cmadd<CF>(acc, coef_a<CF, M, P>(cf, j * M + x), tmp[y][j]);
            if (RELU) acc = acc > 0.f ? acc : 0.f;  // train.cpp:76-83
            r[x] = acc;
        }
        if constexpr (M == 4) {
            if (vec) {
                *reinterpret_cast<float4*>(orow) = make_float4(r[0], r[1], r[2], r[3]);
                continue;
            }
        }
        if (oy0 + y < Ho) {
#pragma unroll
            for (int x = 0; x < M; ++x)
                if (ox0 + x < Wo) orow[x] = r[x];
        }
    }
}

// K4 (dZ = A1·dÕ·A2ᵀ, ψ⁻¹ gather, ReLU mask) runs fused with the exact dW_F digits:
// grad_z_digits_kernel (wino_xdw.cuh).

// ---------------------------------------------------------------------------------
// K7: dI = Σ_φ B1·dĨ_F·B2ᵀ — fused B-transform + deterministic halo gather-sum
//     (layer.cpp:157-169).  Block = (image n, group of CG channels).  Phase 1 writes the
//     transformed tiles of the group to shared memory; phase 2 gives every input pixel
//     its ≤⌈p/m⌉² contributions in ascending t order from +0 (the reference's
//     accumulation order), so no atomics and the result is bitwise deterministic.
// ---------------------------------------------------------------------------------
template <int M, int P, class CF>
__device__ __forceinline__ float tile_grad_entry(const float* __restrict__ dv, int64_t plane,
                                                 const Coefs& cf, int i, int j) {
    // g(i,j) with m1(i,l) = Σ_k b1(i,k)·x(k,l) ; g(i,j) = Σ_l m1(i,l)·b2(j,l)
    float acc = 0.f;
#pragma unroll
    for (int l = 0; l < P; ++l) {
        float m = 0.f;
#pragma unroll
        for (int k = 0; k < P; ++k) m = cmadd<CF>(m, coef_b<CF, M, P>(cf, i * P + k), __ldg(dv + (int64_t)(k * P + l) * plane));
        acc = cmadd<CF>(acc, coef_b<CF, M, P>(cf, j * P + l), m);
    }
    return acc;
}

template <int M, int P, class CF, bool ALIGNED = false>
__global__ void __launch_bounds__(256)
input_grad_kernel(const float* __restrict__ DV, float* __restrict__ dI, const Coefs cf, int C,
                  int H, int W, int pad, int tiles_y, int tiles_x, int T, int NTs, int CG,
                  unsigned long long z) {
    constexpr int TS = P * P + 1;  // odd per-tile stride: conflict-free tile stores
    extern __shared__ float gsm[];  // [CG][T][TS]
    const int n = blockIdx.y;
    const int c0 = blockIdx.x * CG;
    const int64_t plane = (int64_t)C * NTs;
    for (int idx = threadIdx.x; idx < CG * T; idx += blockDim.x) {
        const int cl = idx / T, t = idx - cl * T;
        const int c = c0 + cl;
        if (c >= C) continue;
        const float* src = DV + (int64_t)c * NTs + (int64_t)n * T + t;
        float x[P][P];
#pragma unroll
        for (int k = 0; k < P; ++k)
#pragma unroll
            for (int l = 0; l < P; ++l, src += plane) x[k][l] = __ldg(src);
        float m1[P][P];
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
            for (int l = 0; l < P; ++l) {
                float acc = 0.f;
#pragma unroll
                for (int k = 0; k < P; ++k) acc = cmadd<CF>(acc, coef_b<CF, M, P>(cf, i * P + k), x[k][l]);
                m1[i][l] = acc;
            }
        float* g = gsm + (int64_t)idx * TS;
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
            for (int j = 0; j < P; ++j) {
                float acc = 0.f;
#pragma unroll
                for (int l = 0; l < P; ++l) acc = cmadd<CF>(acc, coef_b<CF, M, P>(cf, j * P + l), m1[i][l]);
                g[i * P + j] = acc;
            }
    }
    __syncthreads();
    // Phase 2, tile-centric: the thread of tile (ty,tx) owns padded pixels
    // [ty·M, ty·M + M) × [tx·M, tx·M + M), extended to P on the last tile row/column.  A pixel
    // at local (i,j) gets its contributions from tiles (ty-1,tx-1), (ty-1,tx), (ty,tx-1),
    // (ty,tx) — ascending t, the reference's order — at compile-time offsets (+M when the
    // pixel lies in a neighbour's overlap band, i.e. local index < P-M).
    constexpr int O = P - M;
    if constexpr (ALIGNED) {
        // F(4x4,3x3), pad 1, H = 4·tiles_y, W = 4·tiles_x: the thread of tile (ty,tx) owns the
        // 16-byte-aligned pixels y = 4ty + a, x = 4tx + b (a, b < 4).  Padded row Y = 4ty + a + 1
        // lies in tile row ty (local a+1), in ty-1 (local 5) when a = 0 and in ty+1 (local 0) when
        // a = 3; columns likewise: ≤ 4 contributions per pixel, all at compile-time offsets, added
        // in ascending t from +0 (the reference's order); one float4 store per pixel row.
        static_assert(!ALIGNED || (M == 4 && P == 6), "aligned K7 is F(4x4,3x3) only");
        for (int idx = threadIdx.x; idx < CG * T; idx += blockDim.x) {
            const int cl = idx / T, t = idx - cl * T;
            const int c = c0 + cl;
            if (c >= C) continue;
            const int ty = t / tiles_x, tx = t - ty * tiles_x;
            const float* g0 = gsm + (int64_t)idx * TS;
            const float* gu = g0 - tiles_x * TS;  // (ty-1, tx)
            const float* gd = g0 + tiles_x * TS;  // (ty+1, tx)
            const bool up = ty > 0, dn = ty < tiles_y - 1, lf = tx > 0, rt = tx < tiles_x - 1;
            float* dst = dI + (((int64_t)n * C + c) * H + 4 * ty) * W + 4 * tx;
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                float r[4];
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    float acc = 0.f;
                    if (a == 0 && up) {
                        if (b == 0 && lf) acc = __fadd_rn(acc, gu[-TS + 5 * P + 5]);
                        acc = __fadd_rn(acc, gu[5 * P + b + 1]);
                        if (b == 3 && rt) acc = __fadd_rn(acc, gu[TS + 5 * P]);
                    }
                    if (b == 0 && lf) acc = __fadd_rn(acc, g0[-TS + (a + 1) * P + 5]);
                    acc = __fadd_rn(acc, g0[(a + 1) * P + b + 1]);
                    if (b == 3 && rt) acc = __fadd_rn(acc, g0[TS + (a + 1) * P]);
                    if (a == 3 && dn) {
                        if (b == 0 && lf) acc = __fadd_rn(acc, gd[-TS + 5]);
                        acc = __fadd_rn(acc, gd[b + 1]);
                        if (b == 3 && rt) acc = __fadd_rn(acc, gd[TS]);
                    }
                    r[b] = acc;
                }
                *reinterpret_cast<float4*>(dst + a * W) = make_float4(r[0], r[1], r[2], r[3]);
            }
        }
        return;
    }
    for (int idx = threadIdx.x; idx < CG * T; idx += blockDim.x) {
        const int cl = idx / T, t = idx - cl * T;
        const int c = c0 + cl;
        if (c >= C) continue;
        const int ty = t / tiles_x, tx = t - ty * tiles_x;
        const float* g0 = gsm + (int64_t)idx * TS;
        const float* gu = g0 - tiles_x * TS;       // (ty-1, tx)
        const float* gl = g0 - TS;                 // (ty, tx-1)
        const float* gul = gu - TS;                // (ty-1, tx-1)
        const bool up = ty > 0, left = tx > 0;
        const int ni = ty == tiles_y - 1 ? P : M, nj = tx == tiles_x - 1 ? P : M;
        const int xb = tx * M - pad;
        float* dst = dI + ((int64_t)n * C + c) * H * W + xb;  // + y·W per row, + j per pixel
#pragma unroll
        for (int i = 0; i < P; ++i) {
            if (i >= ni) break;
            const int y = ty * M + i - pad;
            if ((unsigned)y >= (unsigned)H) continue;
            float* drow = dst + y * W;
#pragma unroll
            for (int j = 0; j < P; ++j) {
                if (j >= nj) break;
                if ((unsigned)(xb + j) >= (unsigned)W) continue;
                float acc = 0.f;
                if (i < O && j < O && up && left) acc = __fadd_rn(acc, gul[(i + M) * P + j + M]);
                if (i < O && up) acc = __fadd_rn(acc, gu[(i + M) * P + j]);
                if (j < O && left) acc = __fadd_rn(acc, gl[i * P + j + M]);
                acc = __fadd_rn(acc, g0[i * P + j]);
                drow[j] = acc;
            }
        }
    }
}

// Same result without shared-memory staging (large T): each pixel recomputes the
// transformed-tile entries it needs (identical operation order, hence identical bits).
template <int M, int P, class CF>
__global__ void __launch_bounds__(256)
input_grad_direct_kernel(const float* __restrict__ DV, float* __restrict__ dI, const Coefs cf,
                         int N, int C, int H, int W, int pad, int tiles_y, int tiles_x, int T,
                         int NTs) {
    const int64_t total = (int64_t)N * C * H * W;
    const int64_t plane = (int64_t)C * NTs;
    for (int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < total;
         gid += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(gid % W);
        const int y = (int)((gid / W) % H);
        const int c = (int)((gid / ((int64_t)W * H)) % C);
        const int n = (int)(gid / ((int64_t)W * H * C));
        const int Y = y + pad, X = x + pad;
        const int ty_lo = Y - P + 1 <= 0 ? 0 : (Y - P + M) / M;
        const int ty_hi = min(tiles_y - 1, Y / M);
        const int tx_lo = X - P + 1 <= 0 ? 0 : (X - P + M) / M;
        const int tx_hi = min(tiles_x - 1, X / M);
        float acc = 0.f;
        for (int ty = ty_lo; ty <= ty_hi; ++ty)
            for (int tx = tx_lo; tx <= tx_hi; ++tx) {
                const int t = ty * tiles_x + tx;
                const float* src = DV + (int64_t)c * NTs + (int64_t)n * T + t;
                acc = __fadd_rn(acc, tile_grad_entry<M, P, CF>(src, plane, cf, Y - ty * M, X - tx * M));
            }
        dI[gid] = acc;
    }
}

// ---------------------------------------------------------------------------------
// K2 / K6: CSR SpMM, one p·q slice per blockIdx.z:  Y(r,:) = Σ_{e∈row r} v_e·X(col_e,:)
//   forward   : rows = K, X = Ĩ_F, CSR of W_F(:,:,i,j)       (sparse.cpp:51-69)
//   backward  : rows = C, X = dZ,  CSR of W_F(:,:,i,j)ᵀ (CSC)  (layer.cpp:145-155 on the mask)
// Block = (TW-wide tile-column chunk, row group, slice).  X(:, chunk) of every input row is
// staged in shared memory with cp.async (16-byte, L1-bypassing).  A warp owns a row, each
// lane R consecutive columns; per nonzero the (col, v) pair arrives as ONE warp-uniform
// 8-byte load (a broadcast on the L1 pipe, no shuffles) and X(col, lane's columns) as one
// conflict-free LDS.{32,64,128}.  Nonzeros are consumed four at a time so their loads are
// in flight together.  Accumulation follows the CSR order from +0 (bitwise = reference).
// ---------------------------------------------------------------------------------
template <int R>
__device__ __forceinline__ void lds_vec(const float* p, float (&x)[R]) {
    if constexpr (R == 4) {
        const float4 v = *reinterpret_cast<const float4*>(p);
        x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
    } else if constexpr (R == 2) {
        const float2 v = *reinterpret_cast<const float2*>(p);
        x[0] = v.x; x[1] = v.y;
    } else {
        x[0] = *p;
    }
}

template <int R>
__device__ __forceinline__ void st_vec(float* p, const float (&x)[R]) {
    if constexpr (R == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(x[0], x[1], x[2], x[3]);
    } else if constexpr (R == 2) {
        *reinterpret_cast<float2*>(p) = make_float2(x[0], x[1]);
    } else {
        *p = x[0];
    }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    const int bytes = pred ? 16 : 0;  // zero-fill when out of range
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// Stage X[0..nrows_x)[t0 .. t0+TW) (row stride NTs, NTs % 4 == 0) into xs[nrows_x][TW].
template <int TW>
__device__ __forceinline__ void stage_rows_async(const float* __restrict__ X, float* xs, int nrows_x,
                                                 int NTs, int t0, int tbound = -1) {
    constexpr int V4 = TW / 4;
    const int tb = tbound < 0 ? NTs : tbound;  // columns ≥ tb are zero-filled, never read
    for (int idx = threadIdx.x; idx < nrows_x * V4; idx += blockDim.x) {
        const int row = idx / V4, q = idx - row * V4;
        const int t = t0 + q * 4;
        const bool ok = t < tb;
        cp_async16(xs + row * TW + q * 4, X + (int64_t)row * NTs + (ok ? t : 0), ok);
    }
}

__device__ __forceinline__ int2 ld_uniform_int2(const int2* p) {
    int2 v;
    asm volatile("ld.global.nc.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}

template <bool STAGED>
__device__ __forceinline__ int4 load_pair(const int2* p) {
    if constexpr (STAGED) return *reinterpret_cast<const int4*>(p);
    else return __ldg(reinterpret_cast<const int4*>(p));
}
template <bool STAGED>
__device__ __forceinline__ int2 load_one(const int2* p) {
    if constexpr (STAGED) return *p;
    else return __ldg(p);
}

// STAGED: the block's CSR segment is copied next to the X chunk (LDS.128 broadcasts); otherwise
// the (col, value) pairs are read warp-uniformly from global memory through L1, which frees the
// shared memory for the whole row range of a slice (one block per (chunk, slice): the X chunk is
// staged once instead of once per row group).
template <int R, bool STAGED>
__global__ void __launch_bounds__(1024)
spmm_kernel(const int* __restrict__ rowptr, const int2* __restrict__ colval,
            const float* __restrict__ X, float* __restrict__ Y, int nrows, int ncols, int NTs,
            int rows_per_block, int NTr) {
    constexpr int TW = 32 * R;
    constexpr int U = 8;  // nonzeros in flight per warp
    extern __shared__ float4 smem_f4[];
    float* xs = reinterpret_cast<float*>(smem_f4);
    const int s = blockIdx.z;
    const int t0 = blockIdx.x * TW;
    const int r0 = blockIdx.y * rows_per_block;
    const int r1 = min(nrows, r0 + rows_per_block);
    const int* rp = rowptr + (int64_t)s * (nrows + 1);
    const int e0 = __ldg(rp + r0), e1 = __ldg(rp + r1);
    // the block's CSR segment (col byte offset, value) lands next to the X chunk
    int2* cvs = reinterpret_cast<int2*>(xs + ncols * TW);
    stage_rows_async<TW>(X + (int64_t)s * ncols * NTs, xs, ncols, NTs, t0, NTr);
    if constexpr (STAGED) {
        const int a0 = e0 & ~1;  // 16-byte aligned start (pairs of int2)
        const int n2 = (e1 - a0 + 1) >> 1;
        const int4* src = reinterpret_cast<const int4*>(colval + a0);
        int4* dst = reinterpret_cast<int4*>(cvs);
        for (int i = threadIdx.x; i < n2; i += blockDim.x) cp_async16(dst + i, src + i, true);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    // index with global entry numbers
    const int2* cvb = STAGED ? cvs - (e0 & ~1) : colval;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    float* yg = Y + (int64_t)s * nrows * NTs;
    const int tl = t0 + lane * R;
    const char* xl = reinterpret_cast<const char*>(xs + lane * R);
    for (int r = r0 + warp; r < r1; r += nw) {
        float acc[R];
#pragma unroll
        for (int q = 0; q < R; ++q) acc[q] = 0.f;
        int e = __ldg(rp + r);
        const int ee = __ldg(rp + r + 1);
        if ((e & 1) && e < ee) {  // peel to a 16-byte-aligned pair boundary
            const int2 cv = load_one<STAGED>(cvb + e);
            float x[R];
            lds_vec<R>(reinterpret_cast<const float*>(xl + cv.x * (TW * 4)), x);
#pragma unroll
            for (int q = 0; q < R; ++q) acc[q] = madd(acc[q], __int_as_float(cv.y), x[q]);
            ++e;
        }
        for (; e + U <= ee; e += U) {
            int2 cv[U];
#pragma unroll
            for (int u = 0; u < U; u += 2) {  // one broadcast LDS.128 per two nonzeros
                const int4 two = load_pair<STAGED>(cvb + e + u);
                cv[u] = make_int2(two.x, two.y);
                cv[u + 1] = make_int2(two.z, two.w);
            }
            float x[U][R];
#pragma unroll
            for (int u = 0; u < U; ++u) lds_vec<R>(reinterpret_cast<const float*>(xl + cv[u].x * (TW * 4)), x[u]);
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int q = 0; q < R; ++q) acc[q] = madd(acc[q], __int_as_float(cv[u].y), x[u][q]);
        }
        if (e + 4 <= ee) {
            int2 cv[4];
#pragma unroll
            for (int u = 0; u < 4; u += 2) {
                const int4 two = load_pair<STAGED>(cvb + e + u);
                cv[u] = make_int2(two.x, two.y);
                cv[u + 1] = make_int2(two.z, two.w);
            }
            float x[4][R];
#pragma unroll
            for (int u = 0; u < 4; ++u) lds_vec<R>(reinterpret_cast<const float*>(xl + cv[u].x * (TW * 4)), x[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int q = 0; q < R; ++q) acc[q] = madd(acc[q], __int_as_float(cv[u].y), x[u][q]);
            e += 4;
        }
        for (; e < ee; ++e) {
            const int2 cv = load_one<STAGED>(cvb + e);
            float x[R];
            lds_vec<R>(reinterpret_cast<const float*>(xl + cv.x * (TW * 4)), x);
#pragma unroll
            for (int q = 0; q < R; ++q) acc[q] = madd(acc[q], __int_as_float(cv.y), x[q]);
        }
        if (tl < NTr) st_vec<R>(yg + (int64_t)r * NTs + tl, acc);
    }
}

// Masked SGD on the CSR values (train.cpp:281-290; L2 term train.cpp:219-223)
__global__ void sgd_kernel(float* __restrict__ vals, const float* __restrict__ grad, int64_t nnz,
                           float lr, float scale, float l2_over_norm) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float v = vals[i];
        const float g = scale * grad[i] + l2_over_norm * v;
        vals[i] = v - lr * g;
    }
}

// Σ v² in fp64 (the layer-wide ‖w‖₂ of train.cpp:225-229), single block for determinism.
__global__ void sumsq_kernel(const float* __restrict__ vals, int64_t nnz, double* __restrict__ out) {
    __shared__ double red[32];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < nnz; i += blockDim.x) {
        const double v = vals[i];
        s += v * v;
    }
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
        if (threadIdx.x == 0) *out = s;
    }
}

// Refresh the value halves of the interleaved SpMM streams from the master CSR values:
// cv[e].y = vals[e], cvT[j].y = vals[perm[j]]
__global__ void refresh_values_kernel(int2* __restrict__ cv, int2* __restrict__ cvT,
                                      const float* __restrict__ vals, const int* __restrict__ perm,
                                      int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        cv[i].y = __float_as_int(vals[i]);
        cvT[i].y = __float_as_int(vals[perm[i]]);
    }
}

// Dense plan: split W[s][k][c] into tf32 hi/lo (rna), both as W and as Wᵀ[s][c][k].
__global__ void split_tf32_kernel(const float* __restrict__ w, float* __restrict__ wh, float* __restrict__ wl,
                                  float* __restrict__ wth, float* __restrict__ wtl, int K, int C, int P2) {
    const int64_t total = (int64_t)P2 * K * C;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float x = w[i];
        uint32_t h, l;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
        const float r = x - __uint_as_float(h);
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(r));
        wh[i] = __uint_as_float(h);
        wl[i] = __uint_as_float(l);
        const int64_t s = i / ((int64_t)K * C), kc = i - s * K * C;
        const int k = (int)(kc / C), c = (int)(kc - (int64_t)k * C);
        const int64_t t = (s * C + c) * K + k;
        wth[t] = __uint_as_float(h);
        wtl[t] = __uint_as_float(l);
    }
}

}  // namespace wino
