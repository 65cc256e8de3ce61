// dW_F = dZ·Ĩ_Fᵀ (layer.cpp:118-128), to the accuracy of the reference's f64 layer, on the int8
// tensor cores.
//
// The reference computes dW_F from f64 Ĩ_F and dZ.  fp32 storage of those operands alone keeps a
// dW_F off the f64 result by more than the strict tolerance (|d| <= 1e-5 + 1e-4·|ref|) on entries
// with heavy cancellation.  So the dW_F operands are NOT the fp32 cache tensors:
// digit kernels recompute Ĩ_F and dZ in f64 (the reference's own f64 coefficients) straight from
// I and dO, and write each value as DIG = 5 balanced base-256 digits (int8):
//     x = 2^(E-38) · m,  m = round(x·2^(38-E)) = Σ_{k<5} d_k·256^k,  d_k ∈ [-128, 127]
// with one exponent E per (segment, slice, row) taken from an a-priori bound: |Ĩ_F(c,·)| <=
// ‖B_i‖₁‖B_j‖₁·max|I(·,c,·,·)| over the segment's images (the max comes from K1 / K4 for free).
// A value keeps 38 bits below its row's bound (~2^-35 of a typical value).
//
// Products: m_a·m_b = Σ_{i,j} d_i e_j 256^(i+j); the 15 digit pairs with i+j >= 4 (weight >=
// 256^4) are formed exactly on tcgen05 kind::i8 into five int32 TMEM accumulators, one per level
// L = i+j-4 (|sum| <= 5·128²·L_cols < 2^31 for chunks of <= kMaxChunkCols columns: exact); the
// 10 pairs below weigh <= 2^-32 of the largest product and are dropped.  A drain combines the
// levels in fp64 and scales by 2^(E_a+E_b-44) exactly.  Measured against the f64 reference the
// result is ~2^-35 of Σ|products| off — the strict bound is met with two orders of margin where
// an fp32-operand dW_F misses it (tools/oz_sim.py reproduces this in numpy).
//
// The GEMM forms the whole K×C product per Winograd coordinate (dense: the int8 MMA rate is far
// above what a masked SIMT product reaches at any density); the surviving entries are gathered in
// CSR order by reduce_sparse_kernel, masked coordinates are never written (train.cpp:281-283).
// Deterministic: fixed digit order, fixed chunk order, no atomics in the values.
//
// Layouts (columns nt = n·T + t, segments padded to KS columns with zero digits):
//   digits  [DIG][P2][R][NTd] int8, R = C (Ĩ_F) or K (dZ)
//   E       [seg][P2][R] int32
//   partial [chunk][P2][K][C] fp64 (already scaled)
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "wino_dense_tc.cuh"
#include "wino_kernels.cuh"

namespace wino {
namespace xdw {

constexpr int DIG = 5;
constexpr int kScaleBits = 38;
// 1.5·2^52 + 0x8080808080: fma(x, 2^(38-E), kMagic) rounds x·2^(38-E) to the integer m and leaves
// m + 0x8080808080 (in [0, 2^40)) in the low 40 bits, whose bytes XOR 0x80 are the digits.
constexpr double kMagic = 6755399441055744.0 + (double)0x8080808080LL;

constexpr int BM = 128;   // UMMA M: rows of dZ (K)
constexpr int BN = 64;    // rows of Ĩ_F (C) per tile: 5 levels x 64 = 320 TMEM columns
constexpr int KS = 64;    // digit columns per stage (one 64-byte swizzled row per operand row)
constexpr int UK = 32;    // K per tcgen05.mma kind::i8
constexpr int STAGES = 3;
constexpr int A_PLANE = BM * KS;              // 8 KB
constexpr int B_PLANE = BN * KS;              // 4 KB
constexpr int A_BYTES = DIG * A_PLANE;        // 40 KB
constexpr int B_BYTES = DIG * B_PLANE;        // 20 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
constexpr int DRAIN_WARPS = 4;
constexpr int THREADS = 64 + 32 * DRAIN_WARPS;
constexpr int TMEM_COLS = 512;
constexpr uint32_t kLayoutSW64 = 4;
constexpr int kMaxChunks = 96;
// per-level |Σ| <= 5 pairs · 128² · cols < 2^31
constexpr int kMaxChunkCols = 26176;
constexpr int kTileItems = 256;  // digit kernels: items per block (one smem transpose)

struct Norms {
    double v[kMaxP * kMaxP];  // ‖row/col of the transform‖₁ products per slice (the exponent bound)
};

struct ChunkTab {
    int n;
    int col0[kMaxChunks];
    int ncols[kMaxChunks];  // multiple of KS
    int seg[kMaxChunks];
};

template <class CF, int M, int P>
__device__ __forceinline__ double coef_ad(const CoefsD& cf, int i) {
    if constexpr (CF::kConst) return BuiltinCoefs<M, P>::AD(i);
    else return cf.a[i];
}
template <class CF, int M, int P>
__device__ __forceinline__ double coef_bd(const CoefsD& cf, int i) {
    if constexpr (CF::kConst) return BuiltinCoefs<M, P>::BD(i);
    else return cf.b[i];
}
template <class CF>
__device__ __forceinline__ double dmadd(double acc, double c, double x) {
    if constexpr (CF::kConst) {
        if (c == 0.0) return acc;
        if (c == 1.0) return acc + x;
        if (c == -1.0) return acc - x;
    }
    return fma(c, x, acc);
}

// smallest E with bound <= 2^E (0 for a zero bound)
__device__ __forceinline__ int bound_exp(double bound) {
    if (!(bound > 0.0)) return 0;
    const int e = (int)((__double_as_longlong(bound) >> 52) & 0x7ff) - 1022;
    return min(e, 1000);
}
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }

// x -> (digits 0..3 as one word, digit 4): the bytes are the int8 digits
__device__ __forceinline__ void to_digits(double x, double scale, uint32_t& lo, uint32_t& hi) {
    const long long b = __double_as_longlong(fma(x, scale, kMagic));
    lo = (uint32_t)b ^ 0x80808080u;
    hi = ((uint32_t)(b >> 32) & 0xffu) ^ 0x80u;
}

// max|x| per (segment, row) of x = [n][R][HW] images: amax[(n / seg_imgs)·R + r] as float bits
// (atomicMax: non-negative floats order as their bits).  One warp per (n, r) plane; the a-priori
// exponent bound of the digits.  For a ReLU-masked dO (train.cpp:193) the callers still pass dO
// itself: max|dO| >= max|dO·mask|, and an upper bound is all the exponent needs.
__global__ void __launch_bounds__(256)
plane_amax_kernel(const float* __restrict__ x, unsigned* __restrict__ amax, int R, int HW, int seg_imgs,
                  int n_planes) {
    const int lane = threadIdx.x & 31;
    for (int pl = blockIdx.x * 8 + (threadIdx.x >> 5); pl < n_planes; pl += gridDim.x * 8) {
        const float* src = x + (int64_t)pl * HW;
        unsigned mx = 0;
        if ((HW & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
            const float4* s4 = reinterpret_cast<const float4*>(src);
#pragma unroll 8
            for (int i = lane; i < (HW >> 2); i += 32) {
                const float4 v = __ldg(s4 + i);
                mx = max(mx, max(max(__float_as_uint(v.x) & 0x7fffffffu, __float_as_uint(v.y) & 0x7fffffffu),
                                 max(__float_as_uint(v.z) & 0x7fffffffu, __float_as_uint(v.w) & 0x7fffffffu)));
            }
        } else {
#pragma unroll 4
            for (int i = lane; i < HW; i += 32) mx = max(mx, __float_as_uint(__ldg(src + i)) & 0x7fffffffu);
        }
        mx = __reduce_max_sync(0xffffffffu, mx);
        const int n = pl / R, r = pl - n * R;
        if (lane == 0) atomicMax(amax + (int64_t)(n / seg_imgs) * R + r, mx);
    }
}

// Shared-memory staging of the digits: [P2][kTileItems] words (digits 0..3) + [P2][kTileItems]
// bytes (digit 4) + the P2 per-slice scales.
template <int P2>
constexpr int digit_smem_bytes() {
    return P2 * kTileItems * 5 + P2 * 8;
}

// Per-block prologue: the scale 2^(38-E) of each slice from the row's segment maximum (E written
// once per (slice, row) by the row's first column block).
__device__ __forceinline__ void slice_scales(double* ssc, const Norms& nrm, int P2, const unsigned* amax, int row,
                                             int R, int* Eout) {
    if ((int)threadIdx.x < P2) {
        const double amx = (double)__uint_as_float(__ldg(amax + row));
        const int E = bound_exp(nrm.v[threadIdx.x] * amx);
        ssc[threadIdx.x] = pow2(kScaleBits - E);
        if (blockIdx.x == 0) Eout[threadIdx.x * R + row] = E;
    }
}

// Block-wide copy-out of the staged digits of row `row`, block columns [jb, jb + kTileItems)
// (only those < ncols_pad): four columns of one slice per thread and step -> one u32 per plane.
__device__ __forceinline__ void store_digit_rows(const uint32_t* slo, const uint8_t* shi, int P2, int R, int row,
                                                 int jb, int ncols_pad, int8_t* __restrict__ dig, int64_t NTd,
                                                 int64_t plane, int col0) {
    constexpr int G = kTileItems / 4;
    for (int idx = threadIdx.x; idx < P2 * G; idx += kTileItems) {
        const int s = idx / G, g = idx - s * G;
        const int col = jb + 4 * g;
        if (col >= ncols_pad) continue;
        const uint4 w = *reinterpret_cast<const uint4*>(slo + s * kTileItems + 4 * g);
        const uint32_t h = *reinterpret_cast<const uint32_t*>(shi + s * kTileItems + 4 * g);
        const uint32_t t01 = __byte_perm(w.x, w.y, 0x5140), t23 = __byte_perm(w.z, w.w, 0x5140);
        const uint32_t u01 = __byte_perm(w.x, w.y, 0x7362), u23 = __byte_perm(w.z, w.w, 0x7362);
        int8_t* dst = dig + ((int64_t)s * R + row) * NTd + col0 + col;
        *reinterpret_cast<uint32_t*>(dst) = __byte_perm(t01, t23, 0x5410);
        *reinterpret_cast<uint32_t*>(dst + plane) = __byte_perm(t01, t23, 0x7632);
        *reinterpret_cast<uint32_t*>(dst + 2 * plane) = __byte_perm(u01, u23, 0x5410);
        *reinterpret_cast<uint32_t*>(dst + 3 * plane) = __byte_perm(u01, u23, 0x7632);
        *reinterpret_cast<uint32_t*>(dst + 4 * plane) = h;
    }
}

// K1 fused with the Ĩ_F digits of one exponent segment.  Grid (column blocks, C): c = blockIdx.y,
// segment column j = n·T + t (`in` and V offset to the segment's first image).  From one φ gather:
//   V(s, c, j)      fp32, bitwise K1 (the reference's f32 order, transforms.cpp:196-210), j < vcols
//                   (columns >= ncols are the batch's zero padding);
//   digits(s, c, j) the reference's f64 B1ᵀ·d·B2 (layer.cpp:55-59) as DIG digits, j < ncols_pad.
// Row i of both products at a time keeps the working set at d plus one row.
template <int M, int P, class CF>
__global__ void __launch_bounds__(kTileItems, (P <= 6) ? 2 : 1)
input_transform_digits_kernel(const float* __restrict__ in, float* __restrict__ V, int8_t* __restrict__ dig,
                              int* __restrict__ Eout, const unsigned* __restrict__ amax, const Coefs cf,
                              const CoefsD cfd, const Norms nrm, int C, int H, int W, int pad, int tiles_x, int T,
                              int ncols, int vcols, int ncols_pad, int64_t NTs, int64_t NTd, int64_t plane,
                              int col0, int pf) {
    constexpr int P2 = P * P;
    extern __shared__ __align__(16) uint32_t xdw_smem[];
    uint32_t* slo = xdw_smem;
    uint8_t* shi = reinterpret_cast<uint8_t*>(xdw_smem + P2 * kTileItems);
    double* ssc = reinterpret_cast<double*>(shi + P2 * kTileItems);
    const int c = blockIdx.y;
    const int jb = blockIdx.x * kTileItems;
    const int j = jb + threadIdx.x;
    slice_scales(ssc, nrm, P2, amax, c, C, Eout);
    float d[P][P];
    if (j < ncols) {
        const int n = j / T, t = j - n * T;
        const int ty = t / tiles_x, tx = t - ty * tiles_x;
        const int y0 = ty * M - pad, x0 = tx * M - pad;
        const float* src = in + ((int64_t)n * C + c) * H * W;
        if (M == 4 && P == 6 && pad == 1 && (W & 3) == 0) {
            // row i of the patch = x0 - 0 .. x0 + 5 = 4tx-1 | 4tx .. 4tx+3 (one aligned 16-byte
            // load, always inside the row) | 4tx+4
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
                    for (int k = 0; k < P; ++k) d[i][k] = 0.f;
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < P; ++i) {
                const int y = y0 + i;
                const bool yok = (unsigned)y < (unsigned)H;
#pragma unroll
                for (int k = 0; k < P; ++k) {
                    const int x = x0 + k;
                    d[i][k] = (yok && (unsigned)x < (unsigned)W) ? __ldg(src + y * W + x) : 0.f;
                }
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
            for (int k = 0; k < P; ++k) d[i][k] = 0.f;
    }
    // The gather is this kernel's exposed latency (2 blocks per SM): pull the patch rows of the
    // block that will run one resident wave of blocks later (launch order, x fastest) into L2 now,
    // behind this block's own loads.
    if (pf > 0) {  // pf = (blocks ahead / gridDim.x) << 16 | (blocks ahead % gridDim.x): no division here
        int pbx = (int)blockIdx.x + (pf & 0xffff), pc = (int)blockIdx.y + (pf >> 16);
        if (pbx >= (int)gridDim.x) pbx -= gridDim.x, ++pc;
        const int pj = pbx * kTileItems + threadIdx.x;
        if (pc < (int)gridDim.y && pj < ncols) {
            const int n = pj / T, t = pj - n * T;
            const int ty = t / tiles_x, tx = t - ty * tiles_x;
            const int y0 = ty * M - pad, x0 = max(tx * M - pad, 0);
            const float* src = in + ((int64_t)n * C + pc) * H * W + x0;
#pragma unroll
            for (int i = 0; i < P; ++i)
                if ((unsigned)(y0 + i) < (unsigned)H) asm volatile("prefetch.global.L2 [%0];" ::"l"(src + (y0 + i) * W));
        }
    }
    __syncthreads();  // scales
    const bool vok = j < vcols;
    float* vp = V + (int64_t)c * NTs + j;
    const int64_t vplane = (int64_t)C * NTs;
#pragma unroll
    for (int i = 0; i < P; ++i) {
        float t32[P];
#pragma unroll
        for (int l = 0; l < P; ++l) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < P; ++k) acc = cmadd<CF>(acc, coef_b<CF, M, P>(cf, k * P + i), d[k][l]);
            t32[l] = acc;
        }
#pragma unroll
        for (int l = 0; l < P; ++l) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < P; ++k) acc = cmadd<CF>(acc, coef_b<CF, M, P>(cf, k * P + l), t32[k]);
            if (vok) *vp = acc;
            vp += vplane;
        }
        double t64[P];
#pragma unroll
        for (int l = 0; l < P; ++l) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < P; ++k) acc = dmadd<CF>(acc, coef_bd<CF, M, P>(cfd, k * P + i), (double)d[k][l]);
            t64[l] = acc;
        }
#pragma unroll
        for (int l = 0; l < P; ++l) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < P; ++k) acc = dmadd<CF>(acc, coef_bd<CF, M, P>(cfd, k * P + l), t64[k]);
            const int s = i * P + l;
            uint32_t lo, hi;
            to_digits(acc, ssc[s], lo, hi);
            slo[s * kTileItems + threadIdx.x] = lo;
            shi[s * kTileItems + threadIdx.x] = (uint8_t)hi;
        }
    }
    __syncthreads();
    store_digit_rows(slo, shi, P2, C, c, jb, ncols_pad, dig, NTd, plane, col0);
}

// K4 fused with the dZ digits of one exponent segment (grid (column blocks, K), k = blockIdx.y):
// the ψ⁻¹ gather of dO (zero at padded positions, optional ReLU mask, train.cpp:193), then
//   DZ(s, k, j)     fp32 A1·dÕ·A2ᵀ, bitwise the reference's f32 order (layer.cpp:107-116), j < vcols;
//   digits(s, k, j) the same product in the reference's f64, j < ncols_pad.
template <int M, int P, bool MASK, class CF>
__global__ void __launch_bounds__(kTileItems, (P <= 6) ? 2 : 1)
grad_z_digits_kernel(const float* __restrict__ dO, const float* __restrict__ relu_out, float* __restrict__ DZ,
                     int8_t* __restrict__ dig, int* __restrict__ Eout, const unsigned* __restrict__ amax,
                     const Coefs cf, const CoefsD cfd, const Norms nrm, int K, int Ho, int Wo, int tiles_x, int T,
                     int ncols, int vcols, int ncols_pad, int64_t NTs, int64_t NTd, int64_t plane, int col0,
                     int pf) {
    constexpr int P2 = P * P;
    extern __shared__ __align__(16) uint32_t xdw_smem[];
    uint32_t* slo = xdw_smem;
    uint8_t* shi = reinterpret_cast<uint8_t*>(xdw_smem + P2 * kTileItems);
    double* ssc = reinterpret_cast<double*>(shi + P2 * kTileItems);
    const int k = blockIdx.y;
    const int jb = blockIdx.x * kTileItems;
    const int j = jb + threadIdx.x;
    slice_scales(ssc, nrm, P2, amax, k, K, Eout);
    float d[M][M];
#pragma unroll
    for (int y = 0; y < M; ++y)
#pragma unroll
        for (int x = 0; x < M; ++x) d[y][x] = 0.f;
    if (j < ncols) {
        const int n = j / T, t = j - n * T;
        const int ty = t / tiles_x, tx = t - ty * tiles_x;
        const int64_t base = ((int64_t)n * K + k) * Ho * Wo;
        const bool al16 = ((reinterpret_cast<uintptr_t>(dO) | (MASK ? reinterpret_cast<uintptr_t>(relu_out) : 0)) & 15) == 0;
        if (M == 4 && (Wo & 3) == 0 && al16 && ty * M + M <= Ho) {
            // whole tile inside the image, 16-byte-aligned rows: one load per tile row
#pragma unroll
            for (int y = 0; y < M; ++y) {
                const int64_t o = base + (ty * M + y) * Wo + tx * M;
                float4 v = __ldg(reinterpret_cast<const float4*>(dO + o));
                if (MASK) {
                    const float4 r = __ldg(reinterpret_cast<const float4*>(relu_out + o));
                    v.x = __fmul_rn(v.x, r.x > 0.f ? 1.f : 0.f);
                    v.y = __fmul_rn(v.y, r.y > 0.f ? 1.f : 0.f);
                    v.z = __fmul_rn(v.z, r.z > 0.f ? 1.f : 0.f);
                    v.w = __fmul_rn(v.w, r.w > 0.f ? 1.f : 0.f);
                }
                d[y][0] = v.x;
                d[y][1] = v.y;
                d[y][2] = v.z;
                d[y][3] = v.w;
            }
        } else {
#pragma unroll
            for (int y = 0; y < M; ++y) {
                const int oy = ty * M + y;
#pragma unroll
                for (int x = 0; x < M; ++x) {
                    const int ox = tx * M + x;
                    if (oy < Ho && ox < Wo) {
                        const int64_t o = base + oy * Wo + ox;
                        float v = __ldg(dO + o);
                        if (MASK) v = __fmul_rn(v, __ldg(relu_out + o) > 0.f ? 1.f : 0.f);
                        d[y][x] = v;
                    }
                }
            }
        }
    }
    if (pf > 0) {  // the dO rows of the block `pf` blocks ahead -> L2 (as in K1; pf packed likewise)
        int pbx = (int)blockIdx.x + (pf & 0xffff), pk = (int)blockIdx.y + (pf >> 16);
        if (pbx >= (int)gridDim.x) pbx -= gridDim.x, ++pk;
        const int pj = pbx * kTileItems + threadIdx.x;
        if (pk < (int)gridDim.y && pj < ncols) {
            const int n = pj / T, t = pj - n * T;
            const int ty = t / tiles_x, tx = t - ty * tiles_x;
            const int64_t o = ((int64_t)n * K + pk) * Ho * Wo + (int64_t)(ty * M) * Wo + min(tx * M, Wo - 1);
#pragma unroll
            for (int y = 0; y < M; ++y)
                if (ty * M + y < Ho) {
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(dO + o + y * Wo));
                    if (MASK) asm volatile("prefetch.global.L2 [%0];" ::"l"(relu_out + o + y * Wo));
                }
        }
    }
    __syncthreads();  // scales
    const bool vok = j < vcols;
    float* zp = DZ + (int64_t)k * NTs + j;
    const int64_t zplane = (int64_t)K * NTs;
#pragma unroll
    for (int i = 0; i < P; ++i) {
        float m32[M];  // row i of A1·dÕ
#pragma unroll
        for (int x = 0; x < M; ++x) {
            float acc = 0.f;
#pragma unroll
            for (int y = 0; y < M; ++y) acc = cmadd<CF>(acc, coef_a<CF, M, P>(cf, i * M + y), d[y][x]);
            m32[x] = acc;
        }
#pragma unroll
        for (int l = 0; l < P; ++l) {
            float acc = 0.f;
#pragma unroll
            for (int x = 0; x < M; ++x) acc = cmadd<CF>(acc, coef_a<CF, M, P>(cf, l * M + x), m32[x]);
            if (vok) *zp = acc;
            zp += zplane;
        }
        double m64[M];
#pragma unroll
        for (int x = 0; x < M; ++x) {
            double acc = 0.0;
#pragma unroll
            for (int y = 0; y < M; ++y) acc = dmadd<CF>(acc, coef_ad<CF, M, P>(cfd, i * M + y), (double)d[y][x]);
            m64[x] = acc;
        }
#pragma unroll
        for (int l = 0; l < P; ++l) {
            double acc = 0.0;
#pragma unroll
            for (int x = 0; x < M; ++x) acc = dmadd<CF>(acc, coef_ad<CF, M, P>(cfd, l * M + x), m64[x]);
            const int s = i * P + l;
            uint32_t lo, hi;
            to_digits(acc, ssc[s], lo, hi);
            slo[s * kTileItems + threadIdx.x] = lo;
            shi[s * kTileItems + threadIdx.x] = (uint8_t)hi;
        }
    }
    __syncthreads();
    store_digit_rows(slo, shi, P2, K, k, jb, ncols_pad, dig, NTd, plane, col0);
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
        "[%2];" ::"r"(tc::smem_u32(dst)),
        "l"((uint64_t)map), "r"(tc::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

// D = S32 (bits 4-5 = 2), A = B = signed 8-bit (bits 7-9, 10-12 = 1), both K-major, N>>3, M>>4
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

// exact int32 -> fp64 on the FP64 pipe (no XU conversion)
__device__ __forceinline__ double i2d(uint32_t v) {
    return __hiloint2double(0x43300000, (int)(v ^ 0x80000000u)) - 4503601774854144.0;
}

// part[ch][s][m][n] = Σ_{t ∈ chunk} dZ(s,m,t)·Ĩ_F(s,n,t) from the digit tensors.  Persistent,
// warp-specialised: warp 0 TMA (5 A and 5 B digit planes of a 64-column stage in two 4-D boxes),
// warp 1 TMEM allocation + MMA issue, 4 drain warps.  Per 32-column step the 15 digit pairs run
// as 6 MMAs: the B planes are stacked along N in shared memory, so A plane i multiplies the
// contiguous planes 4-i..4 at once and each plane's product lands in its own level's columns.
__global__ void __launch_bounds__(THREADS, 1)
gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
            const __grid_constant__ ChunkTab ct, const int* __restrict__ EA, const int* __restrict__ EB,
            double* __restrict__ part, int P2, int M, int N, int tiles_m, int tiles_n, int nunits) {
    extern __shared__ uint8_t xdw_gemm_smem[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(xdw_gemm_smem) + 1023) & ~(uintptr_t)1023);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* full = bars;
    uint64_t* empty = bars + STAGES;
    uint64_t* tfull = bars + 2 * STAGES;
    uint64_t* tempty = bars + 2 * STAGES + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto decode = [&](int u, int& ch, int& s, int& mt, int& nt) {
        nt = u % tiles_n;
        int r = u / tiles_n;
        mt = r % tiles_m;
        r /= tiles_m;
        s = r % P2;
        ch = r / P2;
    };
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&empty[i], 1);
        }
        tc::mbar_init(tfull, 1);
        tc::mbar_init(tempty, 32 * DRAIN_WARPS);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         tc::smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int g = 0;
            for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
                int ch, s, mt, nt;
                decode(u, ch, s, mt, nt);
                const int nk = ct.ncols[ch] / KS;
                for (int kb = 0; kb < nk; ++kb, ++g) {
                    const int st = g % STAGES;
                    if (g >= STAGES) tc::mbar_wait(&empty[st], ((g / STAGES) - 1) & 1);
                    uint8_t* base = smem + st * STAGE_BYTES;
                    tc::mbar_expect_tx(&full[st], STAGE_BYTES);
                    const int col = ct.col0[ch] + kb * KS;
                    tma_load_4d(base, &mapA, &full[st], col, mt * BM, s, 0);
                    tma_load_4d(base + A_BYTES, &mapB, &full[st], col, nt * BN, s, 0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int g = 0, it = 0;
            for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
                int ch, s, mt, nt;
                decode(u, ch, s, mt, nt);
                const int nk = ct.ncols[ch] / KS;
                if (it > 0) tc::mbar_wait(tempty, (it - 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (int kb = 0; kb < nk; ++kb, ++g) {
                    const int st = g % STAGES;
                    tc::mbar_wait(&full[st], (g / STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t a0 = tc::smem_u32(smem + st * STAGE_BYTES);
                    const uint32_t b0 = a0 + A_BYTES;
                    const uint64_t da = tc::make_desc(a0, 16, 512, kLayoutSW64);
                    const uint64_t db = tc::make_desc(b0, 16, 512, kLayoutSW64);
#pragma unroll
                    for (int sub = 0; sub < KS / UK; ++sub) {
                        const uint32_t acc = (kb | sub) ? 1u : 0u;
                        const uint64_t ko = (uint64_t)((sub * UK) >> 4);
                        // A plane 4 x B planes 0..3 (levels 0..3) and x B plane 4 (level 4)
                        mma_i8(tmem, da + ko + (uint64_t)((4 * A_PLANE) >> 4), db + ko, idesc_i8(256), acc);
                        mma_i8(tmem + 256, da + ko + (uint64_t)((4 * A_PLANE) >> 4),
                               db + ko + (uint64_t)((4 * B_PLANE) >> 4), idesc_i8(64), acc);
#pragma unroll
                        for (int i = 3; i >= 0; --i)  // A plane i x B planes 4-i..4 -> levels 0..i
                            mma_i8(tmem, da + ko + (uint64_t)((i * A_PLANE) >> 4),
                                   db + ko + (uint64_t)(((4 - i) * B_PLANE) >> 4), idesc_i8((i + 1) * BN), 1u);
                    }
                    tc::mma_commit(&empty[st]);
                }
                tc::mma_commit(tfull);
            }
        }
    } else {
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        int it = 0;
        for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
            int ch, s, mt, nt;
            decode(u, ch, s, mt, nt);
            const int seg = ct.seg[ch];
            const int row = mt * BM + q * 32 + lane;
            const bool rok = row < M;
            const int ea = rok ? __ldg(EA + ((int64_t)seg * P2 + s) * M + row) : 0;
            const int* eb = EB + ((int64_t)seg * P2 + s) * N;
            double* dst = part + (((int64_t)ch * P2 + s) * M + (rok ? row : 0)) * N;
            tc::mbar_wait(tfull, it & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
            for (int blk = 0; blk < BN / 16; ++blk) {
                uint32_t v[DIG][16];
#pragma unroll
                for (int L = 0; L < DIG; ++L) tc::tmem_ld16(ta + (uint32_t)(L * BN + blk * 16), v[L]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (blk == BN / 16 - 1) {  // accumulators free once the last columns are in registers
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    tc::mbar_arrive(tempty);
                }
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) {
                    const int col = nt * BN + blk * 16 + jj;
                    double t = i2d(v[0][jj]);
                    t = fma(i2d(v[1][jj]), 256.0, t);
                    t = fma(i2d(v[2][jj]), 65536.0, t);
                    t = fma(i2d(v[3][jj]), 16777216.0, t);
                    t = fma(i2d(v[4][jj]), 4294967296.0, t);
                    if (rok && col < N) dst[col] = t * pow2(ea + __ldg(eb + col) - 44);
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

// dW_F on the mask, CSR order: grid (blocks, P2), slice s covers entries [off[s], off[s+1]).
__global__ void reduce_sparse_kernel(const double* __restrict__ part, float* __restrict__ dw,
                                     const int* __restrict__ rowof, const int* __restrict__ colidx,
                                     const int64_t* __restrict__ off, int K, int C, int P2, int nchunks,
                                     int64_t nnz) {
    const int s = blockIdx.y;
    const int64_t e0 = off[s], e1 = s + 1 < P2 ? off[s + 1] : nnz;
    const int64_t cstride = (int64_t)P2 * K * C;
    const double* plane = part + (int64_t)s * K * C;
    for (int64_t e = e0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < e1;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = (int64_t)__ldg(rowof + e) * C + __ldg(colidx + e);
        double a = 0.0;
        for (int ch = 0; ch < nchunks; ++ch) a += plane[ch * cstride + o];
        dw[e] = (float)a;
    }
}

// dense plan: dW_F in the reference's K×C×p×q layout
__global__ void reduce_dense_kernel(const double* __restrict__ part, float* __restrict__ dw, int K, int C, int P2,
                                    int nchunks) {
    const int64_t total = (int64_t)P2 * K * C;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t kc = i / P2;
        const int s = (int)(i - kc * P2);
        const double* src = part + (int64_t)s * K * C + kc;
        double a = 0.0;
        for (int ch = 0; ch < nchunks; ++ch) a += src[ch * total];
        dw[i] = (float)a;
    }
}

}  // namespace xdw
}  // namespace wino
