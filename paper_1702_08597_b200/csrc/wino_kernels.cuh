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

// ---------------------------------------------------------------------------------
// K1: φ gather (pad folded in) + Ĩ_F = B1ᵀ·d·B2   (transforms.cpp:196-210, sparse.cpp:94-120)
// One thread per (c, nt); consecutive threads = consecutive tiles -> coalesced stores.
// ---------------------------------------------------------------------------------
template <int M, int P>
__global__ void __launch_bounds__(256)
input_transform_kernel(const float* __restrict__ in, float* __restrict__ V, const Coefs cf, int C,
                       int H, int W, int pad, int tiles_x, int T, int NT, int NTs) {
    const int64_t plane = (int64_t)C * NTs;
    for (int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < plane;
         gid += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(gid / NTs);
        const int nt = (int)(gid - (int64_t)c * NTs);
        float d[P][P];
        if (nt < NT) {
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
                    d[i][j] = (yok && (unsigned)x < (unsigned)W) ? __ldg(src + y * W + x) : 0.f;
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
                for (int k = 0; k < P; ++k) acc = madd(acc, cf.b[k * P + i], d[k][j]);
                tmp[i][j] = acc;
            }
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
            for (int j = 0; j < P; ++j) {
                float acc = 0.f;
#pragma unroll
                for (int k = 0; k < P; ++k) acc = madd(acc, cf.b[k * P + j], tmp[i][k]);
                V[(int64_t)(i * P + j) * plane + gid] = acc;
            }
    }
}

// ---------------------------------------------------------------------------------
// K3: O = ψ(A1ᵀ·Z·A2), crop, optional ReLU   (sparse.cpp:151-184; layer.cpp:79-95)
// One thread per (k, nt): 36 coalesced loads, 16 outputs.
// ---------------------------------------------------------------------------------
template <int M, int P, bool RELU>
__global__ void __launch_bounds__(256)
output_transform_kernel(const float* __restrict__ Z, float* __restrict__ O, const Coefs cf, int K,
                        int Ho, int Wo, int tiles_x, int T, int NT, int NTs) {
    const int64_t total = (int64_t)K * NT;
    const int64_t plane = (int64_t)K * NTs;
    for (int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < total;
         gid += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(gid / NT);
        const int nt = (int)(gid - (int64_t)k * NT);
        const float* zp = Z + (int64_t)k * NTs + nt;
        float z[P][P];
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
            for (int j = 0; j < P; ++j) z[i][j] = __ldg(zp + (int64_t)(i * P + j) * plane);
        float tmp[M][P];
#pragma unroll
        for (int y = 0; y < M; ++y)
#pragma unroll
            for (int j = 0; j < P; ++j) {
                float acc = 0.f;
#pragma unroll
                for (int i = 0; i < P; ++i) acc = madd(acc, cf.a[i * M + y], z[i][j]);
                tmp[y][j] = acc;
            }
        const int n = nt / T, t = nt - n * T;
        const int ty = t / tiles_x, tx = t - ty * tiles_x;
        float* op = O + ((int64_t)n * K + k) * Ho * Wo;
#pragma unroll
        for (int y = 0; y < M; ++y) {
            const int oy = ty * M + y;
#pragma unroll
            for (int x = 0; x < M; ++x) {
                float acc = 0.f;
#pragma unroll
                for (int j = 0; j < P; ++j) acc = madd(acc, cf.a[j * M + x], tmp[y][j]);
                if (RELU) acc = acc > 0.f ? acc : 0.f;  // train.cpp:76-83
                const int ox = tx * M + x;
                if (oy < Ho && ox < Wo) op[oy * Wo + ox] = acc;
            }
        }
    }
}

// ---------------------------------------------------------------------------------
// K4: dZ = A1·dÕ·A2ᵀ with ψ⁻¹ gather, zero at padded positions, optional ReLU mask
//     (layer.cpp:107-116, transforms.cpp:228-241, train.cpp:193)
// One thread per (k, nt < NTs); padding columns nt ≥ NT are written as zeros.
// ---------------------------------------------------------------------------------
template <int M, int P, bool MASK>
__global__ void __launch_bounds__(256)
grad_z_kernel(const float* __restrict__ dO, const float* __restrict__ relu_out,
              float* __restrict__ DZ, const Coefs cf, int K, int Ho, int Wo, int tiles_x, int T,
              int NT, int NTs) {
    const int64_t plane = (int64_t)K * NTs;
    for (int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < plane;
         gid += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(gid / NTs);
        const int nt = (int)(gid - (int64_t)k * NTs);
        float d[M][M];
        if (nt < NT) {
            const int n = nt / T, t = nt - n * T;
            const int ty = t / tiles_x, tx = t - ty * tiles_x;
            const int64_t base = ((int64_t)n * K + k) * Ho * Wo;
#pragma unroll
            for (int y = 0; y < M; ++y) {
                const int oy = ty * M + y;
#pragma unroll
                for (int x = 0; x < M; ++x) {
                    const int ox = tx * M + x;
                    float v = 0.f;
                    if (oy < Ho && ox < Wo) {
                        const int64_t o = base + oy * Wo + ox;
                        v = __ldg(dO + o);
                        if (MASK) v = __fmul_rn(v, __ldg(relu_out + o) > 0.f ? 1.f : 0.f);
                    }
                    d[y][x] = v;
                }
            }
        } else {
#pragma unroll
            for (int y = 0; y < M; ++y)
#pragma unroll
                for (int x = 0; x < M; ++x) d[y][x] = 0.f;
        }
        float m1[P][M];  // m1(i,x) = Σ_y a1(i,y)·d(y,x)
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
            for (int x = 0; x < M; ++x) {
                float acc = 0.f;
#pragma unroll
                for (int y = 0; y < M; ++y) acc = madd(acc, cf.a[i * M + y], d[y][x]);
                m1[i][x] = acc;
            }
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
            for (int j = 0; j < P; ++j) {  // dz(i,j) = Σ_x m1(i,x)·a2(j,x)
                float acc = 0.f;
#pragma unroll
                for (int x = 0; x < M; ++x) acc = madd(acc, cf.a[j * M + x], m1[i][x]);
                DZ[(int64_t)(i * P + j) * plane + gid] = acc;
            }
    }
}

// ---------------------------------------------------------------------------------
// K7: dI = Σ_φ B1·dĨ_F·B2ᵀ — fused B-transform + deterministic halo gather-sum
//     (layer.cpp:157-169).  Block = (image n, group of CG channels).  Phase 1 writes the
//     transformed tiles of the group to shared memory; phase 2 gives every input pixel
//     its ≤⌈p/m⌉² contributions in ascending t order from +0 (the reference's
//     accumulation order), so no atomics and the result is bitwise deterministic.
// ---------------------------------------------------------------------------------
template <int M, int P>
__device__ __forceinline__ float tile_grad_entry(const float* __restrict__ dv, int64_t plane,
                                                 const Coefs& cf, int i, int j) {
    // g(i,j) with m1(i,l) = Σ_k b1(i,k)·x(k,l) ; g(i,j) = Σ_l m1(i,l)·b2(j,l)
    float acc = 0.f;
#pragma unroll
    for (int l = 0; l < P; ++l) {
        float m = 0.f;
#pragma unroll
        for (int k = 0; k < P; ++k) m = madd(m, cf.b[i * P + k], __ldg(dv + (int64_t)(k * P + l) * plane));
        acc = madd(acc, cf.b[j * P + l], m);
    }
    return acc;
}

template <int M, int P>
__global__ void __launch_bounds__(256)
input_grad_kernel(const float* __restrict__ DV, float* __restrict__ dI, const Coefs cf, int C,
                  int H, int W, int pad, int tiles_y, int tiles_x, int T, int NTs, int CG) {
    extern __shared__ float gsm[];  // [CG][T][P*P]
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
            for (int l = 0; l < P; ++l) x[k][l] = __ldg(src + (int64_t)(k * P + l) * plane);
        float m1[P][P];
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
            for (int l = 0; l < P; ++l) {
                float acc = 0.f;
#pragma unroll
                for (int k = 0; k < P; ++k) acc = madd(acc, cf.b[i * P + k], x[k][l]);
                m1[i][l] = acc;
            }
        float* g = gsm + (int64_t)idx * P * P;
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
            for (int j = 0; j < P; ++j) {
                float acc = 0.f;
#pragma unroll
                for (int l = 0; l < P; ++l) acc = madd(acc, cf.b[j * P + l], m1[i][l]);
                g[i * P + j] = acc;
            }
    }
    __syncthreads();
    const int HW = H * W;
    for (int idx = threadIdx.x; idx < CG * HW; idx += blockDim.x) {
        const int cl = idx / HW, pix = idx - cl * HW;
        const int c = c0 + cl;
        if (c >= C) continue;
        const int y = pix / W, x = pix - y * W;
        const int Y = y + pad, X = x + pad;
        const int ty_lo = Y - P + 1 <= 0 ? 0 : (Y - P + M) / M;
        const int ty_hi = min(tiles_y - 1, Y / M);
        const int tx_lo = X - P + 1 <= 0 ? 0 : (X - P + M) / M;
        const int tx_hi = min(tiles_x - 1, X / M);
        float acc = 0.f;
        for (int ty = ty_lo; ty <= ty_hi; ++ty)
            for (int tx = tx_lo; tx <= tx_hi; ++tx) {
                const int t = ty * tiles_x + tx;
                acc = __fadd_rn(acc, gsm[((int64_t)cl * T + t) * P * P + (Y - ty * M) * P + (X - tx * M)]);
            }
        dI[((int64_t)n * C + c) * HW + pix] = acc;
    }
}

// Same result without shared-memory staging (large T): each pixel recomputes the
// transformed-tile entries it needs (identical operation order, hence identical bits).
template <int M, int P>
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
                acc = __fadd_rn(acc, tile_grad_entry<M, P>(src, plane, cf, Y - ty * M, X - tx * M));
            }
        dI[gid] = acc;
    }
}

// ---------------------------------------------------------------------------------
// K2 / K6: CSR SpMM, one p·q slice per blockIdx.z:  Y(r,:) = Σ_{e∈row r} v_e·X(col_e,:)
//   forward   : rows = K, X = Ĩ_F, CSR of W_F(:,:,i,j)       (sparse.cpp:51-69)
//   backward  : rows = C, X = dZ,  CSR of W_F(:,:,i,j)ᵀ (CSC)  (layer.cpp:145-155 on the mask)
// Block = (TW-wide tile-column chunk, row group, slice).  The chunk X(:, chunk) of every
// input row is staged in shared memory with 16-byte loads; a warp owns a row, each lane
// R consecutive columns, so a nonzero costs one broadcast of (col, v) and one
// conflict-free LDS.{32,64,128}.  Accumulation follows the CSR order from +0.
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

// Stage X[0..nrows_x)[t0 .. t0+TW) (row stride NTs, NTs % 4 == 0) into xs[nrows_x][TW].
template <int TW>
__device__ __forceinline__ void stage_rows(const float* __restrict__ X, float* xs, int nrows_x,
                                           int NTs, int t0) {
    constexpr int V4 = TW / 4;
    for (int idx = threadIdx.x; idx < nrows_x * V4; idx += blockDim.x) {
        const int row = idx / V4, q = idx - row * V4;
        const int t = t0 + q * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (t < NTs) v = __ldg(reinterpret_cast<const float4*>(X + (int64_t)row * NTs + t));
        *reinterpret_cast<float4*>(xs + row * TW + q * 4) = v;
    }
}

template <int R>
__global__ void __launch_bounds__(256)
spmm_kernel(const int* __restrict__ rowptr, const int* __restrict__ colidx,
            const float* __restrict__ vals, const float* __restrict__ X, float* __restrict__ Y,
            int nrows, int ncols, int NTs, int rows_per_block) {
    constexpr int TW = 32 * R;
    extern __shared__ float4 smem_f4[];
    float* xs = reinterpret_cast<float*>(smem_f4);
    const int s = blockIdx.z;
    const int t0 = blockIdx.x * TW;
    const int r0 = blockIdx.y * rows_per_block;
    const int r1 = min(nrows, r0 + rows_per_block);
    stage_rows<TW>(X + (int64_t)s * ncols * NTs, xs, ncols, NTs, t0);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int* rp = rowptr + (int64_t)s * (nrows + 1);
    float* yg = Y + (int64_t)s * nrows * NTs;
    const int tl = t0 + lane * R;
    for (int r = r0 + warp; r < r1; r += nw) {
        float acc[R];
#pragma unroll
        for (int q = 0; q < R; ++q) acc[q] = 0.f;
        const int e0 = __ldg(rp + r), e1 = __ldg(rp + r + 1);
        for (int eb = e0; eb < e1; eb += 32) {
            const int e = eb + lane;
            int cl = 0;
            float vl = 0.f;
            if (e < e1) {
                cl = __ldg(colidx + e);
                vl = __ldg(vals + e);
            }
            const int cnt = min(32, e1 - eb);
            for (int j = 0; j < cnt; ++j) {
                const int c = __shfl_sync(kFull, cl, j);
                const float v = __shfl_sync(kFull, vl, j);
                float x[R];
                lds_vec<R>(xs + c * TW + lane * R, x);
#pragma unroll
                for (int q = 0; q < R; ++q) acc[q] = madd(acc[q], v, x[q]);
            }
        }
        if (tl < NTs) st_vec<R>(yg + (int64_t)r * NTs + tl, acc);
    }
}

// ---------------------------------------------------------------------------------
// K5: masked SDDMM  dW(e=(k,c)) = Σ_t dZ(k,t)·Ĩ_F(c,t)  for surviving (k,c) only
//     (layer.cpp:118-128 restricted to the mask; masked coordinates are never updated,
//     train.cpp:281-283).  Block = (row group, slice), looping over t-chunks of TW.
//     Per chunk Ĩ_F(:, chunk) and dZ(rows, chunk) are staged in shared memory; a warp
//     takes 32 consecutive nonzeros, every lane forms the 32 partial dot products over
//     its R columns, and a 31-shuffle transpose-reduction leaves lane j with nonzero j's
//     chunk sum, which is added to an fp64 accumulator in shared memory (deterministic:
//     each nonzero has one owner, chunks are summed in ascending t).
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void transpose_reduce32(float (&v)[32], int lane) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool hi = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const float send = hi ? v[i] : v[i + o];
            const float keep = hi ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(kFull, send, o);
        }
    }
}

template <int R>
__global__ void __launch_bounds__(256)
sddmm_kernel(const int* __restrict__ rowptr, const int* __restrict__ colidx,
             const int* __restrict__ rowof, const float* __restrict__ DZ,
             const float* __restrict__ V, float* __restrict__ dW, int K, int C, int NT, int NTs,
             int rows_per_block) {
    constexpr int TW = 32 * R;
    extern __shared__ float4 smem_f4[];
    const int s = blockIdx.y;
    const int r0 = blockIdx.x * rows_per_block;
    const int r1 = min(K, r0 + rows_per_block);
    const int nrb = r1 - r0;
    const int* rp = rowptr + (int64_t)s * (K + 1);
    const int e0 = __ldg(rp + r0), e1 = __ldg(rp + r1);
    const int nb = e1 - e0;
    double* acc = reinterpret_cast<double*>(smem_f4);              // [nb]
    float* vs = reinterpret_cast<float*>(acc + ((nb + 1) & ~1));    // [C][TW]
    float* zs = vs + C * TW;                                        // [nrb][TW]
    for (int i = threadIdx.x; i < nb; i += blockDim.x) acc[i] = 0.0;
    const float* vg = V + (int64_t)s * C * NTs;
    const float* zg = DZ + ((int64_t)s * K + r0) * NTs;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int t0 = 0; t0 < NT; t0 += TW) {
        stage_rows<TW>(vg, vs, C, NTs, t0);
        stage_rows<TW>(zg, zs, nrb, NTs, t0);
        __syncthreads();
        for (int b = warp * 32; b < nb; b += nw * 32) {
            const int e = e0 + b + lane;
            int packed = 0;
            if (e < e1) packed = ((__ldg(rowof + e) - r0) << 16) | __ldg(colidx + e);
            float part[32];
            float z[R];
            int rprev = -1;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int pk = __shfl_sync(kFull, packed, j);
                const int rl = pk >> 16, c = pk & 0xffff;
                if (rl != rprev) {
                    lds_vec<R>(zs + rl * TW + lane * R, z);
                    rprev = rl;
                }
                float x[R];
                lds_vec<R>(vs + c * TW + lane * R, x);
                float p = 0.f;
#pragma unroll
                for (int q = 0; q < R; ++q) p = fmaf(z[q], x[q], p);
                part[j] = p;
            }
            transpose_reduce32(part, lane);
            if (b + lane < nb) acc[b + lane] += (double)part[0];
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < nb; i += blockDim.x) dW[e0 + i] = (float)acc[i];
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

// CSC value refresh: valsT[j] = vals[perm[j]]
__global__ void gather_kernel(float* __restrict__ dst, const float* __restrict__ src,
                              const int* __restrict__ perm, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[perm[i]];
}

// dense-plan dW: slice-major compact [s][k][c] -> W_F layout K×C×p×q
__global__ void slice_major_to_kcpq_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                           int K, int C, int P2) {
    const int64_t total = (int64_t)P2 * K * C;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = i / ((int64_t)K * C), kc = i - s * K * C;
        dst[kc * P2 + s] = src[i];
    }
}

}  // namespace wino
