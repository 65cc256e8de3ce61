// dW_F = dZ·Ĩ_Fᵀ on the int8 tensor cores with exact fp32 products (an Ozaki-style split).
//
// The masked SDDMM (wino_kernels.cuh, K5) forms every product exactly in fp64 on the SIMT pipes
// and is bound there (one fp32->fp64 conversion per product).  Here the same exact dot products
// run on tcgen05 kind::i8:
//   * every 128-long block of a dZ / Ĩ_F row gets a shared exponent E (|x| < 2^(E-1)) and is
//     written as DIG = 5 signed base-2^7 digits, x = 2^E·Σ_i d_i·2^(-7(i+1)) + r, |d_i| <= 64
//     (round-to-nearest digits: each remainder is exact in fp32); |r| <= 2^(E-36), i.e. every
//     entry within 2^-12 of its block's max keeps all 24 of its bits;
//   * per 128-long block, digit pairs (i, j) with i + j = w < 5 accumulate exactly in int32 TMEM
//     accumulator w (|sum| <= 5·128·64² < 2^22), pairs with i + j >= 5 (<= 2^-37 of the block's
//     max|a|·max|b| each) are dropped;
//   * drain warps combine T = Σ_w acc_w·2^(7(4-w)) exactly in int64, scale by 2^(E_a+E_b-42)
//     (exact) and accumulate the blocks in fp64 — the dot product of the stored fp32 operands
//     up to the dropped digit pairs and the 2^-29-relative digit remainders, then one rounding.
// The whole K×C product is formed (a GEMM per Winograd coordinate); the surviving entries are
// gathered in CSR order afterwards (gather_kernel), so masked
// coordinates are never written (train.cpp:281-283).  Deterministic: fixed block order.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "wino_dense_tc.cuh"

namespace wino {
namespace oz {

constexpr int DIG = 5;      // base-2^7 digits per value
constexpr int KB = 128;     // reduction block: one 128-byte swizzle row of int8 per operand row
constexpr int BM = 128;     // UMMA M (K rows of dW_F)
constexpr int BN = 48;      // UMMA N (C columns of dW_F): 5 levels x 48 x 2 buffers fit TMEM
constexpr int UK = 32;      // K per tcgen05.mma kind::i8 (32 bytes)
constexpr int STAGES = 2;
constexpr int A_DIG = BM * KB;                       // 16 KB per digit tile
constexpr int B_DIG = BN * KB;                       // 6 KB
constexpr int STAGE_BYTES = DIG * (A_DIG + B_DIG);   // 110 KB
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 256;
constexpr int DRAIN_WARPS = 8;                       // 4 lane quarters x 2 column blocks
constexpr int DCOLS = BN / (DRAIN_WARPS / 4);         // 24 columns per drain thread
constexpr int THREADS = 64 + 32 * DRAIN_WARPS;
constexpr int LEVELS = DIG;                          // accumulators: digit-pair weight i + j < DIG
constexpr int TMEM_COLS = 512;                       // 2 x LEVELS x BN = 480 used (double-buffered)

// D = S32 (bits 4-5 = 2), A = B = signed 8-bit (bits 7-9, 10-12 = 1), both K-major, N>>3, M>>4
__host__ __device__ constexpr uint32_t idesc_i8() {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

// X [S][R][NTs] fp32 (columns >= NT ignored) -> digits [DIG][S][R][NTp] int8 and block exponents
// [S][NTp/KB][R] int32 (rows contiguous: the drain reads a tile's column exponents as int4s).  One warp per (s, r, block); lane l covers t = 4l..4l+3 of the block.
__global__ void __launch_bounds__(256) slice_kernel(const float* __restrict__ X, int8_t* __restrict__ dig,
                                                    int* __restrict__ ex, int S, int R, int NT, int NTs, int NTp) {
    const int nkb = NTp / KB;
    const int64_t warps = (int64_t)S * R * nkb;
    const int lane = threadIdx.x & 31;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < warps;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int kb = (int)(w % nkb);
        const int64_t sr = w / nkb;  // s·R + r
        const int t0 = kb * KB + lane * 4;
        float x[4];
        const float* src = X + sr * NTs;
        if (t0 + 3 < NT) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(src + t0));
            x[0] = v.x, x[1] = v.y, x[2] = v.z, x[3] = v.w;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) x[j] = t0 + j < NT ? __ldg(src + t0 + j) : 0.f;
        }
        uint32_t m = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) m = max(m, __float_as_uint(x[j]) & 0x7fffffffu);
        m = __reduce_max_sync(0xffffffffu, m);
        // |x| < 2^(e-126) for biased exponent e (e >= 1); E = e - 125 gives |x| < 2^(E-1)
        const int e = max(1, (int)(m >> 23));
        const int E = m == 0 ? 0 : e - 125;
        int8_t d[DIG][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float q = ldexpf(x[j], 7 - E);  // |q| < 64, exact
#pragma unroll
            for (int i = 0; i < DIG; ++i) {
                const float di = rintf(q);
                d[i][j] = (int8_t)(int)di;
                q = (q - di) * 128.f;  // |q - di| <= 1/2: the next digit is in [-64, 64]
            }
        }
#pragma unroll
        for (int i = 0; i < DIG; ++i) {
            const uint32_t packed = (uint32_t)(uint8_t)d[i][0] | ((uint32_t)(uint8_t)d[i][1] << 8) |
                                    ((uint32_t)(uint8_t)d[i][2] << 16) | ((uint32_t)(uint8_t)d[i][3] << 24);
            *reinterpret_cast<uint32_t*>(dig + ((int64_t)i * S * R + sr) * NTp + t0) = packed;
        }
        if (lane == 0) ex[((sr / R) * nkb + kb) * R + sr % R] = E;
    }
}

// D[s][m][n] (fp32, row stride N) = Σ_t A[s][m][t]·B[s][n][t] exactly (up to the digit
// truncation above) from the digit tensors; persistent, warp-specialised:
//   warp 0 TMA (the 5 A and 5 B digit tiles of a 128-long block per stage) · warp 1 TMEM alloc
//   + MMA (15 digit pairs x 4 k-steps into 5 level accumulators, double-buffered) · 8 drain
//   warps (int64 combine, exact scaling, fp64 accumulation over the blocks of a tile).
__global__ void __launch_bounds__(THREADS, 1)
gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
            const int* __restrict__ exA, const int* __restrict__ exB, float* __restrict__ D, int S, int M, int N,
            int nkb, int tiles_n, int tiles_m, int ntiles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* full = bars;                   // [STAGES]
    uint64_t* empty = bars + STAGES;         // [STAGES]
    uint64_t* tfull = bars + 2 * STAGES;     // [2]
    uint64_t* tempty = bars + 2 * STAGES + 2;  // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto decode = [&](int tile, int& n0, int& m0, int& s) {
        const int nt = tile % tiles_n, rest = tile / tiles_n;
        m0 = (rest % tiles_m) * BM;
        s = rest / tiles_m;
        n0 = nt * BN;
    };
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&tfull[i], 1);
            tc::mbar_init(&tempty[i], 32 * DRAIN_WARPS);
        }
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
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                int n0, m0, s;
                decode(tile, n0, m0, s);
                for (int kb = 0; kb < nkb; ++kb, ++g) {
                    const int st = g % STAGES;
                    if (g >= STAGES) tc::mbar_wait(&empty[st], ((g / STAGES) - 1) & 1);
                    uint8_t* base = smem + st * STAGE_BYTES;
                    tc::mbar_expect_tx(&full[st], STAGE_BYTES);
#pragma unroll
                    for (int i = 0; i < DIG; ++i) {
                        tc::tma_load_3d(base + i * A_DIG, &mapA, &full[st], kb * KB, m0, i * S + s);
                        tc::tma_load_3d(base + DIG * A_DIG + i * B_DIG, &mapB, &full[st], kb * KB, n0, i * S + s);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t id = idesc_i8();
            int g = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                for (int kb = 0; kb < nkb; ++kb, ++g) {
                    const int st = g % STAGES, b = g & 1;
                    if (g >= 2) tc::mbar_wait(&tempty[b], ((g >> 1) - 1) & 1);
                    tc::mbar_wait(&full[st], (g / STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t a0 = tc::smem_u32(smem + st * STAGE_BYTES);
                    // descriptors of the stage's first digit tiles; the start-address field (addr >> 4,
                    // 14 bits) takes the byte offsets of the other tiles / k-steps without carry
                    const uint64_t da0 = tc::make_desc(a0, 0, 1024, tc::kLayoutSW128);
                    const uint64_t db0 = tc::make_desc(a0 + DIG * A_DIG, 0, 1024, tc::kLayoutSW128);
#pragma unroll
                    for (int w = 0; w < LEVELS; ++w) {
                        const uint32_t acc = tmem + (uint32_t)(b * LEVELS * BN + w * BN);
#pragma unroll
                        for (int i = 0; i <= w; ++i) {
                            const int j = w - i;
#pragma unroll
                            for (int k = 0; k < KB / UK; ++k)
                                mma_i8(acc, da0 + (uint64_t)((i * A_DIG + k * 32) >> 4),
                                       db0 + (uint64_t)((j * B_DIG + k * 32) >> 4), id, (i == 0 && k == 0) ? 0u : 1u);
                        }
                    }
                    tc::mma_commit(&empty[st]);
                    tc::mma_commit(&tfull[b]);
                }
            }
        }
    } else {
        const int qd = warp & 3, cb = (warp - 2) >> 2;  // lane quarter, column block
        int g = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            int n0, m0, s;
            decode(tile, n0, m0, s);
            const int row = m0 + qd * 32 + lane;
            const int col0 = n0 + cb * DCOLS;
            double acc[DCOLS];
#pragma unroll
            for (int j = 0; j < DCOLS; ++j) acc[j] = 0.0;
            for (int kb = 0; kb < nkb; ++kb, ++g) {
                const int b = g & 1;
                const int ea = row < M ? __ldg(exA + ((int64_t)s * nkb + kb) * M + row) : 0;
                const int* exb = exB + ((int64_t)s * nkb + kb) * N;
                tc::mbar_wait(&tfull[b], (g >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t ta = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(b * LEVELS * BN + cb * DCOLS);
#pragma unroll
                for (int h = 0; h < DCOLS / 8; ++h) {
                    uint32_t v0[8], v1[8];
                    long long hm[8];
                    tmem_ld8(ta + 0 * BN + h * 8, v0);
                    tmem_ld8(ta + 1 * BN + h * 8, v1);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int j = 0; j < 8; ++j) hm[j] = (long long)((int)v0[j] * 128 + (int)v1[j]) << 14;  // < 2^43
                    tmem_ld8(ta + 2 * BN + h * 8, v0);
                    tmem_ld8(ta + 3 * BN + h * 8, v1);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int j = 0; j < 8; ++j) hm[j] = (hm[j] + (int)v0[j] * 128 + (int)v1[j]) * 128;  // < 2^50
                    tmem_ld8(ta + 4 * BN + h * 8, v0);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (h == DCOLS / 8 - 1) {  // the buffer is free once the last columns are in registers
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        tc::mbar_arrive(&tempty[b]);
                    }
                    int ebv[8];
                    if (col0 + h * 8 + 8 <= N) {  // N % 4 == 0: 16-byte aligned rows
                        const int4 e0 = __ldg(reinterpret_cast<const int4*>(exb + col0 + h * 8));
                        const int4 e1 = __ldg(reinterpret_cast<const int4*>(exb + col0 + h * 8 + 4));
                        ebv[0] = e0.x, ebv[1] = e0.y, ebv[2] = e0.z, ebv[3] = e0.w;
                        ebv[4] = e1.x, ebv[5] = e1.y, ebv[6] = e1.z, ebv[7] = e1.w;
                    } else {
#pragma unroll
                        for (int j = 0; j < 8; ++j) ebv[j] = col0 + h * 8 + j < N ? __ldg(exb + col0 + h * 8 + j) : 0;
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int eb = ebv[j];
                        const long long T = hm[j] + (int)v0[j];  // Σ_w acc_w·2^(7(4-w)), exact (< 2^51)
                        const double sc = __longlong_as_double((long long)(ea + eb - 42 + 1023) << 52);
                        acc[h * 8 + j] = fma((double)T, sc, acc[h * 8 + j]);
                    }
                }
            }
            if (row < M) {
                float* drow = D + ((int64_t)s * M + row) * N;
#pragma unroll
                for (int j = 0; j < DCOLS; ++j)
                    if (col0 + j < N) drow[col0 + j] = (float)acc[j];
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

// dW_F in CSR order from the dense [S][K][C] product: grid (blocks, S), slice s covers entries
// [off[s], off[s+1]) (rowof = row within the slice, colidx = column).
__global__ void gather_kernel(const float* __restrict__ Dd, float* __restrict__ dw, const int* __restrict__ rowof,
                              const int* __restrict__ colidx, const int64_t* __restrict__ off, int K, int C,
                              int S, int64_t nnz) {
    const int s = blockIdx.y;
    const int64_t e0 = off[s], e1 = s + 1 < S ? off[s + 1] : nnz;
    const float* plane = Dd + (int64_t)s * K * C;
    for (int64_t e = e0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < e1; e += (int64_t)gridDim.x * blockDim.x)
        dw[e] = plane[(int64_t)__ldg(rowof + e) * C + __ldg(colidx + e)];
}

}  // namespace oz
}  // namespace wino
