// K2/K6 with the X operand in tensor memory: Y(r, t) = Σ_{e in CSR row r} w_e·X(c_e, t), the
// reference's association (products rounded, then added from +0 in CSR order, sparse.cpp:51-69),
// bitwise equal to spmm_kernel (wino_kernels.cuh).
//
// Why TMEM: with random masks each nonzero multiplies a whole row of X and no operand is reused
// in registers, so the shared-memory SpMM is bound by shared-memory operand delivery (~24
// multiply-adds/clk/SM measured).  A warp's tcgen05.ld.32x32b.x4 hands each lane 4 consecutive t
// of one X row from TMEM; with the products and sums on packed FFMA2/FADD2 the same loop reaches
// 42 multiply-adds/clk/SM (tools/microbench/spmm_hybrid_bw.cu).
//
// Layout: a block owns a 512-wide t chunk of one Winograd slice and a group of output rows.
// TMEM lane L (quarter q = L/32) holds t = t0 + 4L .. 4L+3; X row c of the current pass sits at
// columns 4(c - c0) .. +3, so one pass holds 128 X rows (512 columns).  Layers with more X rows
// run ceil(ncols/128) passes; CSR rows are sorted by column, so each output row continues where
// the previous pass stopped and the sum keeps the reference order.  Warp (q, g) of the 16 handles
// the lanes of quarter q for output rows g, g+4, ... of the group (RPW rows, accumulators in
// registers across passes).  The X rows of a pass are loaded with float4 loads and written with
// tcgen05.st by the warps of the matching quarter.
//
// Status: opt-in (WINO_SPMM_TMEM=1), bitwise equal to spmm_kernel on every parity test, but
// measured at parity at c2 (705 vs 703 µs) and slower at c1 (59 vs 40 µs) and c3 (696 vs 543 µs):
// the kernel issues more instructions per multiply-add than the microbenchmark loop (row/pass
// boundaries, tails of < 8 nonzeros per row and pass) and the TMEM fill is not overlapped with the
// products (one 512-column buffer per SM); see DESIGN.md §7.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace wino {
namespace st {

constexpr int TW = 512;        // t per block: 128 TMEM lanes x 4 columns
constexpr int PASS_ROWS = 128; // X rows per TMEM fill
constexpr int WARPS = 16;      // 4 lane quarters x 4 row subsets
constexpr int THREADS = 32 * WARPS;
constexpr int U = 8;           // nonzeros in flight per warp

__device__ __forceinline__ unsigned long long pk2(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk2(unsigned long long r, float& a, float& b) {
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
// acc += fl(w·x) on two lanes' t: FFMA2 with a runtime −0 addend gives the rounded product (ptxas
// would otherwise fuse mul.rn.f32x2 + add.rn.f32x2 into one FFMA2), then FADD2
__device__ __forceinline__ unsigned long long madd2(unsigned long long acc, unsigned long long w2,
                                                    unsigned long long x2, unsigned long long n0) {
    unsigned long long p, r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(x2), "l"(w2), "l"(n0));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(acc), "l"(p));
    return r;
}

__device__ __forceinline__ void tld4(uint32_t taddr, float (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
                 : "r"(taddr));
}
__device__ __forceinline__ void tst4(uint32_t taddr, float4 v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}

// grid = (row groups, ceil(NTr / TW), slices); RPW output rows per warp (rows_per_block = 4·RPW)
template <int RPW>
__global__ void __launch_bounds__(THREADS, 1)
spmm_tmem_kernel(const int* __restrict__ rowptr, const int2* __restrict__ colval, const float* __restrict__ X,
                 float* __restrict__ Y, int nrows, int ncols, int NTs, int NTr, float neg0) {
    __shared__ uint32_t tbase;
    extern __shared__ int4 seg4[];  // the block's CSR segment (col, value) pairs, staged once
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = warp & 3, g = warp >> 2;
    const int s = blockIdx.z;
    const int t0 = blockIdx.y * TW;
    const int r0 = blockIdx.x * 4 * RPW;
    const int* rp = rowptr + (int64_t)s * (nrows + 1);
    const float* xs = X + (int64_t)s * ncols * NTs;
    const int tl = t0 + 4 * (32 * q + lane);  // this lane's first t
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tq = tbase + ((uint32_t)(32 * q) << 16);  // this warp's lane quarter
    const unsigned long long n0 = pk2(neg0, neg0);
    // stage the CSR segment of rows [r0, r0 + 4·RPW) (16-byte aligned start: pairs of entries)
    const int rb = min(nrows, r0 + 4 * RPW);
    const int a0 = r0 < nrows ? (__ldg(rp + r0) & ~1) : 0;
    const int a1 = r0 < nrows ? __ldg(rp + rb) : 0;
    for (int i = threadIdx.x; i < (a1 - a0 + 1) >> 1; i += THREADS)
        seg4[i] = __ldg(reinterpret_cast<const int4*>(colval + a0) + i);
    const int2* cvs = reinterpret_cast<const int2*>(seg4) - a0;  // indexed by global entry number

    unsigned long long acc[RPW][2];
#pragma unroll
    for (int i = 0; i < RPW; ++i) acc[i][0] = acc[i][1] = 0ull;  // +0, +0
    // per local row: the CSR entry where each pass starts (columns ascend within a row)
    constexpr int MAXP = 8;  // ncols <= 1024
    __shared__ int bnd[4 * RPW][MAXP + 1];
    const int npass = (ncols + PASS_ROWS - 1) / PASS_ROWS;
    __syncthreads();  // the staged segment
    for (int lr = threadIdx.x; lr < 4 * RPW; lr += THREADS) {
        const int r = r0 + lr;
        int e = r < nrows ? __ldg(rp + r) : 0;
        const int ee = r < nrows ? __ldg(rp + r + 1) : 0;
        bnd[lr][0] = e;
        for (int ps = 1; ps <= npass; ++ps) {
            while (e < ee && cvs[e].x < ps * PASS_ROWS) ++e;
            bnd[lr][ps] = e;
        }
    }
    for (int c0 = 0; c0 < ncols; c0 += PASS_ROWS) {
        const int nr = min(PASS_ROWS, ncols - c0);
        if (c0 > 0) {  // every warp is done reading the previous pass
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncthreads();
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        // fill: the 4 warps of quarter q store rows g, g+4, ... of the pass into their lanes,
        // 8 rows' loads in flight before their stores
        for (int cb = g; cb < nr; cb += 32) {
            float4 v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int cc = cb + 4 * j;
                v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (cc < nr && tl < NTs)
                    v[j] = __ldg(reinterpret_cast<const float4*>(xs + (int64_t)(c0 + cc) * NTs + tl));
            }
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (cb + 4 * j < nr) tst4(tq + 4 * (cb + 4 * j), v[j]);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int ps = c0 / PASS_ROWS;
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            const int lr = g + 4 * i;
            int e = bnd[lr][ps];
            const int ee = bnd[lr][ps + 1];
            for (; e + U <= ee; e += U) {  // full batches: U loads in flight, no predicates
                int2 cv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) cv[u] = cvs[e + u];  // shared-memory broadcasts
                float x[U][4];
#pragma unroll
                for (int u = 0; u < U; ++u) tld4(tq + 4 * (cv[u].x - c0), x[u]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const float w = __int_as_float(cv[u].y);
                    const unsigned long long w2 = pk2(w, w);
                    acc[i][0] = madd2(acc[i][0], w2, pk2(x[u][0], x[u][1]), n0);
                    acc[i][1] = madd2(acc[i][1], w2, pk2(x[u][2], x[u][3]), n0);
                }
            }
            // tail of < U entries in batches of 4, 2, 1: at most three load waits
#pragma unroll
            for (int b = U / 2; b >= 1; b >>= 1) {
                if (ee - e >= b) {
                    int2 cv[U / 2];
                    float x[U / 2][4];
#pragma unroll
                    for (int u = 0; u < b; ++u) cv[u] = cvs[e + u];
#pragma unroll
                    for (int u = 0; u < b; ++u) tld4(tq + 4 * (cv[u].x - c0), x[u]);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int u = 0; u < b; ++u) {
                        const float w = __int_as_float(cv[u].y);
                        const unsigned long long w2 = pk2(w, w);
                        acc[i][0] = madd2(acc[i][0], w2, pk2(x[u][0], x[u][1]), n0);
                        acc[i][1] = madd2(acc[i][1], w2, pk2(x[u][2], x[u][3]), n0);
                    }
                    e += b;
                }
            }
        }
    }
    // write back: lane's 4 t of every row (t < NTr; NTr is a multiple of 4)
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const int r = r0 + g + 4 * i;
        if (r < nrows && tl < NTr) {
            float4 o;
            upk2(acc[i][0], o.x, o.y);
            upk2(acc[i][1], o.z, o.w);
            *reinterpret_cast<float4*>(Y + ((int64_t)s * nrows + r) * NTs + tl) = o;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

}  // namespace st
}  // namespace wino
