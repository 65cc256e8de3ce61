// Dense contraction on the 5th-generation tensor cores (tcgen05), used by the dense plan
// (W_F without zeros, e.g. BASELINE configs[3] at 0% sparsity):
//     D[s] (M×N) = A[s] (M×Kd) · B[s] (Kd×N)      for every Winograd slice s = (i,j)
//   forward    : M=K, Kd=C, A = W_F(:,:,i,j) [K][C],   B = Ĩ_F [C][NT]   -> Z   (layer.cpp:61-71)
//   bwd data   : M=C, Kd=K, A = W_F(:,:,i,j)ᵀ [C][K], B = dZ [K][NT]    -> dĨ_F (layer.cpp:145-155)
//   bwd weights: M=K, N=C, Kd=NT, A = dZ [K][NT] (K-major, split on the fly), B = Ĩ_Fᵀ (Ĩ_F [C][NT]
//                is K-major for this product), split over NT into fp32 partials that
//                reduce_dw_kernel sums in fp64 in split order              -> dW_F (layer.cpp:118-128)
//
// Precision: 3xTF32 (D += Ah·Bh + Ah·Bl + Al·Bh, X = Xh + Xl with Xh = rna_tf32(X),
// Xl = rna_tf32(X − Xh)): ~2^-22 relative error per product, fp32 accumulation in TMEM.  A is
// split once on the host (weights); B is split per stage in shared memory by converter warps
// (an elementwise op, so the TMA swizzle layout is preserved).
//
// Structure (one 128×256 output tile per CTA, 256 threads):
//   warp 0     : TMA producer — A_hi, A_lo (K-major, 128B swizzle) and B (MN-major, 128B swizzle)
//   warp 1     : TMEM allocator + single-thread tcgen05.mma issuer
//   warps 4..7 : B hi/lo split per stage, then the epilogue (tcgen05.ld 32x32b.x32 -> global)
// Two-stage ring: full (TMA tx) -> split (128 arrivals) -> MMA -> tcgen05.commit -> empty.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace wino {
namespace tc {

constexpr int BM = 128;      // UMMA M (cta_group::1)
constexpr int BN = 256;      // UMMA N
constexpr int BK = 32;       // fp32 elements per stage along the reduction (one 128-byte row)
constexpr int UK = 8;        // K per tcgen05.mma for kind::tf32 (32 bytes)
constexpr int STAGES = 2;
constexpr int THREADS = 256;
constexpr int A_TILE = BM * BK * 4;       // 16 KB
constexpr int B_TILE = BK * BN * 4;       // 32 KB
constexpr int STAGE_BYTES = 2 * A_TILE + 2 * B_TILE;   // A_hi, A_lo, B(hi in place), B_lo
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

// TMA store of a shared-memory box into a 3-D tensor (out-of-range rows/columns are clipped)
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     (uint64_t)map),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Shared-memory matrix descriptor (SM100 UMMA): start>>4 [0,14), LBO>>4 [16,30), SBO>>4
// [32,46), version=1 [46,48), layout type [61,64): 2 = SWIZZLE_128B (K-major tf32),
// 1 = SWIZZLE_128B_BASE32B (the layout MN-major 32-bit operands require; produced by TMA's
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B).
constexpr uint32_t kLayoutSW128 = 2;
constexpr uint32_t kLayoutSW128Base32 = 1;
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

// Instruction descriptor, kind::tf32: D f32 (bits 4-5 = 1), A/B tf32 (2), A K-major (bit 15 = 0),
// B major (bit 16: 1 = MN-major, 0 = K-major), N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t make_idesc(bool b_mn_major) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | ((b_mn_major ? 1u : 0u) << 16) |
           ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__device__ __forceinline__ void split_tile(uint8_t* hi_buf, uint8_t* lo_buf, int bytes, int t, int nthreads) {
    const uint32_t h0 = smem_u32(hi_buf), l0 = smem_u32(lo_buf);
#pragma unroll 4
    for (int i = t * 16; i < bytes; i += nthreads * 16) {
        float4 x;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "r"(h0 + i));
        float4 h, l;
#ifdef WINO_TC_NOSPLIT
        h = x;
        l = make_float4(0.f, 0.f, 0.f, 0.f);
#else
        h.x = tf32_rna(x.x); l.x = tf32_rna(x.x - h.x);
        h.y = tf32_rna(x.y); l.y = tf32_rna(x.y - h.y);
        h.z = tf32_rna(x.z); l.z = tf32_rna(x.z - h.z);
        h.w = tf32_rna(x.w); l.w = tf32_rna(x.w - h.w);
#endif
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(h0 + i), "f"(h.x), "f"(h.y), "f"(h.z), "f"(h.w));
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(l0 + i), "f"(l.x), "f"(l.y), "f"(l.z), "f"(l.w));
    }
}

// Same split with integer rounding, bitwise equal to split_tile for finite x: cvt.rna.tf32 (round
// to nearest, ties away from zero) = add half a tf32 ulp to the sign-magnitude bit pattern and
// clear the 13 low bits; hi = rna(x), lo = rna(x - hi) (x - hi is exact).  Five ALU/FP32
// instructions per element instead of two emulated cvt.rna (~10).
__device__ __forceinline__ uint32_t rna_bits(uint32_t x) { return (x + 0x1000u) & 0xffffe000u; }

__device__ __forceinline__ void split_tile_fast(uint8_t* hi_buf, uint8_t* lo_buf, int bytes, int t, int nthreads) {
    const uint32_t h0 = smem_u32(hi_buf), l0 = smem_u32(lo_buf);
#pragma unroll 4
    for (int i = t * 16; i < bytes; i += nthreads * 16) {
        uint32_t x[4], h[4], l[4];
        asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]) : "r"(h0 + i));
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            h[j] = rna_bits(x[j]);
            l[j] = rna_bits(__float_as_uint(__fsub_rn(__uint_as_float(x[j]), __uint_as_float(h[j]))));
        }
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(h0 + i), "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3]));
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(l0 + i), "r"(l[0]), "r"(l[1]), "r"(l[2]), "r"(l[3]));
    }
}

// Kahan step on two lanes of fp32 pairs at once (FADD2): s += v with compensation c.
__device__ __forceinline__ void kahan2(float& s0, float& s1, float& c0, float& c1, float v0, float v1) {
    unsigned long long s, c, v, y, t, d;
    asm("mov.b64 %0, {%1,%2};" : "=l"(s) : "f"(s0), "f"(s1));
    asm("mov.b64 %0, {%1,%2};" : "=l"(c) : "f"(c0), "f"(c1));
    asm("mov.b64 %0, {%1,%2};" : "=l"(v) : "f"(v0), "f"(v1));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(y) : "l"(v), "l"(c));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(s), "l"(y));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(t), "l"(s));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(c) : "l"(d), "l"(y));
    asm("mov.b64 {%0,%1}, %2;" : "=f"(s0), "=f"(s1) : "l"(t));
    asm("mov.b64 {%0,%1}, %2;" : "=f"(c0), "=f"(c1) : "l"(c));
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}


__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}

// ---------------------------------------------------------------------------------------
// The accurate tcgen05 GEMM: every k-block (32 reduction elements × 3 tf32 products) accumulates
// into a FRESH TMEM accumulator, folded outside TMEM (long fp32 accumulation chains inside TMEM
// are what cost 3xTF32 its accuracy — measured error/Σ|p| 2.4e-6 with 63 k-blocks per
// accumulator vs 4.6e-8 with one).  Tile 128×128.  (Earlier generations — single-accumulator,
// non-persistent and persistent-with-shared-epilogue-warps forms — are described with their
// measurements in DESIGN.md §7.)
// ---------------------------------------------------------------------------------------
namespace flush {
constexpr int BN = 128;
constexpr int STAGES = 3;
constexpr int THREADS = 320;
constexpr int A_TILE = BM * BK * 4;   // 16 KB
constexpr int B_TILE = BK * BN * 4;   // 16 KB
constexpr int STAGE_BYTES = 2 * A_TILE + 2 * B_TILE;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 256;
constexpr int WS_SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 8 * 4096;  // + barriers, 8 staging boxes
constexpr int TMEM_COLS = 2 * BN;

__host__ __device__ constexpr uint32_t idesc(bool b_mn_major) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | ((b_mn_major ? 1u : 0u) << 16) |
           ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}
}  // namespace flush

// Persistent and warp-specialised (when one set of epilogue warps both split the operands of
// stage kb+2 and drained the accumulator of k-block kb, the split feeding the MMA waited behind
// every drain — ncu: tensor pipe ~20% active).  The roles are separate warps:
//   warp 0 TMA · warp 1 TMEM alloc + MMA · SW split warps (hi/lo of the stage, runs up to STAGES
//   ahead, gated only by TMA) · DW drain warps (fold each k-block's fresh accumulator; warp w
//   reads TMEM lane quarter w % 4 and column block of COLS = BN/(DW/4) columns).
// NBUF TMEM accumulators let the MMA run NBUF-1 k-blocks ahead of the drain.  Same arithmetic
// per tile as the shared-epilogue form (bitwise, with KAHAN = false).
template <bool A_SPLIT, bool B_MN, int SW, int DW, bool KAHAN, int NBUF>
__global__ void __launch_bounds__(64 + 32 * (SW + DW), 1)
gemm_3xtf32_ws_kernel(const __grid_constant__ CUtensorMap mapAh, const __grid_constant__ CUtensorMap mapAl,
                      const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapD,
                      float* __restrict__ D, int M, int N, int Kd,
                      int64_t ldd, int slices, int splits, int kb_per, int tiles_n, int tiles_m, int ntiles) {
    constexpr int BN = flush::BN, STAGES = flush::STAGES, A_TILE = flush::A_TILE, B_TILE = flush::B_TILE;
    constexpr int STAGE_BYTES = flush::STAGE_BYTES;
    constexpr int TMEM_COLS = NBUF * BN;
    static_assert(TMEM_COLS <= 512 && (NBUF & (NBUF - 1)) == 0, "TMEM holds 512 columns");
    static_assert(SW > 0, "split warps");
    static_assert(DW == 8 || DW == 16, "drain warps: 4 lane quarters x 2 or 4 column blocks");
    constexpr int COLS = BN / (DW / 4);
    // output staging box per drain warp: 32 rows x BOXC columns (4 KB with a 128-byte swizzle for
    // DW = 8, 2 KB with a 64-byte swizzle for DW = 16) — 32 KB of shared memory either way
    constexpr int BOXC = DW == 8 ? 32 : 16;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* full = bars;
    uint64_t* split = bars + STAGES;
    uint64_t* empty = bars + 2 * STAGES;
    uint64_t* tfull = bars + 3 * STAGES;
    uint64_t* tempty = bars + 3 * STAGES + NBUF;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * STAGES + 2 * NBUF);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kb_total = (Kd + BK - 1) / BK;
    struct Tile { int n0, m0, s, q, kb0, kblocks; };
    auto decode = [&](int tile) {
        Tile t;
        const int nt = tile % tiles_n, rest = tile / tiles_n;
        const int mt = rest % tiles_m, z = rest / tiles_m;
        t.n0 = nt * BN;
        t.m0 = mt * BM;
        t.s = z / splits;
        t.q = z - t.s * splits;
        t.kb0 = t.q * kb_per;
        t.kblocks = max(0, min(kb_total, t.kb0 + kb_per) - t.kb0);
        return t;
    };

    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&split[i], SW > 0 ? 32 * SW : 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < NBUF; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 32 * DW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    auto stage_ptr = [&](int st) { return smem + st * STAGE_BYTES; };

    if (warp == 0) {
        if (lane == 0) {
            int kbg = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const Tile t = decode(tile);
                for (int kb = 0; kb < t.kblocks; ++kb, ++kbg) {
                    const int st = kbg % STAGES;
                    if (kbg >= STAGES) mbar_wait(&empty[st], ((kbg / STAGES) - 1) & 1);
                    uint8_t* base = stage_ptr(st);
                    const int kk = (t.kb0 + kb) * BK;
                    mbar_expect_tx(&full[st], (A_SPLIT ? A_TILE : 2 * A_TILE) + B_TILE);
                    tma_load_3d(base, &mapAh, &full[st], kk, t.m0, t.s);
                    if (!A_SPLIT) tma_load_3d(base + A_TILE, &mapAl, &full[st], kk, t.m0, t.s);
                    if (B_MN) {
#pragma unroll
                        for (int j = 0; j < BN / 32; ++j) {
                            tma_load_3d(base + 2 * A_TILE + j * (BK * 128), &mapB, &full[st], t.n0 + 32 * j, kk, t.s);
                        }
                    } else {
                        tma_load_3d(base + 2 * A_TILE, &mapB, &full[st], kk, t.n0, t.s);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t id = flush::idesc(B_MN);
            int kbg = 0, gg = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const Tile t = decode(tile);
                for (int kb = 0; kb < t.kblocks; ++kb, ++kbg, ++gg) {
                    const int st = kbg % STAGES, b = gg % NBUF;
                    if (gg >= NBUF) mbar_wait(&tempty[b], ((gg / NBUF) - 1) & 1);
                    if constexpr (SW > 0)
                        mbar_wait(&split[st], (kbg / STAGES) & 1);
                    else
                        mbar_wait(&full[st], (kbg / STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t a_hi = smem_u32(stage_ptr(st));
                    const uint32_t a_lo = a_hi + A_TILE;
                    const uint32_t b_hi = a_hi + 2 * A_TILE;
                    const uint32_t b_lo = b_hi + B_TILE;
                    const uint32_t acc = tmem + (uint32_t)(b * BN);
#pragma unroll
                    for (int k = 0; k < BK / UK; ++k) {
                        const uint64_t dah = make_desc(a_hi + k * 32, 0, 1024, kLayoutSW128);
                        const uint64_t dal = make_desc(a_lo + k * 32, 0, 1024, kLayoutSW128);
                        uint64_t dbh, dbl;
                        if (B_MN) {
                            dbh = make_desc(b_hi + k * 1024, BK * 128, 512, kLayoutSW128Base32);
                            dbl = make_desc(b_lo + k * 1024, BK * 128, 512, kLayoutSW128Base32);
                        } else {
                            dbh = make_desc(b_hi + k * 32, 0, 1024, kLayoutSW128);
                            dbl = make_desc(b_lo + k * 32, 0, 1024, kLayoutSW128);
                        }
                        mma_tf32(acc, dah, dbh, id, k == 0 ? 0u : 1u);  // fresh accumulator per k-block
                        mma_tf32(acc, dah, dbl, id, 1u);
                        mma_tf32(acc, dal, dbh, id, 1u);
                    }
                    mma_commit(&empty[st]);
                    mma_commit(&tfull[b]);
                }
            }
        }
    } else if (warp < 2 + SW) {
        const int ts = threadIdx.x - 64;
        int kbg = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int kbl = decode(tile).kblocks;
            for (int kb = 0; kb < kbl; ++kb, ++kbg) {
                const int st = kbg % STAGES;
                mbar_wait(&full[st], (kbg / STAGES) & 1);
                uint8_t* base = stage_ptr(st);
                if (A_SPLIT) split_tile_fast(base, base + A_TILE, A_TILE, ts, 32 * SW);
                split_tile_fast(base + 2 * A_TILE, base + 2 * A_TILE + B_TILE, B_TILE, ts, 32 * SW);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(&split[st]);
            }
        }
    } else {
        const int qd = warp & 3, cb = (warp - 2 - SW) >> 2;
        float* stg = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 1024) + (warp - 2 - SW) * 32 * BOXC;
        int gg = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const Tile t = decode(tile);
            using Acc = typename std::conditional<KAHAN, float, double>::type;
            Acc accd[COLS];
            float comp[KAHAN ? COLS : 1];
#pragma unroll
            for (int j = 0; j < COLS; ++j) accd[j] = Acc(0);
#pragma unroll
            for (int j = 0; j < (KAHAN ? COLS : 1); ++j) comp[j] = 0.f;
            for (int kb = 0; kb < t.kblocks; ++kb, ++gg) {
                const int b = gg % NBUF;
                mbar_wait(&tfull[b], (gg / NBUF) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t ta = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(b * BN + cb * COLS);
                // 8-column TMEM loads: fewer live registers next to the 2·COLS accumulator words
#pragma unroll
                for (int c = 0; c < COLS; c += 8) {
                    uint32_t v[8];
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                                   "=r"(v[6]), "=r"(v[7])
                                 : "r"(ta + c));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (c + 8 == COLS) {  // the buffer is free once the last columns are in registers
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        mbar_arrive(&tempty[b]);
                    }
                    if constexpr (KAHAN) {
#pragma unroll
                        for (int j = 0; j < 8; j += 2)
                            kahan2(accd[c + j], accd[c + j + 1], comp[c + j], comp[c + j + 1], __uint_as_float(v[j]),
                                   __uint_as_float(v[j + 1]));
                    } else {
#pragma unroll
                        for (int j = 0; j < 8; ++j) accd[c + j] += (double)__uint_as_float(v[j]);
                    }
                }
            }
            if constexpr (KAHAN) {
#pragma unroll
                for (int j = 0; j < COLS; ++j) accd[j] = __fsub_rn(accd[j], comp[j]);
            }
            // Output through a per-warp 32-row staging box (swizzled: conflict-free float4 writes,
            // lane = row) and TMA stores — row-per-lane global stores hit 32 rows per instruction
            // with half-sector writes (measured: +45% GEMM time at c3).
#pragma unroll
            for (int p = 0; p < COLS / BOXC; ++p) {
                if (lane == 0) bulk_wait_read();  // the previous box has left shared memory
                __syncwarp();
#pragma unroll
                for (int j = 0; j < BOXC / 4; ++j) {
                    // 16-byte chunk j of row `lane`: XOR with address bits 7.. (SW128: lane & 7,
                    // SW64: (lane >> 1) & 3)
                    const int pj = BOXC == 32 ? (j ^ (lane & 7)) : (j ^ ((lane >> 1) & 3));
                    *reinterpret_cast<float4*>(stg + lane * BOXC + (pj << 2)) =
                        make_float4((float)accd[p * BOXC + 4 * j], (float)accd[p * BOXC + 4 * j + 1],
                                    (float)accd[p * BOXC + 4 * j + 2], (float)accd[p * BOXC + 4 * j + 3]);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    tma_store_3d(&mapD, stg, t.n0 + cb * COLS + p * BOXC, t.m0 + qd * 32, t.q * slices + t.s);
                    bulk_commit();
                }
            }
        }
        if (lane == 0) bulk_wait_all();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

}  // namespace tc
}  // namespace wino
