// K2 / K6 with the operand chunk resident in tensor memory (128 < ncols <= 512).
//
//   Y(r, t) = Σ_{e ∈ row r} v_e · X(col_e, t)      (sparse.cpp:51-69; layer.cpp:145-155 on the mask)
//
// The shared-memory SpMM (wino_kernels.cuh) delivers 4 bytes of X per multiply-add through the
// LSU pipe (~100 B/clk/SM for LDS.128), which caps it at ~25 multiply-adds/clk/SM.  TMEM reads
// (tcgen05.ld.32x32b.x4: 4 columns of a warp's 32 lanes) sustain ~156 B/clk/SM, but only with
// four columns per lane and nonzero, i.e. 4 consecutive t per lane -> 128 c of a 512-column TMEM.
// So the X chunk of all ncols rows is spread over the lane quarters by STAGE:
//
//   S = ncols <= 256 ? 2 : 4 stages, stage j holds c ∈ [128j, 128j + 128);  TB = 4/S t-blocks,
//   chunk width TW = 128·TB.  Lane quarter q = warp & 3 holds stage j = q / TB, t-block b = q % TB:
//   TMEM lane 32q + l, columns 4c' .. 4c'+3  =  X(128j + c', t0 + 128b + 4l .. +3).
//
// A row's walk over its (column-sorted) CSR entries therefore passes through the S stages in
// order: the warp of stage j applies the row's entries with c in stage j's range and hands its
// accumulators (4 per lane) to the warp of stage j+1 through a shared-memory slot ring (mbarrier
// full/empty).  Every output element is still one thread's left-to-right sum from +0 in CSR order
// with each product rounded before the add (FFMA2 with a -0 addend = the rounded product, then
// FADD2) — bitwise the reference's order and the shared-memory kernel.
//
// Persistent CTAs, one per SM (the whole TMEM), 16 warps: warp w = (quarter w & 3, row set w >> 2);
// chain (t-block b, row set g) = the S warps that process rows r ≡ g (mod 4) for t-block b.  A
// unit = (slice, chunk); its X chunk is written into TMEM by every warp for its own quarter
// (coalesced 16-byte loads, tcgen05.st.32x32b.x16); the unit's slice of the CSR and its per-row
// stage boundaries (precomputed once per CSR structure) are staged in shared memory when they fit,
// else read warp-uniformly through L1.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace wino {
namespace tm {

constexpr int THREADS = 1024;
constexpr int ROWSETS = 8;   // warps per lane quarter
constexpr int TMEM_COLS = 512;
// R = t per lane (tcgen05.ld.32x32b.xR per entry): a stage holds 512 / R input rows
__host__ __device__ constexpr int stage_rows(int R) { return 512 / R; }
// R for an operand of ncols rows (128 < ncols <= 512): 4.  (R = 8 — twice the multiply-adds per
// entry instruction, but 64-row stages, i.e. 4 stages and 3 handoffs per row for 256 rows — was
// measured slower at 80-95% sparsity: c3 90% 536 vs 439 µs; the kernel stays generic in R.)
__host__ __device__ constexpr int lanes_t(int) { return 4; }
__host__ __device__ constexpr int stages_for(int ncols) {
    return (ncols + stage_rows(lanes_t(ncols)) - 1) / stage_rows(lanes_t(ncols)) <= 2 ? 2 : 4;
}
// rows per visit (one handoff per group of rows; measured: 3 for S = 2, 2 for S = 4)
__host__ __device__ constexpr int group_rows(int S) { return S == 2 ? 3 : 2; }
constexpr int SLOTS = 2;  // handoff ring depth per (chain, stage boundary), in row groups
// a row group's slot: group_rows x 32 lanes x R floats
__host__ __device__ constexpr int slot_bytes(int R, int S) { return 128 * R * group_rows(S); }
// handoff slots: chains x (S-1) boundaries x SLOTS
__host__ __device__ constexpr int handoff_slots(int S) { return (4 / S) * ROWSETS * (S - 1) * SLOTS; }
// handoff ring + barriers, then (STAGED) the slice's stage boundaries and its CSR entries
__host__ __device__ constexpr int smem_fixed(int R, int S) { return handoff_slots(S) * (slot_bytes(R, S) + 16) + 16; }
__host__ __device__ constexpr int smem_bytes(int R, int S, int nrows, int64_t entries) {
    return smem_fixed(R, S) + ((nrows * (S + 1) + 3) & ~3) * 4 + (int)(entries * 8);
}
// > half the SM's shared memory: one CTA per SM (it owns all 512 TMEM columns)
constexpr int kMinSmem = 120 * 1024;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}" ::"r"(su32(b))
                 : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n\t}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}

// the same on 32-bit shared addresses (precomputed once per warp: the row loop stays lean)
__device__ __forceinline__ void mb_arrive_a(uint32_t a) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}" ::"r"(a)
                 : "memory");
}
__device__ __forceinline__ void mb_wait_a(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n\t}" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void sts4(uint32_t a, unsigned long long lo, unsigned long long hi) {
    asm volatile("st.shared.v2.b64 [%0], {%1, %2};" ::"r"(a), "l"(lo), "l"(hi) : "memory");
}
__device__ __forceinline__ void lds4(uint32_t a, unsigned long long& lo, unsigned long long& hi) {
    asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "r"(a) : "memory");
}

__device__ __forceinline__ void tld4(uint32_t taddr, float (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
                 : "r"(taddr));
}
__device__ __forceinline__ void tld8(uint32_t taddr, float (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "r"(taddr));
}
template <int R>
__device__ __forceinline__ void tld(uint32_t taddr, float (&v)[R]) {
    if constexpr (R == 8) tld8(taddr, v);
    else tld4(taddr, v);
}
__device__ __forceinline__ void tst16(uint32_t taddr, const float4 (&v)[4]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "f"(v[0].x), "f"(v[0].y), "f"(v[0].z), "f"(v[0].w), "f"(v[1].x), "f"(v[1].y), "f"(v[1].z), "f"(v[1].w),
        "f"(v[2].x), "f"(v[2].y), "f"(v[2].z), "f"(v[2].w), "f"(v[3].x), "f"(v[3].y), "f"(v[3].z), "f"(v[3].w)
        : "memory");
}

__device__ __forceinline__ int4 ldg_pair(const int2* p) {
    int4 v;
    asm volatile("ld.global.nc.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ int2 ldg_one(const int2* p) {
    int2 v;
    asm volatile("ld.global.nc.v2.s32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}

// acc += round(w·x) for two lanes' t at once: FFMA2 with the runtime -0 addend z is the rounded
// product (ptxas cannot fuse it with the add), FADD2 the reference's rounded sum.
__device__ __forceinline__ void madd2(unsigned long long& acc, float w, float x0, float x1, unsigned long long z) {
    unsigned long long xv, wv, pr;
    asm("mov.b64 %0, {%1,%2};" : "=l"(xv) : "f"(x0), "f"(x1));
    asm("mov.b64 %0, {%1,%1};" : "=l"(wv) : "f"(w));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(pr) : "l"(xv), "l"(wv), "l"(z));
    asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(pr));
}

// ---- the kernel's operand stream: per (slice, row, stage) segments ----
// For every (slice, row) and stage j the row's entries with col in stage j's rows [jW, jW + W)
// (W = 512 / R), in CSR order, as (TMEM column R·(col − jW), value), each segment padded to an even length with (the
// segment's last column, +0) — an exact no-op for finite operands (the accumulator starts at +0
// and is never -0, so adding ±0 leaves it unchanged) — so every segment starts on a 16-byte
// entry pair.  tbnd[(s·nrows + r)·(S+1) + j] = start of segment j (j = S: the row's end), global
// positions in the stream; tpidx = source entry of each stream entry (-1: pad), for value refreshes.
__global__ void tm_count_kernel(const int* __restrict__ rowptr, const int2* __restrict__ cv, int nrows, int P2,
                                int S, int R, int* __restrict__ cnt) {
    const int swc = 512 / R;
    const int64_t total = (int64_t)P2 * nrows;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(i / nrows), r = (int)(i - (int64_t)s * nrows);
        const int e0 = rowptr[(int64_t)s * (nrows + 1) + r], e1 = rowptr[(int64_t)s * (nrows + 1) + r + 1];
        int n = 0, j = 0, len = 0;
        for (int e = e0; e < e1; ++e) {
            const int sj = cv[e].x / swc;
            if (sj != j) {
                n += (len + 1) & ~1;
                len = 0;
                j = sj;
            }
            ++len;
        }
        cnt[i] = n + ((len + 1) & ~1);
    }
}

// in-place exclusive scan of cnt[0..n) (one block of 1024 threads); cnt[n] = the total
__global__ void __launch_bounds__(1024) tm_scan_kernel(int* __restrict__ cnt, int n) {
    __shared__ int part[1024];
    const int per = (n + 1023) / 1024;
    const int a = threadIdx.x * per, b = min(n, a + per);
    int s = 0;
    for (int i = a; i < b; ++i) s += cnt[i];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const int v = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    int run = part[threadIdx.x] - s;
    for (int i = a; i < b; ++i) {
        const int c = cnt[i];
        cnt[i] = run;
        run += c;
    }
    if (threadIdx.x == 1023) cnt[n] = part[1023];
}

__global__ void tm_fill_kernel(const int* __restrict__ rowptr, const int2* __restrict__ cv,
                               const int* __restrict__ off, int nrows, int P2, int S, int R, int2* __restrict__ tcv,
                               int* __restrict__ tpidx, int* __restrict__ tbnd) {
    const int swc = 512 / R;
    const int64_t total = (int64_t)P2 * nrows;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(i / nrows), r = (int)(i - (int64_t)s * nrows);
        const int e0 = rowptr[(int64_t)s * (nrows + 1) + r], e1 = rowptr[(int64_t)s * (nrows + 1) + r + 1];
        int* b = tbnd + i * (S + 1);
        int pos = off[i];
        int e = e0;
        for (int j = 0; j < S; ++j) {
            b[j] = pos;
            int last = 0, len = 0;
            for (; e < e1 && cv[e].x / swc == j; ++e, ++len) {
                last = R * (cv[e].x % swc);
                tcv[pos] = make_int2(last, cv[e].y);
                tpidx[pos++] = e;
            }
            if (len & 1) {
                tcv[pos] = make_int2(last, 0);
                tpidx[pos++] = -1;
            }
        }
        b[S] = pos;
    }
}

// new values (same structure): stream entries take the value of their source entry
__global__ void tm_refresh_kernel(int2* __restrict__ tcv, const int* __restrict__ tpidx, const int2* __restrict__ cv,
                                  int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int e = tpidx[i];
        if (e >= 0) tcv[i].y = cv[e].y;
    }
}

// (col, value) entries from the staged slice in shared memory or warp-uniformly from global
template <bool STAGED>
__device__ __forceinline__ int4 fetch_pair(const int2* p) {
    if constexpr (STAGED) return *reinterpret_cast<const int4*>(p);
    else return ldg_pair(p);
}
template <bool STAGED>
__device__ __forceinline__ int2 fetch_one(const int2* p) {
    if constexpr (STAGED) return *p;
    else return ldg_one(p);
}

// NB entries of the stream from e (NB, e even): their TMEM reads in flight together, one wait
template <int NB, int R, bool STAGED>
__device__ __forceinline__ void batch(const int2* __restrict__ cv, int e, uint32_t tq,
                                      unsigned long long (&acc)[R / 2], unsigned long long z) {
    int2 a[NB];
#pragma unroll
    for (int u = 0; u < NB; u += 2) {
        const int4 two = fetch_pair<STAGED>(cv + e + u);
        a[u] = make_int2(two.x, two.y);
        a[u + 1] = make_int2(two.z, two.w);
    }
    float x[NB][R];
#pragma unroll
    for (int u = 0; u < NB; ++u) tld<R>(tq + (uint32_t)a[u].x, x[u]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int u = 0; u < NB; ++u)
#pragma unroll
        for (int h = 0; h < R / 2; ++h) madd2(acc[h], __int_as_float(a[u].y), x[u][2 * h], x[u][2 * h + 1], z);
}

// One row segment [e, ee) of a stage (e, ee even): acc (R t per lane as R/2 packed pairs) += the
// entries' rounded products in order: batches of 8 and a final 6, 4 or 2 (R = 4); batches of 4
// and a final 2 (R = 8: the same registers per batch)
template <int R, bool STAGED>
__device__ __forceinline__ void walk(const int2* __restrict__ cv, int e, int ee, uint32_t tq,
                                     unsigned long long (&acc)[R / 2], unsigned long long z) {
    if constexpr (R == 4) {
        for (; e + 8 <= ee; e += 8) batch<8, 4, STAGED>(cv, e, tq, acc, z);
        const int rem = ee - e;
        if (rem == 6) batch<6, 4, STAGED>(cv, e, tq, acc, z);
        else if (rem == 4) batch<4, 4, STAGED>(cv, e, tq, acc, z);
        else if (rem == 2) batch<2, 4, STAGED>(cv, e, tq, acc, z);
    } else {
        for (; e + 4 <= ee; e += 4) batch<4, 8, STAGED>(cv, e, tq, acc, z);
        if (e < ee) batch<2, 8, STAGED>(cv, e, tq, acc, z);
    }
}

// R floats of the handoff slot / the output row per lane, as R/2 packed pairs
template <int R>
__device__ __forceinline__ void sts_acc(uint32_t a, const unsigned long long (&acc)[R / 2]) {
#pragma unroll
    for (int h = 0; h < R / 4; ++h) sts4(a + 16 * h, acc[2 * h], acc[2 * h + 1]);
}
template <int R>
__device__ __forceinline__ void lds_acc(uint32_t a, unsigned long long (&acc)[R / 2]) {
#pragma unroll
    for (int h = 0; h < R / 4; ++h) lds4(a + 16 * h, acc[2 * h], acc[2 * h + 1]);
}
template <int R>
__device__ __forceinline__ void stg_acc(float* y, const unsigned long long (&acc)[R / 2]) {
#pragma unroll
    for (int h = 0; h < R / 4; ++h) {
        float4 o;
        asm("mov.b64 {%0,%1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(acc[2 * h]));
        asm("mov.b64 {%0,%1}, %2;" : "=f"(o.z), "=f"(o.w) : "l"(acc[2 * h + 1]));
        *reinterpret_cast<float4*>(y + 4 * h) = o;
    }
}

// X, Y: [P2][ncols or nrows][NTs] (offset to a column range's first column; NTr = owned columns),
// cv / bnd: the padded stage-segment stream and its segment starts (tm_fill_kernel), units =
// P2 · chunks, z = -0.0f pair.  STAGED: each unit copies its slice of the stream (and the slice's
// segment starts) into shared memory; otherwise both are read through L1.
template <int R, int S, bool STAGED>
__global__ void __launch_bounds__(THREADS, 1)
spmm_tmem_kernel(const int2* __restrict__ cv, const int* __restrict__ bnd,
                 const float* __restrict__ X, float* __restrict__ Y, int nrows, int ncols, int NTs, int NTr,
                 int chunks, int units, unsigned long long z) {
    constexpr int TB = 4 / S;
    constexpr int SWC = stage_rows(R);          // input rows per stage
    constexpr int QT = 32 * R;                  // t per lane quarter
    constexpr int TW = QT * TB;                 // chunk width
    constexpr int FILL_C = SWC / ROWSETS;       // stage rows each warp writes into TMEM
    constexpr int NSLOT = handoff_slots(S);
    constexpr int GR = group_rows(S);
    constexpr int SLOT_BYTES = slot_bytes(R, S);
    constexpr int RB = 128 * R;                 // one row's part of a slot
    static_assert(FILL_C * R == 64, "fill: 16 float4 per lane");
    extern __shared__ __align__(16) uint8_t tm_smem[];
    // [NSLOT][GR rows][32 lanes][R floats] handoff slots at tm_smem (addressed through slot_in / slot_out)
    uint64_t* full = reinterpret_cast<uint64_t*>(tm_smem + NSLOT * SLOT_BYTES);
    uint64_t* empty = full + NSLOT;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(empty + NSLOT);
    int* sbnd = reinterpret_cast<int*>(tm_smem + NSLOT * (SLOT_BYTES + 16) + 16);  // [nrows][S+1]
    int2* scv = reinterpret_cast<int2*>(sbnd + ((nrows * (S + 1) + 3) & ~3));     // slice entries
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = warp & 3, g = warp >> 2;
    const int st = q / TB, b = q % TB;
    if (threadIdx.x < NSLOT) {
        mb_init(&full[threadIdx.x], 32);  // every lane arrives after its own slot access
        mb_init(&empty[threadIdx.x], 32);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tq = *tslot + ((uint32_t)(32 * q) << 16);
    // the handoff rings of this warp's chain: into stage st (st > 0) and out of it (st < S-1)
    const int chain = b * ROWSETS + g;
    const int ring_in = (chain * (S - 1) + (st - 1)) * SLOTS;
    const int ring_out = (chain * (S - 1) + st) * SLOTS;
    const uint32_t sbase = su32(tm_smem);
    const uint32_t full_in = sbase + NSLOT * SLOT_BYTES + 8 * ring_in, empty_in = full_in + 8 * NSLOT;
    const uint32_t full_out = sbase + NSLOT * SLOT_BYTES + 8 * ring_out, empty_out = full_out + 8 * NSLOT;
    const uint32_t slot_in = sbase + ring_in * SLOT_BYTES + 4 * R * lane;
    const uint32_t slot_out = sbase + ring_out * SLOT_BYTES + 4 * R * lane;
    int nrow_chain = 0;  // row groups this chain has passed through its rings so far (all units)
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int s = u / chunks, ch = u - s * chunks;
        const int t = ch * TW + QT * b + R * lane;  // this lane's R columns
        const bool tok = t < NTr;
        // ---- stage the slice's boundaries and entries (cp.async, overlaps the fill) ----
        const int* bs = bnd + (int64_t)s * nrows * (S + 1);
        const int e_lo = STAGED ? __ldg(bs) : 0;  // even
        if constexpr (STAGED) {
            const int nb = nrows * (S + 1);
            for (int i = threadIdx.x; i < nb; i += THREADS) sbnd[i] = __ldg(bs + i);
            const int e_hi = __ldg(bs + nb - 1);  // even
            const int n2 = (e_hi - e_lo) >> 1;      // whole 16-byte pairs
            const int4* src = reinterpret_cast<const int4*>(cv + e_lo);
            int4* dst = reinterpret_cast<int4*>(scv);
            for (int i = threadIdx.x; i < n2; i += THREADS) {
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst + i)), "l"(src + i));
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        // ---- fill: X(SWC·st + c', t .. t+R) for this warp's FILL_C rows c' -> TMEM columns R·c' ----
        // (16 float4 per lane; float4 f = row FILL_C·g + f / (R/4), part f % (R/4), column 4f + R·FILL_C·g)
        {
            const int c0 = SWC * st + FILL_C * g;
            const float* xs = X + ((int64_t)s * ncols + c0) * NTs + t;
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                float4 v[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int f = 4 * h + i, cl = f / (R / 4), pt = f % (R / 4);
                    v[i] = (tok && c0 + cl < ncols)
                               ? __ldg(reinterpret_cast<const float4*>(xs + (int64_t)cl * NTs + 4 * pt))
                               : make_float4(0.f, 0.f, 0.f, 0.f);
                }
                tst16(tq + (uint32_t)(R * FILL_C * g + 16 * h), v);
            }
        }
        if constexpr (STAGED) asm volatile("cp.async.wait_all;" ::: "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // ---- the next unit's chunk rows of this warp: L2 prefetch behind this unit's compute ----
        if (u + (int)gridDim.x < units && lane < FILL_C) {
            const int un = u + gridDim.x, sn = un / chunks, chn = un - sn * chunks;
            const int cl = SWC * st + FILL_C * g + lane, tn = chn * TW + QT * b;
            if (cl < ncols && tn < NTr) {
                const float* src = X + ((int64_t)sn * ncols + cl) * NTs + tn;
                const int bytes = 4 * min(QT, NTr - tn);  // multiple of 16
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
            }
        }
        // ---- rows of this chain, in groups (r, r + ROWSETS, ...): one handoff per group ----
        const int* rbp = (STAGED ? sbnd : bs) + g * (S + 1) + st;  // this warp's rows' segment starts
        const int2* cvb = STAGED ? scv - e_lo : cv;               // indexed by global entry numbers
        float* yp = Y + ((int64_t)s * nrows + g) * NTs + t;
        constexpr int PB = ROWSETS * (S + 1);  // segment-start stride between a group's rows
        if constexpr (GR == 2) {
            for (int r = g; r < nrows;
                 r += 2 * ROWSETS, ++nrow_chain, rbp += 2 * PB, yp += 2 * ROWSETS * (int64_t)NTs) {
                const uint32_t k = (uint32_t)nrow_chain & (SLOTS - 1);
                const uint32_t par = (uint32_t)(nrow_chain / SLOTS) & 1u;
                const bool hasb = r + ROWSETS < nrows;
                const int ea = rbp[0], eea = rbp[1];
                const int eb = hasb ? rbp[PB] : 0, eeb = hasb ? rbp[PB + 1] : 0;
                unsigned long long acca[R / 2], accb[R / 2];
#pragma unroll
                for (int h = 0; h < R / 2; ++h) acca[h] = accb[h] = 0ull;
                if (st > 0) {  // the previous stage's accumulators for these rows
                    mb_wait_a(full_in + 8 * k, par);
                    lds_acc<R>(slot_in + SLOT_BYTES * k, acca);
                    lds_acc<R>(slot_in + SLOT_BYTES * k + RB, accb);
                    mb_arrive_a(empty_in + 8 * k);
                }
                walk<R, STAGED>(cvb, ea, eea, tq, acca, z);
                walk<R, STAGED>(cvb, eb, eeb, tq, accb, z);
                if (st == S - 1) {
                    if (tok) {
                        stg_acc<R>(yp, acca);
                        if (hasb) stg_acc<R>(yp + ROWSETS * (int64_t)NTs, accb);
                    }
                } else {
                    if (nrow_chain >= SLOTS) mb_wait_a(empty_out + 8 * k, par ^ 1u);
                    sts_acc<R>(slot_out + SLOT_BYTES * k, acca);
                    sts_acc<R>(slot_out + SLOT_BYTES * k + RB, accb);
                    mb_arrive_a(full_out + 8 * k);
                }
            }
        } else {
            for (int r = g; r < nrows;
                 r += GR * ROWSETS, ++nrow_chain, rbp += GR * PB, yp += GR * ROWSETS * (int64_t)NTs) {
                const uint32_t k = (uint32_t)nrow_chain & (SLOTS - 1);
                const uint32_t par = (uint32_t)(nrow_chain / SLOTS) & 1u;
                unsigned long long acc[GR][R / 2];
#pragma unroll
                for (int i = 0; i < GR; ++i)
#pragma unroll
                    for (int h = 0; h < R / 2; ++h) acc[i][h] = 0ull;
                if (st > 0) {  // the previous stage's accumulators for these rows
                    mb_wait_a(full_in + 8 * k, par);
#pragma unroll
                    for (int i = 0; i < GR; ++i) lds_acc<R>(slot_in + SLOT_BYTES * k + RB * i, acc[i]);
                    mb_arrive_a(empty_in + 8 * k);
                }
#pragma unroll
                for (int i = 0; i < GR; ++i) {
                    const bool has = r + i * ROWSETS < nrows;
                    walk<R, STAGED>(cvb, has ? rbp[i * PB] : 0, has ? rbp[i * PB + 1] : 0, tq, acc[i], z);
                }
                if (st == S - 1) {
                    if (tok) {
#pragma unroll
                        for (int i = 0; i < GR; ++i)
                            if (r + i * ROWSETS < nrows) stg_acc<R>(yp + i * ROWSETS * (int64_t)NTs, acc[i]);
                    }
                } else {
                    if (nrow_chain >= SLOTS) mb_wait_a(empty_out + 8 * k, par ^ 1u);
#pragma unroll
                    for (int i = 0; i < GR; ++i) sts_acc<R>(slot_out + SLOT_BYTES * k + RB * i, acc[i]);
                    mb_arrive_a(full_out + 8 * k);
                }
            }
        }
        // every warp is done reading this chunk (and the staged slice) before the next unit
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tslot), "r"(TMEM_COLS));
}


// ---------------------------------------------------------------------------------------------
// K2 / K6, hybrid operand delivery (128 < ncols <= 256): input rows [0, 128) of the chunk in
// tensor memory, rows [128, ncols) in shared memory.  The staged kernel above is bound by what the
// TMEM read path delivers (every multiply-add needs its own 4-byte operand) and pays a handoff per
// (row, stage); here the two operand halves come through two different pipes (tcgen05.ld and LDS)
// and ONE warp walks a whole row: its stage-0 segment against TMEM, its stage-1 segment against
// shared memory, the same accumulators throughout — no handoff ring, no barriers inside a unit.
// Same operand stream (tm_fill_kernel, S = 2) and the same per-element operation order: bitwise
// the staged kernel, the shared-memory kernel and the reference.
//
// Chunk = 256 t (two 128-t blocks).  Warp w: lane quarter q = w & 3, t-block b = q & 1, row set
// g = (w >> 2) + 8·(q >> 1) of 16.  A warp only reads its own lane quarter of TMEM, so quarters
// q and q + 2 hold the same block b of rows [0, 128): TMEM lane 32q + l, columns 4c .. 4c+3 =
// X(c, t0 + 128b + 4l .. +3).  Shared memory: xs[c − 128][256] floats (a warp's LDS.128 reads 512
// contiguous bytes: conflict-free).
// ---------------------------------------------------------------------------------------------
constexpr int HYB_TW = 256;
__host__ __device__ constexpr int hyb_x_bytes(int ncols) { return (ncols - 128) * HYB_TW * 4; }
__host__ __device__ constexpr int hyb_smem_fixed(int ncols) { return hyb_x_bytes(ncols) + 16; }
__host__ __device__ constexpr int hyb_smem_bytes(int ncols, int nrows, int64_t entries) {
    return hyb_smem_fixed(ncols) + ((nrows * 3 + 3) & ~3) * 4 + (int)(entries * 8);
}

// NB stream entries from e against the shared-memory rows: xl = this lane's 16 bytes of row 128
template <int NB, bool STAGED>
__device__ __forceinline__ void batch_sm(const int2* __restrict__ cv, int e, uint32_t xl,
                                         unsigned long long (&acc)[2], unsigned long long z) {
    int2 a[NB];
#pragma unroll
    for (int u = 0; u < NB; u += 2) {
        const int4 two = fetch_pair<STAGED>(cv + e + u);
        a[u] = make_int2(two.x, two.y);
        a[u + 1] = make_int2(two.z, two.w);
    }
    float x[NB][4];
#pragma unroll
    for (int u = 0; u < NB; ++u) {  // stream column = 4·(c − 128): row stride 1024 bytes
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(x[u][0]), "=f"(x[u][1]), "=f"(x[u][2]), "=f"(x[u][3])
                     : "r"(xl + ((uint32_t)a[u].x << 8)));
    }
#pragma unroll
    for (int u = 0; u < NB; ++u)
#pragma unroll
        for (int h = 0; h < 2; ++h) madd2(acc[h], __int_as_float(a[u].y), x[u][2 * h], x[u][2 * h + 1], z);
}

template <bool STAGED>
__device__ __forceinline__ void walk_sm(const int2* __restrict__ cv, int e, int ee, uint32_t xl,
                                        unsigned long long (&acc)[2], unsigned long long z) {
    for (; e + 8 <= ee; e += 8) batch_sm<8, STAGED>(cv, e, xl, acc, z);
    const int rem = ee - e;
    if (rem == 6) batch_sm<6, STAGED>(cv, e, xl, acc, z);
    else if (rem == 4) batch_sm<4, STAGED>(cv, e, xl, acc, z);
    else if (rem == 2) batch_sm<2, STAGED>(cv, e, xl, acc, z);
}

template <bool STAGED>
__global__ void __launch_bounds__(THREADS, 1)
spmm_hyb_kernel(const int2* __restrict__ cv, const int* __restrict__ bnd, const float* __restrict__ X,
                float* __restrict__ Y, int nrows, int ncols, int NTs, int NTr, int chunks, int units,
                unsigned long long z) {
    constexpr int R = 4, QT = 128, TW = HYB_TW, FILL_C = 16, NSETS = 16;
    extern __shared__ __align__(16) uint8_t tm_smem[];
    const int xbytes = hyb_x_bytes(ncols);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tm_smem + xbytes);
    int* sbnd = reinterpret_cast<int*>(tm_smem + xbytes + 16);    // [nrows][3]
    int2* scv = reinterpret_cast<int2*>(sbnd + ((nrows * 3 + 3) & ~3));  // slice entries
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = warp & 3, b = q & 1, wq = warp >> 2;
    const int g = wq + 8 * (q >> 1);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tq = *tslot + ((uint32_t)(32 * q) << 16);
    const uint32_t xl = su32(tm_smem) + 4 * (QT * b + R * lane);
    const int nsm = ncols - 128;  // rows held in shared memory
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int s = u / chunks, ch = u - s * chunks;
        const int t = ch * TW + QT * b + R * lane;  // this lane's 4 columns
        const bool tok = t < NTr;
        const int* bs = bnd + (int64_t)s * nrows * 3;
        const int e_lo = STAGED ? __ldg(bs) : 0;                    // even
        const int e_hi = STAGED ? __ldg(bs + nrows * 3 - 1) : 0;     // even
        const float* xs = X + (int64_t)s * ncols * NTs;
        // ---- rows [128, ncols) of the chunk -> shared memory (cp.async, zero-filled past NTr) ----
        for (int i = threadIdx.x; i < nsm * (TW / 4); i += THREADS) {
            const int row = i >> 6, c4 = i & 63;
            const int tt = ch * TW + 4 * c4;
            const bool ok = tt < NTr;
            const float* src = xs + (int64_t)(128 + row) * NTs + (ok ? tt : 0);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su32(tm_smem) + 16 * i), "l"(src),
                         "r"(ok ? 16 : 0));
        }
        if constexpr (STAGED) {
            const int nb = nrows * 3;
            for (int i = threadIdx.x; i < nb; i += THREADS)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(su32(sbnd + i)), "l"(bs + i));
            const int n2 = (e_hi - e_lo) >> 1;  // whole 16-byte pairs
            const int4* src = reinterpret_cast<const int4*>(cv + e_lo);
            int4* dst = reinterpret_cast<int4*>(scv);
            for (int i = threadIdx.x; i < n2; i += THREADS)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst + i)), "l"(src + i));
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        // ---- rows [0, 128) -> this warp's lane quarter: its 16 rows c0 .. c0+15, 16 float4 per lane ----
        {
            const int c0 = FILL_C * wq;
            const float* xr = xs + (int64_t)c0 * NTs + t;
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                float4 v[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    v[i] = tok ? __ldg(reinterpret_cast<const float4*>(xr + (int64_t)(4 * h + i) * NTs))
                               : make_float4(0.f, 0.f, 0.f, 0.f);
                tst16(tq + (uint32_t)(R * c0 + 16 * h), v);
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // ---- the next unit's chunk: L2 prefetch behind this unit's compute (quarters 0,1: the TMEM
        //      rows, quarters 2,3: the shared-memory rows) ----
        if (u + (int)gridDim.x < units) {  // 16 rows x 512 bytes per warp: two 128-byte lines per lane
            const int un = u + gridDim.x, sn = un / chunks, chn = un - sn * chunks;
            const int cl = 128 * (q >> 1) + FILL_C * wq + (lane >> 1), tn = chn * TW + QT * b + 64 * (lane & 1);
            if (cl < ncols) {
                const float* src = X + ((int64_t)sn * ncols + cl) * NTs + tn;
                if (tn < NTr) asm volatile("prefetch.global.L2 [%0];" ::"l"(src));
                if (tn + 32 < NTr) asm volatile("prefetch.global.L2 [%0];" ::"l"(src + 32));
            }
        }
        // ---- rows g, g + 16, ...: stage-0 segment from TMEM, stage-1 segment from shared memory ----
        const int* rbp = (STAGED ? sbnd : bs) + g * 3;
        const int2* cvb = STAGED ? scv - e_lo : cv;  // indexed by global entry numbers
        float* yp = Y + ((int64_t)s * nrows + g) * NTs + t;
        for (int r = g; r < nrows; r += NSETS, rbp += 3 * NSETS, yp += NSETS * (int64_t)NTs) {
            const int e0 = rbp[0], e1 = rbp[1], e2 = rbp[2];
            unsigned long long acc[2] = {0ull, 0ull};
            walk<4, STAGED>(cvb, e0, e1, tq, acc, z);
            walk_sm<STAGED>(cvb, e1, e2, xl, acc, z);
            if (tok) stg_acc<4>(yp, acc);
        }
        // every warp is done reading this chunk (and the staged slice) before the next unit
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tslot), "r"(TMEM_COLS));
}

}  // namespace tm
}  // namespace wino
