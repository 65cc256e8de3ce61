// Microbenchmark: SpMM inner loop with the operand rows split between TMEM and shared memory.
// Per nonzero a warp reads a warp-uniform (column, value) pair from a shared-memory broadcast,
// then its lanes' XT operand values from TMEM (tcgen05.ld.32x32b.xXT at column c·XT of the warp's
// lane quarter) and RS values from shared memory (row c of the quarter's region), and does
// XT+RS multiply-then-add steps (no FMA contraction, as the reference-order SpMM).  Reports
// multiply-adds per clock per SM; XT=0 is the shared-memory-only kernel of round 1.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o spmm_hybrid_bw spmm_hybrid_bw.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e = (x);                                                           \
        if (e != cudaSuccess) {                                                        \
            printf("%s: %s\n", #x, cudaGetErrorString(e));                             \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

template <int X>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float (&v)[X]) {
    if constexpr (X == 1)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=f"(v[0]) : "r"(taddr));
    else if constexpr (X == 2)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=f"(v[0]), "=f"(v[1]) : "r"(taddr));
    else if constexpr (X == 4)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
                     : "r"(taddr));
}

template <int R>
__device__ __forceinline__ void lds(const float* p, float (&v)[R]) {
    if constexpr (R == 4) {
        const float4 q = *reinterpret_cast<const float4*>(p);
        v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w;
    } else if constexpr (R == 2) {
        const float2 q = *reinterpret_cast<const float2*>(p);
        v[0] = q.x, v[1] = q.y;
    } else if constexpr (R == 1) {
        v[0] = *p;
    }
}

// C rows; shared memory: CSR-like stream int2[1024] + rows [C][4 quarters][32 lanes][RS]
// P2: paired math — FFMA2 with a runtime -0 addend (the exact rounded product; ptxas would fuse
// mul.rn.f32x2 + add.rn.f32x2 into FFMA2) followed by FADD2: one instruction per two lanes' t.
__device__ __forceinline__ void madd2(float& a0, float& a1, float w, float x0, float x1, unsigned long long z) {
    unsigned long long acc, xv, wv, p;
    asm("mov.b64 %0, {%1,%2};" : "=l"(acc) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1,%2};" : "=l"(xv) : "f"(x0), "f"(x1));
    asm("mov.b64 %0, {%1,%1};" : "=l"(wv) : "f"(w));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(xv), "l"(wv), "l"(z));
    asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(p));
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a0), "=f"(a1) : "l"(acc));
}

template <int XT, int RS, int U, int C, bool P2 = false>
__global__ void __launch_bounds__(1024, 1) hyb_kernel(const int2* __restrict__ cv_g, int iters, float* out,
                                                      unsigned long long z) {
    extern __shared__ __align__(16) float sm[];
    int2* cvs = reinterpret_cast<int2*>(sm);
    float* xs = sm + 2048;
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, qd = warp & 3;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) cvs[i] = cv_g[i];
    for (int i = threadIdx.x; i < C * 128 * RS; i += blockDim.x) xs[i] = (float)(i & 1023) * 1e-3f;
    if constexpr (XT > 0) {
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                (uint32_t)__cvta_generic_to_shared(&tbase)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = XT > 0 ? tbase + ((uint32_t)(qd * 32) << 16) : 0u;
    const float* xl = xs + (qd * 32 + lane) * RS;
    float acc[XT + RS];
#pragma unroll
    for (int j = 0; j < XT + RS; ++j) acc[j] = 0.f;
    for (int it = 0; it < iters; it += U) {
        int2 cv[U];
#pragma unroll
        for (int u = 0; u < U; u += 2) {
            const int4 two = *reinterpret_cast<const int4*>(cvs + ((it + u + warp * 2) & 1023));
            cv[u] = make_int2(two.x, two.y);
            cv[u + 1] = make_int2(two.z, two.w);
        }
        float vt[U][XT > 0 ? XT : 1], vs[U][RS > 0 ? RS : 1];
        if constexpr (XT > 0) {
#pragma unroll
            for (int u = 0; u < U; ++u) tmem_ld<XT>(base + (uint32_t)(cv[u].x * XT), vt[u]);
        }
        if constexpr (RS > 0) {
#pragma unroll
            for (int u = 0; u < U; ++u) lds<RS>(xl + cv[u].x * (128 * RS), vs[u]);
        }
        if constexpr (XT > 0) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const float w = __int_as_float(cv[u].y);
            if constexpr (P2) {
#pragma unroll
                for (int j = 0; j < XT; j += 2) madd2(acc[j], acc[j + 1], w, vt[u][j], vt[u][j + 1], z);
#pragma unroll
                for (int j = 0; j < RS; j += 2)
                    madd2(acc[XT + j], acc[XT + j + 1], w, vs[u][j], vs[u][j + 1], z);
            } else {
#pragma unroll
                for (int j = 0; j < XT; ++j) acc[j] = __fadd_rn(acc[j], __fmul_rn(w, vt[u][j]));
#pragma unroll
                for (int j = 0; j < RS; ++j) acc[XT + j] = __fadd_rn(acc[XT + j], __fmul_rn(w, vs[u][j]));
            }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < XT + RS; ++j) s += acc[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if constexpr (XT > 0) {
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
    }
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    int2* cv;
    float* out;
    CK(cudaMalloc(&cv, 1024 * sizeof(int2)));
    CK(cudaMalloc(&out, sms * 1024 * sizeof(float)));
    int2 h[1024];
    for (int i = 0; i < 1024; ++i) h[i] = make_int2((i * 97 + 13) % 64, [](float f) { int r; memcpy(&r, &f, 4); return r; }(0.5f + (i & 7) * 0.01f));
    CK(cudaMemcpy(cv, h, sizeof h, cudaMemcpyHostToDevice));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 1 << 15;
    auto run = [&](const char* name, auto kern, int threads, int macs_per_lane, size_t smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<sms, threads, smem>>>(cv, iters, out, 0x8000000080000000ull);
        cudaEventRecord(a);
        kern<<<sms, threads, smem>>>(cv, iters, out, 0x8000000080000000ull);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaError_t e = cudaGetLastError();
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double macs = (double)sms * threads * iters * macs_per_lane;
        const double cyc = ms * 1e-3 * clk * 1e3;
        printf("%-34s threads=%4d %8.3f ms %7.1f MAC/clk/SM (%s)\n", name, threads, ms, macs / cyc / sms,
               e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    };
    const size_t cvb = 2048 * 4;
    for (int th : {512, 1024}) {
        run("smem only R=4 (round 1)", hyb_kernel<0, 4, 8, 64>, th, 4, cvb + 64 * 128 * 4 * 4);
        run("smem only R=2", hyb_kernel<0, 2, 8, 64>, th, 2, cvb + 64 * 128 * 2 * 4);
        run("tmem only x2", hyb_kernel<2, 0, 8, 128>, th, 2, cvb);
        run("tmem only x4", hyb_kernel<4, 0, 8, 128>, th, 4, cvb);
        run("tmem x2 + smem R=1", hyb_kernel<2, 1, 8, 64>, th, 3, cvb + 64 * 128 * 1 * 4);
        run("tmem x2 + smem R=2", hyb_kernel<2, 2, 8, 64>, th, 4, cvb + 64 * 128 * 2 * 4);
        run("tmem x4 + smem R=2", hyb_kernel<4, 2, 8, 64>, th, 6, cvb + 64 * 128 * 2 * 4);
        run("tmem x4 + smem R=4", hyb_kernel<4, 4, 8, 64>, th, 8, cvb + 64 * 128 * 4 * 4);
        run("tmem x1 + smem R=1", hyb_kernel<1, 1, 8, 64>, th, 2, cvb + 64 * 128 * 1 * 4);
        run("P2 smem only R=4", hyb_kernel<0, 4, 8, 64, true>, th, 4, cvb + 64 * 128 * 4 * 4);
        run("P2 tmem only x4", hyb_kernel<4, 0, 8, 128, true>, th, 4, cvb);
        run("P2 tmem x2 + smem R=2", hyb_kernel<2, 2, 8, 64, true>, th, 4, cvb + 64 * 128 * 2 * 4);
        run("P2 tmem x4 + smem R=2", hyb_kernel<4, 2, 8, 64, true>, th, 6, cvb + 64 * 128 * 2 * 4);
        run("P2 tmem x4 + smem R=4", hyb_kernel<4, 4, 8, 64, true>, th, 8, cvb + 64 * 128 * 4 * 4);
        run("P2 tmem x4 + smem R=4 U4", hyb_kernel<4, 4, 4, 64, true>, th, 8, cvb + 64 * 128 * 4 * 4);
    }
    printf("clock %d kHz, %d SMs\n", clk, sms);
    return 0;
}
