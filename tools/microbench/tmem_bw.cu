// Microbenchmark: per-SM read throughput of tcgen05.ld (TMEM) vs LDS (shared memory) vs a
// warp-uniform LDG broadcast, for the operand-gather pattern of the CSR SpMM
// (one warp-uniform column/row index per nonzero, each lane reading its own t).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int X>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float (&v)[X]);
template <>
__device__ __forceinline__ void tmem_ld<1>(uint32_t taddr, float (&v)[1]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=f"(v[0]) : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ld<2>(uint32_t taddr, float (&v)[2]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=f"(v[0]), "=f"(v[1]) : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ld<4>(uint32_t taddr, float (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(taddr));
}

template <int X, int UNROLL>
__global__ void __launch_bounds__(512, 1) tmem_kernel(const int* __restrict__ cols, int iters, float* out) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                     :: "r"((uint32_t)__cvta_generic_to_shared(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    float acc = 0.f;
    for (int it = 0; it < iters; it += UNROLL) {
        float v[UNROLL][X];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const int c = __ldg(cols + ((it + u) & 1023));   // warp-uniform "column index"
            tmem_ld<X>(base + (uint32_t)(c * X & 511), v[u]);
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
#pragma unroll
            for (int x = 0; x < X; ++x) acc += v[u][x];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tbase));
}

template <int X, int UNROLL>
__global__ void __launch_bounds__(512, 1) lds_kernel(const int* __restrict__ cols, int iters, float* out) {
    extern __shared__ float sm[];  // 256 rows x 32*X floats
    for (int i = threadIdx.x; i < 256 * 32 * X; i += blockDim.x) sm[i] = (float)i;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    float acc = 0.f;
    for (int it = 0; it < iters; it += UNROLL) {
        float v[UNROLL][X];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const int c = __ldg(cols + ((it + u) & 1023)) & 255;
            const float* p = sm + c * 32 * X + lane * X;
            if constexpr (X == 4) {
                float4 q = *reinterpret_cast<const float4*>(p);
                v[u][0] = q.x; v[u][1] = q.y; v[u][2] = q.z; v[u][3] = q.w;
            } else if constexpr (X == 2) {
                float2 q = *reinterpret_cast<const float2*>(p);
                v[u][0] = q.x; v[u][1] = q.y;
            } else {
                v[u][0] = *p;
            }
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
#pragma unroll
            for (int x = 0; x < X; ++x) acc += v[u][x];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    int* cols;
    float* out;
    CK(cudaMalloc(&cols, 1024 * sizeof(int)));
    CK(cudaMalloc(&out, sms * 512 * sizeof(float)));
    int h[1024];
    for (int i = 0; i < 1024; ++i) h[i] = (i * 97 + 13) % 128;
    CK(cudaMemcpy(cols, h, sizeof h, cudaMemcpyHostToDevice));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 1 << 16;
    auto run = [&](const char* name, auto kern, int threads, int bytes_per_warp_iter, size_t smem) {
        if (smem) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<sms, threads, smem>>>(cols, iters, out);
        cudaEventRecord(a);
        kern<<<sms, threads, smem>>>(cols, iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaError_t e = cudaGetLastError();
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)sms * (threads / 32) * iters * bytes_per_warp_iter;
        const double cyc = ms * 1e-3 * clk * 1e3;
        printf("%-28s threads=%3d  %8.3f ms  %7.1f B/clk/SM  (%s)\n", name, threads, ms, bytes / cyc / sms,
               e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    };
    for (int th : {128, 256, 512}) {
        run("tmem ld 32x32b.x1 u8", tmem_kernel<1, 8>, th, 128, 0);
        run("tmem ld 32x32b.x2 u8", tmem_kernel<2, 8>, th, 256, 0);
        run("tmem ld 32x32b.x4 u4", tmem_kernel<4, 4>, th, 512, 0);
        run("lds.32 u8", lds_kernel<1, 8>, th, 128, 256 * 32 * 4);
        run("lds.64 u8", lds_kernel<2, 8>, th, 256, 256 * 64 * 4);
        run("lds.128 u4", lds_kernel<4, 4>, th, 512, 256 * 128 * 4);
    }
    printf("clock %d kHz, %d SMs\n", clk, sms);
    return 0;
}
