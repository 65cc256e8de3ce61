// Throughput of F2F.F64.F32 (fp32 -> fp64 conversion) and DFMA per SM on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o f2f_tput f2f_tput.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void conv_kernel(const float* in, double* out, int iters) {
    float x[8];
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { x[i] = in[(threadIdx.x + i) & 255]; acc[i] = 0.0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            acc[i] = acc[i] * 0.5 + (double)x[i];   // one F2F + one DFMA per element
            x[i] = fmaf(x[i], 1.0001f, 1e-7f);  // a new value every iteration: no conversion can be hoisted
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_kernel(const float* in, double* out, int iters) {
    double acc[8], y[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { y[i] = in[(threadIdx.x + i) & 255]; acc[i] = 0.0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], 0.5, y[i]);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* in; double* out;
    cudaMalloc(&in, 256 * 4); cudaMemset(in, 0, 256 * 4);
    const int threads = 512, blocks = sms * 4, iters = 4096;
    cudaMalloc(&out, (size_t)blocks * threads * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int k = 0; k < 2; ++k) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (k == 0) conv_kernel<<<blocks, threads>>>(in, out, iters);
            else dfma_kernel<<<blocks, threads>>>(in, out, iters);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double ops = (double)blocks * threads * iters * 8;
            double per_clk_sm = ops / (ms * 1e-3) / sms / (clk * 1e3);
            if (rep == 1) printf("%s: %.2f ops/clk/SM (%.3f ms, %d SMs, clock attr %d MHz)\n",
                                 k == 0 ? "F2F.F64.F32 (+DFMA)" : "DFMA", per_clk_sm, ms, sms, clk / 1000);
        }
    }
    return 0;
}
