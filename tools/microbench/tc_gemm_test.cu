// Standalone check of the 3xTF32 tcgen05 GEMM (csrc/wino_dense_tc.cuh) against an fp64 CPU GEMM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tc_gemm_test tc_gemm_test.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../../paper_1702_08597_b200/csrc/wino_dense_tc.cuh"
#include "../../paper_1702_08597_b200/csrc/wino_tmap.h"

static float tf32_round(float x) {  // host rna to tf32
    uint32_t u;
    memcpy(&u, &x, 4);
    u = (u + 0x1000u) & 0xFFFFE000u;
    float r;
    memcpy(&r, &u, 4);
    return r;
}

static bool g_flush = false;
static int g_F = 1;
template <bool A, bool B>
auto flush_k() {
    return g_F == 1 ? wino::tc::gemm_3xtf32_flush_kernel<A, B, 1>
         : g_F == 2 ? wino::tc::gemm_3xtf32_flush_kernel<A, B, 2> : wino::tc::gemm_3xtf32_flush_kernel<A, B, 4>;
}
int run(int S, int M, int N, int Kd, bool timeit) {
    const int NTs = (N + 3) / 4 * 4;
    std::mt19937 rng(1234 + M + N + Kd);
    std::normal_distribution<float> nd(0.f, 1.f);
    std::vector<float> A((size_t)S * M * Kd), B((size_t)S * Kd * NTs, 0.f), Ah(A.size()), Al(A.size());
    for (auto& v : A) v = nd(rng);
    for (int s = 0; s < S; ++s)
        for (int k = 0; k < Kd; ++k)
            for (int n = 0; n < N; ++n) B[((size_t)s * Kd + k) * NTs + n] = nd(rng);
    for (size_t i = 0; i < A.size(); ++i) {
        Ah[i] = tf32_round(A[i]);
        Al[i] = tf32_round(A[i] - Ah[i]);
    }
    float *dAh, *dAl, *dB, *dD;
    cudaMalloc(&dAh, A.size() * 4);
    cudaMalloc(&dAl, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD, (size_t)S * M * NTs * 4);
    cudaMemcpy(dAh, Ah.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dAl, Al.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, (size_t)S * M * NTs * 4);
    CUtensorMap mAh, mAl, mB;
    bool ok = wino::make_map_3d(&mAh, dAh, Kd, M, S, (uint64_t)Kd * 4, (uint64_t)M * Kd * 4, 32, 128) &&
              wino::make_map_3d(&mAl, dAl, Kd, M, S, (uint64_t)Kd * 4, (uint64_t)M * Kd * 4, 32, 128) &&
              wino::make_map_3d(&mB, dB, NTs, Kd, S, (uint64_t)NTs * 4, (uint64_t)Kd * NTs * 4, 32, 32, true);
    if (!ok) { printf("tensor map creation failed\n"); return 1; }
    auto kern = g_flush ? flush_k<false, true>() : wino::tc::gemm_3xtf32_kernel<false, true>;
    const int smem = g_flush ? wino::tc::flush::SMEM_BYTES : wino::tc::SMEM_BYTES;
    const int bn = g_flush ? 128 : 256, th = g_flush ? wino::tc::flush::THREADS : 256;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    dim3 grid((NTs + bn - 1) / bn, (M + 127) / 128, S);
    const int kbp = (Kd + 31) / 32;
    kern<<<grid, th, smem>>>(mAh, mAl, mB, dD, M, NTs, Kd, NTs, S, 1, kbp);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("kernel error: %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> D((size_t)S * M * NTs);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    if (M == 128 && N == 256 && S == 1) {
        for (int m = 0; m < 3; ++m)
            for (int n = 0; n < 6; ++n) {
                double ref = 0;
                for (int k = 0; k < Kd; ++k) ref += (double)A[(size_t)m * Kd + k] * B[(size_t)k * NTs + n];
                printf("  D[%d][%d]=% .5f ref=% .5f\n", m, n, D[(size_t)m * NTs + n], ref);
            }
        // which (m, n) does D[0][0] match?
        double d00 = D[0];
        for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
            double ref = 0;
            for (int k = 0; k < Kd; ++k) ref += (double)A[(size_t)m * Kd + k] * B[(size_t)k * NTs + n];
            if (fabs(ref - d00) < 1e-3 * (1 + fabs(d00))) printf("  D[0][0] matches ref[%d][%d]\n", m, n);
        }
        long nz = 0; for (size_t i = 0; i < D.size(); ++i) nz += D[i] != 0.f;
        printf("  nonzero outputs: %ld of %zu\n", nz, D.size());
    }
    double max_err = 0, max_ref = 0, max_rel_tol = 0;
    long bad = 0;
    for (int s = 0; s < S; ++s)
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                double ref = 0, aref = 0;
                for (int k = 0; k < Kd; ++k) {
                    const double p = (double)A[((size_t)s * M + m) * Kd + k] * B[((size_t)s * Kd + k) * NTs + n];
                    ref += p;
                    aref += fabs(p);
                }
                const double got = D[((size_t)s * M + m) * NTs + n];
                const double err = fabs(got - ref);
                max_err = std::max(max_err, err);
                max_ref = std::max(max_ref, fabs(ref));
                max_rel_tol = std::max(max_rel_tol, err / (aref + 1e-30));
                if (err > 1e-5 + 1e-4 * fabs(ref)) ++bad;
            }
    printf("S=%d M=%d N=%d Kd=%d: max|err|=%.3e max|ref|=%.3e max err/sum|p|=%.3e strict-fail=%ld\n", S, M, N, Kd,
           max_err, max_ref, max_rel_tol, bad);
    if (timeit) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        for (int i = 0; i < 10; ++i)
            kern<<<grid, th, smem>>>(mAh, mAl, mB, dD, M, NTs, Kd, NTs, S, 1, kbp);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 10;
        const double flops = 2.0 * S * M * (double)N * Kd;
        printf("  %.3f ms  %.1f TFLOP/s useful (x3 issued)  %.0f GB/s (A+B+D)\n", ms, flops / ms / 1e9,
               (A.size() * 4.0 + B.size() * 4.0 + (double)S * M * NTs * 4) / ms / 1e6);
    }
    cudaFree(dAh); cudaFree(dAl); cudaFree(dB); cudaFree(dD);
    return 0;
}

// dW-style: A raw [S][M][R] (split on the fly), B [S][N][R] (K-major), split-K partials.
int run_kk(int S, int M, int N, int R, int splits) {
    std::mt19937 rng(99 + M + N + R);
    std::normal_distribution<float> nd(0.f, 1.f);
    std::vector<float> A((size_t)S * M * R), B((size_t)S * N * R);
    for (auto& v : A) v = nd(rng);
    for (auto& v : B) v = nd(rng);
    float *dA, *dB, *dP;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dP, (size_t)splits * S * M * N * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap mA, mB;
    bool ok = wino::make_map_3d(&mA, dA, R, M, S, (uint64_t)R * 4, (uint64_t)M * R * 4, 32, 128) &&
              wino::make_map_3d(&mB, dB, R, N, S, (uint64_t)R * 4, (uint64_t)N * R * 4, 32, g_flush ? 128 : 256);
    if (!ok) { printf("map failed %d\n", wino::last_tmap_error()); return 1; }
    auto kern = g_flush ? flush_k<true, false>() : wino::tc::gemm_3xtf32_kernel<true, false>;
    const int smem = g_flush ? wino::tc::flush::SMEM_BYTES : wino::tc::SMEM_BYTES;
    const int bn = g_flush ? 128 : 256, th = g_flush ? wino::tc::flush::THREADS : 256;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int kbt = (R + 31) / 32, kbp = (kbt + splits - 1) / splits;
    dim3 grid((N + bn - 1) / bn, (M + 127) / 128, S * splits);
    kern<<<grid, th, smem>>>(mA, mA, mB, dP, M, N, R, N, S, splits, kbp);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("kernel error: %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> P((size_t)splits * S * M * N);
    cudaMemcpy(P.data(), dP, P.size() * 4, cudaMemcpyDeviceToHost);
    double max_rel = 0, worst_err = 0;
    long bad = 0;
    for (int s = 0; s < S; ++s)
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                double ref = 0, aref = 0, got = 0;
                for (int r = 0; r < R; ++r) {
                    const double p = (double)A[((size_t)s * M + m) * R + r] * B[((size_t)s * N + n) * R + r];
                    ref += p;
                    aref += fabs(p);
                }
                for (int q = 0; q < splits; ++q) got += P[(((size_t)q * S + s) * M + m) * N + n];
                const double err = fabs(got - ref);
                worst_err = std::max(worst_err, err);
                max_rel = std::max(max_rel, err / (aref + 1e-30));
                if (err > 1e-5 + 1e-4 * fabs(ref)) ++bad;
            }
    printf("KK S=%d M=%d N=%d R=%d splits=%d: max|err|=%.3e max err/sum|p|=%.3e strict-fail=%ld\n", S, M, N, R,
           splits, worst_err, max_rel, bad);
    cudaFree(dA); cudaFree(dB); cudaFree(dP);
    return 0;
}

int main() {
    int rc0 = 0;
    rc0 |= run_kk(1, 128, 256, 64, 1);
    rc0 |= run_kk(2, 256, 256, 1000, 3);
    rc0 |= run_kk(2, 384, 200, 520, 2);
    // accuracy vs accumulation length: same product, 1 split (TMEM accumulates all 63 k-blocks)
    // vs 63 splits (each k-block a fresh accumulator, partials summed in fp64)
    rc0 |= run_kk(2, 128, 256, 2000, 1);
    rc0 |= run_kk(2, 128, 256, 2000, 8);
    rc0 |= run_kk(2, 128, 256, 2000, 63);
    g_flush = true;
    printf("--- flush variant ---\n");
    rc0 |= run_kk(1, 128, 256, 64, 1);
    rc0 |= run_kk(2, 256, 256, 1000, 3);
    rc0 |= run_kk(2, 384, 200, 520, 2);
    rc0 |= run_kk(2, 128, 256, 2000, 1);
    rc0 |= run(1, 128, 256, 32, false);
    rc0 |= run(3, 256, 520, 256, false);
    rc0 |= run(2, 16, 36, 16, false);
    rc0 |= run(2, 384, 1000, 256, false);
    rc0 |= run(36, 256, 12544, 256, true);
    for (int f : {2, 4}) {
        g_F = f;
        printf("--- flush every %d k-blocks ---\n", f);
        rc0 |= run_kk(2, 128, 256, 2000, 1);
        rc0 |= run(36, 256, 12544, 256, true);
    }
    g_flush = false;
    printf("--- fast variant timing ---\n");
    rc0 |= run(36, 256, 12544, 256, true);
    int rc = 0;
    rc |= run(1, 128, 256, 32, false);
    rc |= run(2, 128, 256, 64, false);
    rc |= run(3, 256, 520, 256, false);
    rc |= run(2, 16, 36, 16, false);
    rc |= run(2, 384, 1000, 256, false);
    // rc |= run(36, 256, 12544, 256, true);
    rc |= rc0;
    return rc;
}
