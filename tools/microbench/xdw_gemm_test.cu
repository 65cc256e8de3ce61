// Standalone check of the exact dW_F kernels (csrc/wino_xdw.cuh) against exact CPU arithmetic:
//   1. gemm_kernel on random int8 digit planes (every level, every tile edge case);
//   2. input_digits_kernel: digits reassembled on the host equal round(x·2^(38-E)) of the f64
//      transform computed on the host.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 --expt-relaxed-constexpr
//        -I../../paper_1702_08597_b200/csrc xdw_gemm_test.cu -o xdw_gemm_test -lcuda
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <random>
#include <vector>

#include "wino_xdw.cuh"
#include "wino_tmap.h"

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e = (x);                                                                   \
        if (e != cudaSuccess) {                                                                \
            std::printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));     \
            std::exit(1);                                                                      \
        }                                                                                      \
    } while (0)

namespace x = wino::xdw;

static int gemm_case(int P2, int M, int N, int ncols, int nchunks) {
    const int64_t NTd = (int64_t)ncols * nchunks;
    std::mt19937 rng(1234 + M + N);
    std::uniform_int_distribution<int> dig(-128, 127);
    std::vector<int8_t> A((size_t)x::DIG * P2 * M * NTd), B((size_t)x::DIG * P2 * N * NTd);
    for (auto& v : A) v = (int8_t)dig(rng);
    for (auto& v : B) v = (int8_t)dig(rng);
    std::vector<int> EA((size_t)nchunks * P2 * M, 22), EB((size_t)nchunks * P2 * N, 22);
    int8_t *dA, *dB;
    int *dEA, *dEB;
    double* dP;
    CK(cudaMalloc(&dA, A.size()));
    CK(cudaMalloc(&dB, B.size()));
    CK(cudaMalloc(&dEA, EA.size() * 4));
    CK(cudaMalloc(&dEB, EB.size() * 4));
    const size_t np = (size_t)nchunks * P2 * M * N;
    CK(cudaMalloc(&dP, np * 8));
    CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dEA, EA.data(), EA.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dEB, EB.data(), EB.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(dP, 0xff, np * 8));
    CUtensorMap ma, mb;
    if (!wino::make_map_4d_u8(&ma, dA, NTd, M, P2, x::DIG, x::KS, x::BM, CU_TENSOR_MAP_SWIZZLE_64B) ||
        !wino::make_map_4d_u8(&mb, dB, NTd, N, P2, x::DIG, x::KS, x::BN, CU_TENSOR_MAP_SWIZZLE_64B)) {
        std::printf("tensor map failed %d\n", wino::last_tmap_error());
        return 1;
    }
    x::ChunkTab ct{};
    ct.n = nchunks;
    for (int c = 0; c < nchunks; ++c) {
        ct.col0[c] = c * ncols;
        ct.ncols[c] = ncols;
        ct.seg[c] = c;
    }
    const int tm = (M + x::BM - 1) / x::BM, tn = (N + x::BN - 1) / x::BN, units = nchunks * P2 * tm * tn;
    CK(cudaFuncSetAttribute(x::gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, x::SMEM_BYTES));
    x::gemm_kernel<<<std::min(units, 148), x::THREADS, x::SMEM_BYTES>>>(ma, mb, ct, dEA, dEB, dP, P2, M, N, tm, tn,
                                                                         units);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<double> P(np);
    CK(cudaMemcpy(P.data(), dP, np * 8, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int ch = 0; ch < nchunks; ++ch)
        for (int s = 0; s < P2; ++s)
            for (int m = 0; m < M; ++m)
                for (int n = 0; n < N; ++n) {
                    long long lv[5] = {};
                    for (int t = ch * ncols; t < (ch + 1) * ncols; ++t)
                        for (int i = 0; i < 5; ++i)
                            for (int j = 4 - i; j < 5; ++j)
                                lv[i + j - 4] += (long long)A[(((size_t)i * P2 + s) * M + m) * NTd + t] *
                                                 B[(((size_t)j * P2 + s) * N + n) * NTd + t];
                    double want = 0;
                    for (int L = 4; L >= 0; --L) want = want * 256.0 + (double)lv[L];
                    const double got = P[(((size_t)ch * P2 + s) * M + m) * N + n];
                    if (std::fabs(got - want) > 1e-12 * std::fabs(want) + 1e-9) {
                        if (bad < 8)
                            std::printf("  mismatch ch %d s %d m %d n %d: got %.17g want %.17g (L0 %lld L4 %lld)\n",
                                        ch, s, m, n, got, want, lv[0], lv[4]);
                        ++bad;
                    }
                }
    std::printf("gemm P2=%d M=%d N=%d cols=%d chunks=%d: %d bad of %zu\n", P2, M, N, ncols, nchunks, bad, np);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dEA);
    cudaFree(dEB);
    cudaFree(dP);
    return bad != 0;
}

// digits of the f64 input transform (m = 4, builtin coefficients) vs the host
static int digits_case() {
    constexpr int M = 4, P = 6, P2 = 36;
    const int N = 2, C = 8, H = 13, W = 13, pad = 1;
    const int hi = H + 2 * pad, tiles_x = (hi - 3 + 1 + M - 1) / M, T = tiles_x * tiles_x;
    const int ncols = N * T, ncols_pad = (ncols + 63) / 64 * 64;
    const int64_t NTd = ncols_pad, plane = (int64_t)P2 * C * NTd;
    std::mt19937 rng(7);
    std::normal_distribution<float> nd(0.f, 1.f);
    std::vector<float> in((size_t)N * C * H * W);
    for (auto& v : in) v = nd(rng);
    std::vector<unsigned> amax(C, 0);
    for (int n = 0; n < N; ++n)
        for (int c = 0; c < C; ++c)
            for (int i = 0; i < H * W; ++i) {
                union { float f; unsigned u; } q{std::fabs(in[((size_t)n * C + c) * H * W + i])};
                amax[c] = std::max(amax[c], q.u);
            }
    wino::CoefsD cf{};
    x::Norms nrm{};
    double nb[6] = {};
    for (int i = 0; i < P; ++i)
        for (int k = 0; k < P; ++k) {
            cf.b[i * P + k] = wino::BuiltinCoefs<4, 6>::BD(i * P + k);
            nb[k] += std::fabs(wino::BuiltinCoefs<4, 6>::BD(i * P + k));  // column k of b
        }
    for (int i = 0; i < P; ++i)
        for (int j = 0; j < P; ++j) nrm.v[i * P + j] = nb[i] * nb[j];
    float* din;
    int8_t* ddig;
    int* dE;
    unsigned* dmax;
    CK(cudaMalloc(&din, in.size() * 4));
    CK(cudaMalloc(&ddig, (size_t)5 * plane));
    CK(cudaMalloc(&dE, (size_t)P2 * C * 4));
    CK(cudaMalloc(&dmax, C * 4));
    CK(cudaMemcpy(din, in.data(), in.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dmax, amax.data(), C * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(ddig, 0x55, (size_t)5 * plane));
    const size_t smem = (size_t)P2 * x::kTileItems * 5;
    auto kern = x::input_digits_kernel<M, P, wino::ConstCoef<4, 6>>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t items = (int64_t)C * ncols_pad;
    kern<<<(unsigned)((items + 255) / 256), 256, smem>>>(din, ddig, dE, dmax, cf, nrm, C, H, W, pad, tiles_x, T,
                                                          ncols, ncols_pad, NTd, plane, 0);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<int8_t> dig((size_t)5 * plane);
    std::vector<int> E((size_t)P2 * C);
    CK(cudaMemcpy(dig.data(), ddig, dig.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(E.data(), dE, E.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int c = 0; c < C; ++c)
        for (int j = 0; j < ncols_pad; ++j) {
            double d[P][P] = {};
            if (j < ncols) {
                const int n = j / T, t = j % T, ty = t / tiles_x, tx = t % tiles_x;
                for (int a = 0; a < P; ++a)
                    for (int b = 0; b < P; ++b) {
                        const int y = ty * M - pad + a, xx = tx * M - pad + b;
                        if (y >= 0 && y < H && xx >= 0 && xx < W) d[a][b] = in[((size_t)n * C + c) * H * W + y * W + xx];
                    }
            }
            for (int i = 0; i < P; ++i)
                for (int l = 0; l < P; ++l) {
                    double acc = 0;
                    for (int a = 0; a < P; ++a)
                        for (int b = 0; b < P; ++b) acc += cf.b[a * P + i] * cf.b[b * P + l] * d[a][b];
                    const int s = i * P + l;
                    long long m = 0;
                    for (int k = 4; k >= 0; --k) m = m * 256 + dig[(size_t)k * plane + ((size_t)s * C + c) * NTd + j];
                    const double got = std::ldexp((double)m, E[(size_t)s * C + c] - 38);
                    const double tol = std::ldexp(1.0, E[(size_t)s * C + c] - 37);  // 2 units of the last digit
                    if (!(std::fabs(got - acc) <= tol)) {
                        if (bad < 8) std::printf("  digits c %d j %d s %d: got %.17g want %.17g E %d\n", c, j, s, got, acc,
                                                 E[(size_t)s * C + c]);
                        ++bad;
                    }
                }
        }
    std::printf("digits: %d bad of %d\n", bad, C * ncols_pad * P2);
    return bad != 0;
}

int main() {
    int fails = 0;
    fails += digits_case();
    fails += gemm_case(1, 128, 64, 64, 1);
    fails += gemm_case(2, 256, 128, 128, 1);
    fails += gemm_case(3, 200, 136, 192, 2);
    std::printf(fails ? "FAIL\n" : "PASS\n");
    return fails != 0;
}
