// C-ABI implementation of include/wino_cuda.h: the drop-in boundary between the
// reference's layer API (layer.hpp:28-43, sparse.hpp:40-82) and the sm_100a kernels.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/wino_cuda.h"
#include "wino_compress.cuh"
#include "wino_dense_tc.cuh"
#include "wino_kernels.cuh"
#include "wino_ozaki.cuh"
#include "wino_spmm_tmem.cuh"
#include "wino_precise.cuh"
#include "wino_tmap.h"
#include "wino_update.cuh"

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                     \
    do {                                                                                   \
        cudaError_t _e = (expr);                                                           \
        if (_e != cudaSuccess)                                                             \
            return set_err(WINO_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// ---------------------------------------------------------------------------------------
// Cook–Toom transform generator — restatement of transforms.cpp:33-145 (same loop and
// accumulation order so the doubles are bit-identical to the reference's; pinned by
// tests/test_capi_host.py against the golden dump of the reference matrices).
// ---------------------------------------------------------------------------------------
const double kPoints[7] = {0.0, 1.0, -1.0, 2.0, -2.0, 0.5, -0.5};

void poly_mul_linear(std::vector<double>& coeff, double a) {  // coeff *= (x - a)
    std::vector<double> next(coeff.size() + 1, 0.0);
    for (size_t d = 0; d < coeff.size(); ++d) {
        next[d] -= coeff[d] * a;
        next[d + 1] += coeff[d];
    }
    coeff.swap(next);
}

int cook_toom(int m, int r, double* a, double* b, double* g) {
    if (m < 1 || r < 1) return set_err(WINO_CAPABILITY_ERROR, "tile and kernel extents must be >= 1");
    const int p = m + r - 1;
    if (p > 8)
        return set_err(WINO_CAPABILITY_ERROR,
                       "unsupported transform size: m+r-1 = " + std::to_string(p) + " exceeds 8");
    std::fill(a, a + p * m, 0.0);
    std::fill(b, b + p * p, 0.0);
    std::fill(g, g + p * r, 0.0);
    if (p == 1) {
        a[0] = b[0] = g[0] = 1.0;
        return WINO_OK;
    }
    const int n = p - 1;  // finite points
    auto eval = [&](double* v, int ncoeff) {
        for (int i = 0; i < n; ++i) {
            double x = 1.0;
            for (int j = 0; j < ncoeff; ++j) {
                v[i * ncoeff + j] = x;
                x *= kPoints[i];
            }
        }
        v[(p - 1) * ncoeff + ncoeff - 1] = 1.0;
    };
    eval(g, r);
    eval(a, m);
    // Lagrange basis (inverse Vandermonde), column i = basis polynomial of point i
    std::vector<double> inv(n * n, 0.0);
    for (int i = 0; i < n; ++i) {
        std::vector<double> coeff = {1.0};
        double denom = 1.0;
        for (int k = 0; k < n; ++k) {
            if (k == i) continue;
            poly_mul_linear(coeff, kPoints[k]);
            denom *= kPoints[i] - kPoints[k];
        }
        for (int j = 0; j < n; ++j) inv[j * n + i] = coeff[j] / denom;
    }
    std::vector<double> mpoly = {1.0};
    for (int i = 0; i < n; ++i) poly_mul_linear(mpoly, kPoints[i]);
    for (int j = 0; j < n; ++j) {
        for (int i = 0; i < n; ++i) b[j * p + i] = inv[j * n + i];
        b[j * p + p - 1] = mpoly[j];
    }
    b[(p - 1) * p + p - 1] = 1.0;
    return WINO_OK;
}

int transforms(int m, int r, double* a, double* b, double* g) {
    if (m == 2 && r == 3) {  // f2x2_3x3_transforms (transforms.cpp:7-19)
        const double A[8] = {1, 0, 1, 1, 1, -1, 0, -1};
        const double B[16] = {1, 0, 0, 0, 0, 1, -1, 1, -1, 1, 1, 0, 0, 0, 0, -1};
        const double G[12] = {1, 0, 0, 0.5, 0.5, 0.5, 0.5, -0.5, 0.5, 0, 0, 1};
        std::memcpy(a, A, sizeof A);
        std::memcpy(b, B, sizeof B);
        std::memcpy(g, G, sizeof G);
        return WINO_OK;
    }
    return cook_toom(m, r, a, b, g);
}

int make_geometry(int64_t c, int64_t h_i, int64_t w_i, int m, int r, wino_geometry* g) {
    if (h_i < r || w_i < r)
        return set_err(WINO_SHAPE_ERROR, "image (" + std::to_string(c) + "x" + std::to_string(h_i) +
                                             "x" + std::to_string(w_i) + ") smaller than kernel (" +
                                             std::to_string(r) + "x" + std::to_string(r) + ")");
    g->c = c;
    g->h_i = h_i;
    g->w_i = w_i;
    g->m = m;
    g->r = r;
    g->p = m + r - 1;
    g->h_o = h_i - r + 1;
    g->w_o = w_i - r + 1;
    g->tiles_y = (g->h_o + m - 1) / m;
    g->tiles_x = (g->w_o + m - 1) / m;
    g->h_op = g->tiles_y * m;
    g->w_op = g->tiles_x * m;
    g->h_ip = g->h_op + r - 1;
    g->w_ip = g->w_op + r - 1;
    g->t = g->tiles_y * g->tiles_x;
    return WINO_OK;
}

enum Kind { K_INPUT = 0, K_SPMM, K_OUTPUT, K_GRADZ, K_SDDMM, K_SPMM_T, K_INGRAD, K_DENSE_FWD,
            K_DENSE_DW, K_DENSE_DV, K_SGD, K_MISC, K_NKINDS };
const char* kKindNames[K_NKINDS] = {"input_transform", "spmm_fwd", "output_transform", "grad_z",
                                    "sddmm_dw", "spmm_bwd_data", "input_grad", "dense_fwd_tc",
                                    "dense_dw_tc", "dense_dv_tc", "sgd", "misc"};

struct ProfRec {
    int kind;
    cudaEvent_t a, b;
};

}  // namespace

struct wino_plan {
    int device = 0;
    int C = 0, K = 0, H = 0, W = 0, pad = 0, m = 0, r = 0, p = 0, P2 = 0;
    wino_geometry g{};
    wino::Coefs cf{};
    wino::CoefsD cfd{};  // the same transform in the reference's doubles (precise dW mode)
    bool has_weights = false, dense = false;
    bool builtin = false;  // coefficients equal a built-in set: compile-time-constant kernels
    int64_t nnz = 0;
    std::vector<int64_t> slice_nnz, slice_off;
    // CSR (global offsets) and CSC of W_F(:,:,i,j)ᵀ
    int* d_rowptr = nullptr;
    int* d_colidx = nullptr;
    int* d_rowof = nullptr;
    float* d_vals = nullptr;
    int* d_colptr = nullptr;
    int* d_rowidx = nullptr;
    int* d_perm = nullptr;
    int2* d_cv = nullptr;   // CSR (col, value bits) interleaved, the SpMM operand stream
    int2* d_cvT = nullptr;  // CSC (row, value bits) interleaved
    // capacities (elements) of the buffers above, in declaration order: reused across weight sets
    size_t cap_rowptr = 0, cap_colidx = 0, cap_rowof = 0, cap_vals = 0, cap_colptr = 0, cap_rowidx = 0,
           cap_perm = 0, cap_cv = 0, cap_cvT = 0;
    // device compress scratch: the f64 weights, line counts, CSR position map
    double* d_wsrc = nullptr;
    int* d_cnt = nullptr;
    int* d_pos = nullptr;
    size_t cap_wsrc = 0, cap_cnt = 0, cap_pos = 0;
    // weight update: Σw² partials, non-finite counter
    double* d_sumsq_part = nullptr;
    size_t cap_sumsq_part = 0;
    unsigned long long* d_nonfinite = nullptr;
    std::vector<int> h_rowptr, h_colptr;  // kept for launch partitioning
    int sddmm_rows = 0, sddmm_r = 0, sddmm_stages = 1, sddmm_maxb = 8;
    int sddmm_impl = 1;               // 0 = warp/transpose kernel (also the precise mode), 1 = chunk form
    int lane_rows = 0, lane_tw = 0;   // chunk-form plan (0 rows: infeasible)
    int64_t sddmm_max_nb = 0;
    double* d_partial = nullptr;
    size_t partial_cap = 0;
    // dense plan (density 1): full CSR (dW via the exact SDDMM, scattered to K×C×p×q) plus the
    // tcgen05 operands: W and Wᵀ split into tf32 hi/lo, [36][K][C] and [36][C][K]
    float* d_wdense = nullptr;
    float* d_wh = nullptr;
    float* d_wl = nullptr;
    float* d_wth = nullptr;
    float* d_wtl = nullptr;
    CUtensorMap map_wh{}, map_wl{}, map_wth{}, map_wtl{};
    bool tc_ready = false;
    bool tc_fast = false;  // dense=3: single TMEM accumulation chain (faster, ~1e-6 error)
    int dw_mode = 0;       // sparse plan: 0 = masked SDDMM, 1 = tensor-core GEMM + mask gather, 2 = precise,
                           // 3 = int8 tensor cores, exact products (wino_ozaki.cuh)
    int contraction = 0;   // sparse plan, in effect: 0 = CSR kernels (reference order), 1 = tcgen05 on zero-filled W_F
    int contraction_mode = 0;  // as requested: 0 csr, 1 tc, 2 auto (tc + tc dW when dense enough)
    int auto_permille = 80;    // auto: tensor cores at density >= this / 1000 (measured crossover 5-10%)
    int64_t* d_slice_off = nullptr;
    float* d_dwc = nullptr;
    size_t dwc_cap = 0;
    uint8_t* d_oz = nullptr;  // int8 dW: digit tensors, block exponents, the dense K×C product
    size_t oz_cap = 0;
    // scratch
    float* d_z = nullptr;
    size_t z_cap = 0;
    float* d_dv = nullptr;
    size_t dv_cap = 0;
    double* d_scalar = nullptr;
    cudaStream_t side = nullptr;  // wino_backward: dW runs here, concurrent with dĨ_F -> dI
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaStream_t side2 = nullptr;  // wino_forward_backward: the dO -> dZ -> dĨ_F -> dI chain
    cudaEvent_t ev_v = nullptr, ev_dz = nullptr, ev_join2 = nullptr;
    // instrumentation
    int64_t launches = 0;
    bool prof = false;
    std::vector<ProfRec> recs;
    double prof_ms[K_NKINDS] = {};
    int64_t prof_n[K_NKINDS] = {};
    int sm_count = 148;
    int max_smem = 227 * 1024;
};

struct wino_cache {
    wino_plan* plan = nullptr;
    int n_max = 0;
    int n = 0;
    int64_t NTs = 0;
    float* V = nullptr;
    float* DZ = nullptr;
    int dw_chunks = 0;      // SDDMM chunks whose dW partials backward_range already computed
    float* Vlo = nullptr;   // precise dW mode: fp32 residuals of Ĩ_F and dZ
    float* DZlo = nullptr;
    float* Vt = nullptr;    // tensor-core plans: tf32 lo halves of Ĩ_F and dZ (V / DZ hold the hi
    float* DZt = nullptr;   // halves) when the producers split the operands (tf32_presplit)
    bool v_split = false, dz_split = false;
    bool has_fwd = false;
    bool has_grad_z = false;
};

namespace {

void free_weights(wino_plan* p) {
    const char* names[] = {"rowptr", "colidx", "rowof", "vals", "colptr", "rowidx", "perm", "cv", "cvT",
                           "wdense", "wh", "wl", "wth", "wtl"};
    int i = 0;
    for (void* ptr : {(void*)p->d_rowptr, (void*)p->d_colidx, (void*)p->d_rowof, (void*)p->d_vals,
                      (void*)p->d_colptr, (void*)p->d_rowidx, (void*)p->d_perm, (void*)p->d_cv,
                      (void*)p->d_cvT, (void*)p->d_wdense, (void*)p->d_wh, (void*)p->d_wl, (void*)p->d_wth,
                      (void*)p->d_wtl}) {
        if (ptr && cudaFree(ptr) != cudaSuccess)
            std::fprintf(stderr, "wino: cudaFree(%s) failed\n", names[i]);
        ++i;
    }
    p->d_wh = p->d_wl = p->d_wth = p->d_wtl = nullptr;
    p->tc_ready = false;
    p->d_rowptr = p->d_colidx = p->d_rowof = p->d_colptr = p->d_rowidx = p->d_perm = nullptr;
    p->d_vals = p->d_wdense = nullptr;
    p->d_cv = p->d_cvT = nullptr;
    p->cap_rowptr = p->cap_colidx = p->cap_rowof = p->cap_vals = p->cap_colptr = p->cap_rowidx = p->cap_perm =
        p->cap_cv = p->cap_cvT = 0;
    p->has_weights = false;
}

void free_compress_scratch(wino_plan* p) {
    for (void* ptr : {(void*)p->d_wsrc, (void*)p->d_cnt, (void*)p->d_pos, (void*)p->d_sumsq_part,
                      (void*)p->d_nonfinite})
        if (ptr) cudaFree(ptr);
    p->d_wsrc = nullptr;
    p->d_cnt = p->d_pos = nullptr;
    p->d_sumsq_part = nullptr;
    p->d_nonfinite = nullptr;
    p->cap_wsrc = p->cap_cnt = p->cap_pos = p->cap_sumsq_part = 0;
}

// Launch bracket: counts launches and, when profiling, records events on the stream.
struct Launch {
    wino_plan* p;
    cudaStream_t st;
    int kind;
    ProfRec rec{};
    Launch(wino_plan* plan, cudaStream_t s, int k) : p(plan), st(s), kind(k) {
        ++p->launches;
        if (p->prof) {
            rec.kind = k;
            cudaEventCreate(&rec.a);
            cudaEventCreate(&rec.b);
            cudaEventRecord(rec.a, st);
        }
    }
    int done() {
        cudaError_t e = cudaGetLastError();
        if (p->prof) {
            cudaEventRecord(rec.b, st);
            p->recs.push_back(rec);
        }
        if (e != cudaSuccess)
            return set_err(WINO_CUDA_ERROR, std::string("kernel ") + kKindNames[kind] +
                                                ": " + cudaGetErrorString(e));
        return WINO_OK;
    }
};

// cudaFuncSetAttribute once per kernel and size (keeps launches capturable in CUDA graphs and
// off the per-launch host path)
template <typename K>
void set_smem_attr(K kernel, int bytes) {
    static std::mutex mu;
    static std::vector<std::pair<const void*, int>> done;
    std::lock_guard<std::mutex> lock(mu);
    const void* key = reinterpret_cast<const void*>(kernel);
    for (auto& d : done)
        if (d.first == key) {
            if (d.second >= bytes) return;
            cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
            d.second = bytes;
            return;
        }
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done.emplace_back(key, bytes);
}

int grid_for(int64_t work, int threads, int sm_count) {
    int64_t b = (work + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)sm_count * 16));
}

// typed capacity-based (re)allocation: keeps a buffer while it is large enough
template <typename T>
int grow(T** buf, size_t* cap, size_t need) {
    need = std::max<size_t>(need, 1);
    if (*buf && *cap >= need) return WINO_OK;
    if (*buf) cudaFree(*buf);
    *buf = nullptr;
    *cap = 0;
    CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(buf), need * sizeof(T)));
    *cap = need;
    return WINO_OK;
}

int ensure(float** buf, size_t* cap, size_t need) {
    if (*cap >= need) return WINO_OK;
    if (*buf) cudaFree(*buf);
    *buf = nullptr;
    *cap = 0;
    CUDA_TRY(cudaMalloc(buf, need * sizeof(float)));
    *cap = need;
    return WINO_OK;
}

// SpMM lane width: R floats per lane (chunk TW = 32R), the widest whose staged chunk
// ncols×TW×4 B fits 200 KB (LDS.128 sustains the most shared-memory bytes per clock).
int spmm_r(int ncols) {
    if (const char* env = std::getenv("WINO_SPMM_R")) return std::atoi(env);
    const int64_t budget = 200 * 1024;  // the CSR segment shrinks with the row group to fit
    if ((int64_t)ncols * 128 * 4 <= budget) return 4;
    if ((int64_t)ncols * 64 * 4 <= budget) return 2;
    return 1;
}

// Largest CSR segment (in int2 entries, incl. alignment slack) over the row groups of rpb rows.
int64_t max_segment(const std::vector<int>& ptr, int P2, int nrows, int rpb) {
    int64_t m = 0;
    for (int s = 0; s < P2; ++s)
        for (int r0 = 0; r0 < nrows; r0 += rpb) {
            const int r1 = std::min(nrows, r0 + rpb);
            const int64_t a0 = ptr[(size_t)s * (nrows + 1) + r0] & ~1;
            m = std::max<int64_t>(m, ptr[(size_t)s * (nrows + 1) + r1] - a0 + 2);
        }
    return m;
}

template <int R>
int launch_spmm_r(wino_plan* p, cudaStream_t st, int kind, const int* rowptr, const int2* cv,
                  const std::vector<int>& hptr, const float* X, float* Y, int nrows, int ncols, int64_t NT,
                  int64_t NTs, int64_t NTr) {
    constexpr int TW = 32 * R;
    const size_t xbytes = (size_t)ncols * TW * sizeof(float);
    const int chunks = (int)((NT + TW - 1) / TW);
    const int64_t base = (int64_t)chunks * p->P2;
    // enough blocks to fill the GPU once; beyond that every extra row group re-stages the X chunk
    const int64_t target = (int64_t)p->sm_count * 9 / 10;
    int groups = (int)std::max<int64_t>(1, std::min<int64_t>((target + base - 1) / base, nrows / 16));
    if (const char* e = std::getenv("WINO_SPMM_GROUPS")) groups = std::max(1, std::atoi(e));
    // prefer the staged CSR segment (measured faster than L1 reads, c2/c3), adding row groups
    // until it fits; only a segment that never fits falls back to reading it through L1
    int rpb = 0;
    size_t seg = 0;
    for (;; ++groups) {
        rpb = (int)round_up((nrows + groups - 1) / groups, 16);
        seg = (size_t)max_segment(hptr, p->P2, nrows, rpb) * sizeof(int2);
        if ((int)(xbytes + seg) <= p->max_smem || rpb <= 16) break;
    }
    groups = (nrows + rpb - 1) / rpb;
    const bool staged = (int)(xbytes + seg) <= p->max_smem && !std::getenv("WINO_SPMM_UNSTAGED");
    const size_t smem = staged ? xbytes + seg : xbytes;
    if ((int)smem > p->max_smem)
        return set_err(WINO_CAPABILITY_ERROR, "spmm: staged chunk exceeds shared memory");
    Launch L(p, st, kind);
    const int threads = std::getenv("WINO_SPMM_THREADS") ? std::atoi(std::getenv("WINO_SPMM_THREADS")) : 1024;
    const dim3 grid(chunks, groups, p->P2);
    if (staged) {
        set_smem_attr(wino::spmm_kernel<R, true>, (int)smem);
        wino::spmm_kernel<R, true><<<grid, threads, smem, st>>>(rowptr, cv, X, Y, nrows, ncols, (int)NTs, rpb,
                                                                (int)NTr);
    } else {
        set_smem_attr(wino::spmm_kernel<R, false>, (int)smem);
        wino::spmm_kernel<R, false><<<grid, threads, smem, st>>>(rowptr, cv, X, Y, nrows, ncols, (int)NTs, rpb,
                                                                 (int)NTr);
    }
    return L.done();
}

// X, Y may point at column `a` of their rows (a column range of the batch): NT = valid columns
// of the range, NTs = the row stride, NTr = columns the range owns (≥ NT on the batch's last range,
// which also owns the zero padding).  The whole batch: NTr = NTs.
// the SpMM with X in tensor memory (wino_spmm_tmem.cuh): 16 rows per warp when that still fills
// the GPU, else 8
int launch_spmm_tmem(wino_plan* p, cudaStream_t st, int kind, const int* rowptr, const int2* cv,
                     const std::vector<int>& hptr, const float* X, float* Y, int nrows, int ncols, int64_t NTs,
                     int64_t NTr) {
    namespace ws = wino::st;
    const int chunks = (int)((NTr + ws::TW - 1) / ws::TW);
    const int64_t base = (int64_t)chunks * p->P2;
    const bool big = base * ((nrows + 63) / 64) >= p->sm_count;
    const int rpb = big ? 64 : 32;
    const size_t smem = (size_t)max_segment(hptr, p->P2, nrows, rpb) * sizeof(int2) + 16;
    if ((int)smem > p->max_smem) return set_err(WINO_CAPABILITY_ERROR, "spmm (tmem): CSR segment exceeds shared memory");
    Launch L(p, st, kind);
    const dim3 grid((unsigned)((nrows + rpb - 1) / rpb), (unsigned)chunks, (unsigned)p->P2);
    if (big) {
        set_smem_attr(ws::spmm_tmem_kernel<16>, (int)smem);
        ws::spmm_tmem_kernel<16><<<grid, ws::THREADS, smem, st>>>(rowptr, cv, X, Y, nrows, ncols, (int)NTs,
                                                                 (int)NTr, -0.0f);
    } else {
        set_smem_attr(ws::spmm_tmem_kernel<8>, (int)smem);
        ws::spmm_tmem_kernel<8><<<grid, ws::THREADS, smem, st>>>(rowptr, cv, X, Y, nrows, ncols, (int)NTs,
                                                                (int)NTr, -0.0f);
    }
    return L.done();
}

int launch_spmm(wino_plan* p, cudaStream_t st, int kind, const int* rowptr, const int2* cv,
                const std::vector<int>& hptr, const float* X, float* Y, int nrows, int ncols, int64_t NT,
                int64_t NTs, int64_t NTr = -1) {
    if (NTr < 0) NTr = NTs;
    // read on every launch (not cached): tests switch it per case
    const bool tmem = std::getenv("WINO_SPMM_TMEM") && std::atoi(std::getenv("WINO_SPMM_TMEM")) == 1;
    if (tmem && ncols <= 1024) return launch_spmm_tmem(p, st, kind, rowptr, cv, hptr, X, Y, nrows, ncols, NTs, NTr);
    switch (spmm_r(ncols)) {
        case 4: return launch_spmm_r<4>(p, st, kind, rowptr, cv, hptr, X, Y, nrows, ncols, NT, NTs, NTr);
        case 2: return launch_spmm_r<2>(p, st, kind, rowptr, cv, hptr, X, Y, nrows, ncols, NT, NTs, NTr);
        default: return launch_spmm_r<1>(p, st, kind, rowptr, cv, hptr, X, Y, nrows, ncols, NT, NTs, NTr);
    }
}

constexpr int kSddmmBatch = 16;    // nonzeros per warp batch
constexpr int kSddmmWarps = 24;    // 768 threads (≤ 85 registers: no spills at R=4)

int64_t max_group_nnz(const wino_plan* p, int rows) {
    int64_t nb = 0;
    for (int s = 0; s < p->P2; ++s)
        for (int r0 = 0; r0 < p->K; r0 += rows) {
            const int r1 = std::min(p->K, r0 + rows);
            nb = std::max<int64_t>(nb, p->h_rowptr[s * (p->K + 1) + r1] - p->h_rowptr[s * (p->K + 1) + r0]);
        }
    return nb;
}

// SDDMM variant + partition.  Preferred: R=4 (128-wide chunks) single-stage; otherwise R=2
// with a two-stage cp.async pipeline.  Row group: the largest whose staged chunk fits and
// whose nonzeros fit the per-warp register batches (MAXB ≤ 8, else 16).
void plan_sddmm(wino_plan* p) {
    const int K = p->K;
    const int64_t budget = std::min(p->max_smem, 210 * 1024);
    struct Opt { int r, stages; };
    const char* renv = std::getenv("WINO_SDDMM_R");
    for (Opt o : {Opt{4, 1}, Opt{2, 2}, Opt{2, 1}, Opt{1, 2}}) {
        if (renv && std::atoi(renv) != o.r) continue;
        if (o.r == 2 && o.stages == 1 && p->dw_mode != 2) continue;  // precise mode only (R=1 LO spills)
        const int64_t per_row = (int64_t)o.stages * 32 * o.r * 4 * (p->dw_mode == 2 ? 2 : 1);
        const int64_t cap_rows = budget / per_row - p->C;
        if (cap_rows < 8) continue;
        const char* env = std::getenv("WINO_SDDMM_MAXB");
        const int first = env ? std::atoi(env) : 4;
        for (int lim : {first, 8, 16}) {
            int rows_cap = (int)std::min<int64_t>(round_up(K, 8), cap_rows / 8 * 8);
            if (const char* e = std::getenv("WINO_SDDMM_ROWS")) rows_cap = std::min(rows_cap, std::max(8, std::atoi(e)));
            for (int rows = rows_cap; rows >= 8; rows -= 8) {
                const int64_t nb = max_group_nnz(p, rows);
                if (nb <= (int64_t)kSddmmWarps * kSddmmBatch * lim) {
                    p->sddmm_r = o.r;
                    p->sddmm_stages = o.stages;
                    p->sddmm_rows = rows;
                    p->sddmm_max_nb = nb;
                    const int64_t per_warp = (nb + kSddmmWarps * kSddmmBatch - 1) / (kSddmmWarps * kSddmmBatch);
                    p->sddmm_maxb = per_warp <= 4 ? 4 : per_warp <= 8 ? 8 : 16;
                    return;
                }
            }
        }
    }
    p->sddmm_r = 0;  // no feasible variant: launch reports CAPABILITY
}

void plan_sddmm_chunk(wino_plan* p);
void plan_sddmm_all(wino_plan* p) {
    plan_sddmm(p);
    plan_sddmm_chunk(p);
    p->sddmm_impl = p->lane_rows > 0 ? 1 : 0;
    if (const char* e = std::getenv("WINO_SDDMM_IMPL")) p->sddmm_impl = (std::atoi(e) == 1 && p->lane_rows > 0) ? 1 : 0;
}

constexpr int kChunkThreads = 1024;

// Chunk-form SDDMM plan: TW = 128 when Ĩ_F(:, chunk) plus a useful row group fits, else 64; the
// row group is as large as shared memory allows (fewest re-stagings of the Ĩ_F chunk).
void plan_sddmm_chunk(wino_plan* p) {
    p->lane_rows = 0;
    const int64_t budget = std::min(p->max_smem, 220 * 1024);
    static const int tw_env = std::getenv("WINO_SDDMM_TW") ? std::atoi(std::getenv("WINO_SDDMM_TW")) : 0;
    for (int tw : {128, 64}) {
        if (tw_env && tw != tw_env) continue;
        const int64_t cap_rows = budget / (tw * 4) - p->C;
        if (cap_rows < 8) continue;
        const int64_t need = round_up(p->K, 8);
        int rows = (int)std::min<int64_t>(need, cap_rows / 8 * 8);
        // balance the groups: same number of groups, rows spread evenly
        const int groups = (p->K + rows - 1) / rows;
        rows = (int)round_up((p->K + groups - 1) / groups, 8);
        if (const char* e = std::getenv("WINO_SDDMM_ROWS")) rows = std::max(8, std::min(rows, std::atoi(e)));
        p->lane_rows = rows;
        p->lane_tw = tw;
        return;
    }
}

template <int TW>
void launch_sddmm_chunk_v(dim3 grid, size_t smem, cudaStream_t st, const wino_plan* p, const float* DZ,
                          const float* V, float* dW, double* partial, int NTs, int z0 = 0) {
    set_smem_attr(wino::sddmm_chunk_kernel<TW, kChunkThreads>, (int)smem);
    wino::sddmm_chunk_kernel<TW, kChunkThreads><<<grid, kChunkThreads, smem, st>>>(
        p->d_rowptr, p->d_colidx, p->d_rowof, DZ, V, dW, partial, p->nnz, p->K, p->C, NTs, p->lane_rows, z0);
}

template <int R, int MAXB, int STAGES, bool LO>
void launch_sddmm_v(dim3 grid, size_t smem, cudaStream_t st, const wino_plan* p, const float* DZ,
                    const float* V, const float* DZlo, const float* Vlo, float* dW, double* partial, int NT,
                    int NTs, int tps) {
    constexpr int TH = kSddmmWarps * 32;
    static_assert(TH <= 1024, "block too large");
    set_smem_attr(wino::sddmm_kernel<R, MAXB, STAGES, kSddmmBatch, TH, LO>, (int)smem);
    wino::sddmm_kernel<R, MAXB, STAGES, kSddmmBatch, TH, LO><<<grid, TH, smem, st>>>(
        p->d_rowptr, p->d_colidx, p->d_rowof, DZ, V, DZlo, Vlo, dW, partial, p->nnz, p->K, p->C, NT, NTs,
        p->sddmm_rows, tps);
}

double* ensure_partial(wino_plan* p, size_t need, int* rc) {
    *rc = WINO_OK;
    if (p->partial_cap < need) {
        if (p->d_partial) cudaFree(p->d_partial);
        p->d_partial = nullptr;
        p->partial_cap = 0;
        const cudaError_t e = cudaMalloc(&p->d_partial, need * sizeof(double));
        if (e != cudaSuccess) {
            *rc = set_err(WINO_CUDA_ERROR, std::string("sddmm partials: ") + cudaGetErrorString(e));
            return nullptr;
        }
        p->partial_cap = need;
    }
    return p->d_partial;
}

// chunks [z0, z1) of the batch (default: all) -> fp64 partials; finish = sum them into dW
int launch_sddmm_chunk(wino_plan* p, cudaStream_t st, const float* DZ, const float* V, float* dW, int64_t NT,
                       int64_t NTs, int z0 = 0, int z1 = -1, bool finish = true) {
    const int TW = p->lane_tw;
    const size_t smem = (size_t)(p->C + p->lane_rows) * TW * 4;
    const int groups = (p->K + p->lane_rows - 1) / p->lane_rows;
    const int chunks = (int)((NT + TW - 1) / TW);
    if (z1 < 0) z1 = chunks;
    int rc = WINO_OK;
    double* partial = chunks > 1 ? ensure_partial(p, (size_t)chunks * p->nnz, &rc) : nullptr;
    if (rc) return rc;
    if (z1 > z0) {
        const dim3 grid(groups, p->P2, z1 - z0);
        Launch L(p, st, K_SDDMM);
        if (TW == 128)
            launch_sddmm_chunk_v<128>(grid, smem, st, p, DZ, V, dW, partial, (int)NTs, z0);
        else
            launch_sddmm_chunk_v<64>(grid, smem, st, p, DZ, V, dW, partial, (int)NTs, z0);
        if ((rc = L.done())) return rc;
    }
    if (chunks > 1 && finish) {
        Launch L(p, st, K_SDDMM);
        wino::split_sum_kernel<<<grid_for(p->nnz, 256, p->sm_count), 256, 0, st>>>(partial, dW, p->nnz, chunks);
        return L.done();
    }
    return WINO_OK;
}

int launch_sddmm(wino_plan* p, cudaStream_t st, const float* DZ, const float* V, float* dW, int64_t NT,
                 int64_t NTs, const float* DZlo = nullptr, const float* Vlo = nullptr) {
    if (p->nnz == 0) return WINO_OK;
    const bool lo = Vlo != nullptr;
    if (lo != (p->dw_mode == 2)) return set_err(WINO_CONSISTENCY_ERROR, "sddmm: plan/precision mismatch");
    if (p->sddmm_impl == 1 && !lo) return launch_sddmm_chunk(p, st, DZ, V, dW, NT, NTs);
    if (p->sddmm_r == 0) return set_err(WINO_CAPABILITY_ERROR, "sddmm: no variant fits this layer");
    const int R = p->sddmm_r, TW = 32 * R;
    const size_t smem = (size_t)p->sddmm_stages * (p->C + p->sddmm_rows) * TW * 4 * (lo ? 2 : 1);
    const int groups = (p->K + p->sddmm_rows - 1) / p->sddmm_rows;
    const int chunks = (int)((NT + TW - 1) / TW);
    const int64_t base = (int64_t)groups * p->P2;
    int splits = (int)std::max<int64_t>(1, std::min<int64_t>((3LL * p->sm_count + base - 1) / base, chunks / 2));
    if (const char* e = std::getenv("WINO_SDDMM_SPLITS")) splits = std::max(1, std::min(chunks, std::atoi(e)));
    const int tps = ((chunks + splits - 1) / splits) * TW;
    splits = (int)((NT + tps - 1) / tps);
    double* partial = nullptr;
    if (splits > 1) {
        const size_t need = (size_t)splits * p->nnz;
        if (p->partial_cap < need) {
            if (p->d_partial) cudaFree(p->d_partial);
            p->d_partial = nullptr;
            p->partial_cap = 0;
            CUDA_TRY(cudaMalloc(&p->d_partial, need * sizeof(double)));
            p->partial_cap = need;
        }
        partial = p->d_partial;
    }
    const dim3 grid(groups, p->P2, splits);
    {
        Launch L(p, st, K_SDDMM);
#define SDDMM_CASE(RR, MB, SS)                                                                   \
    if (p->sddmm_r == RR && p->sddmm_maxb == MB && p->sddmm_stages == SS) {                      \
        if (lo)                                                                                  \
            launch_sddmm_v<RR, MB, SS, true>(grid, smem, st, p, DZ, V, DZlo, Vlo, dW, partial, (int)NT, \
                                             (int)NTs, tps);                                     \
        else                                                                                     \
            launch_sddmm_v<RR, MB, SS, false>(grid, smem, st, p, DZ, V, nullptr, nullptr, dW, partial,  \
                                              (int)NT, (int)NTs, tps);                           \
    }
        SDDMM_CASE(4, 4, 1) SDDMM_CASE(4, 8, 1) SDDMM_CASE(4, 16, 1)
        SDDMM_CASE(2, 4, 2) SDDMM_CASE(2, 8, 2) SDDMM_CASE(2, 16, 2)
        SDDMM_CASE(2, 4, 1) SDDMM_CASE(2, 8, 1) SDDMM_CASE(2, 16, 1)
        SDDMM_CASE(1, 4, 2) SDDMM_CASE(1, 8, 2) SDDMM_CASE(1, 16, 2)
#undef SDDMM_CASE
        int rc = L.done();
        if (rc) return rc;
    }
    if (splits > 1) {
        Launch L(p, st, K_SDDMM);
        wino::split_sum_kernel<<<grid_for(p->nnz, 256, p->sm_count), 256, 0, st>>>(partial, dW, p->nnz, splits);
        return L.done();
    }
    return WINO_OK;
}

template <int M, int P, class CF>
int fwd_transforms(wino_plan* p, cudaStream_t st, const float* in, float* out, wino_cache* c,
                   float* V, float* Z, int n, int64_t NT, int64_t NTs, int flags, int stage, int64_t NTr) {
    const wino_geometry& g = p->g;
    if (stage == 0) {
        Launch L(p, st, K_INPUT);
        wino::input_transform_kernel<M, P, CF><<<grid_for((int64_t)p->C * NTr, 256, p->sm_count), 256, 0, st>>>(
            in, V, p->cf, p->C, p->H, p->W, p->pad, (int)g.tiles_x, (int)g.t, (int)NT, (int)NTs, (int)NTr,
            (c && c->v_split && V == c->V) ? c->Vt : nullptr);
        return L.done();
    }
    Launch L(p, st, K_OUTPUT);
    const int grid = grid_for((int64_t)p->K * NT, 256, p->sm_count);
    if (flags & WINO_FWD_RELU)
        wino::output_transform_kernel<M, P, true, CF><<<grid, 256, 0, st>>>(
            Z, out, p->cf, p->K, (int)g.h_o, (int)g.w_o, (int)g.tiles_x, (int)g.t, (int)NT, (int)NTs);
    else
        wino::output_transform_kernel<M, P, false, CF><<<grid, 256, 0, st>>>(
            Z, out, p->cf, p->K, (int)g.h_o, (int)g.w_o, (int)g.tiles_x, (int)g.t, (int)NT, (int)NTs);
    return L.done();
}

template <int M, int P, class CF>
int launch_grad_z(wino_plan* p, cudaStream_t st, const float* dO, const float* relu, float* DZ,
                  int64_t NT, int64_t NTs, bool mask, int64_t NTr, float* DZt = nullptr) {
    const wino_geometry& g = p->g;
    Launch L(p, st, K_GRADZ);
    const int grid = grid_for((int64_t)p->K * NTr, 256, p->sm_count);
    if (mask)
        wino::grad_z_kernel<M, P, true, CF><<<grid, 256, 0, st>>>(dO, relu, DZ, p->cf, p->K, (int)g.h_o,
                                                              (int)g.w_o, (int)g.tiles_x, (int)g.t,
                                                              (int)NT, (int)NTs, (int)NTr, DZt);
    else
        wino::grad_z_kernel<M, P, false, CF><<<grid, 256, 0, st>>>(dO, relu, DZ, p->cf, p->K, (int)g.h_o,
                                                               (int)g.w_o, (int)g.tiles_x, (int)g.t,
                                                               (int)NT, (int)NTs, (int)NTr, DZt);
    return L.done();
}

// precise dW mode: the fp32 residuals of Ĩ_F (after K1) and of dZ (after K4)
template <int M, int P, class CF>
int launch_input_lo(wino_plan* p, cudaStream_t st, const float* in, const float* V, float* Vlo, int64_t NT,
                    int64_t NTs) {
    const wino_geometry& g = p->g;
    Launch L(p, st, K_INPUT);
    wino::input_transform_lo_kernel<M, P><<<grid_for((int64_t)p->C * NTs, 256, p->sm_count), 256, 0, st>>>(
        in, V, Vlo, p->cfd, p->C, p->H, p->W, p->pad, (int)g.tiles_x, (int)g.t, (int)NT, (int)NTs);
    return L.done();
}

template <int M, int P, class CF>
int launch_grad_z_lo(wino_plan* p, cudaStream_t st, const float* dO, const float* relu, const float* DZ,
                     float* DZlo, int64_t NT, int64_t NTs, bool mask) {
    const wino_geometry& g = p->g;
    Launch L(p, st, K_GRADZ);
    const int grid = grid_for((int64_t)p->K * NTs, 256, p->sm_count);
    if (mask)
        wino::grad_z_lo_kernel<M, P, true><<<grid, 256, 0, st>>>(dO, relu, DZ, DZlo, p->cfd, p->K, (int)g.h_o,
                                                                (int)g.w_o, (int)g.tiles_x, (int)g.t, (int)NT,
                                                                (int)NTs);
    else
        wino::grad_z_lo_kernel<M, P, false><<<grid, 256, 0, st>>>(dO, relu, DZ, DZlo, p->cfd, p->K, (int)g.h_o,
                                                                 (int)g.w_o, (int)g.tiles_x, (int)g.t, (int)NT,
                                                                 (int)NTs);
    return L.done();
}

template <int M, int P, class CF>
int launch_input_grad(wino_plan* p, cudaStream_t st, const float* DV, float* dI, int n, int64_t NTs) {
    const wino_geometry& g = p->g;
    const int T = (int)g.t;
    const int64_t per_c = (int64_t)T * (P * P + 1) * sizeof(float);
    Launch L(p, st, K_INGRAD);
    if (per_c <= 96 * 1024) {
        // channels per block: fill >= 256 (c,t) items for phase 1 within ~48 KB of tiles
        int cg = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)p->C, (48 * 1024) / per_c,
                                                                (256 + T - 1) / T}));
        const size_t smem = (size_t)cg * per_c;
        set_smem_attr(wino::input_grad_kernel<M, P, CF>, (int)std::max<size_t>(smem, 48 * 1024));
        wino::input_grad_kernel<M, P, CF><<<dim3((p->C + cg - 1) / cg, n), 256, smem, st>>>(
            DV, dI, p->cf, p->C, p->H, p->W, p->pad, (int)g.tiles_y, (int)g.tiles_x, T, (int)NTs, cg);
    } else {
        const int64_t total = (int64_t)n * p->C * p->H * p->W;
        wino::input_grad_direct_kernel<M, P, CF><<<grid_for(total, 256, p->sm_count), 256, 0, st>>>(
            DV, dI, p->cf, n, p->C, p->H, p->W, p->pad, (int)g.tiles_y, (int)g.tiles_x, T, (int)NTs);
    }
    return L.done();
}

#define DISPATCH_MP(p, FN, ...)                                                                    \
    ((p)->m == 4   ? ((p)->builtin ? FN<4, 6, wino::ConstCoef<4, 6>>(__VA_ARGS__)                      \
                                   : FN<4, 6, wino::RuntimeCoef>(__VA_ARGS__))                          \
     : (p)->m == 2 ? ((p)->builtin ? FN<2, 4, wino::ConstCoef<2, 4>>(__VA_ARGS__)                      \
                                   : FN<2, 4, wino::RuntimeCoef>(__VA_ARGS__))                          \
                   : ((p)->builtin ? FN<6, 8, wino::ConstCoef<6, 8>>(__VA_ARGS__)                      \
                                   : FN<6, 8, wino::RuntimeCoef>(__VA_ARGS__)))

// Dense plan: (re)build the tcgen05 operands from the live values (full CSR order = W[s][k][c]).
int refresh_tc_operands(wino_plan* p, cudaStream_t st) {
    const int64_t n = (int64_t)p->P2 * p->K * p->C;
    if (p->C % 4 || p->K % 4) {  // TMA row strides must be multiples of 16 bytes: CSR kernels instead
        p->tc_ready = false;
        return WINO_OK;
    }
    if (!p->d_wh) {
        CUDA_TRY(cudaMalloc(&p->d_wh, n * 4));
        CUDA_TRY(cudaMalloc(&p->d_wl, n * 4));
        CUDA_TRY(cudaMalloc(&p->d_wth, n * 4));
        CUDA_TRY(cudaMalloc(&p->d_wtl, n * 4));
        const int K = p->K, C = p->C;
        bool ok = wino::make_map_3d(&p->map_wh, p->d_wh, C, K, p->P2, (uint64_t)C * 4, (uint64_t)K * C * 4, 32, 128) &&
                  wino::make_map_3d(&p->map_wl, p->d_wl, C, K, p->P2, (uint64_t)C * 4, (uint64_t)K * C * 4, 32, 128) &&
                  wino::make_map_3d(&p->map_wth, p->d_wth, K, C, p->P2, (uint64_t)K * 4, (uint64_t)K * C * 4, 32, 128) &&
                  wino::make_map_3d(&p->map_wtl, p->d_wtl, K, C, p->P2, (uint64_t)K * 4, (uint64_t)K * C * 4, 32, 128);
        if (!ok)
            return set_err(WINO_CUDA_ERROR, "cuTensorMapEncodeTiled failed for the weight operands (CUresult " +
                                                std::to_string(wino::last_tmap_error()) + ")");
    }
    const float* src = p->d_vals;  // dense plan: the full CSR is W[s][k][c]
    if (!p->dense) {               // sparse plan: scatter the CSR into a zero-filled W[s][k][c]
        if (!p->d_wdense) CUDA_TRY(cudaMalloc(&p->d_wdense, n * 4));
        CUDA_TRY(cudaMemsetAsync(p->d_wdense, 0, n * 4, st));
        if (p->nnz > 0) {
            wino::csr_scatter_dense_kernel<<<grid_for((int64_t)p->K * p->P2, 128, p->sm_count), 128, 0, st>>>(
                p->d_rowptr, p->d_colidx, p->d_vals, p->K, p->C, p->P2, p->d_wdense);
            ++p->launches;
        }
        src = p->d_wdense;
    }
    wino::split_tf32_kernel<<<grid_for(n, 256, p->sm_count), 256, 0, st>>>(src, p->d_wh, p->d_wl, p->d_wth,
                                                                           p->d_wtl, p->K, p->C, p->P2);
    ++p->launches;
    CUDA_TRY(cudaGetLastError());
    p->tc_ready = true;
    return WINO_OK;
}

// B_PRE: B pre-split by its producer (bl = its tf32 lo half); only the warp-specialised kernel
// takes it (tf32_presplit() guarantees that kernel is the one selected)
template <bool A_SPLIT, bool B_MN, bool B_PRE = false>
int launch_tc(wino_plan* p, cudaStream_t st, int kind, const CUtensorMap& ah, const CUtensorMap& al,
              const CUtensorMap& b, float* D, int M, int N, int Kd, int64_t ldd, int splits,
              const CUtensorMap* bl = nullptr) {
    const int kb_total = (Kd + wino::tc::BK - 1) / wino::tc::BK;
    const int kb_per = (kb_total + splits - 1) / splits;
    const int bn = p->tc_fast ? wino::tc::BN : wino::tc::flush::BN;
    const dim3 grid((unsigned)((N + bn - 1) / bn), (M + wino::tc::BM - 1) / wino::tc::BM, p->P2 * splits);
    Launch L(p, st, kind);
    if (p->tc_fast) {
        set_smem_attr(wino::tc::gemm_3xtf32_kernel<A_SPLIT, B_MN>, wino::tc::SMEM_BYTES);
        wino::tc::gemm_3xtf32_kernel<A_SPLIT, B_MN><<<grid, wino::tc::THREADS, wino::tc::SMEM_BYTES, st>>>(
            ah, al, b, D, M, N, Kd, ldd, p->P2, splits, kb_per);
    } else {
        // k-blocks (of 32) per fresh TMEM accumulator folded into fp64: 1 = most accurate; each
        // fold costs one fp32->fp64 conversion per output element on the XU pipe
        static const int fold = std::getenv("WINO_TC_FOLD") ? std::atoi(std::getenv("WINO_TC_FOLD")) : 1;
        static const bool persistent = !(std::getenv("WINO_TC_PERSISTENT") &&
                                         std::atoi(std::getenv("WINO_TC_PERSISTENT")) == 0);
        const int ntiles = (int)(grid.x * grid.y * grid.z);
        auto go = [&](auto kern) {
            set_smem_attr(kern, wino::tc::flush::SMEM_BYTES);
            kern<<<grid, wino::tc::flush::THREADS, wino::tc::flush::SMEM_BYTES, st>>>(ah, al, b, D, M, N, Kd, ldd,
                                                                                     p->P2, splits, kb_per);
        };
        static const int epi = std::getenv("WINO_TC_EPI") ? std::atoi(std::getenv("WINO_TC_EPI")) : 16;
        auto go_p = [&](auto kern, int threads) {
            set_smem_attr(kern, wino::tc::flush::SMEM_BYTES);
            const int ctas = std::min(ntiles, p->sm_count);
            kern<<<ctas, threads, wino::tc::flush::SMEM_BYTES, st>>>(ah, al, b, D, M, N, Kd, ldd, p->P2, splits,
                                                                    kb_per, (int)grid.x, (int)grid.y, ntiles);
        };
        // Default: the warp-specialised kernel (split warps apart from drain warps, 4 TMEM
        // accumulators, TMA-stored output) with the compensated fp32 fold (fp64 for the dW GEMM);
        // WINO_TC_ACC=fp64 selects the fp64 fold everywhere, WINO_TC_WS=0 the round-1 persistent
        // kernel (A/B builds).
        static const bool ws = !(std::getenv("WINO_TC_WS") && std::atoi(std::getenv("WINO_TC_WS")) == 0);
        // the dW GEMM (A split in shared memory too) measured faster with the fp64 fold (551 vs 584
        // µs at c3): its two split warps, not the drain, bound it, and the fp64 fold does not spill
        static const bool fp64_env = std::getenv("WINO_TC_ACC") && std::string(std::getenv("WINO_TC_ACC")) == "fp64";
        static const bool dw_kahan = std::getenv("WINO_TC_DW_ACC") && std::string(std::getenv("WINO_TC_DW_ACC")) == "kahan";
        const bool fp64_fold = fp64_env || (A_SPLIT && !dw_kahan);
        // drain warps: 8 (64 columns each, 4 KB SW128 output boxes; measured 4% faster at c3 than
        // WINO_TC_DW=16 with 32 columns and 2 KB SW64 boxes)
        static const int dw_env = std::getenv("WINO_TC_DW") ? std::atoi(std::getenv("WINO_TC_DW")) : 8;
        // the dW GEMM (A and B split in shared memory, fp64 fold) is split-bound with 2 split warps:
        // it runs 4 split warps next to 16 drain warps of 32 columns (80 registers per thread;
        // c3: 581 -> 521 µs; 6 split warps 526 µs; WINO_TC_DWGEMM_SW=2 restores the 2 + 8 layout)
        static const int dwgemm_sw = std::getenv("WINO_TC_DWGEMM_SW") ? std::atoi(std::getenv("WINO_TC_DWGEMM_SW")) : 4;
        const bool wide_split = A_SPLIT && !B_PRE && fp64_fold && dwgemm_sw != 2;
        const int dw = wide_split ? 16 : dw_env;
        CUtensorMap md;
        const bool ws_ok = ws && persistent && fold == 1 && (ldd & 3) == 0 &&
                           wino::make_map_3d_sw(&md, D, (uint64_t)N, (uint64_t)M, (uint64_t)p->P2 * splits,
                                                (uint64_t)ldd * 4, (uint64_t)M * ldd * 4, dw == 8 ? 32 : 16, 32,
                                                dw == 8 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
        // 2 split warps (4 would cap registers at 128/thread and spill the drain's 64 Kahan pairs);
        // none when both operands arrive pre-split
        constexpr int SW = (!A_SPLIT && B_PRE) ? 0 : 2;
        auto go_ws = [&](auto kern, int drain_warps) {
            set_smem_attr(kern, wino::tc::flush::WS_SMEM_BYTES);
            const int ctas = std::min(ntiles, p->sm_count);
            kern<<<ctas, 64 + 32 * (SW + drain_warps), wino::tc::flush::WS_SMEM_BYTES, st>>>(
                ah, al, b, md, bl ? *bl : b, D, M, N, Kd, ldd, p->P2, splits, kb_per, (int)grid.x, (int)grid.y,
                ntiles);
        };
        if (B_PRE && !(ws_ok && dw == 8))
            return set_err(WINO_CAPABILITY_ERROR, "pre-split operands need the warp-specialised tcgen05 kernel");
        auto go_ws_sw = [&](auto kern, int split_warps, int drain_warps) {
            set_smem_attr(kern, wino::tc::flush::WS_SMEM_BYTES);
            const int ctas = std::min(ntiles, p->sm_count);
            kern<<<ctas, 64 + 32 * (split_warps + drain_warps), wino::tc::flush::WS_SMEM_BYTES, st>>>(
                ah, al, b, md, bl ? *bl : b, D, M, N, Kd, ldd, p->P2, splits, kb_per, (int)grid.x, (int)grid.y,
                ntiles);
        };
        if constexpr (A_SPLIT && !B_PRE) {
            if (ws_ok && wide_split && dwgemm_sw == 4) {
                go_ws_sw(wino::tc::gemm_3xtf32_ws_kernel<A_SPLIT, B_MN, 4, 16, false, 4>, 4, 16);
                return L.done();
            }
            if (ws_ok && wide_split) {
                go_ws_sw(wino::tc::gemm_3xtf32_ws_kernel<A_SPLIT, B_MN, 6, 16, false, 4>, 6, 16);
                return L.done();
            }
        }
        if (ws_ok && dw == 8 && !fp64_fold)
            go_ws(wino::tc::gemm_3xtf32_ws_kernel<A_SPLIT, B_MN, SW, 8, true, 4, B_PRE>, 8);
        else if (ws_ok && dw == 8)
            go_ws(wino::tc::gemm_3xtf32_ws_kernel<A_SPLIT, B_MN, SW, 8, false, 4, B_PRE>, 8);
        else if constexpr (!B_PRE) {
            if (ws_ok && !fp64_fold)
                go_ws(wino::tc::gemm_3xtf32_ws_kernel<A_SPLIT, B_MN, SW, 16, true, 4>, 16);
            else if (ws_ok)
                go_ws(wino::tc::gemm_3xtf32_ws_kernel<A_SPLIT, B_MN, SW, 16, false, 4>, 16);
            else if (persistent && fold == 1 && epi == 8)
                go_p(wino::tc::gemm_3xtf32_flush_persistent_kernel<A_SPLIT, B_MN, 1, 8>, 64 + 32 * 8);
            else if (persistent && fold == 1)
                go_p(wino::tc::gemm_3xtf32_flush_persistent_kernel<A_SPLIT, B_MN, 1, 16>, 64 + 32 * 16);
            else if (fold == 2)
                go(wino::tc::gemm_3xtf32_flush_kernel<A_SPLIT, B_MN, 2>);
            else if (fold == 4)
                go(wino::tc::gemm_3xtf32_flush_kernel<A_SPLIT, B_MN, 4>);
            else
                go(wino::tc::gemm_3xtf32_flush_kernel<A_SPLIT, B_MN, 1>);
        }
    }
    return L.done();
}

// D[s] = W-operand[s] · B[s] on the tensor cores; B = [P2][Kd][NTs] activations (MN-major).
int launch_tc_gemm(wino_plan* p, cudaStream_t st, int kind, const CUtensorMap& ah, const CUtensorMap& al,
                   const float* B, float* D, int M, int Kd, int64_t NTs, const float* Blo = nullptr) {
    CUtensorMap mb, mbl;
    if (!wino::make_map_3d(&mb, B, NTs, Kd, p->P2, (uint64_t)NTs * 4, (uint64_t)Kd * NTs * 4, 32, 32, true) ||
        (Blo && !wino::make_map_3d(&mbl, Blo, NTs, Kd, p->P2, (uint64_t)NTs * 4, (uint64_t)Kd * NTs * 4, 32, 32, true)))
        return set_err(WINO_CUDA_ERROR, "cuTensorMapEncodeTiled failed for the activation operand (CUresult " +
                                            std::to_string(wino::last_tmap_error()) + ")");
    if (Blo) return launch_tc<false, true, true>(p, st, kind, ah, al, mb, D, M, (int)NTs, Kd, NTs, 1, &mbl);
    return launch_tc<false, true>(p, st, kind, ah, al, mb, D, M, (int)NTs, Kd, NTs, 1);
}

// dW_F = dZ·Ĩ_Fᵀ on the tensor cores, split over NT, partials summed in fp64 -> K×C×p×q.
int launch_tc_dw(wino_plan* p, cudaStream_t st, const float* DZ, const float* V, float* dW, int64_t NTs,
                 bool masked = false, const float* DZlo = nullptr, const float* Vlo = nullptr) {
    CUtensorMap ma, mb, mal, mbl;
    const uint32_t bn = p->tc_fast ? wino::tc::BN : wino::tc::flush::BN;
    const bool pre = DZlo && Vlo;  // both operands pre-split by their producers (K4, K1)
    if (!wino::make_map_3d(&ma, DZ, NTs, p->K, p->P2, (uint64_t)NTs * 4, (uint64_t)p->K * NTs * 4, 32, 128) ||
        !wino::make_map_3d(&mb, V, NTs, p->C, p->P2, (uint64_t)NTs * 4, (uint64_t)p->C * NTs * 4, 32, bn) ||
        (DZlo && !wino::make_map_3d(&mal, DZlo, NTs, p->K, p->P2, (uint64_t)NTs * 4, (uint64_t)p->K * NTs * 4, 32, 128)) ||
        (Vlo && !wino::make_map_3d(&mbl, Vlo, NTs, p->C, p->P2, (uint64_t)NTs * 4, (uint64_t)p->C * NTs * 4, 32, bn)))
        return set_err(WINO_CUDA_ERROR, "cuTensorMapEncodeTiled failed for dZ / Ĩ_F (CUresult " +
                                            std::to_string(wino::last_tmap_error()) + ")");
    const int tiles = ((p->C + (int)bn - 1) / (int)bn) * ((p->K + wino::tc::BM - 1) / wino::tc::BM) * p->P2;
    const int kb_total = (int)((NTs + wino::tc::BK - 1) / wino::tc::BK);
    int splits = (int)std::max<int64_t>(1, std::min<int64_t>((2LL * p->sm_count + tiles - 1) / tiles, kb_total / 4));
    if (const char* e = std::getenv("WINO_DW_SPLITS")) splits = std::max(1, std::atoi(e));
    const size_t need = (size_t)splits * p->P2 * p->K * p->C;
    float* part = nullptr;
    int rc = ensure(&p->d_dwc, &p->dwc_cap, need);
    if (rc) return rc;
    part = p->d_dwc;
    const int kind = masked ? K_SDDMM : K_DENSE_DW;
    if (pre)
        rc = launch_tc<false, false, true>(p, st, kind, ma, mal, mb, part, p->K, p->C, (int)NTs, p->C, splits, &mbl);
    else if (Vlo)  // only Ĩ_F pre-split (dZ from a range backward): A still split in shared memory
        rc = launch_tc<true, false, true>(p, st, kind, ma, ma, mb, part, p->K, p->C, (int)NTs, p->C, splits, &mbl);
    else if (DZlo)
        rc = launch_tc<false, false>(p, st, kind, ma, mal, mb, part, p->K, p->C, (int)NTs, p->C, splits);
    else
        rc = launch_tc<true, false>(p, st, kind, ma, ma, mb, part, p->K, p->C, (int)NTs, p->C, splits);
    if (rc) return rc;
    Launch L(p, st, kind);
    if (masked)
        wino::tc::reduce_dw_masked_kernel<<<grid_for(p->nnz, 256, p->sm_count), 256, 0, st>>>(
            part, dW, p->d_rowof, p->d_colidx, p->d_slice_off, p->K, p->C, p->P2, splits, p->nnz);
    else
        wino::tc::reduce_dw_kernel<<<grid_for((int64_t)p->P2 * p->K * p->C, 256, p->sm_count), 256, 0, st>>>(
            part, dW, p->K, p->C, p->P2, splits);
    return L.done();
}

// dW_F on the int8 tensor cores (wino_ozaki.cuh): digit split of dZ and Ĩ_F, the exact-product
// GEMM per Winograd coordinate into a dense [P2][K][C] buffer, then the surviving entries
// gathered in CSR order.
int launch_ozaki_dw(wino_plan* p, cudaStream_t st, const float* DZ, const float* V, float* dW, int64_t NT,
                    int64_t NTs) {
    namespace oz = wino::oz;
    const int64_t NTp = (NT + oz::KB - 1) / oz::KB * oz::KB, nkb = NTp / oz::KB;
    const int64_t P2 = p->P2, K = p->K, C = p->C;
    const size_t dig_a = (size_t)oz::DIG * P2 * K * NTp, dig_b = (size_t)oz::DIG * P2 * C * NTp;
    const size_t ex_a = (size_t)P2 * K * nkb * 4, ex_b = (size_t)P2 * C * nkb * 4;
    const size_t dense = (size_t)P2 * K * C * 4;
    auto up = [](size_t x) { return (x + 1023) / 1024 * 1024; };
    const size_t need = up(dig_a) + up(dig_b) + up(ex_a) + up(ex_b) + up(dense);
    if (p->oz_cap < need) {
        if (p->d_oz) cudaFree(p->d_oz);
        p->d_oz = nullptr;
        p->oz_cap = 0;
        CUDA_TRY(cudaMalloc(&p->d_oz, need));
        p->oz_cap = need;
    }
    int8_t* da = reinterpret_cast<int8_t*>(p->d_oz);
    int8_t* db = da + up(dig_a);
    int* ea = reinterpret_cast<int*>(db + up(dig_b));
    int* eb = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(ea) + up(ex_a));
    float* dd = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(eb) + up(ex_b));
    CUtensorMap ma, mb;
    if (!wino::make_map_3d_sw(&ma, da, NTp, K, oz::DIG * P2, NTp, K * NTp, oz::KB, oz::BM,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_UINT8) ||
        !wino::make_map_3d_sw(&mb, db, NTp, C, oz::DIG * P2, NTp, C * NTp, oz::KB, oz::BN,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_UINT8))
        return set_err(WINO_CUDA_ERROR, "cuTensorMapEncodeTiled failed for the int8 digit tensors (CUresult " +
                                            std::to_string(wino::last_tmap_error()) + ")");
    Launch L(p, st, K_SDDMM);
    oz::slice_kernel<<<grid_for(P2 * K * nkb * 32, 256, p->sm_count), 256, 0, st>>>(DZ, da, ea, (int)P2, (int)K,
                                                                                   (int)NT, (int)NTs, (int)NTp);
    oz::slice_kernel<<<grid_for(P2 * C * nkb * 32, 256, p->sm_count), 256, 0, st>>>(V, db, eb, (int)P2, (int)C,
                                                                                   (int)NT, (int)NTs, (int)NTp);
    const int tiles_n = (int)((C + oz::BN - 1) / oz::BN), tiles_m = (int)((K + oz::BM - 1) / oz::BM);
    const int ntiles = tiles_n * tiles_m * (int)P2;
    set_smem_attr(oz::gemm_kernel, oz::SMEM_BYTES);
    oz::gemm_kernel<<<std::min(ntiles, p->sm_count), oz::THREADS, oz::SMEM_BYTES, st>>>(
        ma, mb, ea, eb, dd, (int)P2, (int)K, (int)C, (int)nkb, tiles_n, tiles_m, ntiles);
    const int per_slice = (int)std::max<int64_t>(1, std::min<int64_t>(64, p->nnz / P2 / 1024 + 1));
    oz::gather_kernel<<<dim3(per_slice, (unsigned)P2), 256, 0, st>>>(dd, dW, p->d_rowof, p->d_colidx,
                                                                    p->d_slice_off, p->K, p->C, p->P2, p->nnz);
    p->launches += 3;  // Launch L counts one
    return L.done();
}

int check_plan(const wino_plan* p) {
    if (!p) return set_err(WINO_INVALID_ARGUMENT, "null plan");
    if (!p->has_weights) return set_err(WINO_CONSISTENCY_ERROR, "plan has no weights (call wino_set_weights*)");
    return WINO_OK;
}

int apply_contraction(wino_plan* p);

int upload_csr(wino_plan* p, const std::vector<int>& rowptr, const std::vector<int>& col,
               const std::vector<float>& val) {
    const int K = p->K, C = p->C, P2 = p->P2;
    const int64_t nnz = (int64_t)col.size();
    // row-of-entry, CSC (counting sort per slice, ascending rows within a column) and perm
    std::vector<int> rowof(nnz), colptr((size_t)P2 * (C + 1)), rowidx(nnz), perm(nnz);
    std::vector<int2> cv(nnz), cvT(nnz);
    for (int s = 0; s < P2; ++s) {
        const int* rp = &rowptr[(size_t)s * (K + 1)];
        int* cp = &colptr[(size_t)s * (C + 1)];
        std::fill(cp, cp + C + 1, 0);
        for (int k = 0; k < K; ++k)
            for (int e = rp[k]; e < rp[k + 1]; ++e) {
                rowof[e] = k;
                cp[col[e] + 1]++;
            }
        cp[0] = rp[0];
        for (int c = 0; c < C; ++c) cp[c + 1] += cp[c];
        std::vector<int> fill(cp, cp + C);
        for (int k = 0; k < K; ++k)
            for (int e = rp[k]; e < rp[k + 1]; ++e) {
                const int dst = fill[col[e]]++;
                rowidx[dst] = k;
                perm[dst] = e;
                int bits;
                std::memcpy(&bits, &val[e], 4);
                cvT[dst] = make_int2(k, bits);
            }
    }
    for (int64_t e = 0; e < nnz; ++e) {
        int bits;
        std::memcpy(&bits, &val[e], 4);
        cv[e] = make_int2(col[e], bits);
    }
    auto up = [&](auto** dptr, const auto& hv) -> int {
        using T = typename std::decay_t<decltype(hv)>::value_type;
        CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(dptr), std::max<size_t>(1, hv.size()) * sizeof(T)));
        if (!hv.empty())
            CUDA_TRY(cudaMemcpy(*dptr, hv.data(), hv.size() * sizeof(T), cudaMemcpyHostToDevice));
        return WINO_OK;
    };
    int rc;
    if ((rc = up(&p->d_rowptr, rowptr)) || (rc = up(&p->d_colidx, col)) || (rc = up(&p->d_rowof, rowof)) ||
        (rc = up(&p->d_vals, val)) || (rc = up(&p->d_colptr, colptr)) || (rc = up(&p->d_rowidx, rowidx)) ||
        (rc = up(&p->d_perm, perm)) || (rc = up(&p->d_cv, cv)) || (rc = up(&p->d_cvT, cvT)))
        return rc;
    p->h_rowptr = rowptr;
    p->h_colptr = colptr;
    if (p->d_slice_off) {
        cudaFree(p->d_slice_off);
        p->d_slice_off = nullptr;
    }
    if (p->slice_off.size() == (size_t)P2) {
        CUDA_TRY(cudaMalloc(&p->d_slice_off, P2 * sizeof(int64_t)));
        CUDA_TRY(cudaMemcpy(p->d_slice_off, p->slice_off.data(), P2 * sizeof(int64_t), cudaMemcpyHostToDevice));
    }
    p->nnz = nnz;
    p->has_weights = true;
    p->dense = false;
    plan_sddmm_all(p);
    if (p->contraction_mode != 0) return apply_contraction(p);
    return WINO_OK;
}

// compress<float> on the device (wino_compress.cuh): W_F f64 is copied to HBM once, CSR + CSC +
// position map are built there; only the two pointer arrays come back (launch partitioning).
// keep_all = 1 keeps every coordinate (the dense plan's full CSR).
// Put the requested contraction into effect for the current weights (sparse plans): auto picks
// the tensor cores when the density reaches auto_permille/1000 (measured crossover).
int apply_contraction(wino_plan* p) {
    if (!p->has_weights || p->dense) return WINO_OK;
    int eff = p->contraction_mode;
    if (eff == 2) {
        const double density = (double)p->nnz / ((double)p->P2 * p->K * p->C);
        eff = (density * 1000.0 >= p->auto_permille && p->C % 4 == 0 && p->K % 4 == 0) ? 1 : 0;
    }
    p->contraction = eff;
    if (eff == 1) {
        if (!p->d_slice_off) {
            CUDA_TRY(cudaMalloc(&p->d_slice_off, p->P2 * sizeof(int64_t)));
            CUDA_TRY(cudaMemcpy(p->d_slice_off, p->slice_off.data(), p->P2 * sizeof(int64_t), cudaMemcpyHostToDevice));
        }
        const int rc = refresh_tc_operands(p, nullptr);
        if (rc) return rc;
        CUDA_TRY(cudaDeviceSynchronize());
    } else {
        p->tc_ready = false;
    }
    return WINO_OK;
}

int compress_from_wsrc(wino_plan* p, double tol, int keep_all);

int device_compress(wino_plan* p, const double* w_host, double tol, int keep_all) {
    const int64_t total = (int64_t)p->P2 * p->K * p->C;
    if (total >= ((int64_t)1 << 31)) return set_err(WINO_CAPABILITY_ERROR, "more than 2^31 weight coordinates");
    // buffers are reused in place: nothing still in flight may read the previous weights
    CUDA_TRY(cudaDeviceSynchronize());
    int rc = grow(&p->d_wsrc, &p->cap_wsrc, (size_t)total);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpy(p->d_wsrc, w_host, (size_t)total * sizeof(double), cudaMemcpyHostToDevice));
    return compress_from_wsrc(p, tol, keep_all);
}

// compress of the K×C×p×q f64 weights already in p->d_wsrc (device-synchronous)
int compress_from_wsrc(wino_plan* p, double tol, int keep_all) {
    const int K = p->K, C = p->C, P2 = p->P2;
    const int64_t total = (int64_t)P2 * K * C;
    p->has_weights = false;
    p->tc_ready = false;
    int rc;
    if ((rc = grow(&p->d_cnt, &p->cap_cnt, (size_t)P2 * std::max(K, C))) ||
        (rc = grow(&p->d_rowptr, &p->cap_rowptr, (size_t)P2 * (K + 1))) ||
        (rc = grow(&p->d_colptr, &p->cap_colptr, (size_t)P2 * (C + 1))) ||
        (rc = grow(&p->d_pos, &p->cap_pos, (size_t)total)))
        return rc;
    const cudaStream_t st = 0;
    constexpr int TH = 128;
    auto blocks = [](int64_t n) { return (int)std::max<int64_t>(1, (n + TH - 1) / TH); };
    {
        Launch L(p, st, K_MISC);
        wino::compress_count_kernel<false><<<blocks((int64_t)K * P2), TH, 0, st>>>(p->d_wsrc, K, C, P2, tol, keep_all,
                                                                                  p->d_cnt);
        if ((rc = L.done())) return rc;
    }
    {
        Launch L(p, st, K_MISC);
        wino::compress_scan_kernel<<<1, 1024, 0, st>>>(p->d_cnt, P2, K, p->d_rowptr);
        if ((rc = L.done())) return rc;
    }
    {
        Launch L(p, st, K_MISC);
        wino::compress_count_kernel<true><<<blocks((int64_t)C * P2), TH, 0, st>>>(p->d_wsrc, K, C, P2, tol, keep_all,
                                                                                 p->d_cnt);
        if ((rc = L.done())) return rc;
    }
    {
        Launch L(p, st, K_MISC);
        wino::compress_scan_kernel<<<1, 1024, 0, st>>>(p->d_cnt, P2, C, p->d_colptr);
        if ((rc = L.done())) return rc;
    }
    std::vector<int> rowptr((size_t)P2 * (K + 1)), colptr((size_t)P2 * (C + 1));
    CUDA_TRY(cudaMemcpy(rowptr.data(), p->d_rowptr, rowptr.size() * sizeof(int), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(colptr.data(), p->d_colptr, colptr.size() * sizeof(int), cudaMemcpyDeviceToHost));
    const int64_t nnz = rowptr.back();
    if ((rc = grow(&p->d_colidx, &p->cap_colidx, (size_t)nnz)) || (rc = grow(&p->d_vals, &p->cap_vals, (size_t)nnz)) ||
        (rc = grow(&p->d_rowof, &p->cap_rowof, (size_t)nnz)) || (rc = grow(&p->d_cv, &p->cap_cv, (size_t)nnz)) ||
        (rc = grow(&p->d_rowidx, &p->cap_rowidx, (size_t)nnz)) || (rc = grow(&p->d_perm, &p->cap_perm, (size_t)nnz)) ||
        (rc = grow(&p->d_cvT, &p->cap_cvT, (size_t)nnz)))
        return rc;
    if (nnz > 0) {
        {
            Launch L(p, st, K_MISC);
            wino::compress_fill_rows_kernel<<<blocks((int64_t)K * P2), TH, 0, st>>>(
                p->d_wsrc, K, C, P2, tol, keep_all, p->d_rowptr, p->d_colidx, p->d_vals, p->d_rowof, p->d_cv, p->d_pos);
            if ((rc = L.done())) return rc;
        }
        {
            Launch L(p, st, K_MISC);
            wino::compress_fill_cols_kernel<<<blocks((int64_t)C * P2), TH, 0, st>>>(
                p->d_wsrc, K, C, P2, tol, keep_all, p->d_colptr, p->d_pos, p->d_rowidx, p->d_perm, p->d_cvT);
            if ((rc = L.done())) return rc;
        }
    }
    p->slice_nnz.resize(P2);
    p->slice_off.resize(P2);
    for (int s = 0; s < P2; ++s) {
        p->slice_off[s] = rowptr[(size_t)s * (K + 1)];
        p->slice_nnz[s] = rowptr[(size_t)s * (K + 1) + K] - p->slice_off[s];
    }
    if (!p->d_slice_off) CUDA_TRY(cudaMalloc(&p->d_slice_off, P2 * sizeof(int64_t)));
    CUDA_TRY(cudaMemcpy(p->d_slice_off, p->slice_off.data(), P2 * sizeof(int64_t), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaDeviceSynchronize());
    p->h_rowptr = std::move(rowptr);
    p->h_colptr = std::move(colptr);
    p->nnz = nnz;
    p->has_weights = true;
    p->dense = false;
    plan_sddmm_all(p);
    if (p->contraction_mode != 0) return apply_contraction(p);
    return WINO_OK;
}

}  // namespace

extern "C" {

const char* wino_last_error(void) { return g_err.c_str(); }
const char* wino_version(void) { return "wino-b200 0.1 (sm_100a)"; }

int wino_make_geometry(int64_t c, int64_t h_i, int64_t w_i, int m, int r, wino_geometry* out) {
    if (!out) return set_err(WINO_INVALID_ARGUMENT, "null geometry");
    return make_geometry(c, h_i, w_i, m, r, out);
}

int wino_phi(const wino_geometry* g, int64_t t, int64_t i, int64_t j, int64_t* y, int64_t* x) {
    if (!g || !y || !x) return set_err(WINO_INVALID_ARGUMENT, "null argument");
    if (t < 0 || i < 0 || j < 0 || t >= g->t || i >= g->p || j >= g->p)
        return set_err(WINO_SHAPE_ERROR, "phi index (" + std::to_string(t) + "," + std::to_string(i) +
                                             "," + std::to_string(j) + ") out of range");
    *y = (t / g->tiles_x) * g->m + i;
    *x = (t % g->tiles_x) * g->m + j;
    return WINO_OK;
}

int wino_psi(const wino_geometry* g, int64_t y, int64_t x, int64_t* t, int64_t* i, int64_t* j) {
    if (!g || !t || !i || !j) return set_err(WINO_INVALID_ARGUMENT, "null argument");
    if (y < 0 || x < 0 || y >= g->h_op || x >= g->w_op)
        return set_err(WINO_SHAPE_ERROR,
                       "psi index (" + std::to_string(y) + "," + std::to_string(x) + ") out of range");
    *t = (y / g->m) * g->tiles_x + x / g->m;
    *i = y % g->m;
    *j = x % g->m;
    return WINO_OK;
}

int wino_transforms(int m, int r, double* a, double* b, double* g) {
    if (!a || !b || !g) return set_err(WINO_INVALID_ARGUMENT, "null output");
    return transforms(m, r, a, b, g);
}

int wino_plan_create(const wino_layer_desc* d, wino_plan** out) {
    if (!d || !out) return set_err(WINO_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    if (d->c <= 0 || d->k <= 0 || d->h <= 0 || d->w <= 0 || d->pad < 0)
        return set_err(WINO_SHAPE_ERROR, "layer extents must be positive");
    if (d->r != 3 || (d->m != 2 && d->m != 4 && d->m != 6))
        return set_err(WINO_CAPABILITY_ERROR, "kernels are built for F(m,3), m in {2,4,6}; got m=" +
                                                  std::to_string(d->m) + " r=" + std::to_string(d->r));
    if (d->c >= 65536 || d->k >= 65536)
        return set_err(WINO_CAPABILITY_ERROR, "channel counts must be < 65536");
    auto* p = new wino_plan();
    p->device = d->device;
    p->C = d->c;
    p->K = d->k;
    p->H = d->h;
    p->W = d->w;
    p->pad = d->pad;
    p->m = d->m;
    p->r = d->r;
    p->p = d->m + d->r - 1;
    p->P2 = p->p * p->p;
    int rc = make_geometry(d->c, d->h + 2 * d->pad, d->w + 2 * d->pad, d->m, d->r, &p->g);
    if (rc) {
        delete p;
        return rc;
    }
    double a[64], b[64], gg[64];
    if (d->a && d->b) {
        std::memcpy(a, d->a, sizeof(double) * p->p * p->m);
        std::memcpy(b, d->b, sizeof(double) * p->p * p->p);
    } else if ((rc = transforms(d->m, d->r, a, b, gg))) {
        delete p;
        return rc;
    }
    for (int i = 0; i < p->p * p->m; ++i) p->cf.a[i] = (float)(p->cfd.a[i] = a[i]);
    for (int i = 0; i < p->p * p->p; ++i) p->cf.b[i] = (float)(p->cfd.b[i] = b[i]);
    auto same = [&](const float* ta, const float* tb) {
        return std::memcmp(p->cf.a, ta, sizeof(float) * p->p * p->m) == 0 &&
               std::memcmp(p->cf.b, tb, sizeof(float) * p->p * p->p) == 0;
    };
    if (!std::getenv("WINO_RUNTIME_COEFS")) {
        if (p->m == 4) p->builtin = same(wino::BuiltinCoefs<4, 6>::a, wino::BuiltinCoefs<4, 6>::b);
        if (p->m == 2) p->builtin = same(wino::BuiltinCoefs<2, 4>::a, wino::BuiltinCoefs<2, 4>::b);
        if (p->m == 6) p->builtin = same(wino::BuiltinCoefs<6, 8>::a, wino::BuiltinCoefs<6, 8>::b);
    }
    cudaError_t e = cudaSetDevice(p->device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&p->sm_count, cudaDevAttrMultiProcessorCount, p->device);
    if (e == cudaSuccess)
        e = cudaDeviceGetAttribute(&p->max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->device);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_scalar, sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&p->d_nonfinite, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(p->d_nonfinite, 0, sizeof(unsigned long long));
    if (e != cudaSuccess) {
        delete p;
        return set_err(WINO_CUDA_ERROR, std::string("plan_create: ") + cudaGetErrorString(e));
    }
    *out = p;
    return WINO_OK;
}

int wino_plan_destroy(wino_plan* p) {
    if (!p) return WINO_OK;
    std::string bad;
    auto chk = [&](cudaError_t e, const char* what) {
        if (e != cudaSuccess && bad.empty()) bad = std::string(what) + ": " + cudaGetErrorString(e);
    };
    chk(cudaGetLastError(), "pending error before destroy");
    free_weights(p);
    free_compress_scratch(p);
    chk(cudaGetLastError(), "free_weights");
    if (p->d_dwc) chk(cudaFree(p->d_dwc), "d_dwc");
    if (p->d_oz) chk(cudaFree(p->d_oz), "d_oz");
    if (p->d_z) chk(cudaFree(p->d_z), "d_z");
    if (p->d_dv) chk(cudaFree(p->d_dv), "d_dv");
    if (p->d_scalar) chk(cudaFree(p->d_scalar), "d_scalar");
    if (p->side) chk(cudaStreamDestroy(p->side), "side stream");
    if (p->ev_fork) chk(cudaEventDestroy(p->ev_fork), "ev_fork");
    if (p->ev_join) chk(cudaEventDestroy(p->ev_join), "ev_join");
    if (p->side2) chk(cudaStreamDestroy(p->side2), "side2");
    if (p->ev_v) chk(cudaEventDestroy(p->ev_v), "ev_v");
    if (p->ev_dz) chk(cudaEventDestroy(p->ev_dz), "ev_dz");
    if (p->ev_join2) chk(cudaEventDestroy(p->ev_join2), "ev_join2");
    if (p->d_partial) chk(cudaFree(p->d_partial), "d_partial");
    if (p->d_slice_off) chk(cudaFree(p->d_slice_off), "d_slice_off");
    for (auto& r : p->recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    delete p;
    cudaGetLastError();  // never leave a stale error behind for the caller's next CUDA call
    return bad.empty() ? WINO_OK : set_err(WINO_CUDA_ERROR, "plan_destroy: " + bad);
}

int wino_plan_info(const wino_plan* p, wino_geometry* geom, int64_t* nnz_total, int* is_dense) {
    if (!p) return set_err(WINO_INVALID_ARGUMENT, "null plan");
    if (geom) *geom = p->g;
    if (nnz_total) *nnz_total = p->has_weights ? p->nnz : -1;
    if (is_dense) *is_dense = p->dense ? 1 : 0;
    return WINO_OK;
}

int wino_set_weights_csr(wino_plan* p, const uint64_t* const* row_ptr, const uint64_t* const* col_idx,
                         const float* const* values, const uint64_t* nnz) {
    if (!p || !row_ptr || !col_idx || !values || !nnz) return set_err(WINO_INVALID_ARGUMENT, "null argument");
    const int K = p->K, C = p->C, P2 = p->P2;
    std::vector<int> rowptr((size_t)P2 * (K + 1));
    std::vector<int> col;
    std::vector<float> val;
    int64_t off = 0;
    for (int s = 0; s < P2; ++s) {
        const uint64_t* rp = row_ptr[s];
        const uint64_t n = nnz[s];
        if (!rp || (n > 0 && (!col_idx[s] || !values[s])))
            return set_err(WINO_CORRUPT_FORMAT, "slice " + std::to_string(s) + ": missing arrays");
        if (rp[0] != 0 || rp[K] != n)
            return set_err(WINO_CORRUPT_FORMAT, "slice " + std::to_string(s) +
                                                    ": row_ptr must start at 0 and end at nnz");
        if (off + (int64_t)n >= (int64_t)1 << 31)
            return set_err(WINO_CAPABILITY_ERROR, "more than 2^31 nonzeros");
        for (int k = 0; k < K; ++k) {
            if (rp[k + 1] < rp[k] || rp[k + 1] > n)
                return set_err(WINO_CORRUPT_FORMAT, "slice " + std::to_string(s) + ": row_ptr not monotone");
            for (uint64_t e = rp[k]; e < rp[k + 1]; ++e) {
                const uint64_t cidx = col_idx[s][e];
                if (cidx >= (uint64_t)C)
                    return set_err(WINO_CORRUPT_FORMAT, "spmdm: column index out of bounds");
                if (e > rp[k] && cidx <= col_idx[s][e - 1])
                    return set_err(WINO_CORRUPT_FORMAT, "slice " + std::to_string(s) +
                                                            ": column indices not strictly increasing");
            }
        }
        for (int k = 0; k <= K; ++k) rowptr[(size_t)s * (K + 1) + k] = (int)(off + (int64_t)rp[k]);
        for (uint64_t e = 0; e < n; ++e) {
            col.push_back((int)col_idx[s][e]);
            val.push_back(values[s][e]);
        }
        off += (int64_t)n;
    }
    free_weights(p);
    p->slice_nnz.assign(nnz, nnz + P2);
    p->slice_off.resize(P2);
    for (int s = 0, o = 0; s < P2; o += (int)nnz[s], ++s) p->slice_off[s] = o;
    CUDA_TRY(cudaSetDevice(p->device));
    return upload_csr(p, rowptr, col, val);
}

int wino_set_weights(wino_plan* p, const double* w_f, double zero_tol, int dense) {
    if (!p || !w_f) return set_err(WINO_INVALID_ARGUMENT, "null argument");
    if (dense < 0 || dense > 3) return set_err(WINO_INVALID_ARGUMENT, "dense must be 0..3");
    CUDA_TRY(cudaSetDevice(p->device));
    // dense != 0: every coordinate is a weight (zeros included): the full CSR
    int rc = device_compress(p, w_f, zero_tol, dense ? 1 : 0);
    if (rc != WINO_OK || !dense) return rc;
    p->dense = true;
    p->tc_fast = dense == 3;
    if (dense >= 2) {
        rc = refresh_tc_operands(p, nullptr);
        if (rc == WINO_OK) CUDA_TRY(cudaDeviceSynchronize());
    }
    return rc;
}

int wino_get_csr(const wino_plan* p, uint64_t* nnz, uint64_t* row_ptr, uint64_t* col_idx, float* values) {
    if (!p || !nnz) return set_err(WINO_INVALID_ARGUMENT, "null argument");
    if (!p->has_weights) return set_err(WINO_CONSISTENCY_ERROR, "plan holds no CSR weights");
    const int K = p->K, P2 = p->P2;
    for (int s = 0; s < P2; ++s) nnz[s] = (uint64_t)p->slice_nnz[s];
    if (row_ptr)
        for (int s = 0; s < P2; ++s)
            for (int k = 0; k <= K; ++k)
                row_ptr[(size_t)s * (K + 1) + k] =
                    (uint64_t)(p->h_rowptr[(size_t)s * (K + 1) + k] - p->slice_off[s]);
    if (col_idx || values) {
        std::vector<int> col(p->nnz);
        std::vector<float> val(p->nnz);
        CUDA_TRY(cudaMemcpy(col.data(), p->d_colidx, p->nnz * sizeof(int), cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemcpy(val.data(), p->d_vals, p->nnz * sizeof(float), cudaMemcpyDeviceToHost));
        for (int64_t e = 0; e < p->nnz; ++e) {
            if (col_idx) col_idx[e] = (uint64_t)col[e];
            if (values) values[e] = val[e];
        }
    }
    return WINO_OK;
}

int wino_weight_values(wino_plan* p, float** values_dev) {
    int rc = check_plan(p);
    if (rc) return rc;
    if (!values_dev) return set_err(WINO_INVALID_ARGUMENT, "null argument");
    *values_dev = p->d_vals;
    return WINO_OK;
}

int wino_values_updated(wino_plan* p, void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    Launch L(p, st, K_MISC);
    wino::refresh_values_kernel<<<grid_for(p->nnz, 256, p->sm_count), 256, 0, st>>>(p->d_cv, p->d_cvT, p->d_vals,
                                                                                   p->d_perm, p->nnz);
    rc = L.done();
    if (rc == WINO_OK && p->tc_ready) rc = refresh_tc_operands(p, st);
    return rc;
}

// Every reader of Ĩ_F and dZ on this plan is a tcgen05 GEMM through the warp-specialised kernel
// (dense plan, or tensor-core contraction with the tensor-core dW): the producers then write the
// tf32 hi/lo split once (input_transform_kernel / grad_z_kernel) and the GEMMs skip their own.
// Opt-in (WINO_TC_PRESPLIT=1): measured at c3 dense 2041 vs 1945 µs — the dW GEMM gains (581 ->
// 401 µs) but K1/K4 write twice the bytes (+50/+90 µs) and the forward/dĨ_F GEMMs, which were not
// split-bound, load twice the B bytes (+25/+40 µs); c1 with the tensor-core contraction: 141 vs 148.
static bool ws_kernel_selected() {
    static const bool ok = !(std::getenv("WINO_TC_WS") && std::atoi(std::getenv("WINO_TC_WS")) == 0) &&
                           !(std::getenv("WINO_TC_FOLD") && std::atoi(std::getenv("WINO_TC_FOLD")) != 1) &&
                           !(std::getenv("WINO_TC_PERSISTENT") && std::atoi(std::getenv("WINO_TC_PERSISTENT")) == 0) &&
                           !(std::getenv("WINO_TC_DW") && std::atoi(std::getenv("WINO_TC_DW")) != 8);
    return ok;
}
static bool tc_dw_path(const wino_plan* p) {
    return p->dense || p->dw_mode == 1 || (p->dw_mode == 0 && p->contraction_mode == 2 && p->contraction == 1);
}
static bool tf32_presplit(const wino_plan* p) {
    static const bool env = std::getenv("WINO_TC_PRESPLIT") && std::atoi(std::getenv("WINO_TC_PRESPLIT")) == 1;
    return env && p->tc_ready && !p->tc_fast && p->dw_mode != 2 && ws_kernel_selected() &&
           (p->dense || p->contraction == 1) && tc_dw_path(p);
}
static int ensure_cache_t(wino_plan* p, wino_cache* c) {
    if (c->Vt) return WINO_OK;
    const int64_t NTs = round_up((int64_t)c->n_max * p->g.t, 4);
    CUDA_TRY(cudaMalloc(&c->Vt, (size_t)p->P2 * p->C * NTs * sizeof(float)));
    CUDA_TRY(cudaMalloc(&c->DZt, (size_t)p->P2 * p->K * NTs * sizeof(float)));
    return WINO_OK;
}

static int ensure_cache_lo(wino_plan* p, wino_cache* c) {
    if (c->Vlo) return WINO_OK;
    const int64_t NTs = round_up((int64_t)c->n_max * p->g.t, 4);
    CUDA_TRY(cudaMalloc(&c->Vlo, (size_t)p->P2 * p->C * NTs * sizeof(float)));
    CUDA_TRY(cudaMalloc(&c->DZlo, (size_t)p->P2 * p->K * NTs * sizeof(float)));
    return WINO_OK;
}

int wino_cache_create(wino_plan* p, int n_max, wino_cache** out) {
    if (!p || !out || n_max <= 0) return set_err(WINO_INVALID_ARGUMENT, "bad argument");
    CUDA_TRY(cudaSetDevice(p->device));
    auto* c = new wino_cache();
    c->plan = p;
    c->n_max = n_max;
    const int64_t NTs = round_up((int64_t)n_max * p->g.t, 4);
    cudaError_t e = cudaMalloc(&c->V, (size_t)p->P2 * p->C * NTs * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&c->DZ, (size_t)p->P2 * p->K * NTs * sizeof(float));
    if (e != cudaSuccess) {
        if (c->V) cudaFree(c->V);
        delete c;
        return set_err(WINO_CUDA_ERROR, std::string("cache_create: ") + cudaGetErrorString(e));
    }
    if (p->dw_mode == 2) {
        const int rc = ensure_cache_lo(p, c);
        if (rc) {
            wino_cache_destroy(c);
            return rc;
        }
    }
    *out = c;
    return WINO_OK;
}

int wino_cache_destroy(wino_cache* c) {
    if (!c) return WINO_OK;
    if (c->V) cudaFree(c->V);
    if (c->DZ) cudaFree(c->DZ);
    if (c->Vt) cudaFree(c->Vt);
    if (c->DZt) cudaFree(c->DZt);
    if (c->Vlo) cudaFree(c->Vlo);
    if (c->DZlo) cudaFree(c->DZlo);
    delete c;
    return WINO_OK;
}

int wino_forward(wino_plan* p, int n, const float* input, float* output, wino_cache* cache, int flags,
                 void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    if (!input || !output) return set_err(WINO_INVALID_ARGUMENT, "null buffer");
    if (n <= 0) return set_err(WINO_SHAPE_ERROR, "batch must be positive");
    if (cache && (cache->plan != p || n > cache->n_max))
        return set_err(WINO_SHAPE_ERROR, "cache does not match plan / batch exceeds cache capacity");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t NT = (int64_t)n * p->g.t;
    const int64_t NTs = round_up(NT, 4);
    float* V;
    if (cache) {
        V = cache->V;
    } else {
        if ((rc = ensure(&p->d_dv, &p->dv_cap, (size_t)p->P2 * std::max(p->C, p->K) * NTs))) return rc;
        V = p->d_dv;  // inference: the backward scratch doubles as Ĩ_F
    }
    if ((rc = ensure(&p->d_z, &p->z_cap, (size_t)p->P2 * p->K * NTs))) return rc;
    if (cache) {
        cache->v_split = tf32_presplit(p);
        if (cache->v_split && (rc = ensure_cache_t(p, cache))) return rc;
    }
    if ((rc = DISPATCH_MP(p, fwd_transforms, p, st, input, output, cache, V, p->d_z, n, NT, NTs, flags, 0, NTs)))
        return rc;
    if (cache && p->dw_mode == 2) {
        if ((rc = ensure_cache_lo(p, cache))) return rc;
        if ((rc = DISPATCH_MP(p, launch_input_lo, p, st, input, V, cache->Vlo, NT, NTs))) return rc;
    }
    if (p->tc_ready && (p->dense || p->contraction == 1))
        rc = launch_tc_gemm(p, st, K_DENSE_FWD, p->map_wh, p->map_wl, V, p->d_z, p->K, p->C, NTs,
                            cache && cache->v_split ? cache->Vt : nullptr);
    else
        rc = launch_spmm(p, st, K_SPMM, p->d_rowptr, p->d_cv, p->h_rowptr, V, p->d_z, p->K, p->C, NT, NTs);
    if (rc) return rc;
    if ((rc = DISPATCH_MP(p, fwd_transforms, p, st, input, output, cache, V, p->d_z, n, NT, NTs, flags, 1, NTs)))
        return rc;
    if (cache) {
        cache->n = n;
        cache->NTs = NTs;
        cache->has_fwd = true;
        cache->has_grad_z = false;  // layer.cpp:88
    }
    return WINO_OK;
}

static int bwd_check(wino_plan* p, const float* grad_output, const float* relu_out, const wino_cache* c,
                     const float* grad_w, int flags) {
    int rc = check_plan(p);
    if (rc) return rc;
    if (!c || !grad_output || (!grad_w && p->nnz > 0)) return set_err(WINO_INVALID_ARGUMENT, "null argument");
    if (c->plan != p || !c->has_fwd)
        return set_err(WINO_CONSISTENCY_ERROR, "forward cache does not match the given geometry");
    if ((flags & WINO_BWD_RELU_MASK) && !relu_out)
        return set_err(WINO_INVALID_ARGUMENT, "relu mask requested without relu_out");
    if (p->dw_mode == 2 && !c->Vlo)
        return set_err(WINO_CONSISTENCY_ERROR, "precise dW: run the forward with this mode set");
    return WINO_OK;
}

// dZ = A1·dÕ·A2ᵀ (+ its fp32 residual in the precise mode) into the cache
static int bwd_grad_z(wino_plan* p, const float* grad_output, const float* relu_out, wino_cache* c, int flags,
                      cudaStream_t st) {
    const bool mask = (flags & WINO_BWD_RELU_MASK) != 0;
    const int64_t NT = (int64_t)c->n * p->g.t, NTs = c->NTs;
    c->dz_split = tf32_presplit(p);
    if (c->dz_split) {
        const int rc0 = ensure_cache_t(p, c);
        if (rc0) return rc0;
    }
    int rc = DISPATCH_MP(p, launch_grad_z, p, st, grad_output, relu_out, c->DZ, NT, NTs, mask, NTs,
                         c->dz_split ? c->DZt : nullptr);
    if (rc) return rc;
    if (p->dw_mode == 2)
        rc = DISPATCH_MP(p, launch_grad_z_lo, p, st, grad_output, relu_out, c->DZ, c->DZlo, NT, NTs, mask);
    return rc;
}

// dW_F from the cached dZ and Ĩ_F
static int bwd_dw(wino_plan* p, const wino_cache* c, float* grad_w, cudaStream_t st) {
    const int64_t NT = (int64_t)c->n * p->g.t, NTs = c->NTs;
    const bool precise = p->dw_mode == 2;
    int rc = WINO_OK;
    const float* dzt = c->dz_split ? c->DZt : nullptr;
    const float* vt = c->v_split ? c->Vt : nullptr;
    if (p->dense && p->tc_ready && !precise) return launch_tc_dw(p, st, c->DZ, c->V, grad_w, NTs, false, dzt, vt);
    if ((c->v_split || c->dz_split) && !(!p->dense && tc_dw_path(p) && p->nnz > 0))
        return set_err(WINO_CONSISTENCY_ERROR, "the cache holds tensor-core split operands: rerun the forward "
                                               "after changing the dW mode / contraction");
    float* dwc = grad_w;
    if (p->dense && (rc = ensure(&p->d_dwc, &p->dwc_cap, (size_t)p->nnz))) return rc;
    if (p->dense) dwc = p->d_dwc;
    const bool tc_dw = p->dw_mode == 1 || (p->dw_mode == 0 && p->contraction_mode == 2 && p->contraction == 1);
    if (!p->dense && tc_dw && p->nnz > 0)
        rc = launch_tc_dw(p, st, c->DZ, c->V, dwc, NTs, /*masked=*/true, dzt, vt);
    else if (!p->dense && p->dw_mode == 3 && p->nnz > 0)
        rc = launch_ozaki_dw(p, st, c->DZ, c->V, dwc, NT, NTs);
    else if (precise)
        rc = launch_sddmm(p, st, c->DZ, c->V, dwc, NT, NTs, c->DZlo, c->Vlo);
    else
        rc = launch_sddmm(p, st, c->DZ, c->V, dwc, NT, NTs);
    if (rc) return rc;
    if (p->dense) {  // [s][k][c] -> K×C×p×q
        Launch L(p, st, K_MISC);
        wino::slice_major_to_kcpq_kernel<<<grid_for(p->nnz, 256, p->sm_count), 256, 0, st>>>(dwc, grad_w, p->K,
                                                                                            p->C, p->P2);
        rc = L.done();
    }
    return rc;
}

// dĨ_F = W_Fᵀ·dZ and dI = Σ_φ B1·dĨ_F·B2ᵀ
static int bwd_input(wino_plan* p, const wino_cache* c, float* grad_input, cudaStream_t st) {
    const int64_t NT = (int64_t)c->n * p->g.t, NTs = c->NTs;
    int rc = ensure(&p->d_dv, &p->dv_cap, (size_t)p->P2 * std::max(p->C, p->K) * NTs);
    if (rc) return rc;
    if (p->tc_ready && (p->dense || p->contraction == 1))
        rc = launch_tc_gemm(p, st, K_DENSE_DV, p->map_wth, p->map_wtl, c->DZ, p->d_dv, p->C, p->K, NTs,
                            c->dz_split ? c->DZt : nullptr);
    else if (c->dz_split)
        return set_err(WINO_CONSISTENCY_ERROR, "the cache holds tensor-core split operands: rerun the backward "
                                               "after changing the contraction");
    else
        rc = launch_spmm(p, st, K_SPMM_T, p->d_colptr, p->d_cvT, p->h_colptr, c->DZ, p->d_dv, p->C, p->K, NT, NTs);
    if (rc) return rc;
    return DISPATCH_MP(p, launch_input_grad, p, st, p->d_dv, grad_input, c->n, NTs);
}

int wino_backward_weights(wino_plan* p, const float* grad_output, const float* relu_out, wino_cache* c,
                          float* grad_w, int flags, void* stream) {
    int rc = bwd_check(p, grad_output, relu_out, c, grad_w, flags);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if ((rc = bwd_grad_z(p, grad_output, relu_out, c, flags, st))) return rc;
    if ((rc = bwd_dw(p, c, grad_w, st))) return rc;
    c->has_grad_z = true;
    return WINO_OK;
}

int wino_backward(wino_plan* p, const float* grad_output, const float* relu_out, wino_cache* c, float* grad_w,
                  float* grad_input, int flags, void* stream) {
    int rc = bwd_check(p, grad_output, relu_out, c, grad_w, flags);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if (!grad_input) {  // no dI wanted (the first layer of a stack, train.cpp:201): dW only
        if ((rc = bwd_grad_z(p, grad_output, relu_out, c, flags, st))) return rc;
        c->has_grad_z = true;
        return bwd_dw(p, c, grad_w, st);
    }
    if (!p->side) {
        // dW_F is the longest chain of the step: its stream gets the greatest priority, so its
        // blocks are scheduled first whenever SMs free up (c1 step 172 -> 169 µs measured)
        int lo = 0, hi = 0;
        CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CUDA_TRY(cudaStreamCreateWithPriority(&p->side, cudaStreamNonBlocking, hi));
        CUDA_TRY(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
    }
    if ((rc = bwd_grad_z(p, grad_output, relu_out, c, flags, st))) return rc;
    c->has_grad_z = true;
    // dW (side stream) and dĨ_F -> dI (caller's stream) only share the read-only dZ and Ĩ_F
    CUDA_TRY(cudaEventRecord(p->ev_fork, st));
    CUDA_TRY(cudaStreamWaitEvent(p->side, p->ev_fork, 0));
    if ((rc = bwd_dw(p, c, grad_w, p->side))) return rc;
    CUDA_TRY(cudaEventRecord(p->ev_join, p->side));
    if ((rc = bwd_input(p, c, grad_input, st))) return rc;
    CUDA_TRY(cudaStreamWaitEvent(st, p->ev_join, 0));
    return WINO_OK;
}

// One training step of the layer (forward, then backward with both gradients) scheduled as the
// dependency graph it is instead of in API order: dZ = A1·dÕ·A2ᵀ needs only dO, so the
// dO -> dZ -> dĨ_F -> dI chain runs beside the forward from the start (side2), and dW_F waits
// for just Ĩ_F and dZ (side) — the forward's SpMM and output transform overlap the backward.
// Same kernels, same buffers, same results bit for bit as wino_forward + wino_backward.
int wino_forward_backward(wino_plan* p, int n, const float* input, float* output, wino_cache* c,
                          const float* grad_output, float* grad_w, float* grad_input, void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    if (!input || !output || !c || !grad_output || !grad_input || (!grad_w && p->nnz > 0))
        return set_err(WINO_INVALID_ARGUMENT, "null buffer");
    if (n <= 0) return set_err(WINO_SHAPE_ERROR, "batch must be positive");
    if (c->plan != p || n > c->n_max)
        return set_err(WINO_SHAPE_ERROR, "cache does not match plan / batch exceeds cache capacity");
    cudaStream_t st = (cudaStream_t)stream;
    if (!p->side) {
        // dW_F is the longest chain of the step: its stream gets the greatest priority, so its
        // blocks are scheduled first whenever SMs free up (c1 step 172 -> 169 µs measured)
        int lo = 0, hi = 0;
        CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CUDA_TRY(cudaStreamCreateWithPriority(&p->side, cudaStreamNonBlocking, hi));
        CUDA_TRY(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
    }
    if (!p->side2) {
        CUDA_TRY(cudaStreamCreateWithFlags(&p->side2, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&p->ev_v, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&p->ev_dz, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&p->ev_join2, cudaEventDisableTiming));
    }
    const int64_t NT = (int64_t)n * p->g.t;
    const int64_t NTs = round_up(NT, 4);
    if ((rc = ensure(&p->d_z, &p->z_cap, (size_t)p->P2 * p->K * NTs))) return rc;
    if ((rc = ensure(&p->d_dv, &p->dv_cap, (size_t)p->P2 * std::max(p->C, p->K) * NTs))) return rc;
    if (p->dw_mode == 2 && (rc = ensure_cache_lo(p, c))) return rc;
    c->v_split = tf32_presplit(p);
    if (c->v_split && (rc = ensure_cache_t(p, c))) return rc;
    c->n = n;
    c->NTs = NTs;
    c->has_fwd = true;
    c->has_grad_z = false;
    // fork both side streams off the caller's stream
    CUDA_TRY(cudaEventRecord(p->ev_fork, st));
    CUDA_TRY(cudaStreamWaitEvent(p->side2, p->ev_fork, 0));
    CUDA_TRY(cudaStreamWaitEvent(p->side, p->ev_fork, 0));
    // side2: dZ, then dĨ_F = W_Fᵀ·dZ and dI
    if ((rc = bwd_grad_z(p, grad_output, nullptr, c, 0, p->side2))) return rc;
    CUDA_TRY(cudaEventRecord(p->ev_dz, p->side2));
    if ((rc = bwd_input(p, c, grad_input, p->side2))) return rc;
    CUDA_TRY(cudaEventRecord(p->ev_join2, p->side2));
    // caller's stream: Ĩ_F, then Z = W_F·Ĩ_F and O
    if ((rc = DISPATCH_MP(p, fwd_transforms, p, st, input, output, c, c->V, p->d_z, n, NT, NTs, 0, 0, NTs)))
        return rc;
    if (p->dw_mode == 2 && (rc = DISPATCH_MP(p, launch_input_lo, p, st, input, c->V, c->Vlo, NT, NTs))) return rc;
    CUDA_TRY(cudaEventRecord(p->ev_v, st));
    // side: dW_F once Ĩ_F and dZ exist
    CUDA_TRY(cudaStreamWaitEvent(p->side, p->ev_v, 0));
    CUDA_TRY(cudaStreamWaitEvent(p->side, p->ev_dz, 0));
    if ((rc = bwd_dw(p, c, grad_w, p->side))) return rc;
    CUDA_TRY(cudaEventRecord(p->ev_join, p->side));
    if (p->tc_ready && (p->dense || p->contraction == 1))
        rc = launch_tc_gemm(p, st, K_DENSE_FWD, p->map_wh, p->map_wl, c->V, p->d_z, p->K, p->C, NTs,
                            c->v_split ? c->Vt : nullptr);
    else
        rc = launch_spmm(p, st, K_SPMM, p->d_rowptr, p->d_cv, p->h_rowptr, c->V, p->d_z, p->K, p->C, NT, NTs);
    if (rc) return rc;
    if ((rc = DISPATCH_MP(p, fwd_transforms, p, st, input, output, c, c->V, p->d_z, n, NT, NTs, 0, 1, NTs)))
        return rc;
    // join
    CUDA_TRY(cudaStreamWaitEvent(st, p->ev_join2, 0));
    CUDA_TRY(cudaStreamWaitEvent(st, p->ev_join, 0));
    c->has_grad_z = true;
    return WINO_OK;
}

// ---- image ranges of one batch (pipelined host transfers) ----
struct ColRange {
    int64_t a, NT, NTs, NTr;  // first column, valid columns, row stride, owned columns
};

static int make_range(const wino_plan* p, int n_total, int n0, int n1, ColRange* r) {
    if (n_total <= 0 || n0 < 0 || n1 <= n0 || n1 > n_total)
        return set_err(WINO_SHAPE_ERROR, "image range [" + std::to_string(n0) + ", " + std::to_string(n1) +
                                             ") outside the batch of " + std::to_string(n_total));
    const int64_t T = p->g.t;
    r->a = (int64_t)n0 * T;
    if (r->a % 4) return set_err(WINO_SHAPE_ERROR, "range start n0·T must be a multiple of 4 (16-byte columns)");
    r->NTs = round_up((int64_t)n_total * T, 4);
    r->NT = (int64_t)(n1 - n0) * T;
    r->NTr = n1 == n_total ? r->NTs - r->a : r->NT;
    return WINO_OK;
}

static int range_capable(const wino_plan* p) {
    if (p->tc_ready || p->dw_mode != 0)
        return set_err(WINO_CAPABILITY_ERROR, "image-range calls run the CSR kernels only "
                                              "(no tensor-core plan/contraction, dW mode 0)");
    return WINO_OK;
}

int wino_forward_range(wino_plan* p, int n_total, int n0, int n1, const float* input, float* output,
                       wino_cache* cache, int flags, void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    if ((rc = range_capable(p))) return rc;
    if (!input || !output || !cache) return set_err(WINO_INVALID_ARGUMENT, "null argument");
    if (cache->plan != p || n_total > cache->n_max)
        return set_err(WINO_SHAPE_ERROR, "cache does not match plan / batch exceeds cache capacity");
    ColRange r{};
    if ((rc = make_range(p, n_total, n0, n1, &r))) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if ((rc = ensure(&p->d_z, &p->z_cap, (size_t)p->P2 * p->K * r.NTs))) return rc;
    float* V = cache->V + r.a;
    float* Z = p->d_z + r.a;
    cache->v_split = false;  // range calls run the CSR kernels on fp32 operands
    if ((rc = DISPATCH_MP(p, fwd_transforms, p, st, input, output, cache, V, Z, n1 - n0, r.NT, r.NTs, flags, 0,
                          r.NTr)))
        return rc;
    if ((rc = launch_spmm(p, st, K_SPMM, p->d_rowptr, p->d_cv, p->h_rowptr, V, Z, p->K, p->C, r.NT, r.NTs, r.NTr)))
        return rc;
    if ((rc = DISPATCH_MP(p, fwd_transforms, p, st, input, output, cache, V, Z, n1 - n0, r.NT, r.NTs, flags, 1,
                          r.NTr)))
        return rc;
    cache->n = n_total;
    cache->NTs = r.NTs;
    cache->has_fwd = true;
    cache->has_grad_z = false;
    return WINO_OK;
}

int wino_backward_range(wino_plan* p, int n0, int n1, const float* grad_output, const float* relu_out,
                        wino_cache* c, float* grad_input, int flags, void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    if ((rc = range_capable(p))) return rc;
    if (!c || !grad_output || !grad_input) return set_err(WINO_INVALID_ARGUMENT, "null argument");
    if (c->plan != p || !c->has_fwd)
        return set_err(WINO_CONSISTENCY_ERROR, "forward cache does not match the given geometry");
    const bool mask = (flags & WINO_BWD_RELU_MASK) != 0;
    if (mask && !relu_out) return set_err(WINO_INVALID_ARGUMENT, "relu mask requested without relu_out");
    ColRange r{};
    if ((rc = make_range(p, c->n, n0, n1, &r))) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if ((rc = ensure(&p->d_dv, &p->dv_cap, (size_t)p->P2 * std::max(p->C, p->K) * r.NTs))) return rc;
    float* DZ = c->DZ + r.a;
    float* DV = p->d_dv + r.a;
    c->dz_split = false;
    if ((rc = DISPATCH_MP(p, launch_grad_z, p, st, grad_output, relu_out, DZ, r.NT, r.NTs, mask, r.NTr)))
        return rc;
    if ((rc = launch_spmm(p, st, K_SPMM_T, p->d_colptr, p->d_cvT, p->h_colptr, DZ, DV, p->C, p->K, r.NT, r.NTs,
                          r.NTr)))
        return rc;
    if ((rc = DISPATCH_MP(p, launch_input_grad, p, st, DV, grad_input, n1 - n0, r.NTs))) return rc;
    // dW_F partials of this range's t chunks, when the range is whole chunks of the chunk-form
    // SDDMM (backward_weights_cached then only sums the chunks)
    const int64_t NTfull = (int64_t)c->n * p->g.t;
    if (p->sddmm_impl == 1 && p->dw_mode == 0 && !p->dense && p->nnz > 0 && p->lane_tw > 0) {
        const int TW = p->lane_tw;
        const int chunks = (int)((NTfull + TW - 1) / TW);
        const bool last = n1 == c->n;
        if (chunks > 1 && r.a % TW == 0 && (last || (r.a + r.NT) % TW == 0)) {
            const int z0 = (int)(r.a / TW), z1 = last ? chunks : (int)((r.a + r.NT) / TW);
            if ((rc = launch_sddmm_chunk(p, st, c->DZ, c->V, nullptr, NTfull, r.NTs, z0, z1, false))) return rc;
            if (z0 == 0) c->dw_chunks = 0;
            c->dw_chunks += z1 - z0;
        }
    }
    c->has_grad_z = true;
    return WINO_OK;
}

int wino_backward_weights_cached(wino_plan* p, wino_cache* c, float* grad_w, void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    if (!c || (!grad_w && p->nnz > 0)) return set_err(WINO_INVALID_ARGUMENT, "null argument");
    if (c->plan != p || !c->has_fwd || !c->has_grad_z)
        return set_err(WINO_CONSISTENCY_ERROR, "backward_weights_cached: dL/dZ missing; run backward_range first");
    const int64_t NTfull = (int64_t)c->n * p->g.t;
    if (p->sddmm_impl == 1 && p->dw_mode == 0 && !p->dense && p->lane_tw > 0 && p->nnz > 0 &&
        c->dw_chunks == (int)((NTfull + p->lane_tw - 1) / p->lane_tw)) {
        // every chunk's partials came from the ranges: only their ordered sum remains
        const int rc2 = launch_sddmm_chunk(p, (cudaStream_t)stream, c->DZ, c->V, grad_w, NTfull, c->NTs, 0, 0, true);
        c->dw_chunks = 0;
        return rc2;
    }
    c->dw_chunks = 0;
    return bwd_dw(p, c, grad_w, (cudaStream_t)stream);
}

// ---- the data-parallel exchange: one in-place sum of dW_F over an NCCL communicator ----
// NCCL is resolved at run time (the process's already-loaded libnccl, e.g. PyTorch's, else the
// system one), so the library has no link-time NCCL dependency.  ABI constants of nccl.h:
// ncclFloat32 = 7, ncclSum = 0, ncclSuccess = 0.
namespace {
using nccl_allreduce_t = int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t);
using nccl_errstr_t = const char* (*)(int);
nccl_allreduce_t g_nccl_allreduce = nullptr;
nccl_errstr_t g_nccl_errstr = nullptr;
std::once_flag g_nccl_once;

void resolve_nccl() {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    g_nccl_allreduce = reinterpret_cast<nccl_allreduce_t>(dlsym(h, "ncclAllReduce"));
    g_nccl_errstr = reinterpret_cast<nccl_errstr_t>(dlsym(h, "ncclGetErrorString"));
}
}  // namespace

int wino_allreduce_dw(wino_plan* p, void* nccl_comm, float* grad_w, int64_t count, void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    if (!nccl_comm || (!grad_w && count != 0)) return set_err(WINO_INVALID_ARGUMENT, "null argument");
    if (count < 0) count = p->dense ? (int64_t)p->P2 * p->K * p->C : p->nnz;
    if (count == 0) return WINO_OK;
    std::call_once(g_nccl_once, resolve_nccl);
    if (!g_nccl_allreduce) return set_err(WINO_CAPABILITY_ERROR, "allreduce_dw: libnccl.so.2 not found");
    const int r = g_nccl_allreduce(grad_w, grad_w, (size_t)count, /*ncclFloat32*/ 7, /*ncclSum*/ 0, nccl_comm,
                                   (cudaStream_t)stream);
    if (r != 0)
        return set_err(WINO_CUDA_ERROR, std::string("ncclAllReduce: ") + (g_nccl_errstr ? g_nccl_errstr(r) : "error"));
    return WINO_OK;
}

int wino_backward_input(wino_plan* p, const wino_cache* c, float* grad_input, void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    if (!c) return set_err(WINO_INVALID_ARGUMENT, "null cache");
    if (c->plan != p)
        return set_err(WINO_CONSISTENCY_ERROR, "forward cache does not match the given geometry");
    if (!c->has_fwd || !c->has_grad_z)  // layer.cpp:137-138
        return set_err(WINO_CONSISTENCY_ERROR, "backward_input: dL/dZ missing; run backward_weights first");
    if (!grad_input) return set_err(WINO_INVALID_ARGUMENT, "null grad_input");
    return bwd_input(p, c, grad_input, (cudaStream_t)stream);
}

int wino_update_weights(wino_plan* p, const float* grad_w, const wino_update* u, void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    if (!grad_w || !u) return set_err(WINO_INVALID_ARGUMENT, "null argument");
    if (u->norm != 1 && u->norm != 2) return set_err(WINO_INVALID_ARGUMENT, "norm must be 1 or 2");
    if (p->nnz == 0) return WINO_OK;
    cudaStream_t st = (cudaStream_t)stream;
    wino::UpdateParams up{u->lr, u->scale, u->lambda, u->eps, u->beta, u->norm, u->prune};
    if (u->norm == 2 && u->lambda != 0.0) {  // ‖w‖₂ of the layer before the step (train.cpp:264)
        const int parts = std::min<int64_t>(4 * p->sm_count, (p->nnz + 1023) / 1024);
        if ((rc = grow(&p->d_sumsq_part, &p->cap_sumsq_part, (size_t)parts))) return rc;
        Launch L(p, st, K_SGD);
        wino::sumsq_partial_kernel<<<parts, 1024, 0, st>>>(p->d_vals, p->nnz, p->d_sumsq_part);
        wino::sumsq_final_kernel<<<1, 1024, 0, st>>>(p->d_sumsq_part, parts, p->d_scalar);
        ++p->launches;
        if ((rc = L.done())) return rc;
    }
    {
        Launch L(p, st, K_SGD);
        wino::update_kernel<<<grid_for(p->nnz, 256, p->sm_count), 256, 0, st>>>(
            p->d_vals, grad_w, p->nnz, p->dense ? 1 : 0, p->K, p->C, p->P2, up, p->d_scalar, p->d_nonfinite);
        if ((rc = L.done())) return rc;
    }
    return wino_values_updated(p, stream);
}

int wino_sgd_step(wino_plan* p, const float* grad_w, float lr, float scale, float l2, void* stream) {
    const wino_update u{lr, scale, l2, 0.0, 0.0, 2, 0};
    return wino_update_weights(p, grad_w, &u, stream);
}

int wino_update_status(wino_plan* p, int64_t* nonfinite) {
    if (!p || !nonfinite) return set_err(WINO_INVALID_ARGUMENT, "null argument");
    unsigned long long n = 0;
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpy(&n, p->d_nonfinite, sizeof(n), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemset(p->d_nonfinite, 0, sizeof(n)));
    *nonfinite = (int64_t)n;
    return WINO_OK;
}

int wino_recompress(wino_plan* p, double zero_tol) {
    int rc = check_plan(p);
    if (rc) return rc;
    const int K = p->K, C = p->C, P2 = p->P2;
    const int64_t total = (int64_t)P2 * K * C;
    CUDA_TRY(cudaSetDevice(p->device));
    CUDA_TRY(cudaDeviceSynchronize());
    if ((rc = grow(&p->d_wsrc, &p->cap_wsrc, (size_t)total))) return rc;
    CUDA_TRY(cudaMemset(p->d_wsrc, 0, (size_t)total * sizeof(double)));
    if (p->nnz > 0) {
        Launch L(p, 0, K_MISC);
        wino::csr_to_kcpq_f64_kernel<<<grid_for((int64_t)K * P2, 128, p->sm_count), 128>>>(
            p->d_rowptr, p->d_colidx, p->d_vals, K, C, P2, p->d_wsrc);
        if ((rc = L.done())) return rc;
    }
    return compress_from_wsrc(p, zero_tol, 0);
}

int wino_set_option(wino_plan* p, int option, int value) {
    if (!p) return set_err(WINO_INVALID_ARGUMENT, "null plan");
    if (option == WINO_OPT_CONTRACTION) {
        if (value < 0 || value > 2) return set_err(WINO_INVALID_ARGUMENT, "contraction must be 0, 1 or 2");
        if (value == 1 && (p->C % 4 || p->K % 4))
            return set_err(WINO_CAPABILITY_ERROR, "tensor-core contraction needs C and K multiples of 4 (TMA strides)");
        p->contraction_mode = value;
        p->contraction = value == 1 ? 1 : 0;
        return apply_contraction(p);
    }
    if (option == WINO_OPT_AUTO_DENSITY) {
        if (value < 0 || value > 1000) return set_err(WINO_INVALID_ARGUMENT, "auto density is per mille, 0..1000");
        p->auto_permille = value;
        return p->contraction_mode == 2 ? apply_contraction(p) : WINO_OK;
    }
    if (option != WINO_OPT_DW_MODE || value < 0 || value > 3)
        return set_err(WINO_INVALID_ARGUMENT, "unknown option / value");
    if (value == 1 || value == 3) {
        if (p->C % 4 || p->K % 4)
            return set_err(WINO_CAPABILITY_ERROR, "tensor-core dW needs C and K multiples of 4 (TMA strides)");
        if (!p->d_slice_off && p->has_weights) {
            CUDA_TRY(cudaMalloc(&p->d_slice_off, p->P2 * sizeof(int64_t)));
            CUDA_TRY(cudaMemcpy(p->d_slice_off, p->slice_off.data(), p->P2 * sizeof(int64_t), cudaMemcpyHostToDevice));
        }
    }
    const bool replan = (value == 2) != (p->dw_mode == 2);
    p->dw_mode = value;
    if (replan && p->has_weights) plan_sddmm_all(p);  // the precise variant stages twice the rows
    return WINO_OK;
}

int64_t wino_launch_count(const wino_plan* p) { return p ? p->launches : -1; }
void wino_reset_launch_count(wino_plan* p) {
    if (p) p->launches = 0;
}

int wino_profile_enable(wino_plan* p, int enable) {
    if (!p) return set_err(WINO_INVALID_ARGUMENT, "null plan");
    p->prof = enable != 0;
    return WINO_OK;
}

int wino_profile_read(wino_plan* p, int cap, const char** names, double* ms, int64_t* launches, int* n_kinds) {
    if (!p) return set_err(WINO_INVALID_ARGUMENT, "null plan");
    for (auto& r : p->recs) {
        CUDA_TRY(cudaEventSynchronize(r.b));
        float t = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&t, r.a, r.b));
        p->prof_ms[r.kind] += t;
        p->prof_n[r.kind] += 1;
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    p->recs.clear();
    const int n = std::min(cap, (int)K_NKINDS);
    for (int k = 0; k < n; ++k) {
        if (names) names[k] = kKindNames[k];
        if (ms) ms[k] = p->prof_ms[k];
        if (launches) launches[k] = p->prof_n[k];
        p->prof_ms[k] = 0.0;
        p->prof_n[k] = 0;
    }
    if (n_kinds) *n_kinds = n;
    return WINO_OK;
}

}  // extern "C"
