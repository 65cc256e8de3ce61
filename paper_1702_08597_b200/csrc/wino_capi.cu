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
#include "wino_tmap.h"
#include "wino_update.cuh"
#include "wino_xdw.cuh"
#include "wino_spmm_tm.cuh"

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

// input_transform / grad_z: K1 / K4, in training steps fused with the exact dW_F digits;
// amax: the per-(segment, row) max|I| / max|dO| pre-pass that bounds the digit exponents.
enum Kind { K_INPUT = 0, K_SPMM, K_OUTPUT, K_GRADZ, K_AMAX, K_DW_GEMM, K_DW_REDUCE, K_SPMM_T, K_INGRAD,
            K_DENSE_FWD, K_DENSE_DV, K_SGD, K_MISC, K_NKINDS };
const char* kKindNames[K_NKINDS] = {"input_transform", "spmm_fwd",      "output_transform", "grad_z",
                                    "amax",            "dw_gemm_i8",    "dw_reduce",        "spmm_bwd_data",
                                    "input_grad",      "dense_fwd_tc",  "dense_dv_tc",      "sgd",
                                    "misc"};

struct ProfRec {
    int kind;
    cudaEvent_t a, b;
};

// One exponent segment of the batch (images [n0, n1), digit columns [col0, col0 + ncols_pad)):
// the exact dW_F digits of its rows share one exponent per (slice, row) (wino_xdw.cuh).
struct DwSeg {
    int n0, n1;
    int64_t col0, ncols_pad;
};

}  // namespace

struct wino_plan {
    int device = 0;
    int C = 0, K = 0, H = 0, W = 0, pad = 0, m = 0, r = 0, p = 0, P2 = 0;
    wino_geometry g{};
    wino::Coefs cf{};
    wino::CoefsD cfd{};              // the transform in the reference's doubles (exact dW_F digits)
    wino::xdw::Norms nrm_v{}, nrm_z{};  // ‖B_i‖₁‖B_j‖₁ and ‖A_i‖₁‖A_j‖₁ per slice: digit exponent bounds
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
    // tcgen05 contraction operands (dense plan, or a sparse plan with the tensor-core contraction):
    // W and Wᵀ split into tf32 hi/lo, [36][K][C] and [36][C][K]
    float* d_wdense = nullptr;
    float* d_wh = nullptr;
    float* d_wl = nullptr;
    float* d_wth = nullptr;
    float* d_wtl = nullptr;
    CUtensorMap map_wh{}, map_wl{}, map_wth{}, map_wtl{};
    bool tc_ready = false;
    int contraction = 0;       // sparse plan, in effect: 0 = CSR kernels (reference order), 1 = tcgen05 on zero-filled W_F
    int contraction_mode = 0;  // as requested: 0 csr, 1 tc, 2 auto (tc when dense enough)
    int auto_permille = -1;    // auto: tensor cores at density >= this / 1000; -1: the measured default
                               // (110 where the hybrid CSR kernel applies, 128 < C, K <= 256: c3 crossover
                               // 10.7%; 80 elsewhere: c1 9%, c2 6%)
    int64_t* d_slice_off = nullptr;
    // TMEM SpMM (wino_spmm_tm.cuh): the padded stage-segment streams of the CSR [0] and CSC [1],
    // rebuilt whenever the structure changes, values refreshed by wino_values_updated
    int spmm_operands = 0;  // WINO_OPT_SPMM_OPERANDS: 0 auto, 1 shared memory, 2 tensor memory, 3 hybrid
    void* dw_comm = nullptr;  // wino_set_dw_allreduce: ncclComm_t of the in-backward dW_F exchange
    struct TmStream {        // the TMEM SpMM's padded stage-segment stream of one direction
        int2* cv = nullptr;  // (TMEM column, value)
        int* pidx = nullptr; // source entry (-1: pad)
        int* bnd = nullptr;  // [P2][rows][S+1] segment starts
        int* cnt = nullptr;  // [P2·rows + 1] scan scratch
        size_t cap_cv = 0, cap_pidx = 0, cap_bnd = 0, cap_cnt = 0;
        int64_t n = 0;       // stream length
        int64_t max_slice = 0;
        int R = 4, S = 2;    // t per lane and stages of the layout the stream encodes
        bool ready = false;
    } tms[2];
    double* d_xpart = nullptr;  // exact dW_F: scaled fp64 products per accumulation chunk [chunk][P2][K][C]
    size_t xpart_cap = 0;
    // scratch
    float* d_z = nullptr;
    size_t z_cap = 0;
    float* d_dv = nullptr;
    size_t dv_cap = 0;
    double* d_scalar = nullptr;
    cudaStream_t side = nullptr;  // dW_F chain (greatest priority)
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
    float* V = nullptr;   // Ĩ_F [P2][C][NTs] fp32 (the forward's operand, bitwise the reference's f32)
    float* DZ = nullptr;  // dZ  [P2][K][NTs] fp32
    // exact dW_F operands (wino_xdw.cuh): digit planes of the f64 Ĩ_F and dZ, per-segment row
    // maxima of |I| and |dO| (from K1 / K4) and the digit exponents
    int8_t* dig_v = nullptr;
    int8_t* dig_z = nullptr;
    int64_t NTd = 0;  // digit row stride (capacity in columns)
    unsigned* amax_v = nullptr;
    unsigned* amax_z = nullptr;
    int* e_v = nullptr;
    int* e_z = nullptr;
    int seg_cap = 0;
    std::vector<DwSeg> segs;  // the batch's exponent segments in column order (set by the forward)
    int z_segs = 0;           // segments whose dZ digits exist (set by the backward)
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
    const bool staged = (int)(xbytes + seg) <= p->max_smem;
    const size_t smem = staged ? xbytes + seg : xbytes;
    if ((int)smem > p->max_smem)
        return set_err(WINO_CAPABILITY_ERROR, "spmm: staged chunk exceeds shared memory");
    Launch L(p, st, kind);
    constexpr int threads = 1024;
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
bool tm_applies(const wino_plan* p, int ncols) { return p->spmm_operands != 1 && ncols > 128 && ncols <= 512; }

// Build the TMEM SpMM stream of direction dir (0: CSR rows K over C columns, 1: CSC rows C over K)
// for the current structure and values (device-synchronous: at weight-set time only).
int build_tm_stream(wino_plan* p, int dir) {
    namespace t = wino::tm;
    auto& ts = p->tms[dir];
    ts.ready = false;
    const int nrows = dir ? p->C : p->K, ncols = dir ? p->K : p->C;
    if (!(ncols > 128 && ncols <= 512) || p->nnz == 0) return WINO_OK;
    // the layout: R t per lane and S stages (wino_spmm_tm.cuh)
    const int R = t::lanes_t(ncols);
    const int S = (ncols + t::stage_rows(R) - 1) / t::stage_rows(R) <= 2 ? 2 : 4;
    ts.R = R;
    ts.S = S;
    const int* rowptr = dir ? p->d_colptr : p->d_rowptr;
    const int2* cv = dir ? p->d_cvT : p->d_cv;
    const int64_t rows = (int64_t)p->P2 * nrows;
    int rc;
    if ((rc = grow(&ts.cnt, &ts.cap_cnt, (size_t)rows + 1)) || (rc = grow(&ts.bnd, &ts.cap_bnd, (size_t)rows * (S + 1))))
        return rc;
    t::tm_count_kernel<<<grid_for(rows, 128, p->sm_count), 128>>>(rowptr, cv, nrows, p->P2, S, R, ts.cnt);
    t::tm_scan_kernel<<<1, 1024>>>(ts.cnt, (int)rows);
    CUDA_TRY(cudaGetLastError());
    std::vector<int> off((size_t)rows + 1);
    CUDA_TRY(cudaMemcpy(off.data(), ts.cnt, off.size() * sizeof(int), cudaMemcpyDeviceToHost));
    ts.n = off.back();
    ts.max_slice = 0;
    for (int s = 0; s < p->P2; ++s)
        ts.max_slice = std::max<int64_t>(ts.max_slice, off[(size_t)(s + 1) * nrows] - off[(size_t)s * nrows]);
    if ((rc = grow(&ts.cv, &ts.cap_cv, (size_t)ts.n + 2)) || (rc = grow(&ts.pidx, &ts.cap_pidx, (size_t)ts.n + 2)))
        return rc;
    t::tm_fill_kernel<<<grid_for(rows, 128, p->sm_count), 128>>>(rowptr, cv, ts.cnt, nrows, p->P2, S, R, ts.cv, ts.pidx,
                                                                 ts.bnd);
    p->launches += 3;
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
    ts.ready = true;
    return WINO_OK;
}

int build_tm_streams(wino_plan* p) {
    int rc = build_tm_stream(p, 0);
    return rc ? rc : build_tm_stream(p, 1);
}

// K2/K6 with the X chunk in TMEM (wino_spmm_tm.cuh)
int launch_spmm_tm(wino_plan* p, cudaStream_t st, int kind, const float* X, float* Y, int nrows, int ncols,
                   int64_t NTs, int64_t NTr) {
    namespace t = wino::tm;
    const int dir = kind == K_SPMM_T ? 1 : 0;
    const auto& ts = p->tms[dir];
    const int R = ts.R, S = ts.S;
    const int TW = 32 * R * (4 / S);
    const int chunks = (int)((NTr + TW - 1) / TW);
    const int units = chunks * p->P2;
    // stage each slice's stream in shared memory when the largest slice fits
    const int staged_smem = t::smem_bytes(R, S, nrows, ts.max_slice);
    const bool staged = staged_smem <= p->max_smem;
    const int smem = std::max(staged ? staged_smem : t::smem_fixed(R, S), t::kMinSmem);
    const unsigned long long z = 0x8000000080000000ull;  // (-0.f, -0.f)
    const int grid = std::min(units, p->sm_count);
    Launch L(p, st, kind);
    auto go = [&](auto kern) {
        set_smem_attr(kern, smem);
        kern<<<grid, t::THREADS, smem, st>>>(ts.cv, ts.bnd, X, Y, nrows, ncols, (int)NTs, (int)NTr, chunks, units, z);
    };
    if (S == 2) staged ? go(t::spmm_tmem_kernel<4, 2, true>) : go(t::spmm_tmem_kernel<4, 2, false>);
    else staged ? go(t::spmm_tmem_kernel<4, 4, true>) : go(t::spmm_tmem_kernel<4, 4, false>);
    return L.done();
}

// K2/K6 with operand rows [0,128) in TMEM and [128, ncols) in shared memory (128 < ncols <= 256)
bool hyb_applies(const wino_plan* p, int ncols, int dir) {
    return ncols > 128 && ncols <= 256 && p->tms[dir].ready && p->tms[dir].S == 2 && p->tms[dir].R == 4;
}

int launch_spmm_hyb(wino_plan* p, cudaStream_t st, int kind, const float* X, float* Y, int nrows, int ncols,
                    int64_t NTs, int64_t NTr) {
    namespace t = wino::tm;
    const auto& ts = p->tms[kind == K_SPMM_T ? 1 : 0];
    const int chunks = (int)((NTr + t::HYB_TW - 1) / t::HYB_TW);
    const int units = chunks * p->P2;
    const int staged_smem = t::hyb_smem_bytes(ncols, nrows, ts.max_slice);
    const bool staged = staged_smem <= p->max_smem;
    const int smem = std::max(staged ? staged_smem : t::hyb_smem_fixed(ncols), t::kMinSmem);
    const unsigned long long z = 0x8000000080000000ull;  // (-0.f, -0.f)
    const int grid = std::min(units, p->sm_count);
    Launch L(p, st, kind);
    auto go = [&](auto kern) {
        set_smem_attr(kern, smem);
        kern<<<grid, t::THREADS, smem, st>>>(ts.cv, ts.bnd, X, Y, nrows, ncols, (int)NTs, (int)NTr, chunks, units, z);
    };
    staged ? go(t::spmm_hyb_kernel<true>) : go(t::spmm_hyb_kernel<false>);
    return L.done();
}

int launch_spmm(wino_plan* p, cudaStream_t st, int kind, const int* rowptr, const int2* cv,
                const std::vector<int>& hptr, const float* X, float* Y, int nrows, int ncols, int64_t NT,
                int64_t NTs, int64_t NTr = -1) {
    if (NTr < 0) NTr = NTs;
    // TMEM operands where they pay (measured): their per-(row, stage) and per-unit
    // costs are fixed, so they win once a row has enough entries (density >= 4%: c3 95% 317 vs
    // 344 µs, 97% 272 vs 265) and the units fill the GPU at least twice; below that the
    // shared-memory kernel is faster
    const double density = (double)p->nnz / ((double)p->P2 * p->K * p->C);
    const auto& tms = p->tms[kind == K_SPMM_T ? 1 : 0];
    const int64_t tm_w = 32 * tms.R * (4 / tms.S);
    const int64_t tm_units = (NTr + tm_w - 1) / tm_w * p->P2;  // CTA-units
    // hybrid operands (TMEM + shared memory, no stage handoffs) when its staged stream fits next to
    // the shared-memory half of the chunk (c3: 90% 428 vs 441 µs, 95% 284 vs 315; unstaged it loses)
    const int dir = kind == K_SPMM_T ? 1 : 0;
    if (hyb_applies(p, ncols, dir) &&
        (p->spmm_operands == 3 ||
         (p->spmm_operands == 0 && density >= 0.04 && tm_units >= 2 * p->sm_count &&
          wino::tm::hyb_smem_bytes(ncols, nrows, tms.max_slice) <= p->max_smem)))
        return launch_spmm_hyb(p, st, kind, X, Y, nrows, ncols, NTs, NTr);
    if (tm_applies(p, ncols) && p->tms[kind == K_SPMM_T ? 1 : 0].ready &&
        (p->spmm_operands == 2 || (density >= 0.04 && tm_units >= 2 * p->sm_count)))
        return launch_spmm_tm(p, st, kind, X, Y, nrows, ncols, NTs, NTr);
    switch (spmm_r(ncols)) {
        case 4: return launch_spmm_r<4>(p, st, kind, rowptr, cv, hptr, X, Y, nrows, ncols, NT, NTs, NTr);
        case 2: return launch_spmm_r<2>(p, st, kind, rowptr, cv, hptr, X, Y, nrows, ncols, NT, NTs, NTr);
        default: return launch_spmm_r<1>(p, st, kind, rowptr, cv, hptr, X, Y, nrows, ncols, NT, NTs, NTr);
    }
}

// stage 0: K1 (Ĩ_F only: inference; training steps run K1 fused with the dW_F digits);
// stage 1: K3 (O)
template <int M, int P, class CF>
int fwd_transforms(wino_plan* p, cudaStream_t st, const float* in, float* out, float* V, float* Z, int n,
                   int64_t NT, int64_t NTs, int flags, int stage, int64_t NTr) {
    const wino_geometry& g = p->g;
    if (stage == 0) {
        Launch L(p, st, K_INPUT);
        wino::input_transform_kernel<M, P, CF><<<dim3((unsigned)((NTr + 255) / 256), (unsigned)p->C), 256, 0, st>>>(
            in, V, p->cf, p->C, p->H, p->W, p->pad, (int)g.tiles_x, (int)g.t, (int)NT, (int)NTs, (int)NTr);
        return L.done();
    }
    Launch L(p, st, K_OUTPUT);
    const dim3 grid((unsigned)((NT + 255) / 256), (unsigned)p->K);
    if (flags & WINO_FWD_RELU)
        wino::output_transform_kernel<M, P, true, CF><<<grid, 256, 0, st>>>(
            Z, out, p->cf, p->K, (int)g.h_o, (int)g.w_o, (int)g.tiles_x, (int)g.t, (int)NT, (int)NTs);
    else
        wino::output_transform_kernel<M, P, false, CF><<<grid, 256, 0, st>>>(
            Z, out, p->cf, p->K, (int)g.h_o, (int)g.w_o, (int)g.tiles_x, (int)g.t, (int)NT, (int)NTs);
    return L.done();
}

template <int M, int P, class CF>
int launch_input_grad(wino_plan* p, cudaStream_t st, const float* DV, float* dI, int n, int64_t NTs) {
    const wino_geometry& g = p->g;
    const int T = (int)g.t;
    const int64_t per_c = (int64_t)T * (P * P + 1) * sizeof(float);
    Launch L(p, st, K_INGRAD);
    if (per_c <= 96 * 1024) {
        // channels per block: as many whole (c, all tiles) planes as fit 256 threads in one pass
        // (c4: T = 49 -> 5 channels, 245 items; 6 would leave a second pass 15% full), within ~48 KB
        int cg = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)p->C, (48 * 1024) / per_c, 256 / T}));
        const size_t smem = (size_t)cg * per_c;
        const dim3 grid((p->C + cg - 1) / cg, n);
        // whole warps over the block's (channel, tile) items (c3: 196 tiles -> 224 threads)
        const int threads = (int)std::min<int64_t>(256, round_up((int64_t)cg * T, 32));
        bool aligned = false;
        if constexpr (M == 4 && P == 6)
            aligned = p->pad == 1 && p->H == 4 * (int)g.tiles_y && p->W == 4 * (int)g.tiles_x &&
                      (reinterpret_cast<uintptr_t>(dI) & 15) == 0;
        if (aligned) {
            if constexpr (M == 4 && P == 6) {
                set_smem_attr(wino::input_grad_kernel<M, P, CF, true>, (int)std::max<size_t>(smem, 48 * 1024));
                wino::input_grad_kernel<M, P, CF, true><<<grid, threads, smem, st>>>(
                    DV, dI, p->cf, p->C, p->H, p->W, p->pad, (int)g.tiles_y, (int)g.tiles_x, T, (int)NTs, cg,
                    0x8000000080000000ull);
            }
        } else {
            set_smem_attr(wino::input_grad_kernel<M, P, CF>, (int)std::max<size_t>(smem, 48 * 1024));
            wino::input_grad_kernel<M, P, CF><<<grid, threads, smem, st>>>(
                DV, dI, p->cf, p->C, p->H, p->W, p->pad, (int)g.tiles_y, (int)g.tiles_x, T, (int)NTs, cg,
                0x8000000080000000ull);
        }
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

// D[s] = W-operand[s] · B[s] on the tensor cores (forward: W_F·Ĩ_F; backward data: W_Fᵀ·dZ), B =
// [P2][Kd][NTs] activations (MN-major): the warp-specialised 3xTF32 tcgen05 kernel
// (wino_dense_tc.cuh; 2 split warps, 8 drain warps with a compensated fp32 fold, TMA-stored output).
int launch_tc_gemm(wino_plan* p, cudaStream_t st, int kind, const CUtensorMap& ah, const CUtensorMap& al,
                   const float* B, float* D, int M, int Kd, int64_t NTs) {
    namespace tc = wino::tc;
    CUtensorMap mb, md;
    const int N = (int)NTs;
    if (!wino::make_map_3d(&mb, B, NTs, Kd, p->P2, (uint64_t)NTs * 4, (uint64_t)Kd * NTs * 4, 32, 32, true) ||
        !wino::make_map_3d_sw(&md, D, (uint64_t)N, (uint64_t)M, (uint64_t)p->P2, (uint64_t)NTs * 4,
                              (uint64_t)M * NTs * 4, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B))
        return set_err(WINO_CUDA_ERROR, "cuTensorMapEncodeTiled failed for the activation operand (CUresult " +
                                            std::to_string(wino::last_tmap_error()) + ")");
    const int kb = (Kd + tc::BK - 1) / tc::BK;
    const int tiles_n = (N + tc::flush::BN - 1) / tc::flush::BN, tiles_m = (M + tc::BM - 1) / tc::BM;
    const int ntiles = tiles_n * tiles_m * p->P2;
    auto kern = tc::gemm_3xtf32_ws_kernel<false, true, 2, 8, true, 4>;
    set_smem_attr(kern, tc::flush::WS_SMEM_BYTES);
    Launch L(p, st, kind);
    kern<<<std::min(ntiles, p->sm_count), 64 + 32 * (2 + 8), tc::flush::WS_SMEM_BYTES, st>>>(
        ah, al, mb, md, D, M, N, Kd, NTs, p->P2, 1, kb, tiles_n, tiles_m, ntiles);
    return L.done();
}

// ---- exact dW_F (wino_xdw.cuh): segments, digits, the int8 GEMM, the masked reduce ----

// images per exponent segment: one segment's columns fit one exact accumulation chunk
int seg_images(const wino_plan* p) {
    return (int)std::max<int64_t>(1, wino::xdw::kMaxChunkCols / std::max<int64_t>(1, p->g.t));
}

// digit buffers for `cols` columns and `nseg` segments (contents are lost when they grow)
int ensure_digits(wino_plan* p, wino_cache* c, int64_t cols, int nseg) {
    namespace x = wino::xdw;
    cols = round_up(std::max<int64_t>(cols, x::KS), x::KS);
    if (c->NTd < cols) {
        if (c->dig_v) cudaFree(c->dig_v);
        if (c->dig_z) cudaFree(c->dig_z);
        c->dig_v = c->dig_z = nullptr;
        c->NTd = 0;
        CUDA_TRY(cudaMalloc(&c->dig_v, (size_t)x::DIG * p->P2 * p->C * cols));
        CUDA_TRY(cudaMalloc(&c->dig_z, (size_t)x::DIG * p->P2 * p->K * cols));
        c->NTd = cols;
    }
    if (c->seg_cap < nseg) {
        for (void* q : {(void*)c->amax_v, (void*)c->amax_z, (void*)c->e_v, (void*)c->e_z})
            if (q) cudaFree(q);
        c->amax_v = c->amax_z = nullptr;
        c->e_v = c->e_z = nullptr;
        c->seg_cap = 0;
        CUDA_TRY(cudaMalloc(&c->amax_v, (size_t)nseg * p->C * sizeof(unsigned)));
        CUDA_TRY(cudaMalloc(&c->amax_z, (size_t)nseg * p->K * sizeof(unsigned)));
        CUDA_TRY(cudaMalloc(&c->e_v, (size_t)nseg * p->P2 * p->C * sizeof(int)));
        CUDA_TRY(cudaMalloc(&c->e_z, (size_t)nseg * p->P2 * p->K * sizeof(int)));
        c->seg_cap = nseg;
    }
    return WINO_OK;
}

// Append the segments of images [n0, n1) (after the ones already planned, which must end at n0).
// full: the whole batch in one call (exact column capacity); otherwise a range of a pipelined
// batch (capacity for the worst case, so later ranges never reallocate).
int plan_segments(wino_plan* p, wino_cache* c, int n0, int n1, bool full) {
    namespace x = wino::xdw;
    if (n0 == 0) {
        c->segs.clear();
        c->z_segs = 0;
    }
    if ((c->segs.empty() ? 0 : c->segs.back().n1) != n0)
        return set_err(WINO_CONSISTENCY_ERROR, "image ranges of a batch must be issued in order from image 0");
    const int per = seg_images(p);
    const int64_t T = p->g.t;
    int64_t col = c->segs.empty() ? 0 : c->segs.back().col0 + c->segs.back().ncols_pad;
    for (int a = n0; a < n1; a += per) {
        const int b = std::min(n1, a + per);
        const int64_t pad = round_up((int64_t)(b - a) * T, x::KS);
        c->segs.push_back(DwSeg{a, b, col, pad});
        col += pad;
    }
    const int nseg = full ? (int)c->segs.size() : c->n_max;
    const int64_t cols = full ? col : (int64_t)c->n_max * round_up(T, x::KS);
    if (n0 == 0) return ensure_digits(p, c, cols, nseg);
    if (c->NTd < col || c->seg_cap < (int)c->segs.size())
        return set_err(WINO_CONSISTENCY_ERROR, "exact dW_F digit buffers too small for this range");
    return WINO_OK;
}

// segments [g0, g1) of the cache covering images [n0, n1) exactly
int find_segments(const wino_cache* c, int n0, int n1, int* g0, int* g1) {
    int a = -1, b = -1;
    for (int i = 0; i < (int)c->segs.size(); ++i) {
        if (c->segs[i].n0 == n0) a = i;
        if (c->segs[i].n1 == n1) b = i + 1;
    }
    if (a < 0 || b <= a)
        return set_err(WINO_CONSISTENCY_ERROR, "backward image range [" + std::to_string(n0) + ", " +
                                                   std::to_string(n1) + ") differs from the forward's ranges");
    *g0 = a;
    *g1 = b;
    return WINO_OK;
}

// max|x| per (segment, row) over images [0, n) of x = [n][R][HW] (segments of seg_images(p)
// images from amax[0]).  A ReLU-masked dO is passed unmasked: an upper bound is all the digit
// exponent needs, and it saves the pass over the ReLU output.
int launch_amax(wino_plan* p, cudaStream_t st, const float* x, unsigned* amax, int R, int64_t HW, int n) {
    const int64_t planes = (int64_t)n * R;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((planes + 7) / 8, (int64_t)p->sm_count * 16));
    Launch L(p, st, K_AMAX);
    wino::xdw::plane_amax_kernel<<<grid, 256, 0, st>>>(x, amax, R, (int)HW, seg_images(p), (int)planes);
    return L.done();
}

// gather prefetch distance of the fused K1 / K4 (blocks ahead in launch order, x fastest) as
// (rows ahead) << 16 | (column blocks ahead); 0 = off (distances that do not fit the fields)
static int pack_prefetch(int blocks, unsigned gx) {
    if (blocks <= 0 || gx == 0 || gx > 0xffffu || blocks / gx > 0x7fffu) return 0;
    return (int)((blocks / gx) << 16 | (blocks % gx));
}

// K1 fused with the Ĩ_F digits, segments [g0, g1) of the cache: `in` holds images from n_base on,
// V points at image n_base's first column (row stride NTs), `owned` = V columns this call writes
// (from image n_base on; beyond the last image: the batch's zero padding).
template <int M, int P, class CF>
int launch_input_fused(wino_plan* p, cudaStream_t st, const float* in, float* V, int64_t NTs, int64_t owned,
                       int n_base, wino_cache* c, int g0, int g1) {
    namespace x = wino::xdw;
    const int64_t T = p->g.t;
    constexpr int smem = x::digit_smem_bytes<P * P>();
    auto kern = x::input_transform_digits_kernel<M, P, CF>;
    set_smem_attr(kern, smem);
    static int per_sm = 0;  // resident blocks per SM: the L2 prefetch distance of the gather
    if (!per_sm && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, x::kTileItems, smem) != cudaSuccess)
        per_sm = 2;
    const int pf_blocks = per_sm * p->sm_count;
    const int64_t plane = (int64_t)p->P2 * p->C * c->NTd;
    for (int g = g0; g < g1; ++g) {
        const DwSeg& sg = c->segs[g];
        const int64_t ncols = (int64_t)(sg.n1 - sg.n0) * T, voff = (int64_t)(sg.n0 - n_base) * T;
        const int64_t vcols = g == g1 - 1 ? owned - voff : ncols;
        const int64_t cols = std::max(vcols, sg.ncols_pad);
        Launch L(p, st, K_INPUT);
        const unsigned gx = (unsigned)((cols + x::kTileItems - 1) / x::kTileItems);
        const int pf = pack_prefetch(pf_blocks, gx);
        kern<<<dim3(gx, (unsigned)p->C), x::kTileItems, smem, st>>>(
            in + (int64_t)(sg.n0 - n_base) * p->C * p->H * p->W, V + voff, c->dig_v,
            c->e_v + (int64_t)g * p->P2 * p->C, c->amax_v + (int64_t)g * p->C, p->cf, p->cfd, p->nrm_v, p->C, p->H,
            p->W, p->pad, (int)p->g.tiles_x, (int)T, (int)ncols, (int)vcols, (int)sg.ncols_pad, NTs, c->NTd, plane,
            (int)sg.col0, pf);
        int rc = L.done();
        if (rc) return rc;
    }
    return WINO_OK;
}

// K4 fused with the dZ digits, segments [g0, g1): dO (and relu) hold images from n_base on, DZ
// points at image n_base's first column, `owned` as launch_input_fused
template <int M, int P, class CF>
int launch_grad_fused(wino_plan* p, cudaStream_t st, const float* dO, const float* relu, bool mask, float* DZ,
                      int64_t NTs, int64_t owned, int n_base, wino_cache* c, int g0, int g1) {
    namespace x = wino::xdw;
    const int64_t T = p->g.t, HW = p->g.h_o * p->g.w_o;
    constexpr int smem = x::digit_smem_bytes<P * P>();
    const int64_t plane = (int64_t)p->P2 * p->K * c->NTd;
    for (int g = g0; g < g1; ++g) {
        const DwSeg& sg = c->segs[g];
        const int64_t ncols = (int64_t)(sg.n1 - sg.n0) * T, voff = (int64_t)(sg.n0 - n_base) * T;
        const int64_t vcols = g == g1 - 1 ? owned - voff : ncols;
        const int64_t cols = std::max(vcols, sg.ncols_pad);
        const int64_t off = (int64_t)(sg.n0 - n_base) * p->K * HW;
        const dim3 grid((unsigned)((cols + x::kTileItems - 1) / x::kTileItems), (unsigned)p->K);
        Launch L(p, st, K_GRADZ);
        auto go = [&](auto kern) {
            set_smem_attr(kern, smem);
            int per_sm = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, x::kTileItems, smem) != cudaSuccess)
                per_sm = 3;
            kern<<<grid, x::kTileItems, smem, st>>>(
                dO + off, relu ? relu + off : nullptr, DZ + voff, c->dig_z, c->e_z + (int64_t)g * p->P2 * p->K,
                c->amax_z + (int64_t)g * p->K, p->cf, p->cfd, p->nrm_z, p->K, (int)p->g.h_o, (int)p->g.w_o,
                (int)p->g.tiles_x, (int)T, (int)ncols, (int)vcols, (int)sg.ncols_pad, NTs, c->NTd, plane,
                (int)sg.col0, pack_prefetch(per_sm * p->sm_count, grid.x));
        };
        if (mask) go(x::grad_z_digits_kernel<M, P, true, CF>);
        else go(x::grad_z_digits_kernel<M, P, false, CF>);
        int rc = L.done();
        if (rc) return rc;
    }
    return WINO_OK;
}

int dw_exchange(wino_plan* p, float* grad_w, cudaStream_t st);

// dW_F from the digits of every segment: the int8 GEMM per accumulation chunk, then the ordered
// chunk sum gathered on the mask (CSR order) or into K×C×p×q (dense plan).
int launch_xdw(wino_plan* p, cudaStream_t st, const wino_cache* c, float* grad_w) {
    namespace x = wino::xdw;
    x::ChunkTab ct{};
    constexpr int64_t maxc = x::kMaxChunkCols / x::KS * x::KS;
    for (int g = 0; g < (int)c->segs.size(); ++g)
        for (int64_t a = 0; a < c->segs[g].ncols_pad; a += maxc) {
            if (ct.n == x::kMaxChunks)
                return set_err(WINO_CAPABILITY_ERROR, "exact dW_F: more than " + std::to_string(x::kMaxChunks) +
                                                          " accumulation chunks (too many image ranges)");
            ct.col0[ct.n] = (int)(c->segs[g].col0 + a);
            ct.ncols[ct.n] = (int)std::min(maxc, c->segs[g].ncols_pad - a);
            ct.seg[ct.n] = g;
            ++ct.n;
        }
    if (p->nnz == 0 || ct.n == 0) return WINO_OK;
    const int K = p->K, C = p->C, P2 = p->P2;
    const size_t need = (size_t)ct.n * P2 * K * C;
    if (p->xpart_cap < need) {
        if (p->d_xpart) cudaFree(p->d_xpart);
        p->d_xpart = nullptr;
        p->xpart_cap = 0;
        CUDA_TRY(cudaMalloc(&p->d_xpart, need * sizeof(double)));
        p->xpart_cap = need;
    }
    CUtensorMap ma, mb;
    if (!wino::make_map_4d_u8(&ma, c->dig_z, c->NTd, K, P2, x::DIG, x::KS, x::BM, CU_TENSOR_MAP_SWIZZLE_64B) ||
        !wino::make_map_4d_u8(&mb, c->dig_v, c->NTd, C, P2, x::DIG, x::KS, x::BN, CU_TENSOR_MAP_SWIZZLE_64B))
        return set_err(WINO_CUDA_ERROR, "cuTensorMapEncodeTiled failed for the dW_F digit tensors (CUresult " +
                                            std::to_string(wino::last_tmap_error()) + ")");
    const int tiles_m = (K + x::BM - 1) / x::BM, tiles_n = (C + x::BN - 1) / x::BN;
    const int units = ct.n * P2 * tiles_m * tiles_n;
    set_smem_attr(x::gemm_kernel, x::SMEM_BYTES);
    {
        Launch L(p, st, K_DW_GEMM);
        x::gemm_kernel<<<std::min(units, p->sm_count), x::THREADS, x::SMEM_BYTES, st>>>(
            ma, mb, ct, c->e_z, c->e_v, p->d_xpart, P2, K, C, tiles_m, tiles_n, units);
        int rc = L.done();
        if (rc) return rc;
    }
    Launch L(p, st, K_DW_REDUCE);
    if (p->dense)
        x::reduce_dense_kernel<<<grid_for((int64_t)P2 * K * C, 256, p->sm_count), 256, 0, st>>>(p->d_xpart, grad_w, K,
                                                                                              C, P2, ct.n);
    else {
        const int per_slice = (int)std::max<int64_t>(1, std::min<int64_t>(64, p->nnz / P2 / 1024 + 1));
        x::reduce_sparse_kernel<<<dim3(per_slice, (unsigned)P2), 256, 0, st>>>(
            p->d_xpart, grad_w, p->d_rowof, p->d_colidx, p->d_slice_off, K, C, P2, ct.n, p->nnz);
    }
    const int rc = L.done();
    return rc ? rc : dw_exchange(p, grad_w, st);
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
    // one zero pad entry: the shared-memory SpMM stages whole 16-byte (col, value) pairs
    cv.push_back(make_int2(0, 0));
    cvT.push_back(make_int2(0, 0));
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
    int rc2 = build_tm_streams(p);
    if (rc2) return rc2;
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
        const bool hyb_shape = p->C > 128 && p->C <= 256 && p->K > 128 && p->K <= 256;
        const int thr = p->auto_permille >= 0 ? p->auto_permille : (hyb_shape ? 110 : 80);
        eff = (density * 1000.0 >= thr && p->C % 4 == 0 && p->K % 4 == 0) ? 1 : 0;
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
        (rc = grow(&p->d_rowof, &p->cap_rowof, (size_t)nnz)) || (rc = grow(&p->d_cv, &p->cap_cv, (size_t)nnz + 1)) ||
        (rc = grow(&p->d_rowidx, &p->cap_rowidx, (size_t)nnz)) || (rc = grow(&p->d_perm, &p->cap_perm, (size_t)nnz)) ||
        (rc = grow(&p->d_cvT, &p->cap_cvT, (size_t)nnz + 1)))
        return rc;
    // one zero pad entry after the (col, value) streams: the shared-memory SpMM stages whole pairs
    CUDA_TRY(cudaMemset(p->d_cv + nnz, 0, sizeof(int2)));
    CUDA_TRY(cudaMemset(p->d_cvT + nnz, 0, sizeof(int2)));
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
    if ((rc = build_tm_streams(p))) return rc;
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
    // the f64 digit kernels take the built-in doubles too: the doubles must match as well
    auto same_d = [&](auto tag) {
        using B = decltype(tag);
        for (int i = 0; i < p->p * p->m; ++i)
            if (p->cfd.a[i] != B::AD(i)) return false;
        for (int i = 0; i < p->p * p->p; ++i)
            if (p->cfd.b[i] != B::BD(i)) return false;
        return true;
    };
    // WINO_RUNTIME_COEFS (debug): run the runtime-coefficient kernel variants
    if (!std::getenv("WINO_RUNTIME_COEFS")) {
        if (p->m == 4)
            p->builtin = same(wino::BuiltinCoefs<4, 6>::a, wino::BuiltinCoefs<4, 6>::b) &&
                         same_d(wino::BuiltinCoefs<4, 6>{});
        if (p->m == 2)
            p->builtin = same(wino::BuiltinCoefs<2, 4>::a, wino::BuiltinCoefs<2, 4>::b) &&
                         same_d(wino::BuiltinCoefs<2, 4>{});
        if (p->m == 6)
            p->builtin = same(wino::BuiltinCoefs<6, 8>::a, wino::BuiltinCoefs<6, 8>::b) &&
                         same_d(wino::BuiltinCoefs<6, 8>{});
    }
    // exponent bounds of the exact dW_F digits: |Ĩ_F(i,j)| <= ‖B col i‖₁‖B col j‖₁·max|d|,
    // |dZ(i,j)| <= ‖A row i‖₁‖A row j‖₁·max|dÕ| (the kernels' own sums, wino_xdw.cuh)
    {
        double nb[8] = {}, na[8] = {};
        for (int i = 0; i < p->p; ++i) {
            for (int k = 0; k < p->p; ++k) nb[i] += std::fabs(p->cfd.b[k * p->p + i]);
            for (int y = 0; y < p->m; ++y) na[i] += std::fabs(p->cfd.a[i * p->m + y]);
        }
        for (int i = 0; i < p->p; ++i)
            for (int j = 0; j < p->p; ++j) {
                p->nrm_v.v[i * p->p + j] = nb[i] * nb[j];
                p->nrm_z.v[i * p->p + j] = na[i] * na[j];
            }
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
    if (p->d_xpart) chk(cudaFree(p->d_xpart), "d_xpart");
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
    if (p->d_slice_off) chk(cudaFree(p->d_slice_off), "d_slice_off");
    for (auto& ts : p->tms)
        for (void* q : {(void*)ts.cv, (void*)ts.pidx, (void*)ts.bnd, (void*)ts.cnt})
            if (q) chk(cudaFree(q), "tmem spmm stream");
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
    if (dense < 0 || dense > 2) return set_err(WINO_INVALID_ARGUMENT, "dense must be 0, 1 or 2");
    CUDA_TRY(cudaSetDevice(p->device));
    // dense != 0: every coordinate is a weight (zeros included): the full CSR
    int rc = device_compress(p, w_f, zero_tol, dense ? 1 : 0);
    if (rc != WINO_OK || !dense) return rc;
    p->dense = true;
    if (dense == 2) {
        rc = refresh_tc_operands(p, nullptr);
        if (rc == WINO_OK) CUDA_TRY(cudaDeviceSynchronize());
    }
    return rc;
}

int wino_get_csr(const wino_plan* p, uint64_t* nnz, uint64_t* row_ptr, uint64_t* col_idx, float* values) {
    if (!p || !nnz) return set_err(WINO_INVALID_ARGUMENT, "null argument");
    if (!p->has_weights) return set_err(WINO_CONSISTENCY_ERROR, "plan holds no CSR weights");
    CUDA_TRY(cudaSetDevice(p->device));
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
    CUDA_TRY(cudaSetDevice(p->device));
    cudaStream_t st = (cudaStream_t)stream;
    Launch L(p, st, K_MISC);
    wino::refresh_values_kernel<<<grid_for(p->nnz, 256, p->sm_count), 256, 0, st>>>(p->d_cv, p->d_cvT, p->d_vals,
                                                                                   p->d_perm, p->nnz);
    rc = L.done();
    for (int dir = 0; dir < 2 && rc == WINO_OK; ++dir) {
        auto& ts = p->tms[dir];
        if (!ts.ready) continue;
        Launch L2(p, st, K_MISC);
        wino::tm::tm_refresh_kernel<<<grid_for(ts.n, 256, p->sm_count), 256, 0, st>>>(ts.cv, ts.pidx,
                                                                                      dir ? p->d_cvT : p->d_cv, ts.n);
        rc = L2.done();
    }
    if (rc == WINO_OK && p->tc_ready) rc = refresh_tc_operands(p, st);
    return rc;
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
        wino_cache_destroy(c);
        return set_err(WINO_CUDA_ERROR, std::string("cache_create: ") + cudaGetErrorString(e));
    }
    *out = c;
    return WINO_OK;
}

int wino_cache_destroy(wino_cache* c) {
    if (!c) return WINO_OK;
    for (void* q : {(void*)c->V, (void*)c->DZ, (void*)c->dig_v, (void*)c->dig_z, (void*)c->amax_v,
                    (void*)c->amax_z, (void*)c->e_v, (void*)c->e_z})
        if (q) cudaFree(q);
    delete c;
    return WINO_OK;
}

// the dW_F stream (greatest priority: the longest chain of a step) and the dI stream, on the
// plan's device
static int ensure_streams(wino_plan* p) {
    if (!p->side) {
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
    return WINO_OK;
}

// After a fork, every exit (errors included) joins the side streams back into the caller's
// stream, so a CUDA-graph capture stays joined and eager callers stay ordered after the side work.
struct JoinGuard {
    wino_plan* p;
    cudaStream_t st;
    bool side, side2;
    ~JoinGuard() {
        if (side) {
            cudaEventRecord(p->ev_join, p->side);
            cudaStreamWaitEvent(st, p->ev_join, 0);
        }
        if (side2) {
            cudaEventRecord(p->ev_join2, p->side2);
            cudaStreamWaitEvent(st, p->ev_join2, 0);
        }
    }
};

static int zero_rows(unsigned* a, int g0, int g1, int rows, cudaStream_t st) {
    CUDA_TRY(cudaMemsetAsync(a + (int64_t)g0 * rows, 0, (size_t)(g1 - g0) * rows * sizeof(unsigned), st));
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
    CUDA_TRY(cudaSetDevice(p->device));
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
    if (cache) {  // training: K1 fused with the exact dW_F digits of Ĩ_F
        cache->has_fwd = false;
        if ((rc = plan_segments(p, cache, 0, n, true))) return rc;
        const int nseg = (int)cache->segs.size();
        if ((rc = zero_rows(cache->amax_v, 0, nseg, p->C, st)) ||
            (rc = launch_amax(p, st, input, cache->amax_v, p->C, (int64_t)p->H * p->W, n)) ||
            (rc = DISPATCH_MP(p, launch_input_fused, p, st, input, V, NTs, NTs, 0, cache, 0, nseg)))
            return rc;
    } else if ((rc = DISPATCH_MP(p, fwd_transforms, p, st, input, output, V, p->d_z, n, NT, NTs, flags, 0, NTs))) {
        return rc;
    }
    if (p->tc_ready && (p->dense || p->contraction == 1))
        rc = launch_tc_gemm(p, st, K_DENSE_FWD, p->map_wh, p->map_wl, V, p->d_z, p->K, p->C, NTs);
    else
        rc = launch_spmm(p, st, K_SPMM, p->d_rowptr, p->d_cv, p->h_rowptr, V, p->d_z, p->K, p->C, NT, NTs);
    if (rc) return rc;
    if ((rc = DISPATCH_MP(p, fwd_transforms, p, st, input, output, V, p->d_z, n, NT, NTs, flags, 1, NTs)))
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
    CUDA_TRY(cudaSetDevice(p->device));
    return WINO_OK;
}

// K4: dZ = A1·dÕ·A2ᵀ into the cache fused with its exact dW_F digits (after the max|dO| pre-pass)
static int bwd_grad_z(wino_plan* p, const float* grad_output, const float* relu_out, wino_cache* c, int flags,
                      cudaStream_t st, bool zero = true) {
    const bool mask = (flags & WINO_BWD_RELU_MASK) != 0;
    const int nseg = (int)c->segs.size();
    c->z_segs = 0;
    int rc;
    if ((zero && (rc = zero_rows(c->amax_z, 0, nseg, p->K, st))) ||
        (rc = launch_amax(p, st, grad_output, c->amax_z, p->K, p->g.h_o * p->g.w_o, c->n)) ||
        (rc = DISPATCH_MP(p, launch_grad_fused, p, st, grad_output, relu_out, mask, c->DZ, c->NTs, c->NTs, 0, c, 0,
                          nseg)))
        return rc;
    c->z_segs = nseg;
    return WINO_OK;
}

// dW_F from the digits of Ĩ_F and dZ (exact, wino_xdw.cuh)
static int bwd_dw(wino_plan* p, wino_cache* c, float* grad_w, cudaStream_t st) { return launch_xdw(p, st, c, grad_w); }

// dĨ_F = W_Fᵀ·dZ and dI = Σ_φ B1·dĨ_F·B2ᵀ
static int bwd_input(wino_plan* p, const wino_cache* c, float* grad_input, cudaStream_t st) {
    const int64_t NT = (int64_t)c->n * p->g.t, NTs = c->NTs;
    int rc = ensure(&p->d_dv, &p->dv_cap, (size_t)p->P2 * std::max(p->C, p->K) * NTs);
    if (rc) return rc;
    if (p->tc_ready && (p->dense || p->contraction == 1))
        rc = launch_tc_gemm(p, st, K_DENSE_DV, p->map_wth, p->map_wtl, c->DZ, p->d_dv, p->C, p->K, NTs);
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
    c->has_grad_z = true;
    return bwd_dw(p, c, grad_w, st);
}

int wino_backward(wino_plan* p, const float* grad_output, const float* relu_out, wino_cache* c, float* grad_w,
                  float* grad_input, int flags, void* stream) {
    int rc = bwd_check(p, grad_output, relu_out, c, grad_w, flags);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if ((rc = bwd_grad_z(p, grad_output, relu_out, c, flags, st))) return rc;
    c->has_grad_z = true;
    if (!grad_input)  // no dI wanted (the first layer of a stack, train.cpp:201): dW only
        return bwd_dw(p, c, grad_w, st);
    if ((rc = ensure_streams(p))) return rc;
    // dW (side stream) and dĨ_F -> dI (caller's stream) only share the read-only dZ / dO
    CUDA_TRY(cudaEventRecord(p->ev_fork, st));
    CUDA_TRY(cudaStreamWaitEvent(p->side, p->ev_fork, 0));
    JoinGuard join{p, st, true, false};
    if ((rc = bwd_dw(p, c, grad_w, p->side))) return rc;
    return bwd_input(p, c, grad_input, st);
}

// One training step of the layer (forward, then backward with both gradients) scheduled as the
// dependency graph it is instead of in API order: dZ = A1·dÕ·A2ᵀ needs only dO, so the
// dO -> dZ -> dĨ_F -> dI chain runs beside the forward from the start (side2), and the dW_F chain
// (digits of Ĩ_F and dZ, the int8 GEMM) waits for just K1 and K4 (side).
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
    CUDA_TRY(cudaSetDevice(p->device));
    cudaStream_t st = (cudaStream_t)stream;
    if ((rc = ensure_streams(p))) return rc;
    const int64_t NT = (int64_t)n * p->g.t;
    const int64_t NTs = round_up(NT, 4);
    if ((rc = ensure(&p->d_z, &p->z_cap, (size_t)p->P2 * p->K * NTs))) return rc;
    if ((rc = ensure(&p->d_dv, &p->dv_cap, (size_t)p->P2 * std::max(p->C, p->K) * NTs))) return rc;
    c->has_fwd = false;
    if ((rc = plan_segments(p, c, 0, n, true))) return rc;
    const int nseg = (int)c->segs.size();
    if ((rc = zero_rows(c->amax_v, 0, nseg, p->C, st)) || (rc = zero_rows(c->amax_z, 0, nseg, p->K, st))) return rc;
    c->n = n;
    c->NTs = NTs;
    c->has_fwd = true;
    c->has_grad_z = false;
    // fork both side streams off the caller's stream
    CUDA_TRY(cudaEventRecord(p->ev_fork, st));
    CUDA_TRY(cudaStreamWaitEvent(p->side2, p->ev_fork, 0));
    CUDA_TRY(cudaStreamWaitEvent(p->side, p->ev_fork, 0));
    JoinGuard join{p, st, true, true};
    // side2: dZ and its digits, then dĨ_F = W_Fᵀ·dZ and dI
    if ((rc = bwd_grad_z(p, grad_output, nullptr, c, 0, p->side2, false))) return rc;
    CUDA_TRY(cudaEventRecord(p->ev_dz, p->side2));
    if ((rc = bwd_input(p, c, grad_input, p->side2))) return rc;
    // caller's stream: Ĩ_F and its digits, then Z = W_F·Ĩ_F and O
    if ((rc = launch_amax(p, st, input, c->amax_v, p->C, (int64_t)p->H * p->W, n)) ||
        (rc = DISPATCH_MP(p, launch_input_fused, p, st, input, c->V, NTs, NTs, 0, c, 0, nseg)))
        return rc;
    CUDA_TRY(cudaEventRecord(p->ev_v, st));
    // side: the dW_F GEMM once both digit sets exist
    CUDA_TRY(cudaStreamWaitEvent(p->side, p->ev_v, 0));
    CUDA_TRY(cudaStreamWaitEvent(p->side, p->ev_dz, 0));
    if ((rc = bwd_dw(p, c, grad_w, p->side))) return rc;
    if (p->tc_ready && (p->dense || p->contraction == 1))
        rc = launch_tc_gemm(p, st, K_DENSE_FWD, p->map_wh, p->map_wl, c->V, p->d_z, p->K, p->C, NTs);
    else
        rc = launch_spmm(p, st, K_SPMM, p->d_rowptr, p->d_cv, p->h_rowptr, c->V, p->d_z, p->K, p->C, NT, NTs);
    if (rc) return rc;
    if ((rc = DISPATCH_MP(p, fwd_transforms, p, st, input, output, c->V, p->d_z, n, NT, NTs, 0, 1, NTs)))
        return rc;
    c->has_grad_z = true;
    return WINO_OK;  // the guard joins side and side2 into st
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
    if (p->tc_ready)
        return set_err(WINO_CAPABILITY_ERROR, "image-range calls run the CSR kernels only "
                                              "(no tensor-core plan/contraction)");
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
    CUDA_TRY(cudaSetDevice(p->device));
    cudaStream_t st = (cudaStream_t)stream;
    if ((rc = ensure(&p->d_z, &p->z_cap, (size_t)p->P2 * p->K * r.NTs))) return rc;
    if (n0 == 0) cache->has_fwd = false;
    const int g0 = n0 == 0 ? 0 : (int)cache->segs.size();
    if ((rc = plan_segments(p, cache, n0, n1, false))) return rc;
    const int g1 = (int)cache->segs.size();
    if ((rc = zero_rows(cache->amax_v, g0, g1, p->C, st))) return rc;
    float* V = cache->V + r.a;
    float* Z = p->d_z + r.a;
    if ((rc = launch_amax(p, st, input, cache->amax_v + (int64_t)g0 * p->C, p->C,
                          (int64_t)p->H * p->W, n1 - n0)) ||
        (rc = DISPATCH_MP(p, launch_input_fused, p, st, input, V, r.NTs, r.NTr, n0, cache, g0, g1)))
        return rc;
    if ((rc = launch_spmm(p, st, K_SPMM, p->d_rowptr, p->d_cv, p->h_rowptr, V, Z, p->K, p->C, r.NT, r.NTs, r.NTr)))
        return rc;
    if ((rc = DISPATCH_MP(p, fwd_transforms, p, st, input, output, V, Z, n1 - n0, r.NT, r.NTs, flags, 1, r.NTr)))
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
    int g0 = 0, g1 = 0;
    if ((rc = find_segments(c, n0, n1, &g0, &g1))) return rc;
    CUDA_TRY(cudaSetDevice(p->device));
    cudaStream_t st = (cudaStream_t)stream;
    if ((rc = ensure(&p->d_dv, &p->dv_cap, (size_t)p->P2 * std::max(p->C, p->K) * r.NTs))) return rc;
    float* DZ = c->DZ + r.a;
    float* DV = p->d_dv + r.a;
    if (n0 == 0) c->z_segs = 0;
    if (g0 != c->z_segs)
        return set_err(WINO_CONSISTENCY_ERROR, "backward image ranges of a batch must be issued in order from image 0");
    if ((rc = zero_rows(c->amax_z, g0, g1, p->K, st)) ||
        (rc = launch_amax(p, st, grad_output, c->amax_z + (int64_t)g0 * p->K, p->K,
                          p->g.h_o * p->g.w_o, n1 - n0)) ||
        (rc = DISPATCH_MP(p, launch_grad_fused, p, st, grad_output, relu_out, mask, DZ, r.NTs, r.NTr, n0, c, g0, g1)))
        return rc;
    if ((rc = launch_spmm(p, st, K_SPMM_T, p->d_colptr, p->d_cvT, p->h_colptr, DZ, DV, p->C, p->K, r.NT, r.NTs,
                          r.NTr)))
        return rc;
    if ((rc = DISPATCH_MP(p, launch_input_grad, p, st, DV, grad_input, n1 - n0, r.NTs))) return rc;
    c->z_segs = g1;
    c->has_grad_z = c->z_segs == (int)c->segs.size();
    return WINO_OK;
}

int wino_backward_weights_cached(wino_plan* p, wino_cache* c, float* grad_w, void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    if (!c || (!grad_w && p->nnz > 0)) return set_err(WINO_INVALID_ARGUMENT, "null argument");
    if (c->plan != p || !c->has_fwd || !c->has_grad_z || c->segs.empty() || c->segs.back().n1 != c->n ||
        c->z_segs != (int)c->segs.size())
        return set_err(WINO_CONSISTENCY_ERROR, "backward_weights_cached: dL/dZ missing; run backward_range first");
    CUDA_TRY(cudaSetDevice(p->device));
    return launch_xdw(p, (cudaStream_t)stream, c, grad_w);
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

}  // extern "C"

namespace {
// the in-backward exchange (wino_set_dw_allreduce): sum grad_w over the plan's communicator
int dw_exchange(wino_plan* p, float* grad_w, cudaStream_t st) {
    if (!p->dw_comm || !grad_w) return WINO_OK;
    const int64_t count = p->dense ? (int64_t)p->P2 * p->K * p->C : p->nnz;
    if (count == 0) return WINO_OK;
    std::call_once(g_nccl_once, resolve_nccl);
    if (!g_nccl_allreduce) return set_err(WINO_CAPABILITY_ERROR, "dW_F exchange: libnccl.so.2 not found");
    ++p->launches;
    const int r = g_nccl_allreduce(grad_w, grad_w, (size_t)count, /*ncclFloat32*/ 7, /*ncclSum*/ 0, p->dw_comm, st);
    if (r != 0)
        return set_err(WINO_CUDA_ERROR, std::string("ncclAllReduce: ") + (g_nccl_errstr ? g_nccl_errstr(r) : "error"));
    return WINO_OK;
}
}  // namespace

extern "C" {

int wino_set_dw_allreduce(wino_plan* p, void* nccl_comm) {
    if (!p) return set_err(WINO_INVALID_ARGUMENT, "null plan");
    p->dw_comm = nccl_comm;
    return WINO_OK;
}

int wino_allreduce_dw(wino_plan* p, void* nccl_comm, float* grad_w, int64_t count, void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    if (!nccl_comm || (!grad_w && count != 0)) return set_err(WINO_INVALID_ARGUMENT, "null argument");
    if (count < 0) count = p->dense ? (int64_t)p->P2 * p->K * p->C : p->nnz;
    if (count == 0) return WINO_OK;
    CUDA_TRY(cudaSetDevice(p->device));
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
    CUDA_TRY(cudaSetDevice(p->device));
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
    CUDA_TRY(cudaSetDevice(p->device));
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
    CUDA_TRY(cudaSetDevice(p->device));
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
    CUDA_TRY(cudaSetDevice(p->device));
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
    if (option == WINO_OPT_SPMM_OPERANDS) {
        if (value < 0 || value > 3)
            return set_err(WINO_INVALID_ARGUMENT, "spmm operands: 0 auto, 1 shared memory, 2 tensor memory, 3 hybrid");
        p->spmm_operands = value;
        return p->has_weights && !p->dense ? build_tm_streams(p) : WINO_OK;
    }
    if (option == WINO_OPT_DW_MODE) {  // one dW_F path: the exact int8 digit GEMM (wino_xdw.cuh)
        if (value != 0) return set_err(WINO_INVALID_ARGUMENT, "dW mode: only 0 (exact) exists");
        return WINO_OK;
    }
    return set_err(WINO_INVALID_ARGUMENT, "unknown option / value");
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
