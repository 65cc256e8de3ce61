// TEST INFRASTRUCTURE ONLY — never linked into or called by the product path.
//
// extern "C" shim over the UNMODIFIED reference implementation in
// /root/reference/proj/src (compiled from its own sources by oracle/Makefile into
// oracle/_ref/libwino_ref.so).  The shim only marshals plain pointers into the
// reference's own C++ API; every number it returns is computed by reference code:
//
//   winograd_forward / _backward_weights / _backward_input   proj/src/layer.cpp:45,98,134
//   compress<T>, sparse_forward<T>, build_tiled_layout<T>    proj/src/sparse.cpp:10,190,81
//   cook_toom_transforms, f2x2_3x3_transforms, make_geometry proj/src/transforms.cpp:7,124,147
//   direct_conv, lift_spatial_weights                        proj/src/reference.cpp:7, layer.cpp:29
//
// The only logic of its own is `wref_layer_fwd_bwd_batch`, which runs the
// reference's single-image dense f64 API over a batch on a std::thread pool
// (per-sample concurrency is allowed by SPEC.md:316-317) — that is the CPU
// baseline of the fwd+bwd path (the reference trainer calls the same three
// functions per sample at train.cpp:169-202).
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include <random>

#include "wino/harness.hpp"
#include "wino/layer.hpp"
#include "wino/reference.hpp"
#include "wino/sparse.hpp"
#include "wino/tensor.hpp"
#include "wino/train.hpp"
#include "wino/transforms.hpp"

using namespace wino;

namespace {

thread_local std::string g_err;

// bindings.cpp:41-44: the fixed F(2x2,3x3) set for m=2,r=3, Cook-Toom otherwise.
TransformSet transforms_for(std::size_t m, std::size_t r) {
    if (m == 2 && r == 3) return f2x2_3x3_transforms();
    return cook_toom_transforms(m, r);
}

Tensor wrap(std::vector<std::size_t> shape, const double* p) {
    std::size_t n = 1;
    for (auto e : shape) n *= e;
    return Tensor(std::move(shape), std::vector<double>(p, p + n));
}

void copy_out(const Tensor& t, double* dst) {
    if (dst) std::memcpy(dst, t.data().data(), t.size() * sizeof(double));
}

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const ShapeError*>(&e)) return 1;
    if (dynamic_cast<const ConsistencyError*>(&e)) return 2;
    if (dynamic_cast<const CorruptFormatError*>(&e)) return 3;
    if (dynamic_cast<const CapabilityError*>(&e)) return 4;
    return 9;
}

#define GUARD(...)                            \
    try {                                     \
        __VA_ARGS__;                          \
        return 0;                             \
    } catch (const std::exception& e) {       \
        return fail(e);                       \
    }

}  // namespace

extern "C" {

const char* wref_last_error() { return g_err.c_str(); }

// a: p x m, b: p x p, g: p x r (row-major doubles, exactly the reference's Matrix entries)
int wref_transforms(int m, int r, double* a, double* b, double* g) {
    GUARD({
        TransformSet t = transforms_for(m, r);
        std::memcpy(a, t.a1.entries().data(), t.a1.entries().size() * sizeof(double));
        std::memcpy(b, t.b1.entries().data(), t.b1.entries().size() * sizeof(double));
        std::memcpy(g, t.g1.entries().data(), t.g1.entries().size() * sizeof(double));
    })
}

// out[0..13] = c,h_i,w_i,h_o,w_o,h_op,w_op,h_ip,w_ip,p,q,tiles_y,tiles_x,t
int wref_geometry(int c, int h_i, int w_i, int m, int r, long* out) {
    GUARD({
        TileGeometry g = make_geometry(c, h_i, w_i, m, m, r, r);
        const std::size_t v[] = {g.c,    g.h_i,  g.w_i,  g.h_o, g.w_o,     g.h_op,    g.w_op,
                                 g.h_ip, g.w_ip, g.p,    g.q,   g.tiles_y, g.tiles_x, g.t};
        for (int i = 0; i < 14; ++i) out[i] = static_cast<long>(v[i]);
    })
}

int wref_phi(int c, int h_i, int w_i, int m, int r, long t, long i, long j, long* yx) {
    GUARD({
        TileGeometry g = make_geometry(c, h_i, w_i, m, m, r, r);
        auto [y, x] = phi(g, t, i, j);
        yx[0] = static_cast<long>(y);
        yx[1] = static_cast<long>(x);
    })
}

int wref_psi(int c, int h_i, int w_i, int m, int r, long y, long x, long* tij) {
    GUARD({
        TileGeometry g = make_geometry(c, h_i, w_i, m, m, r, r);
        TileIndex ti = psi(g, y, x);
        tij[0] = static_cast<long>(ti.t);
        tij[1] = static_cast<long>(ti.i);
        tij[2] = static_cast<long>(ti.j);
    })
}

// Dense f64 layer, one image (layer.cpp:45-171). Any output pointer may be null.
// i_f/z/grad_z are C x T x p x q / K x T x p x q exactly as ForwardCache holds them.
int wref_layer(int m, int c, int h_i, int w_i, int k, const double* img, const double* w_f,
               const double* grad_o, double* out_o, double* out_i_f, double* out_z,
               double* out_grad_wf, double* out_grad_in, double* out_grad_z) {
    GUARD({
        TransformSet t = transforms_for(m, 3);
        TileGeometry g = make_geometry(c, h_i, w_i, t);
        Tensor im = wrap({(std::size_t)c, (std::size_t)h_i, (std::size_t)w_i}, img);
        Tensor wf = wrap({(std::size_t)k, (std::size_t)c, t.p, t.q}, w_f);
        ForwardCache cache;
        Tensor o = winograd_forward(im, wf, t, g, &cache);
        copy_out(o, out_o);
        copy_out(cache.i_f, out_i_f);
        copy_out(cache.z, out_z);
        if (grad_o) {
            Tensor go = wrap({(std::size_t)k, g.h_o, g.w_o}, grad_o);
            Tensor gw = winograd_backward_weights(go, cache, t, g);
            copy_out(gw, out_grad_wf);
            copy_out(*cache.grad_z, out_grad_z);
            Tensor gi = winograd_backward_input(cache, wf, t, g);
            copy_out(gi, out_grad_in);
        }
    })
}

// backward_input without a preceding backward_weights must raise ConsistencyError
// (layer.cpp:137-138); exposed so the host mirror's error contract can be pinned.
int wref_backward_input_without_grad_z(int m, int c, int h_i, int w_i, int k, const double* img,
                                       const double* w_f) {
    GUARD({
        TransformSet t = transforms_for(m, 3);
        TileGeometry g = make_geometry(c, h_i, w_i, t);
        Tensor im = wrap({(std::size_t)c, (std::size_t)h_i, (std::size_t)w_i}, img);
        Tensor wf = wrap({(std::size_t)k, (std::size_t)c, t.p, t.q}, w_f);
        ForwardCache cache;
        winograd_forward(im, wf, t, g, &cache);
        winograd_backward_input(cache, wf, t, g);
    })
}

// compress<float> (sparse.cpp:10-36): nnz per slice -> counts[p*q]; if the
// buffers are non-null they receive row_ptr (p*q*(K+1)), col_idx, values (total nnz)
int wref_compress_f32(int k, int c, int p, const double* w_f, double zero_tol, long* counts,
                      long* row_ptr, long* col_idx, float* values) {
    GUARD({
        Tensor wf = wrap({(std::size_t)k, (std::size_t)c, (std::size_t)p, (std::size_t)p}, w_f);
        PointwiseCsr<float> csr = compress<float>(wf, zero_tol);
        std::size_t off = 0;
        for (std::size_t s = 0; s < csr.slices.size(); ++s) {
            const auto& sl = csr.slices[s];
            counts[s] = static_cast<long>(sl.values.size());
            if (row_ptr)
                for (std::size_t r = 0; r <= (std::size_t)k; ++r)
                    row_ptr[s * (k + 1) + r] = static_cast<long>(sl.row_ptr[r]);
            if (col_idx)
                for (std::size_t e = 0; e < sl.values.size(); ++e) {
                    col_idx[off + e] = static_cast<long>(sl.col_idx[e]);
                    values[off + e] = sl.values[e];
                }
            off += sl.values.size();
        }
    })
}

// build_tiled_layout<float> (sparse.cpp:81-122) of one image: out is (p*q) x C x T floats
int wref_tiled_layout_f32(int m, int c, int h_i, int w_i, const double* img, float* out) {
    GUARD({
        TransformSet t = transforms_for(m, 3);
        TileGeometry g = make_geometry(c, h_i, w_i, t);
        Tensor im = wrap({(std::size_t)c, (std::size_t)h_i, (std::size_t)w_i}, img);
        auto lay = build_tiled_layout<float>(im, t, g);
        std::memcpy(out, lay.buffer.data(), lay.buffer.size() * sizeof(float));
    })
}

// sparse_forward<T> (sparse.cpp:190-253) over a batch: compress<T>(w_f) then the
// reference's own thread pool with `workers` workers. precision: 32 or 64.
int wref_sparse_forward(int m, int n, int c, int h_i, int w_i, int k, const double* batch,
                        const double* w_f, unsigned workers, int precision, double* out,
                        unsigned long long* mults) {
    GUARD({
        TransformSet t = transforms_for(m, 3);
        TileGeometry g = make_geometry(c, h_i, w_i, t);
        Tensor b = wrap({(std::size_t)n, (std::size_t)c, (std::size_t)h_i, (std::size_t)w_i}, batch);
        Tensor wf = wrap({(std::size_t)k, (std::size_t)c, t.p, t.q}, w_f);
        OpCounter ops;
        Tensor o;
        if (precision == 32) {
            auto csr = compress<float>(wf);
            o = sparse_forward<float>(b, csr, t, g, workers, &ops);
        } else {
            auto csr = compress<double>(wf);
            o = sparse_forward<double>(b, csr, t, g, workers, &ops);
        }
        copy_out(o, out);
        if (mults) *mults = ops.multiplications;
    })
}

// direct_conv (reference.cpp:7-34): img C x H x W, w K x C x r x s
int wref_direct_conv(int c, int h, int w, int k, int r, const double* img, const double* wt,
                     double* out) {
    GUARD({
        Tensor im = wrap({(std::size_t)c, (std::size_t)h, (std::size_t)w}, img);
        Tensor kw = wrap({(std::size_t)k, (std::size_t)c, (std::size_t)r, (std::size_t)r}, wt);
        copy_out(direct_conv(im, kw), out);
    })
}

// lift_spatial_weights (layer.cpp:29-43)
int wref_lift(int m, int k, int c, const double* w, double* out) {
    GUARD({
        TransformSet t = transforms_for(m, 3);
        Tensor kw = wrap({(std::size_t)k, (std::size_t)c, 3, 3}, w);
        copy_out(lift_spatial_weights(kw, t), out);
    })
}

// CPU baseline of the fwd+bwd path through the reference API: for each of the
// first `n` images of the batch, winograd_forward (with cache) ->
// winograd_backward_weights -> winograd_backward_input, images spread over
// `threads` std::threads.  grad_wf_sum receives sum_n dW_F (train.cpp:200 order
// is per-sample; the sum is accumulated per thread then merged in thread order).
// Per-image outputs are written when the pointers are non-null.
int wref_layer_fwd_bwd_batch(int m, int n, int c, int h_i, int w_i, int k, const double* batch,
                             const double* w_f, const double* grad_o, unsigned threads,
                             double* out_o, double* out_grad_in, double* grad_wf_sum) {
    GUARD({
        TransformSet t = transforms_for(m, 3);
        TileGeometry g = make_geometry(c, h_i, w_i, t);
        Tensor wf = wrap({(std::size_t)k, (std::size_t)c, t.p, t.q}, w_f);
        const std::size_t in_sz = (std::size_t)c * h_i * w_i;
        const std::size_t out_sz = (std::size_t)k * g.h_o * g.w_o;
        const std::size_t wf_sz = wf.size();
        if (threads == 0) threads = 1;
        threads = std::min<unsigned>(threads, (unsigned)std::max(1, n));
        std::vector<std::vector<double>> partial(threads, std::vector<double>(wf_sz, 0.0));
        std::atomic<int> next{0};
        std::vector<std::string> errs(threads);
        auto work = [&](unsigned w) {
            try {
                for (;;) {
                    const int i = next.fetch_add(1);
                    if (i >= n) break;
                    Tensor im = wrap({(std::size_t)c, (std::size_t)h_i, (std::size_t)w_i}, batch + i * in_sz);
                    Tensor go = wrap({(std::size_t)k, g.h_o, g.w_o}, grad_o + i * out_sz);
                    ForwardCache cache;
                    Tensor o = winograd_forward(im, wf, t, g, &cache);
                    Tensor gw = winograd_backward_weights(go, cache, t, g);
                    Tensor gi = winograd_backward_input(cache, wf, t, g);
                    if (out_o) std::memcpy(out_o + i * out_sz, o.data().data(), out_sz * sizeof(double));
                    if (out_grad_in) std::memcpy(out_grad_in + i * in_sz, gi.data().data(), in_sz * sizeof(double));
                    auto& acc = partial[w];
                    for (std::size_t e = 0; e < wf_sz; ++e) acc[e] += gw[e];
                }
            } catch (const std::exception& e) {
                errs[w] = e.what();
            }
        };
        std::vector<std::thread> pool;
        for (unsigned w = 0; w < threads; ++w) pool.emplace_back(work, w);
        for (auto& th : pool) th.join();
        for (auto& e : errs)
            if (!e.empty()) throw std::runtime_error(e);
        if (grad_wf_sum) {
            std::fill(grad_wf_sum, grad_wf_sum + wf_sz, 0.0);
            for (unsigned w = 0; w < threads; ++w)
                for (std::size_t e = 0; e < wf_sz; ++e) grad_wf_sum[e] += partial[w][e];
        }
    })
}

// WGT1 I/O (tensor.cpp:166-216): dtype 1 = f64, 2 = f32
int wref_write_wgt1(const char* path, const long* shape, int ndim, const double* data, int dtype) {
    GUARD({
        std::vector<std::size_t> sh(shape, shape + ndim);
        std::size_t n = 1;
        for (auto e : sh) n *= e;
        Tensor t(sh, std::vector<double>(data, data + n));
        write_wgt1(path, t, dtype == 2 ? Dtype::f32 : Dtype::f64);
    })
}

// The reference's seeded inputs of infer-bench (tools/wino.cpp:338-343): mt19937_64 seeded with
// train::stream_seed(seed, name), uniform_real_distribution<double>(-1, 1), n draws.
int wref_uniform_stream(unsigned long long seed, const char* name, long n, double* out) {
    GUARD({
        std::mt19937_64 rng(train::stream_seed(seed, name));
        std::uniform_real_distribution<double> dist(-1.0, 1.0);
        for (long i = 0; i < n; ++i) out[i] = dist(rng);
    })
}

// magnitude_threshold_to_density (train.cpp:419-429), in place on a flat f64 array
int wref_threshold_to_density(double* w, long n, double density) {
    GUARD({
        Tensor t({(std::size_t)n}, std::vector<double>(w, w + n));
        train::magnitude_threshold_to_density(t, density);
        std::memcpy(w, t.data().data(), n * sizeof(double));
    })
}

// harness::load_checkpoint then harness::save_checkpoint (harness.cpp:152-212): what the
// reference makes of a checkpoint directory, written back out in its own format.
int wref_checkpoint_roundtrip(const char* dir_in, const char* dir_out) {
    GUARD({ harness::save_checkpoint(dir_out, harness::load_checkpoint(dir_in)); })
}


// The reference's own trainer: `steps` plain-mode SGD steps of make_toy_network (Winograd
// domain) on synth_dataset, minibatches in order; losses[i] = train_step's minibatch loss.
int wref_train_steps(unsigned long long seed, int steps, int batch, int mode, double* losses) {
    GUARD({
        train::Network net = train::make_toy_network(seed, train::Domain::winograd);
        for (auto& conv : net.convs) conv.lambda = mode == 1 ? 1e-3 : 0.0;
        train::Dataset data = train::synth_dataset(seed, (std::size_t)(steps * batch));
        train::PruneConfig cfg;
        cfg.batch_size = (std::size_t)batch;
        const train::StepMode sm = mode == 1 ? train::StepMode::prune : train::StepMode::plain;
        for (int s = 0; s < steps; ++s) {
            std::vector<std::size_t> idx;
            for (int b = 0; b < batch; ++b) idx.push_back((std::size_t)(s * batch + b));
            losses[s] = train::train_step(net, data, idx, cfg, cfg.base_lr, sm);
        }
    })
}

}  // extern "C"
