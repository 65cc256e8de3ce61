// Test entry points of the shim library (extern "C", pointer marshalling only): they call the
// reference's own C++ API — winograd_forward/_backward_*, sparse_forward<float>, compress, and the
// reference trainer's train_step — which this library resolves to the B200 shim
// (layer_cuda.cpp).  tests/test_gpu_shim.py compares them with oracle/_ref (the reference on the
// CPU) on the same inputs.
#include <atomic>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "wino/layer.hpp"
#include "wino/sparse.hpp"
#include "wino/train.hpp"

using namespace wino;

namespace {
std::string g_err;
int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}
#define SHIM_GUARD(...)                                                  \
    try {                                                                \
        __VA_ARGS__                                                      \
        return 0;                                                        \
    } catch (const ShapeError& e) {                                      \
        return fail(e, 1);                                               \
    } catch (const ConsistencyError& e) {                                \
        return fail(e, 2);                                               \
    } catch (const CorruptFormatError& e) {                              \
        return fail(e, 3);                                               \
    } catch (const CapabilityError& e) {                                 \
        return fail(e, 4);                                               \
    } catch (const std::exception& e) {                                  \
        return fail(e, 9);                                               \
    }

Tensor wrap(std::vector<std::size_t> shape, const double* p) {
    std::size_t n = 1;
    for (auto e : shape) n *= e;
    return Tensor(std::move(shape), std::vector<double>(p, p + n));
}
// the reference CLI's choice (tools/wino.cpp): the fixed F(2x2,3x3) set for m = 2, Cook–Toom otherwise
TransformSet transforms_for(std::size_t m) { return m == 2 ? f2x2_3x3_transforms() : cook_toom_transforms(m, 3); }
void copy_out(const Tensor& t, double* out) { std::memcpy(out, t.data().data(), t.size() * sizeof(double)); }
}  // namespace

namespace wino {
extern std::atomic<long long> shim_gpu_calls;
}

extern "C" {

const char* shim_last_error() { return g_err.c_str(); }
long long shim_gpu_call_count() { return wino::shim_gpu_calls.load(); }

// One image through the reference layer API: O, then (grad_o != NULL) dW_F and dI.
int shim_layer(int m, int c, int h_i, int w_i, int k, const double* img, const double* w_f, const double* grad_o,
               double* o, double* grad_wf, double* grad_in) {
    SHIM_GUARD({
        TransformSet t = transforms_for(m);
        TileGeometry g = make_geometry(c, h_i, w_i, t);
        Tensor im = wrap({(std::size_t)c, (std::size_t)h_i, (std::size_t)w_i}, img);
        Tensor wf = wrap({(std::size_t)k, (std::size_t)c, t.p, t.q}, w_f);
        ForwardCache cache;
        copy_out(winograd_forward(im, wf, t, g, &cache), o);
        if (grad_o) {
            Tensor go = wrap({(std::size_t)k, g.h_o, g.w_o}, grad_o);
            copy_out(winograd_backward_weights(go, cache, t, g), grad_wf);
            copy_out(winograd_backward_input(cache, wf, t, g), grad_in);
        }
    })
}

// backward_input before backward_weights must raise the reference's ConsistencyError.
int shim_backward_input_without_grad_z(int m, int c, int h_i, int w_i, int k, const double* img,
                                       const double* w_f) {
    SHIM_GUARD({
        TransformSet t = transforms_for(m);
        TileGeometry g = make_geometry(c, h_i, w_i, t);
        Tensor im = wrap({(std::size_t)c, (std::size_t)h_i, (std::size_t)w_i}, img);
        Tensor wf = wrap({(std::size_t)k, (std::size_t)c, t.p, t.q}, w_f);
        ForwardCache cache;
        winograd_forward(im, wf, t, g, &cache);
        winograd_backward_input(cache, wf, t, g);
    })
}

// compress<float> (the reference's) + sparse_forward<float> (the shim's) over a batch.
int shim_sparse_forward(int m, int n, int c, int h_i, int w_i, int k, const double* batch, const double* w_f,
                        double* out) {
    SHIM_GUARD({
        TransformSet t = transforms_for(m);
        TileGeometry g = make_geometry(c, h_i, w_i, t);
        Tensor b = wrap({(std::size_t)n, (std::size_t)c, (std::size_t)h_i, (std::size_t)w_i}, batch);
        Tensor wf = wrap({(std::size_t)k, (std::size_t)c, t.p, t.q}, w_f);
        copy_out(sparse_forward<float>(b, compress<float>(wf), t, g, 4), out);
    })
}


// The reference's own trainer: `steps` plain-mode SGD steps of make_toy_network (Winograd
// domain) on synth_dataset, minibatches in order; losses[i] = train_step's minibatch loss.
int shim_train_steps(unsigned long long seed, int steps, int batch, int mode, double* losses) {
    SHIM_GUARD({
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
