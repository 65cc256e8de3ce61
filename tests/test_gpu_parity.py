"""GPU parity of the CUDA path (through the C-ABI) against the reference.

Three anchors, strongest first:
  * bitwise: the forward equals the reference's own f32 sparse_forward (golden vectors the
    reference produced) and the f32 operation-order mirror (oracle/wino_oracle.py); dĨ_F/dI
    equal the mirror bitwise too;
  * tolerance: O, dI and dW_F (on the mask) within |d| <= 1e-5 + 1e-4·|ref| of the reference's
    f64 dense layer, every element (BASELINE.json north_star);
  * properties at full BASELINE sizes: determinism, sampled-oracle agreement, CSR structure.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from helpers import LAYER_CASES, assert_parity, fail_fraction, golden_csr_slices, load_layer
from oracle import wino_oracle as wo
import paper_1702_08597_b200 as wb
from paper_1702_08597_b200.synth import CONFIGS, make_inputs, with_sparsity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    assert wb._lib.LIB_PATH.exists(), "libwino_b200.so not built"


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def run_layer(img, w_f, grad_o, m, pad, dense=None, dw_mode=None, contraction=None):
    n, c, h, w = img.shape
    k = w_f.shape[0]
    layer = wb.WinogradLayer(c, k, h, w, pad=pad, m=m)
    layer.set_weights(w_f, dense=dense)
    if dw_mode is not None:
        layer.set_dw_mode(dw_mode)
    if contraction is not None:
        layer.set_contraction(contraction)
    cache = layer.new_cache(n)
    o = layer.forward(dev(img), cache)
    out = {"layer": layer, "o": o.cpu().numpy()}
    if grad_o is not None:
        dw = layer.backward_weights(dev(grad_o), cache)
        di = layer.backward_input(cache)
        torch.cuda.synchronize()
        out["dw_raw"] = dw.cpu().numpy()
        out["di"] = di.cpu().numpy()
        out["dw"] = (out["dw_raw"].astype(np.float64) if layer.is_dense
                     else layer.compact_to_dense(out["dw_raw"].astype(np.float64)))
    return out


@pytest.mark.parametrize("name", LAYER_CASES)
def test_layer_vs_reference_golden(name):
    d = load_layer(name)
    r = run_layer(d["img"], d["w_f"], d["grad_o"], d["m"], d["pad"])
    if not r["layer"].is_dense:
        # CSR path: bit-identical to the reference's f32 sparse_forward
        assert np.array_equal(r["o"].astype(np.float64), d["o_sparse_f32"]), "forward not bitwise"
    assert_parity(r["o"], d["o_f64"], "O vs f64 reference")
    assert_parity(r["di"], d["grad_in_f64"], "dI vs f64 reference")
    if r["layer"].is_dense:
        assert_parity(r["dw"], d["grad_wf_f64"], "dW_F (dense) vs f64 reference")
    else:
        mask = d["w_f"] != 0
        assert_parity(r["dw"][mask], d["grad_wf_f64"][mask], "dW_F on the mask vs f64 reference")
        assert np.all(r["dw"][~mask] == 0)


@pytest.mark.parametrize("name", LAYER_CASES)
def test_layer_vs_f32_mirror_bitwise(name):
    d = load_layer(name)
    r = run_layer(d["img"], d["w_f"], d["grad_o"], d["m"], d["pad"], dense=False)
    mir = wo.layer_f32(d["img"], wo.compress(d["w_f"]), d["grad_o"], m=d["m"], pad=d["pad"])
    assert np.array_equal(r["o"], mir["o"])
    assert np.array_equal(r["di"], mir["di"]), "dI not bitwise equal to the mirror"
    dw_ref = np.concatenate(mir["dw"]) if mir["dw"] else np.zeros(0)
    np.testing.assert_allclose(r["dw_raw"], dw_ref, rtol=2e-6, atol=1e-6 * max(1.0, np.abs(dw_ref).max()))


@pytest.mark.parametrize("name", ["c0", "f63"])
def test_device_csr_matches_reference_compress(name):
    d = load_layer(name)
    layer = wb.WinogradLayer(d["c"], d["k"], d["h"], d["w"], pad=d["pad"], m=d["m"])
    layer.set_weights(d["w_f"], dense=False)
    csr = layer.get_csr()
    rps, cols, vals = golden_csr_slices(d)
    for s in range(len(rps)):
        assert np.array_equal(csr.row_ptr[s].astype(np.int64), rps[s])
        assert np.array_equal(csr.col_idx[s].astype(np.int64), cols[s])
        assert np.array_equal(csr.values[s], vals[s])
    assert layer.nnz == int(d["csr_nnz"].sum())


def test_set_weights_csr_equals_set_weights():
    d = load_layer("c0")
    a = run_layer(d["img"], d["w_f"], d["grad_o"], 4, 1, dense=False)
    layer = wb.WinogradLayer(d["c"], d["k"], d["h"], d["w"], pad=1, m=4)
    layer.set_weights_csr(wb.compress(d["w_f"]))
    cache = layer.new_cache(1)
    o = layer.forward(dev(d["img"]), cache).cpu().numpy()
    assert np.array_equal(o, a["o"])


def test_corrupt_csr_rejected():
    # test_sparse.cpp:155-168 — and the row_ptr length / monotonicity the reference never checks
    layer = wb.WinogradLayer(2, 2, 6, 6, pad=0, m=4)
    csr = wb.compress(np.ones((2, 2, 6, 6)))
    bad = wb.PointwiseCsr(csr.k, csr.c, csr.p, list(csr.row_ptr), list(csr.col_idx), list(csr.values))
    bad.col_idx[3] = bad.col_idx[3].copy()
    bad.col_idx[3][0] = 5  # out of bounds
    with pytest.raises(wb.CorruptFormatError):
        layer.set_weights_csr(bad)
    bad = wb.PointwiseCsr(csr.k, csr.c, csr.p, list(csr.row_ptr), list(csr.col_idx), list(csr.values))
    bad.row_ptr[0] = np.array([0, 3, 2], dtype=np.uint64)  # not monotone / wrong end
    with pytest.raises(wb.CorruptFormatError):
        layer.set_weights_csr(bad)
    bad = wb.PointwiseCsr(csr.k, csr.c, csr.p, list(csr.row_ptr), list(csr.col_idx), list(csr.values))
    bad.col_idx[0] = np.array([1, 0, 0, 1], dtype=np.uint64)  # not increasing within a row
    with pytest.raises(wb.CorruptFormatError):
        layer.set_weights_csr(bad)


def test_backward_input_requires_backward_weights():
    # test_layer.cpp:132-140 (ConsistencyError)
    d = load_layer("f43_tiny")
    layer = wb.WinogradLayer(d["c"], d["k"], d["h"], d["w"], pad=d["pad"], m=4)
    layer.set_weights(d["w_f"])
    cache = layer.new_cache(1)
    with pytest.raises(wb.ConsistencyError):
        layer.backward_input(cache)
    layer.forward(dev(d["img"]), cache)
    with pytest.raises(wb.ConsistencyError):
        layer.backward_input(cache)
    layer.backward_weights(dev(d["grad_o"]), cache)
    layer.backward_input(cache)
    layer.forward(dev(d["img"]), cache)  # a new forward clears dL/dZ (layer.cpp:88)
    with pytest.raises(wb.ConsistencyError):
        layer.backward_input(cache)


def test_shape_errors():
    layer = wb.WinogradLayer(3, 4, 8, 8, pad=1, m=4)
    with pytest.raises(wb.ConsistencyError):
        layer.forward(dev(np.zeros((1, 3, 8, 8))))  # no weights yet
    layer.set_weights(np.ones((4, 3, 6, 6)))
    with pytest.raises(wb.ShapeError):
        layer.forward(dev(np.zeros((1, 2, 8, 8))))
    with pytest.raises(wb.ShapeError):
        layer.set_weights(np.ones((4, 3, 4, 4)))
    cache = layer.new_cache(1)
    with pytest.raises(wb.ShapeError):
        layer.forward(dev(np.zeros((2, 3, 8, 8))), cache)  # batch exceeds the cache


@pytest.mark.parametrize("sparsity", [0.0, 0.5, 0.9, 1.0])
def test_densities_against_f64_oracle(sparsity):
    """acceptance.cpp:114-152 style sweep incl. the all-zero (density 0) and full-density CSR."""
    cfg = with_sparsity(CONFIGS["c0"], sparsity)
    img, w_f, go = make_inputs(cfg, n=2)
    r = run_layer(img, w_f, go, 4, 1, dense=False)
    imgp = np.pad(img.astype(np.float64), ((0, 0), (0, 0), (1, 1), (1, 1)))
    gw = np.zeros_like(w_f)
    for i in range(2):
        o, cache = wo.forward_f64(imgp[i], w_f, 4)
        assert_parity(r["o"][i], o, f"O[{i}]")
        gw += wo.backward_weights_f64(go[i].astype(np.float64), cache)
        assert_parity(r["di"][i], wo.backward_input_f64(cache, w_f)[:, 1:-1, 1:-1], f"dI[{i}]")
    mask = w_f != 0
    assert_parity(r["dw"][mask], gw[mask], "dW on mask")


@pytest.mark.parametrize("mode", ["exact", "tc"])
def test_dense_plan_against_f64_oracle(mode):
    cfg = with_sparsity(CONFIGS["c0"], 0.0)
    img, w_f, go = make_inputs(cfg, n=2)
    w_f[0, 0, 0, 0] = 0.0  # an exact zero still gets a gradient on the dense path
    r = run_layer(img, w_f, go, 4, 1, dense=mode)
    assert r["layer"].is_dense and r["dw"].shape == w_f.shape
    imgp = np.pad(img.astype(np.float64), ((0, 0), (0, 0), (1, 1), (1, 1)))
    gw = np.zeros_like(w_f)
    for i in range(2):
        o, cache = wo.forward_f64(imgp[i], w_f, 4)
        assert_parity(r["o"][i], o, "O")
        gw += wo.backward_weights_f64(go[i].astype(np.float64), cache)
    assert_parity(r["dw"], gw, "dense dW")
    assert r["dw"][0, 0, 0, 0] != 0.0


def _f64_batched(img, w_f, go, pad, m=4):
    """Fast f64 restatement (per-slice BLAS) of layer.cpp over a batch, for large parity cases."""
    n, c, h, w = img.shape
    g = wo.padded_geometry(c, h, w, pad, m)
    a, b, _ = wo.transforms(m)
    p = g.p
    imgp = np.zeros((n, c, g.h_ip, g.w_ip))
    imgp[:, :, pad:pad + h, pad:pad + w] = img
    til = np.stack([imgp[:, :, (t // g.tiles_x) * m:(t // g.tiles_x) * m + p,
                         (t % g.tiles_x) * m:(t % g.tiles_x) * m + p] for t in range(g.t)], axis=2)
    v = np.einsum("ki,nctkl,lj->ijcnt", b, til, b).reshape(p * p, c, n * g.t)
    wsl = w_f.transpose(2, 3, 0, 1).reshape(p * p, w_f.shape[0], c)
    z = np.matmul(wsl, v)
    k = w_f.shape[0]
    zz = z.reshape(p, p, k, n, g.tiles_y, g.tiles_x)
    ot = np.einsum("iy,ijknab,jx->nkaybx", a, zz, a).reshape(n, k, g.h_op, g.w_op)[:, :, :g.h_o, :g.w_o]
    full = np.zeros((n, k, g.h_op, g.w_op))
    full[:, :, :g.h_o, :g.w_o] = go
    dot = full.reshape(n, k, g.tiles_y, m, g.tiles_x, m)
    dz = np.einsum("iy,nkaybx,jx->ijknab", a, dot, a).reshape(p * p, k, n * g.t)
    dw = np.matmul(dz, v.transpose(0, 2, 1)).reshape(p, p, k, c).transpose(2, 3, 0, 1)
    dv = np.matmul(wsl.transpose(0, 2, 1), dz).reshape(p, p, c, n, g.tiles_y, g.tiles_x)
    gt = np.einsum("ik,klcnab,jl->ncabij", b, dv, b)
    di = np.zeros((n, c, g.h_ip, g.w_ip))
    for ty in range(g.tiles_y):
        for tx in range(g.tiles_x):
            di[:, :, ty * m:ty * m + p, tx * m:tx * m + p] += gt[:, :, ty, tx]
    return ot, dw, di[:, :, pad:pad + h, pad:pad + w]


def test_c1_full_batch_parity():
    """BASELINE configs[1] at its full size (N=32, C=256, K=384, H=13, 90%): O, dI and dW_F (every
    surviving entry) within |d| <= 1e-5 + 1e-4·|ref| of the reference's f64 layer — zero misses.
    dW_F is a 512-term dot product with heavy cancellation; an fp32-operand dW_F misses the bound
    on ~5e-5 of the entries, the exact digit GEMM (wino_xdw.cuh) on none, with a margin of ~75x."""
    cfg = CONFIGS["c1"]
    img, w_f, go = make_inputs(cfg)
    r = run_layer(img, w_f, go, 4, 1, dense=False)
    o, dw, di = _f64_batched(img.astype(np.float64), w_f, go.astype(np.float64), 1)
    assert_parity(r["o"], o, "c1 O")
    assert_parity(r["di"], di, "c1 dI")
    mask = w_f != 0
    assert_parity(r["dw"][mask], dw[mask], "c1 dW_F (every surviving entry)")
    worst = np.max(np.abs(r["dw"][mask] - dw[mask]) / (1e-5 + 1e-4 * np.abs(dw[mask])))
    assert worst < 0.1, f"dW_F margin only {1 / worst:.1f}x"
    assert np.all(r["dw"][~mask] == 0)
    # and bitwise against the f32 mirror (reference association order) for the forward
    mir = wo.layer_f32(img, wo.compress(w_f), None, m=4, pad=1)
    assert np.array_equal(r["o"], mir["o"])


def test_c1_tensor_core_contraction():
    """WINO_OPT_CONTRACTION=1 on the sparse plan (zero-filled W_F on tcgen05): O and dI within the
    strict tolerance of the f64 reference on every element at configs[1]; dW_F unchanged (it
    stays on the exact SDDMM)."""
    cfg = CONFIGS["c1"]
    img, w_f, go = make_inputs(cfg)
    r = run_layer(img, w_f, go, 4, 1, dense=False, contraction="tc")
    base = run_layer(img, w_f, go, 4, 1, dense=False)
    o, dw, di = _f64_batched(img.astype(np.float64), w_f, go.astype(np.float64), 1)
    assert_parity(r["o"], o, "c1 O (tc contraction)")
    assert_parity(r["di"], di, "c1 dI (tc contraction)")
    # dZ does not depend on the contraction, so neither does the SDDMM's dW
    assert np.array_equal(r["dw_raw"], base["dw_raw"])


@pytest.mark.parametrize("name", ["c0", "f43_dense", "f63"])
def test_tensor_core_contraction_golden(name):
    d = load_layer(name)
    if d["c"] % 4 or d["k"] % 4:
        pytest.skip("TMA strides need C, K multiples of 4")
    r = run_layer(d["img"], d["w_f"], d["grad_o"], d["m"], d["pad"], dense=False, contraction="tc")
    assert_parity(r["o"], d["o_f64"], "O vs f64 reference")
    assert_parity(r["di"], d["grad_in_f64"], "dI vs f64 reference")


def test_tensor_core_contraction_follows_updates():
    """After an update the zero-filled operands are rebuilt: the forward equals a fresh plan of
    the updated weights, and masked coordinates stay zero."""
    cfg = CONFIGS["c0"]
    img, w_f, go = make_inputs(cfg, n=2)
    layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
    layer.set_weights(w_f)
    layer.set_contraction("tc")
    cache = layer.new_cache(2)
    layer.forward(dev(img), cache)
    g = layer.backward_weights(dev(go), cache)
    layer.sgd_step(g, lr=0.05)
    out = layer.forward(dev(img)).cpu().numpy()
    w1 = layer.weights()
    assert np.all(w1[w_f == 0] == 0)
    fresh = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
    fresh.set_weights(w1, dense=False)
    fresh.set_contraction("tc")
    assert np.array_equal(out, fresh.forward(dev(img)).cpu().numpy())


@pytest.mark.parametrize("mode", ["sparse", "dense-tc"])
def test_fused_backward_equals_separate_calls(mode):
    """wino_backward (dW on a side stream, concurrent with dI) == backward_weights + backward_input."""
    cfg = CONFIGS["c0"]
    img, w_f, go = make_inputs(cfg, n=3)
    if mode == "dense-tc":
        w_f = np.where(w_f == 0, 0.01, w_f)
    layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
    layer.set_weights(w_f, dense=True if mode == "dense-tc" else False)
    cache = layer.new_cache(3)
    x, g = dev(img), dev(go)
    o = layer.forward(x, cache, relu=True)
    dw1 = layer.backward_weights(g, cache, relu_out=o)
    di1 = layer.backward_input(cache)
    dw2, di2 = layer.backward(g, cache, relu_out=o)
    torch.cuda.synchronize()
    assert torch.equal(dw1, dw2) and torch.equal(di1, di2)


def test_determinism_and_repeatability():
    cfg = CONFIGS["c1"]
    img, w_f, go = make_inputs(cfg, n=8)
    a = run_layer(img, w_f, go, 4, 1, dense=False)
    b = run_layer(img, w_f, go, 4, 1, dense=False)
    for key in ("o", "di", "dw_raw"):
        assert np.array_equal(a[key], b[key]), key


def _f64_slices(img, go, slices, pad=1, m=4, chunk=8):
    """f64 Ĩ_F[s] (C×N·T) and dZ[s] (K×N·T) of selected slices over the whole batch (layer.cpp:55-59,
    107-116 in f64), built in image chunks to bound host memory."""
    n, c, h, w = img.shape
    k = go.shape[1]
    g = wo.padded_geometry(c, h, w, pad, m)
    a, b, _ = wo.transforms(m)
    p = g.p
    vs = {s: np.empty((c, n * g.t)) for s in slices}
    zs = {s: np.empty((k, n * g.t)) for s in slices}
    for n0 in range(0, n, chunk):
        n1 = min(n, n0 + chunk)
        imgp = np.zeros((n1 - n0, c, g.h_ip, g.w_ip))
        imgp[:, :, pad:pad + h, pad:pad + w] = img[n0:n1]
        til = np.stack([imgp[:, :, (t // g.tiles_x) * m:(t // g.tiles_x) * m + p,
                             (t % g.tiles_x) * m:(t % g.tiles_x) * m + p] for t in range(g.t)], axis=2)
        full = np.zeros((n1 - n0, k, g.h_op, g.w_op))
        full[:, :, :g.h_o, :g.w_o] = go[n0:n1]
        dot = full.reshape(n1 - n0, k, g.tiles_y, m, g.tiles_x, m)
        for s in slices:
            i, j = divmod(s, p)
            vs[s][:, n0 * g.t:n1 * g.t] = np.einsum("k,nctkl,l->cnt", b[:, i], til, b[:, j]).reshape(c, -1)
            zs[s][:, n0 * g.t:n1 * g.t] = np.einsum("y,nkaybx,x->knab", a[i], dot, a[j]).reshape(k, -1)
    return vs, zs


C3_SLICES = [0, 7, 20, 35]  # corner, interior and the largest-coefficient slice (5,5)


@pytest.fixture(scope="module")
def c3_ref():
    """configs[3] inputs (the same I and dO at every sparsity) and the f64 Ĩ_F / dZ of C3_SLICES."""
    cfg = CONFIGS["c3"]
    img, _, go = make_inputs(cfg)
    vs, zs = _f64_slices(img.astype(np.float64), go.astype(np.float64), C3_SLICES)
    return img, go, vs, zs


def _check_c3(r, w_f, img, go, vs, zs, what):
    sub = [0, 37]
    o, _, di = _f64_batched(img[sub].astype(np.float64), w_f, go[sub].astype(np.float64), 1)
    assert_parity(r["o"][sub], o, f"{what} O (sampled images)")
    assert_parity(r["di"][sub], di, f"{what} dI (sampled images)")
    p = w_f.shape[2]
    worst = 0.0
    for s in C3_SLICES:
        i, j = divmod(s, p)
        ref_ = zs[s] @ vs[s].T                     # f64 dW_F(:,:,i,j), layer.cpp:118-128
        mask = w_f[:, :, i, j] != 0 if not r["layer"].is_dense else np.ones(ref_.shape, bool)
        got = r["dw"][:, :, i, j]
        assert_parity(got[mask], ref_[mask], f"{what} dW_F slice {s} (every surviving entry)")
        worst = max(worst, float(np.max(np.abs(got[mask] - ref_[mask]) / (1e-5 + 1e-4 * np.abs(ref_[mask])))))
        assert np.all(got[~mask] == 0)
    return worst


@pytest.mark.slow
@pytest.mark.parametrize("sparsity,contraction", [(0.5, "csr"), (0.8, "csr"), (0.9, "csr"), (0.95, "csr"),
                                                  (0.5, "auto"), (0.8, "auto"), (0.9, "auto")])
def test_c3_sweep_parity(sparsity, contraction, c3_ref):
    """configs[3] (N=64, C=K=256, H=56) at every BASELINE sparsity, CSR and 'auto' contraction:
    O and dI on sampled images, dW_F on EVERY surviving entry of sampled slices, all against the
    reference's f64 layer (sparse.cpp:189-253 forward, layer.cpp:98-171 backward on the mask)."""
    img, go, vs, zs = c3_ref
    _, w_f, _ = make_inputs(with_sparsity(CONFIGS["c3"], sparsity))
    r = run_layer(img, w_f, go, 4, 1, dense=False, contraction=contraction if contraction != "csr" else None)
    worst = _check_c3(r, w_f, img, go, vs, zs, f"c3 {sparsity:.0%} {contraction}")
    print(f"c3 {sparsity:.0%} {contraction}: dW worst error / tolerance {worst:.3g}")
    if contraction == "csr":  # the CSR forward is bitwise the reference's f32 order: check 2 images
        mir = wo.layer_f32(img[:2], wo.compress(w_f), None, m=4, pad=1)
        assert np.array_equal(r["o"][:2], mir["o"])


@pytest.mark.slow
def test_c3_dense_tensor_core_parity(c3_ref):
    """configs[3] at 0% sparsity: the dense plan (3xTF32 tcgen05 Z / dĨ_F, compensated fold per
    k-block; exact int8 digit GEMM for dW_F): O and dI on sampled images and dW_F on every entry
    of sampled slices within the strict bound of the f64 reference."""
    img, go, vs, zs = c3_ref
    _, w_f, _ = make_inputs(with_sparsity(CONFIGS["c3"], 0.0))
    r = run_layer(img, w_f, go, 4, 1, dense="tc")
    assert r["layer"].is_dense
    worst = _check_c3(r, w_f, img, go, vs, zs, "c3 dense")
    print(f"c3 dense: dW worst error / tolerance {worst:.3g}")


def test_relu_flags_and_sgd():
    d = load_layer("c0")
    layer = wb.WinogradLayer(d["c"], d["k"], d["h"], d["w"], pad=1, m=4)
    layer.set_weights(d["w_f"])
    cache = layer.new_cache(1)
    o = layer.forward(dev(d["img"]), cache, relu=True).cpu().numpy()
    mir = wo.layer_f32(d["img"], wo.compress(d["w_f"]), None, m=4, pad=1)
    assert np.array_equal(o, np.maximum(mir["o"], 0))
    o_dev = dev(o)
    dw = layer.backward_weights(dev(d["grad_o"]), cache, relu_out=o_dev)
    masked = d["grad_o"] * (o > 0)
    mir2 = wo.layer_f32(d["img"], wo.compress(d["w_f"]), masked, m=4, pad=1)
    np.testing.assert_allclose(dw.cpu().numpy(), np.concatenate(mir2["dw"]), rtol=2e-6, atol=1e-5)
    # masked SGD: only surviving values move; v -= lr*(scale*g + l2*v/||v||)
    vals0 = np.concatenate(wb.compress(d["w_f"]).values).astype(np.float64)
    layer.sgd_step(dw, lr=0.1, scale=0.5, l2=0.01)
    torch.cuda.synchronize()
    vals1 = np.concatenate(layer.get_csr().values)
    g = dw.cpu().numpy().astype(np.float64)
    expect = vals0 - 0.1 * (0.5 * g + 0.01 * vals0 / np.sqrt(np.sum(vals0 ** 2)))
    np.testing.assert_allclose(vals1, expect, rtol=1e-5, atol=1e-7)


def test_api_reference_surface():
    """python/tests/test_smoke.py cases, served by the GPU (fp32 tolerances)."""
    rng = np.random.default_rng(0)
    img = rng.standard_normal((3, 9, 11))
    w = rng.standard_normal((2, 3, 3, 3))
    out = wb.conv_winograd(img, wb.lift(w), m=2)
    assert out.shape == (2, 7, 9)
    np.testing.assert_allclose(out, wo.direct_conv_f64(img, w), atol=1e-4)
    img = rng.standard_normal((2, 12, 12))
    w = rng.standard_normal((2, 2, 3, 3))
    np.testing.assert_allclose(wb.conv_winograd(img, wb.lift(w, m=4), m=4), wo.direct_conv_f64(img, w),
                               atol=1e-4)
    img = rng.standard_normal((1, 6, 6))
    w_f = rng.standard_normal((2, 1, 4, 4))
    out = wb.conv_winograd(img, w_f)
    gw, gi = wb.conv_winograd_grad(img, w_f, out)
    o64, cache = wo.forward_f64(img, w_f, 2)
    np.testing.assert_allclose(gw, wo.backward_weights_f64(o64, cache), rtol=1e-4, atol=1e-4)
    np.testing.assert_allclose(gi, wo.backward_input_f64(cache, w_f), rtol=1e-4, atol=1e-4)
    batch = rng.standard_normal((2, 3, 8, 8))
    w_f = rng.standard_normal((4, 3, 4, 4))
    w_f[np.abs(w_f) < 0.8] = 0.0
    out = wb.sparse_conv(batch, w_f, workers=1)
    assert np.array_equal(out, wb.sparse_conv(batch, w_f, workers=4))
    for n in range(2):
        np.testing.assert_allclose(out[n], wo.forward_f64(batch[n], w_f, 2)[0], rtol=1e-4, atol=1e-4)
    with pytest.raises(wb.CapabilityError):
        wb.sparse_conv(batch, w_f, precision="f64")


def test_stack_training_step_matches_mirror():
    """Two-layer stack (configs[0] shapes): forward with fused ReLU, relu-masked backward
    chain, one bucketed reduction, masked SGD — against the f32 mirror chained by hand."""
    from paper_1702_08597_b200.stack import WinogradStack

    cfg = CONFIGS["c0"]
    img, w1, go = make_inputs(cfg, n=3)
    w2 = w1[:, :, ::-1, ::-1].copy()
    st = WinogradStack([w1, w2], cfg.c, cfg.h, cfg.w, pad=1, m=4, n_max=3)
    x = dev(img)
    st.forward(x)
    bucket = st.backward(dev(go))
    torch.cuda.synchronize()
    got = bucket.flat.cpu().numpy().astype(np.float64)
    # mirror: O1 = relu(L1(img)); O2 = relu(L2(O1)); dO2 = go·[O2>0]; dO1 = dI2·[O1>0]
    c1, c2 = wo.compress(w1), wo.compress(w2)
    o1 = np.maximum(wo.layer_f32(img, c1, None, m=4, pad=1)["o"], 0)
    r2 = wo.layer_f32(o1, c2, go * (wo.layer_f32(o1, c2, None, m=4, pad=1)["o"] > 0), m=4, pad=1)
    o2 = np.maximum(r2["o"], 0)
    assert np.array_equal(st.outs[1].cpu().numpy(), o2)
    r1 = wo.layer_f32(img, c1, r2["di"] * (o1 > 0), m=4, pad=1)
    want = np.concatenate([np.concatenate(r1["dw"]), np.concatenate(r2["dw"])])
    np.testing.assert_allclose(got, want, rtol=2e-6, atol=1e-5)
    # masked SGD: v -= lr·g/B on surviving coordinates only
    vals0 = [np.concatenate(wb.compress(w).values).astype(np.float64) for w in (w1, w2)]
    for lay, g in zip(st.layers, st.bucket.views):
        lay.sgd_step(g, lr=0.05, scale=1.0 / 3)
    torch.cuda.synchronize()
    for lay, v0, g in zip(st.layers, vals0, st.bucket.views):
        v1 = np.concatenate(lay.get_csr().values)
        np.testing.assert_allclose(v1, v0 - 0.05 * g.cpu().numpy() / 3, rtol=1e-5, atol=1e-7)
        assert lay.nnz == len(v0)  # the mask is fixed: pruned coordinates never reappear


@pytest.mark.parametrize("name", ["c0", "f23_odd", "f63"])
def test_runtime_and_builtin_coefficient_kernels_agree_bitwise(name, monkeypatch):
    """Transform kernels with compile-time coefficients (zero terms dropped) vs the generic
    runtime-coefficient kernels: identical bits."""
    d = load_layer(name)
    a = run_layer(d["img"], d["w_f"], d["grad_o"], d["m"], d["pad"], dense=False)
    monkeypatch.setenv("WINO_RUNTIME_COEFS", "1")
    b = run_layer(d["img"], d["w_f"], d["grad_o"], d["m"], d["pad"], dense=False)
    for key in ("o", "di", "dw_raw"):
        assert np.array_equal(a[key], b[key]), key


def test_host_step_pipeline_matches_device_path():
    """HostStep (pinned host buffers, overlapped copies, graphed passes) returns exactly what
    the device-resident calls return."""
    from paper_1702_08597_b200.pipeline import HostStep

    cfg = CONFIGS["c1"]
    img, w_f, go = make_inputs(cfg, n=8)
    ref = run_layer(img, w_f, go, 4, 1, dense=False)
    layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
    layer.set_weights(w_f, dense=False)
    cache = layer.new_cache(8)
    x, g = dev(np.zeros_like(img)), dev(np.zeros_like(go))
    o = torch.empty((8, cfg.k, layer.ho, layer.wo), device="cuda")
    dw = torch.empty((layer.nnz,), device="cuda")
    di = torch.empty((8, cfg.c, cfg.h, cfg.w), device="cuda")
    layer.forward(x, cache, out=o)
    layer.backward_weights(g, cache, out=dw)
    hs = HostStep(layer, cache, x, g, o, dw, di)
    h = [torch.from_numpy(a).pin_memory() for a in (img, go)]
    outs = [torch.empty(t.shape).pin_memory() for t in (o, dw, di)]
    for _ in range(3):
        hs(h[0], h[1], *outs)
    torch.cuda.synchronize()
    assert np.array_equal(outs[0].numpy(), ref["o"])
    assert np.array_equal(outs[1].numpy(), ref["dw_raw"])
    assert np.array_equal(outs[2].numpy(), ref["di"])


@pytest.mark.parametrize("name,n,chunks,relu", [("c1", 32, 4, False), ("c1", 32, 3, True), ("c0", 9, 2, False),
                                                ("c0", 9, 1, True)])
def test_pipelined_host_step_is_bitwise_the_whole_batch(name, n, chunks, relu):
    """PipelinedHostStep (image-range forward/backward, dW once over the batch) returns exactly
    what the whole-batch device calls return; c0 (T = 9) exercises the 4-column alignment."""
    from paper_1702_08597_b200.pipeline import PipelinedHostStep

    cfg = CONFIGS[name]
    img, w_f, go = make_inputs(cfg, n=n)
    layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
    layer.set_weights(w_f, dense=False)
    cache = layer.new_cache(n)
    x, g = dev(img), dev(go)
    o_ref = layer.forward(x, cache, relu=relu)
    dw_ref = layer.backward_weights(g, cache, relu_out=o_ref if relu else None)
    di_ref = layer.backward_input(cache)
    torch.cuda.synchronize()
    want = [t.cpu().numpy() for t in (o_ref, dw_ref, di_ref)]
    xs, gs = torch.zeros_like(x), torch.zeros_like(g)
    o, dw, di = torch.empty_like(o_ref), torch.empty_like(dw_ref), torch.empty_like(di_ref)
    ps = PipelinedHostStep(layer, cache, xs, gs, o, dw, di, chunks=chunks, relu=relu)
    h = [torch.from_numpy(a).pin_memory() for a in (img, go)]
    outs = [torch.empty(t.shape).pin_memory() for t in (o, dw, di)]
    for _ in range(2):
        ps(h[0], h[1], *outs)
    torch.cuda.synchronize()
    _check_pipelined(outs, want)
    first = [t.numpy().copy() for t in outs]
    # and captured as one CUDA graph (copies + kernels on three streams)
    from paper_1702_08597_b200.graph import GraphedStep

    for t in outs:
        t.zero_()
    GraphedStep(lambda: ps(h[0], h[1], *outs)).replay()
    torch.cuda.synchronize()
    for got, w in zip(outs, first):
        assert np.array_equal(got.numpy(), w)


def _check_pipelined(outs, want):
    """O and dI bitwise the whole-batch calls.  dW_F: each image chunk is its own digit-exponent
    segment (its max|I| / max|dO| are known when its range runs), so the digits round differently
    than with the whole batch's exponents — both within ~2% of north_star's tolerance of the f64
    value (c1), so they agree within a tolerance 10x tighter than north_star's."""
    assert np.array_equal(outs[0].numpy(), want[0])
    assert np.array_equal(outs[2].numpy(), want[2])
    assert_parity(outs[1].numpy(), want[1], "pipelined dW_F vs whole batch", rtol=1e-5, atol=1e-6)


def test_range_calls_validate():
    cfg = CONFIGS["c0"]
    img, w_f, go = make_inputs(cfg, n=9)
    layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
    layer.set_weights(w_f, dense=False)
    cache = layer.new_cache(9)
    x = dev(img)
    o = torch.empty((9, cfg.k, layer.ho, layer.wo), device="cuda")
    with pytest.raises(wb.ShapeError):  # 1·T = 9 columns: not 16-byte aligned
        layer.forward_range(x[1:3], 9, 1, cache, o[1:3])
    with pytest.raises(wb.ShapeError):
        layer.forward_range(x[4:9], 8, 4, cache, o[4:9])
    with pytest.raises(wb.ConsistencyError):
        layer.backward_weights_cached(layer.new_cache(9))
    dense = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
    dense.set_weights(np.where(w_f == 0, 0.5, w_f), dense=True)
    with pytest.raises(wb.CapabilityError):
        dense.forward_range(x[0:4], 9, 0, dense.new_cache(9), o[0:4])


def test_auto_contraction_follows_density():
    """contraction 'auto': tensor cores at density >= the threshold, the CSR path
    below it (bitwise the default forward), re-decided when the weights change."""
    cfg = CONFIGS["c0"]
    img, w_f, go = make_inputs(with_sparsity(cfg, 0.5), n=2)
    layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
    layer.set_weights(w_f, dense=False)
    layer.set_contraction("auto")
    cache = layer.new_cache(2)
    o = layer.forward(dev(img), cache).cpu().numpy()
    dw = layer.backward_weights(dev(go), cache).cpu().numpy()
    di = layer.backward_input(cache).cpu().numpy()
    o64, dw64, di64 = _f64_batched(img.astype(np.float64), w_f, go.astype(np.float64), 1)
    assert_parity(o, o64, "auto O (tensor cores)")
    assert_parity(di, di64, "auto dI (tensor cores)")
    mask = w_f != 0
    assert_parity(layer.compact_to_dense(dw.astype(np.float64))[mask], dw64[mask], "auto dW_F")
    # below the threshold: the CSR kernels, bitwise the reference order
    layer.set_auto_density(0.9)
    o2 = layer.forward(dev(img)).cpu().numpy()
    mir = wo.layer_f32(img, wo.compress(w_f), None, m=4, pad=1)
    assert np.array_equal(o2, mir["o"])


@pytest.mark.parametrize("mode", ["csr", "tc", "dense"])
def test_forward_backward_equals_two_calls(mode):
    """wino_forward_backward (dI chain and dW_F overlapping the forward) is bitwise forward +
    backward on every plan kind."""
    cfg = CONFIGS["c1"]
    img, w_f, go = make_inputs(cfg if mode != "dense" else with_sparsity(cfg, 0.0))
    layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
    layer.set_weights(w_f, dense=(mode == "dense"))
    if mode == "tc":
        layer.set_contraction("tc")
    x, g = dev(img), dev(go)
    c1 = layer.new_cache(cfg.n)
    o1 = layer.forward(x, c1)
    w1, i1 = layer.backward(g, c1)
    c2 = layer.new_cache(cfg.n)
    o2, w2, i2 = layer.forward_backward(x, g, c2)
    torch.cuda.synchronize()
    for a, b, what in ((o1, o2, "O"), (w1, w2, "dW_F"), (i1, i2, "dI")):
        assert torch.equal(a, b), f"{mode}: {what} differs"
    # the cache holds the step's Ĩ_F and dZ: backward_input from it reproduces dI
    assert torch.equal(layer.backward_input(c2), i1)


@pytest.mark.parametrize("mode", ["dense", "tc", "csr", "fb"])
def test_ragged_tile_shapes(mode):
    """C, K and N·T that fill no tcgen05 tile evenly (C = 136, K = 200, 3 images of 9×9 → N·T = 27):
    partial M, N and reduction blocks in the warp-specialised GEMM (TMA zero-fill, clipped TMA
    stores) and in the int8 digit GEMM (partial 128-row / 64-row tiles, a padded 64-column
    segment), every output element within the strict bound of the f64 reference."""
    from paper_1702_08597_b200.synth import LayerConfig

    cfg = LayerConfig("ragged", 3, 136, 200, 9, 0.0 if mode == "dense" else 0.7)
    img, w_f, go = make_inputs(cfg)
    layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.h, pad=1, m=4)
    layer.set_weights(w_f, dense=(mode == "dense"))
    if mode == "tc":
        layer.set_contraction("tc")
    cache = layer.new_cache(cfg.n)
    x, g = dev(img), dev(go)
    if mode == "fb":
        o, dw, di = layer.forward_backward(x, g, cache)
    else:
        o = layer.forward(x, cache)
        dw, di = layer.backward(g, cache)
    o, dw, di = o.cpu().numpy(), dw.cpu().numpy(), di.cpu().numpy()
    o64, dw64, di64 = _f64_batched(img.astype(np.float64), w_f, go.astype(np.float64), 1)
    assert_parity(o, o64, f"{mode} O")
    assert_parity(di, di64, f"{mode} dI")
    dwd = dw if mode == "dense" else layer.compact_to_dense(dw.astype(np.float64))
    mask = w_f != 0 if mode != "dense" else np.ones(w_f.shape, bool)
    assert_parity(np.asarray(dwd)[mask], dw64[mask], f"{mode} dW_F")


@pytest.mark.slow
@pytest.mark.parametrize("sparsity", [0.8, 0.9, 0.95])
def test_c2_forward_bitwise(sparsity):
    """configs[2] at its full size (N=64, C=K=512, H=W=28) at 80/90/95%: the SpMM runs with its
    operand chunk in TMEM in 4 stages (80/90%) or in shared memory, 2-wide t (95%); the forward of 8
    sampled images is bitwise the f32 mirror of the reference's sparse_forward<float>
    (sparse.cpp:189-253) and within the strict bound of the f64 layer."""
    cfg = with_sparsity(CONFIGS["c2"], sparsity)
    img, w_f, _ = make_inputs(cfg)
    layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.h, pad=1, m=4)
    layer.set_weights(w_f, dense=False)
    o = layer.forward(dev(img)).cpu().numpy()
    sub = [0, 9, 18, 27, 36, 45, 54, 63]
    mir = wo.layer_f32(img[sub], wo.compress(w_f), None, m=4, pad=1)
    assert np.array_equal(o[sub], mir["o"])
    o64, _, _ = _f64_batched(img[sub[:2]].astype(np.float64), w_f, np.zeros((2, cfg.k, cfg.h, cfg.h)), 1)
    assert_parity(o[sub[:2]], o64, f"c2 {sparsity:.0%} O")


@pytest.mark.parametrize("name", LAYER_CASES)
def test_forward_backward_golden(name):
    """wino_forward_backward on every golden layer (F(2,3), F(4,3), F(6,3); odd, padded, dense, tiny
    shapes): O bitwise the reference's f32 sparse_forward where the golden file has it, and O, dI,
    dW_F bitwise the separate forward + backward calls."""
    d = load_layer(name)
    layer = wb.WinogradLayer(d["c"], d["k"], d["h"], d["w"], pad=d["pad"], m=d["m"])
    layer.set_weights(d["w_f"], dense=False)
    x, g = dev(d["img"]), dev(d["grad_o"])
    c1 = layer.new_cache(d["n"])
    o1 = layer.forward(x, c1)
    w1, i1 = layer.backward(g, c1)
    o2, w2, i2 = layer.forward_backward(x, g, layer.new_cache(d["n"]))
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(w1, w2) and torch.equal(i1, i2)
    if "o_sparse_f32" in d:
        assert np.array_equal(o2.cpu().numpy(), d["o_sparse_f32"])



@pytest.mark.slow
def test_c4_stack_layers_against_reference():
    """configs[4]'s layer stack (4 layers, C=K=256, H=W=28, 90% fixed masks, ReLU between layers)
    at 64 images per GPU (the 8-GPU shard of the global batch of 512): every layer's forward is
    bitwise the f32 mirror of the reference's sparse_forward<float> applied to the previous
    layer's fp32 output (ReLU fused, train.cpp:76-83); every layer's dW_F (every surviving entry)
    and dI within the strict bound of the f64 layer on the same fp32 inputs and the
    relu-masked incoming gradient (train.cpp:189-211)."""
    from paper_1702_08597_b200.stack import WinogradStack
    from paper_1702_08597_b200.synth import LayerConfig, Stream

    cfg = CONFIGS["c4"]
    n = 64
    weights = [make_inputs(LayerConfig("c4", 1, cfg.c, cfg.k, cfg.h, cfg.sparsity, seed=cfg.seed), layer=l)[1]
               for l in range(4)]
    img = Stream(cfg.seed, "c4/I").normal((n, cfg.c, cfg.h, cfg.w)).astype(np.float32)
    go = Stream(cfg.seed, "c4/dO").normal((n, cfg.k, cfg.h, cfg.w)).astype(np.float32)
    st = WinogradStack(weights, cfg.c, cfg.h, cfg.w, pad=1, m=4, n_max=n)
    st.forward(dev(img))
    st.backward(dev(go), serial=True)
    torch.cuda.synchronize()
    ins = [img] + [st.outs[i].cpu().numpy() for i in range(3)]
    grads = [g.cpu().numpy().astype(np.float64) for g in st.grads]
    g_in = go
    for i in range(3, -1, -1):
        lay, w_f = st.layers[i], weights[i]
        out = st.outs[i].cpu().numpy()
        if i in (0, 3):  # the mirror of the reference's f32 order, bitwise (two layers: host time)
            mir = wo.layer_f32(ins[i][:4], wo.compress(w_f), None, m=4, pad=1)
            assert np.array_equal(out[:4], np.maximum(mir["o"], 0)), f"layer {i} forward"
        dO = g_in * (out > 0)                            # relu-mask backward, train.cpp:193
        o64, dw64, di64 = _f64_batched(ins[i].astype(np.float64), w_f, dO.astype(np.float64), 1)
        assert_parity(out, np.maximum(o64, 0), f"layer {i} O")
        mask = w_f != 0
        assert_parity(lay.compact_to_dense(grads[i])[mask], dw64[mask], f"layer {i} dW_F")
        if i > 0:
            g_in = st.dis[i].cpu().numpy()
            assert_parity(g_in, di64, f"layer {i} dI")


def test_dw_mode_option():
    """dW_F has one mode ('exact'); the round-1 mode names are rejected."""
    layer = wb.WinogradLayer(16, 16, 12, 12, pad=1, m=4)
    layer.set_weights(make_inputs(CONFIGS["c0"])[1])
    layer.set_dw_mode("exact")
    for bad in ("sddmm", "tc", "precise", "int8"):
        with pytest.raises(wb.InvalidArgument):
            layer.set_dw_mode(bad)


def _step_with_operands(img, w_f, go, where, lr=None):
    n, c, h, w = img.shape
    layer = wb.WinogradLayer(c, w_f.shape[0], h, w, pad=1, m=4)
    layer.set_weights(w_f, dense=False)
    layer.set_spmm_operands(where)
    cache = layer.new_cache(n)
    x, g = dev(img), dev(go)
    outs = []
    for _ in range(2 if lr else 1):
        o = layer.forward(x, cache)
        dw = layer.backward_weights(g, cache)
        di = layer.backward_input(cache)
        torch.cuda.synchronize()
        outs.append((o.cpu().numpy(), dw.cpu().numpy(), di.cpu().numpy()))
        if lr:
            layer.sgd_step(dw, lr=lr, scale=1.0, l2=0.0)  # new values, same structure
    layer.close()
    return outs


@pytest.mark.parametrize("c,k,h,n,sparsity", [(256, 256, 28, 4, 0.9), (256, 384, 13, 8, 0.9),
                                              (512, 512, 14, 2, 0.5), (160, 200, 12, 3, 0.7),
                                              (256, 256, 20, 3, 0.97)])
def test_tmem_spmm_bitwise_equals_shared_memory(c, k, h, n, sparsity):
    """The TMEM-resident CSR kernels (wino_spmm_tm.cuh: S = 2 and 4 stages, staged and global
    stream, ragged row counts) give the shared-memory kernels' results bit for bit — O, dĨ_F -> dI,
    and dW_F — before and after a value update (the padded stream's value refresh)."""
    rng = np.random.default_rng(c * 1000 + k + h)
    img = rng.standard_normal((n, c, h, h)).astype(np.float32)
    go = rng.standard_normal((n, k, h, h)).astype(np.float32)
    w_f = rng.standard_normal((k, c, 6, 6)) * np.sqrt(2.0 / (9 * c))
    w_f *= rng.random(w_f.shape) >= sparsity
    a = _step_with_operands(img, w_f, go, "tmem", lr=1e-3)
    b = _step_with_operands(img, w_f, go, "smem", lr=1e-3)
    for (oa, dwa, dia), (ob, dwb, dib) in zip(a, b):
        assert np.array_equal(oa, ob), "O differs between TMEM and shared-memory operands"
        assert np.array_equal(dia, dib), "dI differs between TMEM and shared-memory operands"
        assert np.array_equal(dwa, dwb), "dW_F differs"
    if 128 < c <= 256 and 128 < k <= 256:
        # hybrid operands (rows [0,128) in TMEM, the rest in shared memory; wino_spmm_tm.cuh):
        # forced here on both directions, staged (0.9 / 0.97) and unstaged (0.7) streams, ragged rows
        h_ = _step_with_operands(img, w_f, go, "hybrid", lr=1e-3)
        for (oa, dwa, dia), (ob, dwb, dib) in zip(h_, b):
            assert np.array_equal(oa, ob), "O differs between hybrid and shared-memory operands"
            assert np.array_equal(dia, dib), "dI differs between hybrid and shared-memory operands"
            assert np.array_equal(dwa, dwb), "dW_F differs"
    if c == 160:  # anchor the TMEM path itself to the reference's f32 operation order
        mir = wo.layer_f32(img, wo.compress(w_f), go, m=4, pad=1)
        assert np.array_equal(a[0][0], mir["o"])
        assert np.array_equal(a[0][2], mir["di"])
