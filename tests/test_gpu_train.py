"""The batched training step's weight update on the GPU, through the C-ABI:
prune-mode steps (L1 regulariser + gradient threshold) on dense plans, the on-device
re-derivation of the CSR (bit-exact with the reference's compress), fine-tune steps (L2) on
the sparse plans, and divergence detection — each checked against oracle.train_update_f64,
the restatement of train.cpp:255-290, applied to the same fp32 weights and gradients."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import ref
from oracle import wino_oracle as wo
import paper_1702_08597_b200 as wb
from paper_1702_08597_b200.stack import WinogradStack
from paper_1702_08597_b200.synth import CONFIGS, make_inputs

pytestmark = pytest.mark.gpu


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def _weights(stack):
    return [lay.weights() for lay in stack.layers]


def _grads(stack):
    out = []
    for lay, g in zip(stack.layers, stack.grads):
        g = g.cpu().numpy().astype(np.float64)
        out.append(g if lay.is_dense else lay.compact_to_dense(g))
    return out


def _stack(dense):
    cfg = CONFIGS["c0"]
    img, w1, go = make_inputs(cfg, n=3)
    rng = np.random.default_rng(5)
    w1 = (rng.standard_normal(w1.shape) * 0.2).astype(np.float32).astype(np.float64)
    w2 = (rng.standard_normal(w1.shape) * 0.2).astype(np.float32).astype(np.float64)
    st = WinogradStack([w1, w2], cfg.c, cfg.h, cfg.w, pad=1, m=4, n_max=3, dense=dense)
    return st, dev(img), dev(go * 1e-3)  # small gradients: |g| << β, so the threshold bites


@pytest.mark.parametrize("dense", [True, "exact"])
def test_prune_steps_then_recompress_then_finetune(dense):
    st, x, go = _stack(dense)
    lam, eps, beta, lr = 0.02, 2e-3, 0.05, 0.05
    for step in range(3):
        w0 = _weights(st)
        st.step(x, go, lr=lr, n_global=3, mode="prune", lmbda=lam, norm=1, eps=eps, beta=beta)
        torch.cuda.synchronize()
        g = _grads(st)
        for lay, w_before, gr, w_after in zip(st.layers, w0, g, _weights(st)):
            want, bad = wo.train_update_f64(w_before.ravel(), gr.ravel(), lr, 1.0 / 3, lam, 1, True, eps, beta)
            assert bad == 0
            # norm 1 involves no reduction: the update is bit-exact
            assert np.array_equal(w_after.ravel().astype(np.float32), want), f"step {step}"
    st.check_finite()
    dens = [np.count_nonzero(w) / w.size for w in _weights(st)]
    assert all(0.0 < d < 1.0 for d in dens), dens  # the threshold pruned something
    assert st.densities() == [1.0, 1.0]  # ... but a dense plan still holds every coordinate
    # set_masks_from_zeros + compress, on the device: equal to the reference's compress<float>
    wts = _weights(st)
    st.prune_to_sparse()
    assert st.densities() == pytest.approx(dens)
    for lay, w in zip(st.layers, wts):
        assert not lay.is_dense
        rp, cols, vals = ref.compress_f32(w)
        csr = lay.get_csr()
        for s in range(lay.p * lay.p):
            assert np.array_equal(csr.row_ptr[s].astype(np.int64), rp[s])
            assert np.array_equal(csr.col_idx[s].astype(np.int64), cols[s])
            assert np.array_equal(csr.values[s], vals[s])
    # fine-tune: L2 regulariser on the survivors, masked coordinates stay exactly zero
    w0 = _weights(st)
    st.step(x, go, lr=lr, n_global=3, mode="finetune", lmbda=0.01)
    torch.cuda.synchronize()
    for lay, w_before, g in zip(st.layers, w0, st.grads):
        vals0 = np.concatenate(wb.compress(w_before).values)
        want, _ = wo.train_update_f64(vals0, g.cpu().numpy(), lr, 1.0 / 3, 0.01, 2)
        got = np.concatenate(lay.get_csr().values)
        # ‖w‖₂ is reduced in a different order than numpy's: at most one fp32 ulp apart
        assert np.max(np.abs(got.view(np.int32).astype(np.int64) - want.view(np.int32).astype(np.int64))) <= 1
        assert np.all(lay.weights()[w_before == 0] == 0)


def test_update_matches_oracle_sparse_l2_and_plain():
    cfg = CONFIGS["c0"]
    img, w_f, go = make_inputs(cfg, n=2)
    layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
    layer.set_weights(w_f)
    cache = layer.new_cache(2)
    layer.forward(dev(img), cache)
    g = layer.backward_weights(dev(go), cache)
    gh = g.cpu().numpy()
    for kw in ({"lmbda": 0.0}, {"lmbda": 0.3, "norm": 1}, {"lmbda": 0.3, "norm": 2},
               {"lmbda": 0.3, "norm": 1, "prune": True, "eps": 1e-3, "beta": 0.2}):
        v0 = np.concatenate(layer.get_csr().values)
        layer.update(g, lr=0.01, scale=0.5, **kw)
        torch.cuda.synchronize()
        want, _ = wo.train_update_f64(v0, gh, 0.01, 0.5, kw.get("lmbda", 0.0), kw.get("norm", 1),
                                      kw.get("prune", False), kw.get("eps", 0.0), kw.get("beta", 0.0))
        got = np.concatenate(layer.get_csr().values)
        ulp = np.abs(got.view(np.int32).astype(np.int64) - want.view(np.int32).astype(np.int64))
        assert ulp.max() <= (1 if kw.get("norm") == 2 else 0), kw
    layer.check_finite()


def test_divergence_raises_training_error():
    cfg = CONFIGS["c0"]
    _, w_f, _ = make_inputs(cfg, n=1)
    layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
    layer.set_weights(w_f)
    g = torch.full((layer.nnz,), float("nan"), device="cuda")
    layer.update(g, lr=0.1)
    with pytest.raises(wb._lib.TrainingError):
        layer.check_finite()
    layer.check_finite()  # the counter was reset
    layer.set_weights(w_f)
    big = torch.full((layer.nnz,), 3e38, device="cuda")
    layer.update(big, lr=10.0)  # finite in f64, beyond fp32
    with pytest.raises(wb._lib.TrainingError):
        layer.check_finite()


def test_dense_plan_sgd_uses_kcpq_gradient_layout():
    """A dense plan's gradient is K×C×p×q (what backward_weights returns); the update must pair
    it with the right coordinates."""
    cfg = CONFIGS["c0"]
    img, w_f, go = make_inputs(cfg, n=1)
    rng = np.random.default_rng(1)
    w_f = rng.standard_normal(w_f.shape).astype(np.float32).astype(np.float64)
    layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
    layer.set_weights(w_f, dense="exact")
    g = rng.standard_normal(w_f.shape).astype(np.float32)
    layer.sgd_step(dev(g), lr=0.1)
    torch.cuda.synchronize()
    lr = float(np.float32(0.1))  # wino_sgd_step takes fp32 scalars
    np.testing.assert_array_equal(layer.weights().astype(np.float32),
                                  (w_f - lr * g.astype(np.float64)).astype(np.float32))


def test_recompress_with_tolerance_matches_compress():
    cfg = CONFIGS["c0"]
    _, w_f, _ = make_inputs(cfg, n=1)
    layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
    layer.set_weights(w_f, dense=True)
    layer.recompress(zero_tol=0.05)
    rp, cols, vals = ref.compress_f32(w_f.astype(np.float32).astype(np.float64), zero_tol=0.05)
    csr = layer.get_csr()
    assert layer.nnz == sum(len(c) for c in cols)
    for s in range(layer.p * layer.p):
        assert np.array_equal(csr.col_idx[s].astype(np.int64), cols[s])
        assert np.array_equal(csr.values[s], vals[s])


# -- the torch operator surface ---------------------------------------------
@pytest.mark.parametrize("dense", [False, "exact", True])
def test_winograd_conv2d_module_matches_torch_conv2d(dense):
    """W_F = lift(w): the module is conv2d(x, w, padding=1); its gradients chain back to the
    spatial kernel as dL/dw = Gᵀ·dL/dW_F·G (f64 torch reference, fp32 tolerance)."""
    from paper_1702_08597_b200.autograd import WinogradConv2d

    rng = np.random.default_rng(7)
    n, c, k, h = 2, 8, 12, 10
    w = rng.standard_normal((k, c, 3, 3)) * 0.3
    w_f = wb.lift(w, m=4).astype(np.float32).astype(np.float64)
    if dense is False:
        w_f[np.abs(w_f) < 0.15] = 0.0  # a pruned W_F is no longer a lifted kernel: compare to itself
    mod = WinogradConv2d(w_f, h, h, pad=1, m=4, dense=dense)
    x = torch.tensor(rng.standard_normal((n, c, h, h)), dtype=torch.float32, device="cuda", requires_grad=True)
    out = mod(x)
    go = torch.tensor(rng.standard_normal(out.shape), dtype=torch.float32, device="cuda")
    out.backward(go)
    _, _, g = wb.transforms(4)
    if dense is not False:
        xr = x.detach().double().cpu().requires_grad_(True)
        wr = torch.tensor(w, requires_grad=True)
        ref_out = torch.nn.functional.conv2d(xr, wr, padding=1)
        ref_out.backward(go.double().cpu())
        np.testing.assert_allclose(out.detach().cpu().numpy(), ref_out.detach().numpy(), rtol=1e-4, atol=1e-4)
        np.testing.assert_allclose(x.grad.cpu().numpy(), xr.grad.numpy(), rtol=1e-4, atol=1e-4)
        dwf = mod.values.grad.double().cpu().numpy().reshape(6, 6, k, c).transpose(2, 3, 0, 1)
        dw = np.einsum("iu,kcij,jv->kcuv", g, dwf, g)
        np.testing.assert_allclose(dw, wr.grad.numpy(), rtol=1e-4, atol=1e-3)
    else:
        lay = wb.WinogradLayer(c, k, h, h, pad=1, m=4)
        lay.set_weights(w_f)
        cache = lay.new_cache(n)
        o2 = lay.forward(x.detach(), cache)
        assert torch.equal(out, o2)
        dw2 = lay.backward_weights(go, cache)
        dx2 = lay.backward_input(cache)
        assert torch.equal(mod.values.grad, dw2) and torch.equal(x.grad, dx2)


def test_winograd_conv2d_optimizer_updates_live_weights():
    from paper_1702_08597_b200.autograd import WinogradConv2d

    rng = np.random.default_rng(3)
    w_f = rng.standard_normal((8, 4, 6, 6)).astype(np.float32).astype(np.float64)
    w_f[np.abs(w_f) < 0.7] = 0.0
    mod = WinogradConv2d(w_f, 9, 9, pad=1, m=4, relu=True)
    opt = torch.optim.SGD(mod.parameters(), lr=0.05)
    x = torch.tensor(rng.standard_normal((3, 4, 9, 9)), dtype=torch.float32, device="cuda")
    before = mod.weight()
    loss = mod(x).square().sum()
    loss.backward()
    g = mod.values.grad.clone()
    opt.step()
    after = mod.weight()
    assert np.all(after[w_f == 0] == 0)  # pruned coordinates do not exist in the parameter
    v0 = np.concatenate(wb.compress(before).values)
    want = (v0.astype(np.float64) - np.float64(np.float32(0.05)) * g.cpu().numpy()).astype(np.float32)
    got = np.concatenate(wb.compress(after).values)
    # torch's fp32 add_(alpha) may fuse: within one fp32 ulp of the exact update
    assert np.abs(got.view(np.int32).astype(np.int64) - want.view(np.int32).astype(np.int64)).max() <= 1
    # the next forward sees the update (CSC / operands refreshed): compare with a fresh layer
    out = mod(x)
    lay = wb.WinogradLayer(4, 8, 9, 9, pad=1, m=4)
    lay.set_weights(after)
    assert torch.equal(out, lay.forward(x, relu=True))


def _nccl():
    import ctypes
    import os
    import site

    try:
        return ctypes.CDLL("libnccl.so.2", mode=os.RTLD_NOLOAD | os.RTLD_NOW)
    except OSError:
        for sp in site.getsitepackages():
            p = os.path.join(sp, "nvidia", "nccl", "lib", "libnccl.so.2")
            if os.path.exists(p):
                return ctypes.CDLL(p, mode=os.RTLD_GLOBAL)
        return ctypes.CDLL("libnccl.so.2", mode=os.RTLD_GLOBAL)


def test_allreduce_dw_over_a_single_rank_communicator():
    """wino_allreduce_dw through a real (one-rank) NCCL communicator: the sum over one rank is the
    identity, in place, on the given stream; the default count is the plan's dW length."""
    import ctypes

    nccl = _nccl()

    class UniqueId(ctypes.Structure):
        _fields_ = [("internal", ctypes.c_char * 128)]

    uid = UniqueId()
    assert nccl.ncclGetUniqueId(ctypes.byref(uid)) == 0
    comm = ctypes.c_void_p()
    nccl.ncclCommInitRank.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, UniqueId, ctypes.c_int]
    assert nccl.ncclCommInitRank(ctypes.byref(comm), 1, uid, 0) == 0
    try:
        cfg = CONFIGS["c0"]
        _, w_f, _ = make_inputs(cfg, n=1)
        layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
        layer.set_weights(w_f)
        g = torch.randn(layer.nnz, device="cuda")
        want = g.clone()
        layer.allreduce_dw(g, comm.value)
        torch.cuda.synchronize()
        assert torch.equal(g, want)
        bucket = torch.randn(3 * layer.nnz, device="cuda")  # a bucket of several layers: explicit count
        want = bucket.clone()
        layer.allreduce_dw(bucket, comm.value, count=bucket.numel())
        torch.cuda.synchronize()
        assert torch.equal(bucket, want)
    finally:
        nccl.ncclCommDestroy(comm)


def test_backward_without_input_gradient():
    cfg = CONFIGS["c0"]
    img, w_f, go = make_inputs(cfg, n=2)
    layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
    layer.set_weights(w_f)
    cache = layer.new_cache(2)
    layer.forward(dev(img), cache)
    dw_ref = layer.backward_weights(dev(go), cache)
    dw, di = layer.backward(dev(go), cache, want_input_grad=False)
    assert di is None and torch.equal(dw, dw_ref)


def test_in_backward_exchange_over_a_torch_nccl_group():
    """wino_set_dw_allreduce with the communicator of a real torch.distributed NCCL group (one
    rank): the exchange runs inside forward_backward / backward on the dW_F stream — eagerly and
    captured in a CUDA graph, as bench.py runs it at N > 1 — and the sum over one rank leaves
    dW_F bit for bit; the stack's per-layer exchange replaces its bucket all-reduce."""
    import os
    import socket

    import torch.distributed as dist

    from paper_1702_08597_b200.graph import GraphedStep
    from paper_1702_08597_b200.stack import WinogradStack

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        cfg = CONFIGS["c0"]
        img, w_f, go = make_inputs(cfg, n=3)
        x, g = dev(img), dev(go)
        ref = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
        ref.set_weights(w_f)
        rc = ref.new_cache(3)
        o0 = torch.empty((3, cfg.k, ref.ho, ref.wo), device="cuda")
        dw0 = torch.empty(ref.grad_w_shape(), device="cuda")
        di0 = torch.empty((3, cfg.c, cfg.h, cfg.w), device="cuda")
        ref.forward_backward(x, g, rc, out=o0, out_w=dw0, out_i=di0)

        lay = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
        lay.set_weights(w_f)
        lay.set_dw_allreduce(dist.group.WORLD)
        cache = lay.new_cache(3)
        o, dw, di = torch.empty_like(o0), torch.empty_like(dw0), torch.empty_like(di0)

        def step():
            lay.forward_backward(x, g, cache, out=o, out_w=dw, out_i=di)

        step()
        torch.cuda.synchronize()
        assert torch.equal(dw, dw0) and torch.equal(di, di0) and torch.equal(o, o0)
        dw.zero_()
        GraphedStep(step).replay()
        torch.cuda.synchronize()
        assert torch.equal(dw, dw0), "graph-captured in-backward exchange changed dW_F"
        dw2, _ = lay.backward(g, cache)
        torch.cuda.synchronize()
        assert torch.equal(dw2, dw0)

        st = WinogradStack([w_f, w_f], cfg.c, cfg.h, cfg.w, pad=1, m=4, n_max=3)
        st.set_dw_allreduce(dist.group.WORLD)
        assert st.in_backward_exchange
        st.forward(x)
        st.backward(g)
        torch.cuda.synchronize()
        assert torch.isfinite(st.bucket.flat).all()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("h,world", [(24, 3), (22, 4)])
def test_tile_split_bands_match_the_whole_layer(h, world):
    """Tile-axis split (dist.py: bands of tile rows, one per rank; here the ranks' bands run one
    after another on the one GPU): every band through the unchanged kernels on its window of the
    zero-padded image (pad=0 plan).  O is bitwise the whole-image layer's rows; the summed dW_F
    (what the all-reduce forms) and the halo-merged dI meet the tolerance against the f64 oracle
    and the whole-image layer."""
    from paper_1702_08597_b200.dist import band_input, band_rows, merge_bands, tile_bands
    from helpers import assert_parity

    rng = np.random.default_rng(h * 10 + world)
    c, k, n, w = 24, 40, 2, 20
    img = rng.standard_normal((n, c, h, w)).astype(np.float32)
    go = rng.standard_normal((n, k, h, w)).astype(np.float32)
    w_f = rng.standard_normal((k, c, 6, 6)) * np.sqrt(2.0 / (9 * c)) * (rng.random((k, c, 6, 6)) >= 0.7)
    whole = wb.WinogradLayer(c, k, h, w, pad=1, m=4)
    whole.set_weights(w_f, dense=False)
    cache = whole.new_cache(n)
    o_ref = whole.forward(dev(img), cache).cpu().numpy()
    dw_ref, di_ref = whole.backward(dev(go), cache)
    dw_ref, di_ref = dw_ref.cpu().numpy().astype(np.float64), di_ref.cpu().numpy()
    bands = tile_bands(h, world)
    x = dev(img)
    o_parts, di_parts, dw_sum = [], [], np.zeros_like(dw_ref)
    for a, b in bands:
        _, rows, o0, on = band_rows(h, a, b)
        if rows == 0:
            di_parts.append(None)
            continue
        lay = wb.WinogradLayer(c, k, rows, w + 2, pad=0, m=4)
        lay.set_weights(w_f, dense=False)
        cb = lay.new_cache(n)
        o_parts.append(lay.forward(band_input(x, a, b), cb).cpu().numpy())
        dw, di = lay.backward(dev(go[:, :, o0:o0 + on, :]), cb)
        dw_sum += dw.cpu().numpy().astype(np.float64)
        di_parts.append(di.clone())
        lay.close()
    assert np.array_equal(np.concatenate(o_parts, axis=2), o_ref), "band O differs from the whole-image O"
    assert_parity(dw_sum, dw_ref, "tile-split dW_F vs whole layer")
    di = merge_bands(di_parts, bands, h).cpu().numpy()
    assert_parity(di, di_ref, "tile-split dI vs whole layer")
    whole.close()
