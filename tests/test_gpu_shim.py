"""The drop-in at the reference's own C++ API: shim/layer_cuda.cpp compiled in place of the
reference's src/layer.cpp (shim/_build/libwino_refapi_cuda.so).  The reference types and calls
(wino::Tensor, winograd_forward/_backward_*, compress<float> + sparse_forward<float>) run on the
GPU through the C-ABI and are compared with the reference itself on the CPU (oracle/_ref)."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np
import pytest

from helpers import LAYER_CASES, assert_parity, load_layer
from oracle import ref

SHIM = Path(__file__).resolve().parents[1] / "shim" / "_build" / "libwino_refapi_cuda.so"
_d = C.POINTER(C.c_double)


def _lib():
    if not SHIM.exists():
        pytest.skip("shim/_build not built (needs /root/reference at build time)")
    lib = C.CDLL(str(SHIM))
    lib.shim_last_error.restype = C.c_char_p
    lib.shim_gpu_call_count.restype = C.c_longlong
    return lib


def _p(a):
    return None if a is None else a.ctypes.data_as(_d)


def test_shim_library_exports_the_test_entry_points():
    lib = _lib()
    for name in ("shim_layer", "shim_sparse_forward", "shim_backward_input_without_grad_z",
                 "shim_train_steps", "shim_last_error", "shim_gpu_call_count"):
        assert hasattr(lib, name)


@pytest.mark.gpu
@pytest.mark.parametrize("name", LAYER_CASES)
def test_reference_layer_api_on_the_gpu_matches_the_reference(name):
    lib = _lib()
    d = load_layer(name)
    m, pad = d["m"], d["pad"]
    img = np.pad(d["img"][0].astype(np.float64), ((0, 0), (pad, pad), (pad, pad)))
    w_f = np.ascontiguousarray(d["w_f"], dtype=np.float64)
    go = np.ascontiguousarray(d["grad_o"][0], dtype=np.float64)
    c, h_i, w_i = img.shape
    k = w_f.shape[0]
    want = ref.layer(img, w_f, go, m=m)
    o = np.zeros_like(want["o"])
    gw = np.zeros_like(want["grad_wf"])
    gi = np.zeros_like(want["grad_in"])
    before = lib.shim_gpu_call_count()
    rc = lib.shim_layer(m, c, h_i, w_i, k, _p(img), _p(w_f), _p(go), _p(o), _p(gw), _p(gi))
    assert rc == 0, lib.shim_last_error().decode()
    assert lib.shim_gpu_call_count() - before == 3  # forward, backward_weights, backward_input
    assert_parity(o, want["o"], f"{name}: O through the reference API")
    assert_parity(gw, want["grad_wf"], f"{name}: dW_F through the reference API")
    assert_parity(gi, want["grad_in"], f"{name}: dI through the reference API")


@pytest.mark.gpu
@pytest.mark.parametrize("name", LAYER_CASES)
def test_reference_sparse_forward_on_the_gpu_is_bitwise_the_reference(name):
    lib = _lib()
    d = load_layer(name)
    m, pad = d["m"], d["pad"]
    batch = np.pad(d["img"].astype(np.float64), ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    w_f = np.ascontiguousarray(d["w_f"], dtype=np.float64)
    n, c, h_i, w_i = batch.shape
    k = w_f.shape[0]
    want = ref.sparse_forward(batch, w_f, m=m, workers=1, precision=32)
    out = np.zeros_like(want)
    before = lib.shim_gpu_call_count()
    rc = lib.shim_sparse_forward(m, n, c, h_i, w_i, k, _p(batch), _p(w_f), _p(out))
    assert rc == 0, lib.shim_last_error().decode()
    assert lib.shim_gpu_call_count() - before == 1
    assert np.array_equal(out, want)


@pytest.mark.gpu
def test_reference_consistency_error_through_the_shim():
    lib = _lib()
    d = load_layer("c0")
    img = np.pad(d["img"][0].astype(np.float64), ((0, 0), (1, 1), (1, 1)))
    w_f = np.ascontiguousarray(d["w_f"], dtype=np.float64)
    c, h_i, w_i = img.shape
    rc = lib.shim_backward_input_without_grad_z(4, c, h_i, w_i, w_f.shape[0], _p(img), _p(w_f))
    assert rc == 2 and b"dL/dZ missing" in lib.shim_last_error()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1])
def test_reference_trainer_runs_on_the_gpu(mode):
    """The reference's own train_step (train.cpp:255-290) on its toy Winograd network: every
    winograd_forward/_backward_* it makes lands on the GPU through the shim, and the minibatch
    losses follow the all-f64 CPU run (mode 1 = prune: L1 + gradient thresholding)."""
    lib = _lib()
    steps, batch = 6, 8
    want = ref.train_steps(3, steps, batch, mode)
    got = np.zeros(steps)
    before = lib.shim_gpu_call_count()
    rc = lib.shim_train_steps(C.c_ulonglong(3), steps, batch, mode, _p(got))
    assert rc == 0, lib.shim_last_error().decode()
    calls = lib.shim_gpu_call_count() - before
    assert calls >= steps * batch * 2 * 2  # ≥ forward + backward_weights per conv layer per sample
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-6)


# -- the reference's own pybind11 module (python/bindings.cpp) built over the shim ----------------
def _module():
    import importlib
    import sys

    build = str(SHIM.parent)
    if not any(p.name.startswith("_wino") for p in SHIM.parent.glob("_wino*.so")):
        pytest.skip("shim/_build/_wino not built")
    if build not in sys.path:
        sys.path.insert(0, build)
    return importlib.import_module("_wino")


@pytest.mark.gpu
def test_reference_python_module_on_the_gpu():
    """bindings.cpp unchanged, its layer calls served by the GPU: conv_winograd against the
    reference's direct convolution, conv_winograd_grad and sparse_conv against the reference on
    the CPU, worker-count invariance, and the reference's error mapping."""
    wino = _module()
    rng = np.random.default_rng(0)
    img = rng.standard_normal((3, 9, 11))
    w = rng.standard_normal((2, 3, 3, 3))
    for m in (2, 4):
        w_f = wino.lift(w, m=m)
        np.testing.assert_allclose(wino.conv_winograd(img, w_f, m=m), wino.conv_direct(img, w), atol=1e-4)
    img = rng.standard_normal((2, 10, 10))
    w_f = rng.standard_normal((3, 2, 6, 6))
    go = rng.standard_normal((3, 8, 8))
    gw, gi = wino.conv_winograd_grad(img, w_f, go, m=4)
    want = ref.layer(img, w_f, go, m=4)
    assert_parity(gw, want["grad_wf"], "module dW_F")
    assert_parity(gi, want["grad_in"], "module dI")
    batch = rng.standard_normal((3, 2, 10, 10))
    w_f[np.abs(w_f) < 0.8] = 0.0
    out = wino.sparse_conv(batch, w_f, m=4, workers=1, precision="f32")  # GPU (the shim)
    assert np.array_equal(out, wino.sparse_conv(batch, w_f, m=4, workers=4, precision="f32"))
    assert np.array_equal(out, ref.sparse_forward(batch, w_f, m=4, workers=1, precision=32))
    # the module's default precision is f64: sparse_forward<double> is served by the GPU too (fp32
    # arithmetic, f64 values cast at the edge like winograd_forward): within north_star's tolerance
    # of the reference's f64 result
    assert_parity(wino.sparse_conv(batch, w_f, m=4), ref.sparse_forward(batch, w_f, m=4, precision=64),
                  "module sparse_conv f64")
    with pytest.raises(ValueError):
        wino.conv_winograd(rng.standard_normal((4, 10, 10)), w_f, m=4)


@pytest.mark.gpu
def test_reference_acceptance_gate_on_the_gpu():
    """The reference's own acceptance gate (tests/acceptance.cpp, unmodified) linked against the
    shim: its winograd_forward and sparse_forward<double> calls run on the GPU.  Criteria 3
    (sparse == dense across densities, bitwise worker-stable), 4 (16 multiplications per
    (tile, c, k) from the OpCounter) and 9 (multiplication ratio <= 0.12 and sparse faster than
    dense) must pass.  Criteria 1-2 pin 1e-10 absolute / 1e-6 finite-difference tolerances that
    only an f64 layer meets (the B200 layer computes in fp32); they are reported, not asserted."""
    import subprocess

    exe = SHIM.parent / "acceptance_cuda"
    if not exe.exists():
        pytest.skip("shim/_build/acceptance_cuda not built")
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    lines = {ln.split(":")[0].split()[-1]: ln for ln in out.stdout.splitlines() if ln.startswith(("PASS", "FAIL"))}
    print(out.stdout)
    for c in ("criterion-3", "criterion-4", "criterion-9"):
        assert c in lines and lines[c].startswith("PASS"), lines.get(c, out.stdout[-2000:])
