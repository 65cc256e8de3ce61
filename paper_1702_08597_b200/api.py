"""The reference's Python surface (python/bindings.cpp:55-204, python/wino/__init__.py)
served by the B200 kernels.

Same names, argument meaning and error classes as the reference module `wino`:
    gen_transforms, lift, conv_winograd, conv_winograd_grad, sparse_conv, density
Inputs/outputs are numpy f64 host arrays as in the reference; the work runs on the GPU
in fp32 (the C-ABI's storage and compute type).  There is no CPU fallback: without the
built library or a CUDA device these raise.
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .layer import WinogradLayer, transforms

ShapeError = _lib.ShapeError
CapabilityError = _lib.CapabilityError
ConsistencyError = _lib.ConsistencyError
CorruptFormatError = _lib.CorruptFormatError


def _square(m, n, r, s):
    n = n or m
    s = s or r
    if n != m or s != r:
        raise CapabilityError(f"only square tiles/kernels are built (m={m}, n={n}, r={r}, s={s})")
    return m, r


def gen_transforms(m: int = 2, n: int = 0, r: int = 3, s: int = 0) -> dict:
    """bindings.cpp:59-73."""
    m, r = _square(m, n, r, s)
    a, b, g = transforms(m, r)
    return {"A1": a, "A2": a.copy(), "B1": b, "B2": b.copy(), "G1": g, "G2": g.copy()}


def lift(weights, m: int = 2, n: int = 0):
    """bindings.cpp:75-84: spatial K×C×r×s -> Winograd-domain K×C×p×q (G1·W·G2ᵀ, layer.cpp:29-43)."""
    w = np.asarray(weights, dtype=np.float64)
    if w.ndim != 4:
        raise ShapeError("expected K x C x r x s spatial weights")
    m, r = _square(m, n, w.shape[2], w.shape[3])
    _, _, g = transforms(m, r)
    return np.einsum("iu,kcuv,jv->kcij", g, w, g)


def _weights_transform(w_f, m, n):
    """bindings.cpp:46-51."""
    if w_f.ndim != 4:
        raise ShapeError("expected K x C x p x q Winograd weights")
    p, q = w_f.shape[2], w_f.shape[3]
    n = n or m
    if p < m or q < n:
        raise ShapeError("tile larger than the Winograd weight extent")
    return _square(m, n, p - m + 1, q - n + 1)


def _to_dev(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def conv_winograd(image, weights_winograd, m: int = 2, n: int = 0):
    """bindings.cpp:94-106: forward of one C×H×W image (no padding: the caller pads)."""
    img = np.asarray(image, dtype=np.float64)
    w_f = np.asarray(weights_winograd, dtype=np.float64)
    if img.ndim != 3:
        raise ShapeError("expected a C x H x W image")
    m, r = _weights_transform(w_f, m, n)
    if w_f.shape[1] != img.shape[0]:
        raise ShapeError(f"winograd_forward: weights expect {w_f.shape[1]} channels, image has {img.shape[0]}")
    layer = WinogradLayer(img.shape[0], w_f.shape[0], img.shape[1], img.shape[2], pad=0, m=m, r=r)
    layer.set_weights(w_f, dense="exact")
    out = layer.forward(_to_dev(img[None]))
    return out[0].double().cpu().numpy()


def conv_winograd_grad(image, weights_winograd, grad_output, m: int = 2, n: int = 0):
    """bindings.cpp:108-125: (dL/dW_F over every coordinate, dL/dI) for upstream dL/dO."""
    img = np.asarray(image, dtype=np.float64)
    w_f = np.asarray(weights_winograd, dtype=np.float64)
    if img.ndim != 3:
        raise ShapeError("expected a C x H x W image")
    m, r = _weights_transform(w_f, m, n)
    layer = WinogradLayer(img.shape[0], w_f.shape[0], img.shape[1], img.shape[2], pad=0, m=m, r=r)
    layer.set_weights(w_f, dense="exact")
    go = np.asarray(grad_output, dtype=np.float64)
    if go.shape != (w_f.shape[0], layer.ho, layer.wo):
        raise ShapeError(f"backward_weights: upstream gradient {go.shape} does not match output "
                         f"{(w_f.shape[0], layer.ho, layer.wo)}")
    cache = layer.new_cache(1)
    layer.forward(_to_dev(img[None]), cache)
    gw = layer.backward_weights(_to_dev(go[None]), cache)
    gi = layer.backward_input(cache)
    return gw.double().cpu().numpy(), gi[0].double().cpu().numpy()


def sparse_conv(batch, weights_winograd, m: int = 2, n: int = 0, workers: int = 1,
                precision: str = "f32"):
    """bindings.cpp:127-146: sparse inference over an N×C×H×W batch; exact zeros skipped.
    `workers` is accepted for signature compatibility (the GPU result does not depend on it,
    as the reference's does not, sparse.hpp:77-78).  Only precision='f32' exists on the GPU."""
    b = np.asarray(batch, dtype=np.float64)
    w_f = np.asarray(weights_winograd, dtype=np.float64)
    if b.ndim != 4:
        raise ShapeError("expected an N x C x H x W batch")
    if precision not in ("f32", "f64"):
        raise ValueError("precision must be f32 or f64")
    if precision != "f32":
        raise CapabilityError("the B200 path stores and computes in fp32 (precision='f32')")
    m, r = _weights_transform(w_f, m, n)
    layer = WinogradLayer(b.shape[1], w_f.shape[0], b.shape[2], b.shape[3], pad=0, m=m, r=r)
    layer.set_weights(w_f, dense=False)
    return layer.forward(_to_dev(b)).double().cpu().numpy()


def density(weights) -> float:
    """bindings.cpp:148-156."""
    w = np.asarray(weights, dtype=np.float64)
    return float(np.count_nonzero(w)) / float(w.size)
