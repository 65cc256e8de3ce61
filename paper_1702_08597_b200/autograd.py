"""PyTorch operator surface over the C-ABI: the reference's
conv_winograd / conv_winograd_grad (python/bindings.cpp:94-125) as a differentiable module.

`WinogradConv2d` owns one WinogradLayer plan.  Its trainable parameter `values` IS the plan's
live weight buffer on the device (zero-copy, via __cuda_array_interface__), in plan order:
the CSR values of a sparse plan (only unmasked coordinates exist, so an optimizer can never
revive a pruned one — the fine-tune invariant of train.cpp:280), or the slice-major [p·p][K][C]
weights of a dense plan.  In-place optimizer updates are picked up before the next forward
(wino_values_updated refreshes the CSC copy and tensor-core operands).

Forward runs the Winograd layer (optionally with the ReLU fused); backward runs
backward_weights (dW_F on the plan's coordinates) then, if the input needs a gradient,
backward_input — exactly the order layer.cpp:134-138 requires.
"""
from __future__ import annotations

import numpy as np
import torch

from .layer import WinogradLayer


class _DeviceArray:
    """Minimal __cuda_array_interface__ exporter for a raw device pointer."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3, "strides": None}


class _WinogradConvFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, values, mod):
        layer = mod.layer
        mod._sync_values()
        cache = mod._take_cache(x.shape[0]) if any(ctx.needs_input_grad[:2]) else None
        out = layer.forward(x.contiguous(), cache if cache is not None else mod._scratch(x.shape[0]),
                            relu=mod.relu)
        ctx.mod, ctx.cache = mod, cache
        ctx.save_for_backward(out if mod.relu else None)
        return out

    @staticmethod
    @torch.autograd.function.once_differentiable
    def backward(ctx, grad_out):
        mod, cache = ctx.mod, ctx.cache
        (relu_out,) = ctx.saved_tensors
        layer = mod.layer
        dw = layer.backward_weights(grad_out.contiguous(), cache, relu_out=relu_out)
        if layer.is_dense:  # K×C×p×q -> the plan's slice-major order
            dw = dw.permute(2, 3, 0, 1).reshape(-1)
        dx = layer.backward_input(cache)[:cache.n] if ctx.needs_input_grad[0] else None
        mod._give_cache(cache)
        ctx.cache = None
        return dx, dw, None


class WinogradConv2d(torch.nn.Module):
    """3×3 convolution (stride 1, padding `pad`) computed as a Winograd F(m×m, 3×3) layer with
    Winograd-domain weights W_F (K×C×p×p) — sparse (exact zeros pruned) or dense."""

    def __init__(self, w_f, h: int, w: int, pad: int = 1, m: int = 4, dense=None, relu: bool = False,
                 device: int = 0):
        super().__init__()
        w_f = np.asarray(w_f, dtype=np.float64)
        k, c, p, _ = w_f.shape
        self.layer = WinogradLayer(c, k, h, w, pad=pad, m=m, device=device)
        self.layer.set_weights(w_f, dense=dense)
        self.relu = relu
        self._pool: list = []
        self._scratch_cache = None
        self._bind()

    # -- weight buffer aliasing -----------------------------------------------------
    def _bind(self):
        n = self.layer.nnz
        ptr = self.layer.weight_values()
        t = torch.as_tensor(_DeviceArray(ptr, n), device=f"cuda:{self.layer.device}") if n else \
            torch.zeros(0, device=f"cuda:{self.layer.device}")
        self.values = torch.nn.Parameter(t, requires_grad=True)
        self._seen = self.values._version

    def _sync_values(self):
        if self.values._version != self._seen:
            self.layer.values_updated()
            self._seen = self.values._version

    def set_weights(self, w_f, dense=None):
        """Replace W_F (the parameter is re-bound to the new buffer: re-create optimizers)."""
        self.layer.set_weights(np.asarray(w_f, dtype=np.float64), dense=dense)
        self._bind()

    def prune(self, zero_tol: float = 0.0):
        """Keep only nonzero coordinates (on-device recompress); re-binds `values`."""
        self._sync_values()
        self.layer.recompress(zero_tol)
        self._bind()

    def weight(self) -> np.ndarray:
        """W_F as K×C×p×q f64."""
        self._sync_values()
        return self.layer.weights()

    # -- caches -------------------------------------------------------------------
    def _take_cache(self, n):
        for i, c in enumerate(self._pool):
            if c.n_max >= n:
                return self._pool.pop(i)
        return self.layer.new_cache(max(n, 1))

    def _give_cache(self, cache):
        if len(self._pool) < 4:
            self._pool.append(cache)

    def _scratch(self, n):
        if self._scratch_cache is None or self._scratch_cache.n_max < n:
            self._scratch_cache = self.layer.new_cache(max(n, 1))
        return self._scratch_cache

    def forward(self, x):
        if not self.values.requires_grad and not x.requires_grad:
            with torch.no_grad():
                self._sync_values()
                return self.layer.forward(x.contiguous(), self._scratch(x.shape[0]), relu=self.relu)
        return _WinogradConvFn.apply(x, self.values, self)

    def extra_repr(self):
        l_ = self.layer
        return (f"c={l_.c}, k={l_.k}, h={l_.h}, w={l_.w}, pad={l_.pad}, m={l_.m}, nnz={l_.nnz}, "
                f"dense={l_.is_dense}, relu={self.relu}")
