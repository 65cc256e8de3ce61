"""Batched training step of a stack of Winograd layers (BASELINE configs[4]).

The reference trainer runs one sample at a time (train.cpp:167) through run_forward
(conv -> ReLU per layer, train.cpp:66-87) and the backward chain (relu-mask multiply,
backward_weights, Σ_n·(1/B), backward_input for l > 0; train.cpp:189-211), then the masked
SGD update of train_step (train.cpp:281-290).  Here one call per layer and minibatch does the
same on the device: ReLU is fused into the output-transform epilogue, the mask into the dZ
kernel, dW_F of all layers lands in one GradBucket that is all-reduced once (data parallel; or,
with set_dw_allreduce, each layer's slice is summed inside its own backward, overlapping its dI chain),
and the update runs on the live CSR values (masked coordinates do not exist in the CSR, so
they stay exactly zero — the fine-tune invariant check_masks enforces, train.cpp:340-347).
"""
from __future__ import annotations

import numpy as np

from .dist import GradBucket
from .layer import WinogradLayer


class WinogradStack:
    def __init__(self, weights, c, h, w, pad=1, m=4, device=0, n_max=1, dense=False):
        """weights: list of K×C×p×p W_F arrays.  dense=False: exact zeros are pruned (masked)
        coordinates — the fine-tune network.  dense=True: every coordinate is trainable — the
        pruning phase (StepMode::prune); prune_to_sparse() then keeps the survivors."""
        import torch

        self.device = device
        self.layers = []
        self.caches = []
        cin = c
        for w_f in weights:
            w_f = np.asarray(w_f)
            lay = WinogradLayer(cin, w_f.shape[0], h, w, pad=pad, m=m, device=device)
            lay.set_weights(w_f, dense=dense if isinstance(dense, str) else bool(dense))
            self.layers.append(lay)
            self.caches.append(lay.new_cache(n_max))
            cin = w_f.shape[0]
            h, w = lay.ho, lay.wo
        self._alloc_bucket()
        self.n_max = n_max
        self.outs = [None] * len(self.layers)
        self.dis = [None] * len(self.layers)
        self._torch = torch
        self.in_backward_exchange = False

    def _alloc_bucket(self):
        self.bucket = GradBucket.allocate([lay.nnz for lay in self.layers], device=f"cuda:{self.device}")
        self.grads = [v.view(lay.grad_w_shape()) for v, lay in zip(self.bucket.views, self.layers)]

    def set_dw_allreduce(self, comm=None):
        """Move the data-parallel exchange into the backward: every layer sums its own dW_F over
        `comm` (an NCCL process group or ncclComm_t address; None: back to the one bucketed
        all-reduce after the backward) right after its dW_F kernels, overlapping that layer's dI
        chain (WinogradLayer.set_dw_allreduce).  step() then skips the bucket all-reduce."""
        for lay in self.layers:
            lay.set_dw_allreduce(comm)
        self.in_backward_exchange = comm is not None

    def forward(self, x):
        """run_forward (train.cpp:66-87): conv -> ReLU for every layer; returns the last output."""
        cur = x
        for i, (lay, cache) in enumerate(zip(self.layers, self.caches)):
            if self.outs[i] is None or self.outs[i].shape[0] != cur.shape[0]:
                self.outs[i] = self._torch.empty((cur.shape[0], lay.k, lay.ho, lay.wo), device=cur.device)
            cur = lay.forward(cur, cache, relu=True, out=self.outs[i])
        return cur

    def backward(self, grad_out, serial: bool = False):
        """The backward chain of minibatch_grad (train.cpp:189-211) for the whole minibatch:
        fills the gradient bucket with Σ_n dW_F per layer; no dI for layer 0 (train.cpp:201).
        serial=True runs dW_F and dI one after the other (same results; per-kernel timing)."""
        g = grad_out
        for i in range(len(self.layers) - 1, -1, -1):
            lay, cache = self.layers[i], self.caches[i]
            if i > 0:  # dW_F concurrently with dI (wino_backward)
                if self.dis[i] is None or self.dis[i].shape[0] != g.shape[0]:
                    self.dis[i] = self._torch.empty((g.shape[0], lay.c, lay.h, lay.w), device=g.device)
                if serial:
                    lay.backward_weights(g, cache, relu_out=self.outs[i], out=self.grads[i])
                    g = lay.backward_input(cache, out=self.dis[i])
                else:
                    _, g = lay.backward(g, cache, relu_out=self.outs[i], out_w=self.grads[i], out_i=self.dis[i])
            else:
                lay.backward_weights(g, cache, relu_out=self.outs[i], out=self.grads[i])
        return self.bucket

    def step(self, x, grad_out, lr, n_global, l2=0.0, group=None, mode=None, lmbda=0.0, norm=1,
             eps=0.0, beta=0.0):
        """One data-parallel training step: forward, backward, ONE all-reduce of the bucket,
        then the update of train_step (train.cpp:255-290) with the 1/B scaling of
        train.cpp:166,200.  mode=None: masked SGD with L2 factor l2 (the fine-tune step).
        'prune': λ‖w‖_norm regulariser + the gradient threshold (ε, β).  'finetune': λ‖w‖₂.
        'train': λ‖w‖_norm without threshold."""
        self.forward(x)
        self.backward(grad_out)
        if not self.in_backward_exchange:
            self.bucket.allreduce(group)
        scale = 1.0 / float(n_global)
        for lay, g in zip(self.layers, self.grads):
            if mode is None:
                lay.sgd_step(g, lr=lr, scale=scale, l2=l2)
            elif mode in ("prune", "finetune", "train"):
                lay.update(g, lr=lr, scale=scale, lmbda=lmbda, norm=2 if mode == "finetune" else norm,
                           prune=mode == "prune", eps=eps, beta=beta)
            else:
                raise ValueError(f"unknown mode {mode!r}")

    def check_finite(self):
        """TrainingError if any layer's update diverged since the last check (synchronizes)."""
        for i, lay in enumerate(self.layers):
            lay.check_finite(f"conv{i + 1}")

    def prune_to_sparse(self, zero_tol=0.0):
        """After the pruning phase: every layer keeps only its nonzero coordinates (the masks of
        set_masks_from_zeros, train.cpp:322-330), re-derived on the device; the gradient
        bucket shrinks to the new nnz."""
        for lay in self.layers:
            lay.recompress(zero_tol)
        self._alloc_bucket()

    def densities(self):
        return [lay.nnz / float(lay.k * lay.c * lay.p * lay.p) for lay in self.layers]

    def launch_count(self):
        return sum(lay.launch_count() for lay in self.layers)
