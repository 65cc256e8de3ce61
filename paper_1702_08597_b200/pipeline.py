"""Host-buffer layer step with transfers overlapped against compute.

The reference API takes host tensors and returns host tensors (layer.hpp:28-43).  On a GPU
the copies over PCIe dominate a small layer, so `HostStep` runs one fwd+bwd step from pinned
host buffers with three streams:

    copy-in : I  ──┐            dO ───────────────┐
    compute :      └─► forward ──► backward_weights ─► backward_input ──┐
    copy-out:                 └─► O        └─► dW_F                     └─► dI

i.e. dO uploads while the forward runs, O downloads during backward_weights, dW_F during
backward_input.  Forward and backward are each captured as a CUDA graph (one launch each).
"""
from __future__ import annotations


class HostStep:
    def __init__(self, layer, cache, x, grad_o, out, grad_w, grad_in, graphs: bool = True):
        """x, grad_o, out, grad_w, grad_in: the layer's fixed device buffers."""
        import torch

        self.layer, self.cache = layer, cache
        self.x, self.g, self.o, self.dw, self.di = x, grad_o, out, grad_w, grad_in
        self.s_in = torch.cuda.Stream()
        self.s_out = torch.cuda.Stream()
        self.ev = {k: torch.cuda.Event() for k in ("x", "g", "fwd", "bw", "bi", "o", "dw", "di")}

        def fwd():
            layer.forward(x, cache, out=out)

        def bwd_w():
            layer.backward_weights(grad_o, cache, out=grad_w)

        def bwd_i():
            layer.backward_input(cache, out=grad_in)

        self.fwd, self.bwd_w, self.bwd_i = fwd, bwd_w, bwd_i
        if graphs:
            from .graph import GraphedStep

            self.fwd = GraphedStep(fwd).replay
            self.bwd_w = GraphedStep(bwd_w).replay
            self.bwd_i = GraphedStep(bwd_i).replay

    def __call__(self, h_x, h_g, h_o, h_dw, h_di):
        """One step from pinned host inputs into pinned host outputs (asynchronous; call
        torch.cuda.synchronize() or .wait() on the returned event before reading)."""
        import torch

        main = torch.cuda.current_stream()
        ev = self.ev
        # the step starts after everything already queued on the caller's stream (the previous
        # step, a timing event): inputs are never overwritten while still being read
        self.s_in.wait_stream(main)
        with torch.cuda.stream(self.s_in):
            self.x.copy_(h_x, non_blocking=True)
            ev["x"].record()
            self.g.copy_(h_g, non_blocking=True)
            ev["g"].record()
        main.wait_event(ev["x"])
        self.fwd()
        ev["fwd"].record(main)
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(ev["fwd"])
            h_o.copy_(self.o, non_blocking=True)
            ev["o"].record()
        main.wait_event(ev["g"])
        self.bwd_w()
        ev["bw"].record(main)
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(ev["bw"])
            h_dw.copy_(self.dw, non_blocking=True)
            ev["dw"].record()
        self.bwd_i()
        ev["bi"].record(main)
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(ev["bi"])
            h_di.copy_(self.di, non_blocking=True)
            ev["di"].record()
        main.wait_stream(self.s_out)  # the caller's stream sees the whole step (downloads included)
        return ev["di"]
