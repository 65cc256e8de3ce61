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


class PipelinedHostStep:
    """HostStep with the batch cut into image chunks so every transfer overlaps compute:

        copy-in : I0 dO0 I1 dO1 I2 dO2 ...
        compute :    f0 b0   f1 b1   f2 b2 ...            dW (whole batch)
        copy-out:       O0 dI0  O1 dI1  O2 dI2 ...              dW

    forward_range / backward_range run the CSR kernels on each chunk's columns of the one batch
    cache; dW_F runs once over the whole batch, so results are bitwise those of HostStep.
    The step is PCIe-bound (H2D ≈ D2H ≈ 55 GB/s on the B200 box): chunking hides all compute but
    the last chunk's behind the transfers."""

    def __init__(self, layer, cache, x, grad_o, out, grad_w, grad_in, chunks=4, relu: bool = False):
        import torch

        self.layer, self.cache = layer, cache
        self.x, self.g, self.o, self.dw, self.di = x, grad_o, out, grad_w, grad_in
        self.relu = relu
        n = x.shape[0]
        t = layer.geometry["t"]
        # chunk boundaries: image counts with n0·T a multiple of 4 (16-byte column alignment)
        step = 1
        while (step * t) % 4:
            step += 1
        if chunks == "auto":
            # large uploads (>= 64 MB per tensor): equal chunks, then a shrinking tail (3u x4, 2u, u, u
            # with u = n/16), so little work is left once the last upload lands (c3: 10.07 vs 10.44 ms
            # with 4 equal chunks; both directions together run at ~80% of either alone, so the
            # copy-only floor is 9.3 ms); small batches: 4 equal chunks (measured best at c1)
            u = n // 16
            big = x.numel() * x.element_size() >= (64 << 20)
            chunks = [3 * u] * 4 + [2 * u, u, u] if big and n % 16 == 0 and u % step == 0 else 4
        if isinstance(chunks, (list, tuple)):
            # explicit image counts (each a multiple of `step`, summing to n): e.g. large chunks
            # first and small ones last, so little work is left after the last upload lands
            if sum(chunks) != n or any(c <= 0 or c % step for c in chunks):
                raise ValueError(f"chunk sizes must be positive multiples of {step} summing to {n}")
            edges = [0]
            for c in chunks:
                edges.append(edges[-1] + c)
            self.bounds = list(zip(edges[:-1], edges[1:]))
        else:
            per = max(step, -(-n // chunks) // step * step or step)
            self.bounds = [(a, min(n, a + per)) for a in range(0, n, per)]
        self.s_in = torch.cuda.Stream()
        self.s_out = torch.cuda.Stream()
        nb = len(self.bounds)
        E = torch.cuda.Event
        self.ev_x = [E() for _ in range(nb)]
        self.ev_g = [E() for _ in range(nb)]
        self.ev_f = [E() for _ in range(nb)]
        self.ev_b = [E() for _ in range(nb)]
        self.ev_w = E()
        self.ev_done = E()

    def __call__(self, h_x, h_g, h_o, h_dw, h_di):
        import torch

        main = torch.cuda.current_stream()
        lay, cache, n = self.layer, self.cache, self.x.shape[0]
        self.s_in.wait_stream(main)
        with torch.cuda.stream(self.s_in):
            for i, (a, b) in enumerate(self.bounds):
                self.x[a:b].copy_(h_x[a:b], non_blocking=True)
                self.ev_x[i].record()
                self.g[a:b].copy_(h_g[a:b], non_blocking=True)
                self.ev_g[i].record()
        self.s_out.wait_stream(main)
        for i, (a, b) in enumerate(self.bounds):
            main.wait_event(self.ev_x[i])
            lay.forward_range(self.x[a:b], n, a, cache, self.o[a:b], relu=self.relu)
            self.ev_f[i].record(main)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(self.ev_f[i])
                h_o[a:b].copy_(self.o[a:b], non_blocking=True)
            main.wait_event(self.ev_g[i])
            lay.backward_range(self.g[a:b], a, cache, self.di[a:b],
                               relu_part=self.o[a:b] if self.relu else None)
            self.ev_b[i].record(main)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(self.ev_b[i])
                h_di[a:b].copy_(self.di[a:b], non_blocking=True)
        lay.backward_weights_cached(cache, out=self.dw)
        self.ev_w.record(main)
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(self.ev_w)
            h_dw.copy_(self.dw, non_blocking=True)
            self.ev_done.record()
        main.wait_stream(self.s_out)
        return self.ev_done
