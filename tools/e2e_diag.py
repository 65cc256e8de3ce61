"""Diagnostics of the pipelined host step (default c1; `python tools/e2e_diag.py c3:0.9`): times (CUDA events) of copy-only, compute-only and
full variants, each captured as a CUDA graph."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1702_08597_b200 as wb  # noqa: E402
from paper_1702_08597_b200.graph import GraphedStep  # noqa: E402
from paper_1702_08597_b200.pipeline import PipelinedHostStep  # noqa: E402
from paper_1702_08597_b200.synth import CONFIGS, make_inputs, with_sparsity  # noqa: E402

_nm, _, _sp = (sys.argv[1] if len(sys.argv) > 1 else "c1").partition(":")
cfg = CONFIGS[_nm]
if _sp:
    cfg = with_sparsity(cfg, float(_sp))
img, w_f, go = make_inputs(cfg)
n = cfg.n
layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
layer.set_weights(w_f, dense=False)
cache = layer.new_cache(n)
x, g = torch.from_numpy(img).cuda(), torch.from_numpy(go).cuda()
o = torch.empty((n, cfg.k, layer.ho, layer.wo), device="cuda")
dw = torch.empty((layer.nnz,), device="cuda")
di = torch.empty_like(x)
h = [torch.from_numpy(a).pin_memory() for a in (img, go)]
outs = [torch.empty(t.shape).pin_memory() for t in (o, dw, di)]
flush = torch.empty(64 * 1024 * 1024, device="cuda")


def timeit(fn, k=20):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    for a, b in ev:
        flush.zero_()
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    print(f"    [min {ts[0]:.0f} median {ts[k // 2]:.0f} mean {sum(ts) / k:.0f} max {ts[-1]:.0f} us]")
    return ts[k // 2]


for chunks in (1, 2, 4, 8) if cfg.n < 64 else (1, 4, 8, [16, 16, 16, 8, 4, 4], [12, 12, 12, 12, 8, 4, 4], [8] * 7 + [4, 4]):
    ps = PipelinedHostStep(layer, cache, x, g, o, dw, di, chunks=chunks)
    full = GraphedStep(lambda: ps(h[0], h[1], *outs)).replay
    print(f"chunks {chunks}: full {timeit(full):.0f} us")

s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()


def copies():
    m = torch.cuda.current_stream()
    s_in.wait_stream(m)
    s_out.wait_stream(m)
    with torch.cuda.stream(s_in):
        x.copy_(h[0], non_blocking=True)
        g.copy_(h[1], non_blocking=True)
    with torch.cuda.stream(s_out):
        outs[0].copy_(o, non_blocking=True)
        outs[1].copy_(dw, non_blocking=True)
        outs[2].copy_(di, non_blocking=True)
    m.wait_stream(s_in)
    m.wait_stream(s_out)


print(f"copies only (H2D ∥ D2H): {timeit(GraphedStep(copies).replay):.0f} us")


def h2d():
    x.copy_(h[0], non_blocking=True)
    g.copy_(h[1], non_blocking=True)


def d2h():
    outs[0].copy_(o, non_blocking=True)
    outs[1].copy_(dw, non_blocking=True)
    outs[2].copy_(di, non_blocking=True)


print(f"H2D only: {timeit(GraphedStep(h2d).replay):.0f} us, D2H only: {timeit(GraphedStep(d2h).replay):.0f} us")


def compute():
    layer.forward(x, cache, out=o)
    layer.backward(g, cache, out_w=dw, out_i=di)


print(f"compute only: {timeit(GraphedStep(compute).replay):.0f} us")
ps = PipelinedHostStep(layer, cache, x, g, o, dw, di, chunks=4)


def in_then_out():
    m = torch.cuda.current_stream()
    s_in.wait_stream(m)
    s_out.wait_stream(m)
    e = torch.cuda.Event()
    with torch.cuda.stream(s_in):
        x.copy_(h[0], non_blocking=True)
        e.record()
        g.copy_(h[1], non_blocking=True)
    with torch.cuda.stream(s_out):
        s_out.wait_event(e)
        outs[0].copy_(o, non_blocking=True)
        outs[2].copy_(di, non_blocking=True)
    m.wait_stream(s_in)
    m.wait_stream(s_out)


print(f"copies, D2H starting after the first H2D tensor: {timeit(GraphedStep(in_then_out).replay):.0f} us")


def ranges_only():
    for i, (a, b) in enumerate(ps.bounds):
        layer.forward_range(x[a:b], n, a, cache, o[a:b])
        layer.backward_range(g[a:b], a, cache, di[a:b])
    layer.backward_weights_cached(cache, out=dw)


print(f"range kernels only (4 chunks): {timeit(GraphedStep(ranges_only).replay):.0f} us")
