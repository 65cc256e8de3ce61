"""Quick GPU check of the exact dW_F path (wino_xdw.cuh): strict parity against the f64
reference on the golden layers and BASELINE configs, plus step / kernel times.

    python tools/xdw_check.py [--configs c0,c1] [--time c1,c3]
"""
from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

import paper_1702_08597_b200 as wb  # noqa: E402
from helpers import LAYER_CASES, load_layer  # noqa: E402
from paper_1702_08597_b200.synth import CONFIGS, make_inputs, with_sparsity  # noqa: E402
from test_gpu_parity import _f64_batched, run_layer  # noqa: E402


def ratio(got, ref):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    r = np.abs(got - ref) / (1e-5 + 1e-4 * np.abs(ref))
    return int((r > 1).sum()), float(r.max()) if r.size else 0.0


def golden():
    for name in LAYER_CASES:
        d = load_layer(name)
        for dense in ([False, True] if name != "f43_dense" else [True]):
            r = run_layer(d["img"], d["w_f"], d["grad_o"], d["m"], d["pad"], dense=dense)
            mask = d["w_f"] != 0 if not r["layer"].is_dense else np.ones_like(d["w_f"], bool)
            nb, worst = ratio(r["dw"][mask], d["grad_wf_f64"][mask])
            no, wo_ = ratio(r["o"], d["o_f64"])
            ni, wi = ratio(r["di"], d["grad_in_f64"])
            print(f"golden {name:10s} dense={dense!s:5s} dW miss {nb} worst {worst:.3g} | O {no} {wo_:.3g} | "
                  f"dI {ni} {wi:.3g}", flush=True)


def full(cfgname, sparsity=None, sub=None, dense=False):
    cfg = CONFIGS[cfgname] if sparsity is None else with_sparsity(CONFIGS[cfgname], sparsity)
    img, w_f, go = make_inputs(cfg)
    r = run_layer(img, w_f, go, 4, 1, dense=dense)
    if sub is None:
        o, dw, di = _f64_batched(img.astype(np.float64), w_f, go.astype(np.float64), 1)
        mask = w_f != 0
        nb, worst = ratio(r["dw"][mask], dw[mask])
        print(f"{cfgname} sp={cfg.sparsity} dW strict miss {nb}/{mask.sum()} worst {worst:.3g} | "
              f"O {ratio(r['o'], o)} dI {ratio(r['di'], di)}", flush=True)


def timing(cfgname, sparsity=None, steps=20, contraction=None, dense=False):
    cfg = CONFIGS[cfgname] if sparsity is None else with_sparsity(CONFIGS[cfgname], sparsity)
    img, w_f, go = make_inputs(cfg)
    layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
    layer.set_weights(w_f, dense=dense)
    if contraction:
        layer.set_contraction(contraction)
    cache = layer.new_cache(cfg.n)
    x, g = torch.from_numpy(img).cuda(), torch.from_numpy(go).cuda()
    o = torch.empty((cfg.n, cfg.k, cfg.h, cfg.w), device="cuda")
    dw = torch.empty(layer.grad_w_shape(), device="cuda")
    di = torch.empty_like(x)
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    for _ in range(3):
        layer.forward_backward(x, g, cache, out=o, out_w=dw, out_i=di)
    ts = []
    for _ in range(steps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        layer.forward_backward(x, g, cache, out=o, out_w=dw, out_i=di)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    layer.profile(True)
    flush.fill_(1.0)
    torch.cuda.synchronize()
    layer.forward_backward(x, g, cache, out=o, out_w=dw, out_i=di)
    torch.cuda.synchronize()
    prof = layer.profile_read()
    layer.profile(False)
    med = float(np.median(ts))
    eff = 3 * 2.0 * cfg.c * cfg.k * cfg.h * cfg.w * 9 * cfg.n / (med * 1e-3) / 1e12
    ks = ", ".join(f"{k} {v[0] * 1e3:.0f}" for k, v in prof.items() if v[1])
    print(f"time {cfgname} sp={cfg.sparsity} contraction={contraction} dense={dense}: {med * 1e3:.0f} us/step "
          f"({eff:.0f} eff TFLOP/s) | kernels (us, concurrent): {ks}", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--golden", action="store_true")
    ap.add_argument("--full", default="")
    ap.add_argument("--time", default="")
    a = ap.parse_args()
    t0 = time.time()
    if a.golden:
        golden()
    for c in filter(None, a.full.split(",")):
        full(c)
    for c in filter(None, a.time.split(",")):
        name, _, sp = c.partition(":")
        if sp == "dense":
            timing(name, 0.0, dense=True)
        elif sp == "auto":
            timing(name, None, contraction="auto")
        else:
            timing(name, float(sp) if sp else None)
    print(f"done in {time.time() - t0:.0f} s")
