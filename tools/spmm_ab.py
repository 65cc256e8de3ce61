"""A/B of the CSR kernels' operand store on the GPU: TMEM (WINO_OPT_SPMM_OPERANDS forced) vs shared
memory.  For each config: forward O, dW_F and dI of one fwd+bwd step must be bitwise equal between
the two; prints the per-kind times (profiled serial step) of both.

    python tools/spmm_ab.py [c1 c2:0.9 c3:0.9 ...]
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1702_08597_b200 as wb  # noqa: E402
from paper_1702_08597_b200.synth import CONFIGS, make_inputs, with_sparsity  # noqa: E402


def run(cfg, where):
    img, w_f, go = make_inputs(cfg)
    lay = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=cfg.pad, m=cfg.m, device=0)
    lay.set_weights(w_f, dense=False)
    lay.set_spmm_operands(where)
    x = torch.from_numpy(img).cuda()
    g = torch.from_numpy(go).cuda()
    cache = lay.new_cache(cfg.n) if cfg.backward else None
    out = lay.forward(x, cache)
    dw = di = None
    if cfg.backward:
        dw = lay.backward_weights(g, cache)
        di = lay.backward_input(cache)
    torch.cuda.synchronize()
    res = [t.cpu().numpy() for t in (out, dw, di) if t is not None]
    flush = torch.empty(64 << 20, device="cuda")
    lay.profile(True)
    for _ in range(3):
        flush.zero_()
        lay.forward(x, cache)
        if cfg.backward:
            lay.backward_weights(g, cache)
            lay.backward_input(cache)
    torch.cuda.synchronize()
    prof = lay.profile_read()
    lay.profile(False)
    lay.close()
    return res, {k: v[0] / 3 * 1e3 for k, v in prof.items() if k.startswith("spmm")}


def main():
    names = sys.argv[1:] or ["c1", "c2:0.9", "c3:0.9", "c3:0.5", "c3:0.95"]
    ok = True
    for nm in names:
        base, _, sp = nm.partition(":")
        cfg = CONFIGS[base]
        if sp:
            cfg = with_sparsity(cfg, float(sp))
        a, ta = run(cfg, "tmem")
        b, tb = run(cfg, "smem")
        c, tc = run(cfg, "hybrid")
        same = all(np.array_equal(x, y) for x, y in zip(a, b)) and all(np.array_equal(x, y) for x, y in zip(c, b))
        ok &= same
        print(f"{nm:8s} bitwise={'yes' if same else 'NO'}  tmem {ta}  smem {tb}  hybrid {tc}", flush=True)
    sys.exit(0 if ok or os.environ.get("SPMM_AB_NOFAIL") else 1)


if __name__ == "__main__":
    main()
