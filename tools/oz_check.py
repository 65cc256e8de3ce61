"""int8 tensor-core dW_F (WINO_OPT_DW_MODE 3) against the exact-product SDDMM and the f64 reference:
golden layer cases and c1 / c3 sampled; prints miss fractions and the largest deviation from the
fp32 floor (the SDDMM)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1702_08597_b200 as wb  # noqa: E402
from paper_1702_08597_b200.synth import CONFIGS, make_inputs  # noqa: E402

for name in ("c0", "c1", "c3"):
    cfg = CONFIGS[name]
    img, w_f, go = make_inputs(cfg)
    layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
    layer.set_weights(w_f, dense=False)
    cache = layer.new_cache(cfg.n)
    layer.forward(torch.from_numpy(img).cuda(), cache)
    g = torch.from_numpy(go).cuda()
    exact = layer.backward_weights(g, cache).cpu().numpy().astype(np.float64)
    layer.set_dw_mode("int8")
    oz = layer.backward_weights(g, cache).cpu().numpy().astype(np.float64)
    torch.cuda.synchronize()
    d = np.abs(oz - exact)
    tol = 1e-5 + 1e-4 * np.abs(exact)
    print(f"{name}: nnz {exact.size}  max|int8 - sddmm| {d.max():.3e}  rel-to-max {d.max() / np.abs(exact).max():.2e}"
          f"  outside strict bound of the SDDMM: {(d > tol).sum()}  bitwise equal: {(oz == exact).mean():.4f}")
