"""One forward of a config with a chosen CSR operand store (for ncu captures of K2).

    python tools/spmm_one.py c3:0.9 hybrid
"""
from __future__ import annotations

import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1702_08597_b200 as wb  # noqa: E402
from paper_1702_08597_b200.synth import CONFIGS, make_inputs, with_sparsity  # noqa: E402

nm, where = sys.argv[1], sys.argv[2]
base, _, sp = nm.partition(":")
cfg = CONFIGS[base]
if sp:
    cfg = with_sparsity(cfg, float(sp))
img, w_f, _ = make_inputs(cfg)
lay = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=cfg.pad, m=cfg.m, device=0)
lay.set_weights(w_f, dense=False)
lay.set_spmm_operands(where)
x = torch.from_numpy(img).cuda()
for _ in range(2):
    lay.forward(x, None)
torch.cuda.synchronize()
print("done")
