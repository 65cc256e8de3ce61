"""Small cases over every kernel family, for compute-sanitizer (memcheck / synccheck):
sparse CSR step, forward_backward DAG, dense tcgen05 plan (warp-specialised GEMM), tensor-core
contraction on a sparse plan, int8 dW mode, precise dW mode, pipelined host step."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1702_08597_b200 as wb  # noqa: E402
from paper_1702_08597_b200.synth import CONFIGS, make_inputs, with_sparsity  # noqa: E402

cfg = CONFIGS["c1"]
for mode in ("csr", "fb", "dense", "tc", "int8", "precise"):
    c = with_sparsity(cfg, 0.0) if mode == "dense" else cfg
    img, w_f, go = make_inputs(c)
    n = 4
    img, go = img[:n], go[:n]
    layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4)
    layer.set_weights(w_f, dense=(mode == "dense"))
    if mode == "tc":
        layer.set_contraction("tc")
    if mode in ("int8", "precise"):
        layer.set_dw_mode(mode)
    cache = layer.new_cache(n)
    x, g = torch.from_numpy(img).cuda(), torch.from_numpy(go).cuda()
    if mode == "fb":
        layer.forward_backward(x, g, cache)
    else:
        layer.forward(x, cache)
        layer.backward(g, cache)
    torch.cuda.synchronize()
    print(mode, "ok", flush=True)
