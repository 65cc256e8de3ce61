"""Small cases over every kernel family, for compute-sanitizer (memcheck / synccheck / racecheck):
sparse CSR step with the shared-memory and the TMEM SpMM (2 and 4 stages, staged and unstaged
stream), forward_backward DAG, dense tcgen05 plan, tensor-core contraction on a sparse plan,
ragged shapes (odd C, K, H), the exact dW_F digits/int8 GEMM in every case, a value update."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1702_08597_b200 as wb  # noqa: E402

rng = np.random.default_rng(0)
CASES = [  # (name, C, K, H, n, sparsity, mode, operands)
    ("csr-smem", 256, 384, 13, 2, 0.9, "csr", "smem"),
    ("csr-tmem-s2", 256, 256, 12, 2, 0.9, "csr", "tmem"),
    ("csr-tmem-s4-unstaged", 384, 512, 9, 2, 0.5, "csr", "tmem"),
    ("ragged-tmem", 161, 203, 11, 3, 0.7, "csr", "tmem"),
    ("csr-hybrid", 256, 256, 12, 2, 0.9, "csr", "hybrid"),
    ("ragged-hybrid-unstaged", 161, 203, 11, 3, 0.3, "csr", "hybrid"),
    ("fb", 256, 256, 12, 2, 0.9, "fb", "auto"),
    ("dense", 128, 128, 12, 2, 0.0, "dense", "auto"),
    ("tc", 256, 256, 12, 2, 0.9, "tc", "auto"),
]
for name, c, k, h, n, sp, mode, ops in CASES:
    w_f = rng.standard_normal((k, c, 6, 6)) * np.sqrt(2.0 / (9 * c))
    w_f *= rng.random(w_f.shape) >= sp
    img = rng.standard_normal((n, c, h, h)).astype(np.float32)
    go = rng.standard_normal((n, k, h, h)).astype(np.float32)
    layer = wb.WinogradLayer(c, k, h, h, pad=1, m=4)
    layer.set_weights(w_f, dense=(mode == "dense"))
    layer.set_spmm_operands(ops)
    if mode == "tc":
        layer.set_contraction("tc")
    cache = layer.new_cache(n)
    x, g = torch.from_numpy(img).cuda(), torch.from_numpy(go).cuda()
    if mode == "fb":
        layer.forward_backward(x, g, cache)
    else:
        layer.forward(x, cache)
        dw, _ = layer.backward(g, cache)
        layer.sgd_step(dw, lr=1e-3)
        layer.forward(x, cache)
    torch.cuda.synchronize()
    layer.close()
    print(name, "ok", flush=True)
