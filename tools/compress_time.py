"""Time set_weights (device compress incl. the host->device copy) and recompress at c1 / vgg4_2 shapes."""
import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1702_08597_b200 as wb  # noqa: E402

for (c, k, h) in [(256, 384, 13), (512, 512, 28)]:
    rng = np.random.default_rng(0)
    w = rng.standard_normal((k, c, 6, 6))
    w[rng.random(w.shape) < 0.9] = 0.0
    lay = wb.WinogradLayer(c, k, h, h, pad=1, m=4)
    for _ in range(2):
        lay.set_weights(w, dense=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); lay.set_weights(w, dense=False); torch.cuda.synchronize(); t1 = time.perf_counter()
    lay.recompress(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"C={c} K={k}: set_weights {1e3*(t1-t0):.2f} ms, recompress {1e3*(t2-t1):.2f} ms")
