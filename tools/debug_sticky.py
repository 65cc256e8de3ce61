import sys, numpy as np, torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import paper_1702_08597_b200 as wb
from paper_1702_08597_b200.synth import CONFIGS, make_inputs

def probe(tag):
    try:
        torch.zeros(1, device="cuda"); torch.cuda.synchronize(); print("ok  ", tag, flush=True)
    except Exception as e:
        print("FAIL", tag, str(e).splitlines()[0], flush=True); sys.exit(1)

cfg = CONFIGS["c1"]
img, w_f, go = make_inputs(cfg)
probe("start")
layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=1, m=4); probe("plan")
layer.set_weights(w_f, dense=False); probe("set_weights")
cache = layer.new_cache(cfg.n); probe("cache")
x = torch.from_numpy(img).cuda(); g = torch.from_numpy(go).cuda(); probe("inputs")
o = layer.forward(x, cache); probe("forward")
dw = layer.backward_weights(g, cache); probe("bwd_w")
di = layer.backward_input(cache); probe("bwd_i")
csr = layer.get_csr(); probe("get_csr")
del cache; probe("del cache")
try:
    layer.close()
except Exception as e:
    print("close raised:", e)
probe("close layer")
