"""Numpy simulation of the exact dW_F digit scheme (csrc/wino_xdw.cuh): 5 balanced base-256
digits per value from the f64 transform, exponents from the ‖B‖₁/‖A‖₁ bounds, the 15 digit pairs
of weight >= 256^4; strict-tolerance misses against the f64 layer vs the fp32-operand floor.
    python tools/oz_sim.py c1        python tools/oz_sim.py c3 12   (first 12 images)"""
import sys, numpy as np
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import wino_oracle as wo
from paper_1702_08597_b200.synth import CONFIGS, make_inputs
cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
nimg = int(sys.argv[2]) if len(sys.argv) > 2 else None
img, w_f, go = make_inputs(CONFIGS[cfg])
if nimg: img, go = img[:nimg], go[:nimg]
m, pad = 4, 1
n, c, h, w = img.shape; k = w_f.shape[0]
g = wo.padded_geometry(c, h, w, pad, m)
a, b, _ = wo.transforms(m); p = g.p
imgp = np.zeros((n, c, g.h_ip, g.w_ip)); imgp[:, :, pad:pad+h, pad:pad+w] = img
til = np.stack([imgp[:, :, (t//g.tiles_x)*m:(t//g.tiles_x)*m+p, (t%g.tiles_x)*m:(t%g.tiles_x)*m+p] for t in range(g.t)], axis=2)
v = np.einsum("ki,nctkl,lj->ijcnt", b, til, b).reshape(p*p, c, n*g.t)
full = np.zeros((n, k, g.h_op, g.w_op)); full[:, :, :g.h_o, :g.w_o] = go
dot = full.reshape(n, k, g.tiles_y, m, g.tiles_x, m)
dz = np.einsum("iy,nkaybx,jx->ijknab", a, dot, a).reshape(p*p, k, n*g.t)
ref = np.matmul(dz, v.transpose(0, 2, 1))  # [36][K][C]
nb = np.abs(b).sum(0); na = np.abs(a).sum(1)  # column l1 norms of B (over rows a), rows of A
imax = np.abs(img).max(axis=(0, 2, 3)); omax = np.abs(go).max(axis=(0, 2, 3))
bound_v = (nb[:, None] * nb[None, :]).reshape(-1)[:, None] * imax[None, :]   # [36][C]
bound_z = (na[:, None] * na[None, :]).reshape(-1)[:, None] * omax[None, :]   # [36][K]
def digits(x, bound, L=38):
    E = np.ceil(np.log2(np.maximum(bound, 1e-300))).astype(np.int64)
    mm = np.rint(x * np.ldexp(1.0, L - E)[:, :, None]).astype(np.int64)
    assert np.abs(mm).max() <= 2**38
    mp = mm + 0x8080808080
    d = [((mp >> (8*j)) & 255).astype(np.int64) - 128 for j in range(5)]
    assert np.array_equal(sum(d[j] << (8*j) for j in range(5)), mm)
    return d, E
dv_, Ev = digits(v, bound_v); dz_, Ez = digits(dz, bound_z)
acc = np.zeros_like(ref)
for i in range(5):
    for j in range(5):
        if i + j >= 4:
            acc += np.matmul(dz_[i].astype(np.float64), dv_[j].astype(np.float64).transpose(0, 2, 1)) * 2.0**(8*(i+j))
got = acc * np.ldexp(1.0, (Ez[:, :, None] + Ev[:, None, :] - 76))
mask = (w_f.transpose(2, 3, 0, 1).reshape(p*p, k, c) != 0)
err = np.abs(got - ref); tol = 1e-5 + 1e-4 * np.abs(ref)
r = (err / tol)[mask]
print(cfg, "entries", mask.sum(), "misses", (r > 1).sum(), "max err/tol", r.max(), "p99.99", np.quantile(r, 0.9999))
# fp32 floor for comparison
v32 = v.astype(np.float32).astype(np.float64); dz32 = dz.astype(np.float32).astype(np.float64)
fl = np.matmul(dz32, v32.transpose(0, 2, 1))
rf = (np.abs(fl - ref) / tol)[mask]
print("floor misses", (rf > 1).sum(), "max", rf.max())
