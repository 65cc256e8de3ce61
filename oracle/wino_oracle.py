"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference Winograd layer.

Parity status: PINNED.  Every function here is checked in tests/test_oracle.py
against (a) the compiled reference (oracle/_ref, built from /root/reference by
oracle/Makefile) where it is available, and (b) the golden vectors in
tests/golden/ that the reference itself produced (tests/golden/make_golden.py).

Two families:

* f64 restatement of the dense layer, following the reference line by line:
  transforms.cpp (Cook–Toom generator, geometry, φ/ψ, tiling) and layer.cpp
  (forward / backward_weights / backward_input).  Matches the reference to
  ~1e-13 (numpy's summation order differs from the reference's left-to-right loops).

* f32 "operation-order mirror" of what the CUDA kernels compute: the same
  association order as the reference's own f32 path (sparse.cpp:81-185) —
  products rounded to f32, sums accumulated left to right from +0, no fused
  multiply-add — extended to the backward pass with the dense layer's
  association order (layer.cpp:107-169).  The GPU forward, dĨ_F and dI must be
  BITWISE equal to these functions; dW_F is accumulated in f64 on both sides.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import
this module.  The product path never does.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

F32 = np.float32

# ----------------------------------------------------------------------------------
# Transforms (transforms.cpp:7-145)
# ----------------------------------------------------------------------------------

_POINTS = (0.0, 1.0, -1.0, 2.0, -2.0, 0.5, -0.5)  # transforms.cpp:23


def f2x2_3x3():
    """transforms.cpp:7-19 — the fixed F(2x2,3x3) matrices."""
    a = np.array([[1, 0], [1, 1], [1, -1], [0, -1]], dtype=np.float64)
    b = np.array([[1, 0, 0, 0], [0, 1, -1, 1], [-1, 1, 1, 0], [0, 0, 0, -1]], dtype=np.float64)
    g = np.array([[1, 0, 0], [0.5, 0.5, 0.5], [0.5, -0.5, 0.5], [0, 0, 1]], dtype=np.float64)
    return a, b, g


def _inverse_vandermonde(pts):
    """transforms.cpp:33-53 (same loop order, so the doubles match bit for bit)."""
    n = len(pts)
    inv = np.zeros((n, n))
    for i in range(n):
        coeff = [1.0]
        denom = 1.0
        for k in range(n):
            if k == i:
                continue
            nxt = [0.0] * (len(coeff) + 1)
            for d in range(len(coeff)):
                nxt[d] -= coeff[d] * pts[k]
                nxt[d + 1] += coeff[d]
            coeff = nxt
            denom *= pts[i] - pts[k]
        for j in range(n):
            inv[j, i] = coeff[j] / denom
    return inv


def _product_poly(pts):
    """transforms.cpp:56-67."""
    coeff = [1.0]
    for a in pts:
        nxt = [0.0] * (len(coeff) + 1)
        for d in range(len(coeff)):
            nxt[d] -= coeff[d] * a
            nxt[d + 1] += coeff[d]
        coeff = nxt
    return coeff


def cook_toom_1d(m: int, r: int):
    """transforms.cpp:71-120 -> (a p×m, b p×p, g p×r)."""
    if m < 1 or r < 1:
        raise ValueError("tile and kernel extents must be >= 1")
    p = m + r - 1
    if p > 8:
        raise ValueError(f"unsupported transform size: m+r-1 = {p} exceeds 8")
    if p == 1:
        return np.eye(1), np.eye(1), np.eye(1)
    pts = list(_POINTS[: p - 1])

    def eval_matrix(ncoeff):
        v = np.zeros((p, ncoeff))
        for i in range(p - 1):
            x = 1.0
            for j in range(ncoeff):
                v[i, j] = x
                x *= pts[i]
        v[p - 1, ncoeff - 1] = 1.0
        return v

    g = eval_matrix(r)
    a = eval_matrix(m)
    inv = _inverse_vandermonde(pts)
    mpoly = _product_poly(pts)
    c = np.zeros((p, p))
    for j in range(p - 1):
        for i in range(p - 1):
            c[j, i] = inv[j, i]
        c[j, p - 1] = mpoly[j]
    c[p - 1, p - 1] = 1.0
    return a, c, g


def transforms(m: int, r: int = 3):
    """bindings.cpp:41-44: fixed F(2,3) for m=2,r=3; Cook–Toom otherwise."""
    if m == 2 and r == 3:
        return f2x2_3x3()
    return cook_toom_1d(m, r)


# ----------------------------------------------------------------------------------
# Geometry, φ, ψ, tiling (transforms.cpp:147-241)
# ----------------------------------------------------------------------------------


@dataclass(frozen=True)
class Geometry:
    c: int
    h_i: int
    w_i: int
    h_o: int
    w_o: int
    h_op: int
    w_op: int
    h_ip: int
    w_ip: int
    m: int
    r: int
    p: int
    tiles_y: int
    tiles_x: int
    t: int


def make_geometry(c, h_i, w_i, m, r=3) -> Geometry:
    """transforms.cpp:147-172 (square tiles/kernels)."""
    if h_i < r or w_i < r:
        raise ValueError(f"image ({c}x{h_i}x{w_i}) smaller than kernel ({r}x{r})")
    h_o, w_o = h_i - r + 1, w_i - r + 1
    ty, tx = (h_o + m - 1) // m, (w_o + m - 1) // m
    h_op, w_op = ty * m, tx * m
    return Geometry(c, h_i, w_i, h_o, w_o, h_op, w_op, h_op + r - 1, w_op + r - 1, m, r,
                    m + r - 1, ty, tx, ty * tx)


def phi(g: Geometry, t, i, j):
    """transforms.cpp:179-187."""
    if t >= g.t or i >= g.p or j >= g.p or min(t, i, j) < 0:
        raise ValueError(f"phi index ({t},{i},{j}) out of range")
    return (t // g.tiles_x) * g.m + i, (t % g.tiles_x) * g.m + j


def psi(g: Geometry, y, x):
    """transforms.cpp:189-194."""
    if y >= g.h_op or x >= g.w_op or min(y, x) < 0:
        raise ValueError(f"psi index ({y},{x}) out of range")
    return (y // g.m) * g.tiles_x + (x // g.m), y % g.m, x % g.m


def tile_input(img, g: Geometry):
    """transforms.cpp:196-210: C×Hi×Wi -> C×T×p×p, zero outside the image."""
    c = img.shape[0]
    xp = np.zeros((c, g.h_ip, g.w_ip), dtype=img.dtype)
    xp[:, : g.h_i, : g.w_i] = img
    out = np.empty((c, g.t, g.p, g.p), dtype=img.dtype)
    for t in range(g.t):
        y0, x0 = (t // g.tiles_x) * g.m, (t % g.tiles_x) * g.m
        out[:, t] = xp[:, y0 : y0 + g.p, x0 : x0 + g.p]
    return out


def untile_output(tiled, g: Geometry):
    """transforms.cpp:212-226: K×T×m×m -> K×Ho×Wo (crop)."""
    k = tiled.shape[0]
    full = tiled.reshape(k, g.tiles_y, g.tiles_x, g.m, g.m).transpose(0, 1, 3, 2, 4)
    return full.reshape(k, g.h_op, g.w_op)[:, : g.h_o, : g.w_o].copy()


def tile_output(img, g: Geometry):
    """transforms.cpp:228-241: K×Ho×Wo -> K×T×m×m (zero fill padding)."""
    k = img.shape[0]
    full = np.zeros((k, g.h_op, g.w_op), dtype=img.dtype)
    full[:, : g.h_o, : g.w_o] = img
    return full.reshape(k, g.tiles_y, g.m, g.tiles_x, g.m).transpose(0, 1, 3, 2, 4).reshape(
        k, g.t, g.m, g.m).copy()


# ----------------------------------------------------------------------------------
# Dense f64 layer (layer.cpp:45-171)
# ----------------------------------------------------------------------------------


def forward_f64(img, w_f, m=4):
    """layer.cpp:45-96 -> (O K×Ho×Wo, cache {i_f C×T×p×p, z K×T×p×p})."""
    a, b, _ = transforms(m)
    img = np.asarray(img, dtype=np.float64)
    g = make_geometry(img.shape[0], img.shape[1], img.shape[2], m)
    til = tile_input(img, g)
    i_f = np.einsum("ki,ctkl,lj->ctij", b, til, b)          # B1ᵀ Ĩ B2
    z = np.einsum("kcij,ctij->ktij", w_f, i_f)               # layer.cpp:61-71
    o_t = np.einsum("iy,ktij,jx->ktyx", a, z, a)             # A1ᵀ Z A2
    return untile_output(o_t, g), {"i_f": i_f, "z": z, "g": g, "m": m}


def backward_weights_f64(grad_o, cache):
    """layer.cpp:98-132 -> dW_F; stores grad_z in the cache (layer.cpp:130)."""
    a, _, _ = transforms(cache["m"])
    go_t = tile_output(np.asarray(grad_o, dtype=np.float64), cache["g"])
    grad_z = np.einsum("iy,ktyx,jx->ktij", a, go_t, a)        # A1 dÕ A2ᵀ
    cache["grad_z"] = grad_z
    return np.einsum("ktij,ctij->kcij", grad_z, cache["i_f"])


def backward_input_f64(cache, w_f):
    """layer.cpp:134-171 -> dI (C×Hi×Wi)."""
    if "grad_z" not in cache:
        raise RuntimeError("backward_input: dL/dZ missing; run backward_weights first")
    g = cache["g"]
    _, b, _ = transforms(cache["m"])
    grad_if = np.einsum("kcij,ktij->ctij", w_f, cache["grad_z"])
    gt = np.einsum("ik,ctkl,jl->ctij", b, grad_if, b)         # B1 dĨ_F B2ᵀ
    out = np.zeros((g.c, g.h_ip, g.w_ip))
    for t in range(g.t):
        y0, x0 = (t // g.tiles_x) * g.m, (t % g.tiles_x) * g.m
        out[:, y0 : y0 + g.p, x0 : x0 + g.p] += gt[:, t]
    return out[:, : g.h_i, : g.w_i].copy()


def direct_conv_f64(img, w):
    """reference.cpp:7-34 (correlation, no flip)."""
    c, h, wd = img.shape
    k, _, r, s = w.shape
    ho, wo = h - r + 1, wd - s + 1
    out = np.zeros((k, ho, wo))
    for u in range(r):
        for v in range(s):
            out += np.einsum("kc,chw->khw", w[:, :, u, v], img[:, u : u + ho, v : v + wo])
    return out


def lift_f64(w, m=4):
    """layer.cpp:29-43: W_F = G1 W G2ᵀ."""
    _, _, gm = transforms(m, w.shape[2])
    return np.einsum("iu,kcuv,jv->kcij", gm, w, gm)


# ----------------------------------------------------------------------------------
# CSR (sparse.cpp:9-69)
# ----------------------------------------------------------------------------------


@dataclass
class Csr:
    """PointwiseCsr<float> (sparse.hpp:19-38): slices in row-major (i,j) order."""
    k: int
    c: int
    p: int
    row_ptr: list  # p*p arrays of K+1 int64
    col_idx: list  # p*p arrays int64
    values: list   # p*p arrays float32

    def nnz(self):
        return sum(len(v) for v in self.values)


def compress(w_f, zero_tol=0.0) -> Csr:
    """sparse.cpp:9-36 (keep rule at sparse.cpp:27, cast at :29)."""
    w_f = np.asarray(w_f, dtype=np.float64)
    k, c, p, _ = w_f.shape
    rps, cols, vals = [], [], []
    for i in range(p):
        for j in range(p):
            sl = w_f[:, :, i, j]
            keep = (np.abs(sl) > zero_tol) | ((zero_tol == 0.0) & (sl != 0.0))
            rk, ck = np.nonzero(keep)            # row-major order == the reference loop order
            rp = np.zeros(k + 1, dtype=np.int64)
            np.add.at(rp, rk + 1, 1)
            rps.append(np.cumsum(rp))
            cols.append(ck.astype(np.int64))
            vals.append(sl[rk, ck].astype(F32))
    return Csr(k, c, p, rps, cols, vals)


def reconstruct(csr: Csr):
    """sparse.cpp:38-49."""
    w = np.zeros((csr.k, csr.c, csr.p, csr.p))
    for s in range(csr.p * csr.p):
        i, j = divmod(s, csr.p)
        rows = np.repeat(np.arange(csr.k), np.diff(csr.row_ptr[s]))
        w[rows, csr.col_idx[s], i, j] = csr.values[s].astype(np.float64)
    return w


def csr_positions(row_ptr):
    """Position of every entry inside its row (for order-preserving vectorisation)."""
    lens = np.diff(row_ptr)
    rows = np.repeat(np.arange(len(lens)), lens)
    pos = np.arange(int(row_ptr[-1])) - np.repeat(row_ptr[:-1], lens)
    return rows, pos, lens


def transpose_slice(row_ptr, col_idx, values, c):
    """CSR of W_F(:,:,i,j)ᵀ (i.e. CSC of the slice): rows sorted ascending within a column."""
    k = len(row_ptr) - 1
    rows = np.repeat(np.arange(k), np.diff(row_ptr))
    order = np.lexsort((rows, col_idx))   # by column, then ascending row
    cp = np.zeros(c + 1, dtype=np.int64)
    np.add.at(cp, col_idx + 1, 1)
    return np.cumsum(cp), rows[order], values[order], order


# ----------------------------------------------------------------------------------
# f32 operation-order mirror of the CUDA kernels (batched, pad folded into φ)
# ----------------------------------------------------------------------------------


def padded_geometry(c, h, w, pad, m, r=3) -> Geometry:
    """Geometry of the reference called on the explicitly zero-padded (H+2pad)×(W+2pad) image
    (tools/wino.cpp:337 convention)."""
    return make_geometry(c, h + 2 * pad, w + 2 * pad, m, r)


def _tiles_f32(batch, g: Geometry, pad):
    n, c, h, w = batch.shape
    xp = np.zeros((n, c, g.h_ip, g.w_ip), dtype=F32)
    xp[:, :, pad : pad + h, pad : pad + w] = batch
    out = np.empty((n, c, g.t, g.p, g.p), dtype=F32)
    for t in range(g.t):
        y0, x0 = (t // g.tiles_x) * g.m, (t % g.tiles_x) * g.m
        out[:, :, t] = xp[:, :, y0 : y0 + g.p, x0 : x0 + g.p]
    return out


def input_transform_f32(batch, m=4, pad=0):
    """K1 mirror: Ĩ_F[(i,j)][c][n·T+t] = (B1ᵀ·d·B2) in the order of sparse.cpp:103-116."""
    batch = np.asarray(batch, dtype=F32)
    n, c, h, w = batch.shape
    g = padded_geometry(c, h, w, pad, m)
    _, b, _ = transforms(m)
    b = b.astype(F32)
    d = _tiles_f32(batch, g, pad)                      # n,c,t,p,p
    p = g.p
    tmp = np.zeros_like(d)
    for k in range(p):                                 # tmp[i][j] = Σ_k b[k][i]·d[k][j]
        tmp = tmp + b[k][:, None] * d[..., k, None, :]
    u = np.zeros_like(d)
    for k in range(p):                                 # u[i][j] = Σ_k tmp[i][k]·b[k][j]
        u = u + tmp[..., :, k, None] * b[k][None, :]
    # -> [(i,j)][c][n,t]
    return np.ascontiguousarray(u.transpose(3, 4, 1, 0, 2).reshape(p * p, c, n * g.t)), g


def spmm_rows_f32(row_ptr, col_idx, values, dense):
    """out(k,:) = Σ_{e∈row k} v_e·dense(col_e,:), accumulated left to right from +0 in f32
    (sparse.cpp:51-69)."""
    k = len(row_ptr) - 1
    out = np.zeros((k, dense.shape[1]), dtype=F32)
    rows, pos, lens = csr_positions(row_ptr)
    if len(rows) == 0:
        return out
    for q in range(int(lens.max())):
        sel = pos == q
        r = rows[sel]
        out[r] = out[r] + values[sel][:, None].astype(F32) * dense[col_idx[sel]]
    return out


def contraction_f32(csr: Csr, v):
    """K2 mirror: Z[(i,j)] = W_F(i,j)·Ĩ_F(i,j) for every slice."""
    return np.stack([spmm_rows_f32(csr.row_ptr[s], csr.col_idx[s], csr.values[s], v[s])
                     for s in range(csr.p * csr.p)])


def output_transform_f32(z, g: Geometry, n, m=4):
    """K3 mirror (sparse.cpp:151-184): tmp[y][j] = Σ_i a1[i][y]·z[i][j]; o[y][x] = Σ_j a2[j][x]·tmp[y][j]."""
    a, _, _ = transforms(m)
    a = a.astype(F32)
    p = g.p
    k = z.shape[1]
    zz = z.reshape(p, p, k, n, g.t)                    # i,j,k,n,t
    tmp = np.zeros((m, p, k, n, g.t), dtype=F32)       # y,j,...
    for i in range(p):
        tmp = tmp + a[i][:, None, None, None, None] * zz[i][None]
    o = np.zeros((m, m, k, n, g.t), dtype=F32)         # y,x,...
    for j in range(p):
        o = o + a[j][None, :, None, None, None] * tmp[:, j][:, None]
    o = o.reshape(m, m, k, n, g.tiles_y, g.tiles_x).transpose(3, 2, 4, 0, 5, 1)
    return np.ascontiguousarray(o.reshape(n, k, g.h_op, g.w_op)[:, :, : g.h_o, : g.w_o])


def grad_z_f32(grad_o, g: Geometry, m=4):
    """K4 mirror (layer.cpp:107-116): dZ = (A1·dÕ)·A2ᵀ, zero for padded positions."""
    a, _, _ = transforms(m)
    a = a.astype(F32)
    grad_o = np.asarray(grad_o, dtype=F32)
    n, k = grad_o.shape[:2]
    full = np.zeros((n, k, g.h_op, g.w_op), dtype=F32)
    full[:, :, : g.h_o, : g.w_o] = grad_o
    d = full.reshape(n, k, g.tiles_y, m, g.tiles_x, m).transpose(0, 1, 2, 4, 3, 5)  # n,k,ty,tx,y,x
    p = g.p
    m1 = np.zeros(d.shape[:4] + (p, m), dtype=F32)      # [i][x] = Σ_y a1[i][y]·d[y][x]
    for y in range(m):
        m1 = m1 + a[:, y][:, None] * d[..., y, None, :]
    dz = np.zeros(d.shape[:4] + (p, p), dtype=F32)      # [i][j] = Σ_x m1[i][x]·a2[j][x]
    for x in range(m):
        dz = dz + m1[..., :, x, None] * a[:, x][None, :]
    dz = dz.reshape(n, k, g.t, p, p)
    return np.ascontiguousarray(dz.transpose(3, 4, 1, 0, 2).reshape(p * p, k, n * g.t))


def sddmm_f64(csr: Csr, dz, v):
    """K5 reference value: dW_F(k,c,i,j) = Σ_t dZ(k,t)·Ĩ_F(c,t) for surviving (k,c) only,
    exact f64 sum of the f32 operands (layer.cpp:118-128 restricted to the mask)."""
    out = []
    for s in range(csr.p * csr.p):
        rows, _, _ = csr_positions(csr.row_ptr[s])
        a = dz[s].astype(np.float64)
        b = v[s].astype(np.float64)
        out.append(np.einsum("et,et->e", a[rows], b[csr.col_idx[s]]))
    return out  # list of f64 arrays, CSR order


def backward_data_f32(csr: Csr, dz):
    """K6 mirror (layer.cpp:145-155 on the mask): dĨ_F(c,t) = Σ_k W_F(k,c)·dZ(k,t), k ascending."""
    outs = []
    for s in range(csr.p * csr.p):
        cp, rows, vals, _ = transpose_slice(csr.row_ptr[s], csr.col_idx[s], csr.values[s], csr.c)
        outs.append(spmm_rows_f32(cp, rows, vals, dz[s]))
    return np.stack(outs)


def input_grad_f32(dv, g: Geometry, n, h, w, pad, m=4):
    """K7 mirror (layer.cpp:157-169): dĨ = (B1·dĨ_F)·B2ᵀ, then the φ scatter-add in ascending
    t order from +0; positions outside the (unpadded) image are dropped."""
    _, b, _ = transforms(m)
    b = b.astype(F32)
    p = g.p
    c = dv.shape[1]
    x = dv.reshape(p, p, c, n, g.t).transpose(3, 2, 4, 0, 1)   # n,c,t,i,j
    m1 = np.zeros_like(x)                                      # [i][j] = Σ_k b[i][k]·x[k][j]
    for k in range(p):
        m1 = m1 + b[:, k][:, None] * x[..., k, None, :]
    gt = np.zeros_like(x)                                      # [i][j] = Σ_k m1[i][k]·b[j][k]
    for k in range(p):
        gt = gt + m1[..., :, k, None] * b[:, k][None, :]
    out = np.zeros((n, c, g.h_ip, g.w_ip), dtype=F32)
    for t in range(g.t):
        y0, x0 = (t // g.tiles_x) * g.m, (t % g.tiles_x) * g.m
        out[:, :, y0 : y0 + p, x0 : x0 + p] = out[:, :, y0 : y0 + p, x0 : x0 + p] + gt[:, :, t]
    return np.ascontiguousarray(out[:, :, pad : pad + h, pad : pad + w])


def layer_f32(batch, csr: Csr, grad_o=None, m=4, pad=0):
    """The whole sparse layer as the GPU computes it (forward, and backward if grad_o)."""
    batch = np.asarray(batch, dtype=F32)
    n, c, h, w = batch.shape
    v, g = input_transform_f32(batch, m, pad)
    z = contraction_f32(csr, v)
    res = {"v": v, "z": z, "o": output_transform_f32(z, g, n, m), "g": g}
    if grad_o is not None:
        dz = grad_z_f32(grad_o, g, m)
        res["dz"] = dz
        res["dw"] = sddmm_f64(csr, dz, v)
        res["dv"] = backward_data_f32(csr, dz)
        res["di"] = input_grad_f32(res["dv"], g, n, h, w, pad, m)
    return res


def train_update_f64(w, g, lr, scale=1.0, lmbda=0.0, norm=1, prune=False, eps=0.0, beta=0.0):
    """The per-coordinate update of train_step (train.cpp:255-290) on the coordinates given
    (a sparse plan's values, or all of a dense layer's), in the reference's f64 expression order:
    reg_grad (train.cpp:213-218; λ·w/‖w‖₂ with ‖w‖ over the given values, l2_norm
    train.cpp:220-224), v = w − lr·(g + reg) (train.cpp:284), threshold_value
    (train.cpp:108-110, applied in prune mode when λ > 0, train.cpp:285-286).
    Returns (new values rounded to f32, number of non-finite results)."""
    w = np.asarray(w, dtype=np.float64)
    g = scale * np.asarray(g, dtype=np.float64)
    if lmbda == 0.0:
        reg = np.zeros_like(w)
    elif norm == 1:
        reg = np.where(w > 0, lmbda, np.where(w < 0, -lmbda, 0.0))
    else:
        nrm = np.sqrt(np.sum(w * w))
        reg = (lmbda * w) / nrm if nrm > 0 else np.zeros_like(w)
    with np.errstate(over="ignore", invalid="ignore"):
        v = w - lr * (g + reg)
        if prune and lmbda > 0:
            v = np.where(np.abs(v) * (np.abs(g) + beta) < eps, 0.0, v)
        f = v.astype(np.float32)
    return f, int(np.count_nonzero(~np.isfinite(f)))


def flops_baseline(c, k, h, r=3):
    """perfmodel.cpp:6-9: 2·C·K·H²·r² per image and pass (the 'effective FLOP' numerator)."""
    return 2.0 * c * k * h * h * r * r
