"""TEST INFRASTRUCTURE ONLY — ctypes access to the compiled reference (oracle/_ref).

`oracle/_ref/libwino_ref.so` is the unmodified reference implementation
(/root/reference/proj/src, built by oracle/Makefile) plus the marshalling shim
oracle/ref_shim.cpp.  Only tests/, __graft_entry__.smoke() and bench.py's CPU
baseline / reference arm may import this module, and only as the checker or the
timed CPU baseline — never as the product path.

Every function returns f64 numpy arrays in the reference's own layouts.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "_ref" / "libwino_ref.so"
_lib = None

_d = C.POINTER(C.c_double)
_f = C.POINTER(C.c_float)
_l = C.POINTER(C.c_long)


class RefError(RuntimeError):
    """Exception thrown inside the reference; .code follows ref_shim.cpp:fail()."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[ref code {code}] {msg}")
        self.code = code


def available() -> bool:
    return LIB_PATH.exists()


def build() -> None:
    """Compile oracle/_ref from /root/reference (only possible where it exists)."""
    if not Path("/root/reference/proj/src").exists():
        return
    import subprocess

    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise FileNotFoundError(f"{LIB_PATH} not built (run `make -C oracle`)")
        _lib = C.CDLL(str(LIB_PATH))
        _lib.wref_last_error.restype = C.c_char_p
    return _lib


def _ptr(a, t=_d):
    return None if a is None else a.ctypes.data_as(t)


def _check(rc: int):
    if rc != 0:
        raise RefError(rc, lib().wref_last_error().decode())


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def transforms(m: int, r: int = 3):
    """(A p×m, B p×p, G p×r) doubles exactly as the reference builds them."""
    p = m + r - 1
    a, b, g = np.zeros((p, m)), np.zeros((p, p)), np.zeros((p, r))
    _check(lib().wref_transforms(m, r, _ptr(a), _ptr(b), _ptr(g)))
    return a, b, g


GEOM_FIELDS = ("c", "h_i", "w_i", "h_o", "w_o", "h_op", "w_op", "h_ip", "w_ip", "p", "q",
               "tiles_y", "tiles_x", "t")


def geometry(c, h_i, w_i, m, r=3) -> dict:
    out = np.zeros(14, dtype=np.int64)
    _check(lib().wref_geometry(c, h_i, w_i, m, r, _ptr(out, _l)))
    return dict(zip(GEOM_FIELDS, (int(v) for v in out)))


def phi(c, h_i, w_i, m, t, i, j, r=3):
    out = np.zeros(2, dtype=np.int64)
    _check(lib().wref_phi(c, h_i, w_i, m, r, C.c_long(t), C.c_long(i), C.c_long(j), _ptr(out, _l)))
    return int(out[0]), int(out[1])


def psi(c, h_i, w_i, m, y, x, r=3):
    out = np.zeros(3, dtype=np.int64)
    _check(lib().wref_psi(c, h_i, w_i, m, r, C.c_long(y), C.c_long(x), _ptr(out, _l)))
    return int(out[0]), int(out[1]), int(out[2])


def layer(img, w_f, grad_o=None, m=4):
    """Dense f64 layer on one image: dict with o, i_f, z (+ grad_wf, grad_in, grad_z)."""
    img, w_f = _c64(img), _c64(w_f)
    c, h_i, w_i = img.shape
    k, _, p, _ = w_f.shape
    g = geometry(c, h_i, w_i, m)
    t = g["t"]
    res = {"o": np.zeros((k, g["h_o"], g["w_o"])), "i_f": np.zeros((c, t, p, p)),
           "z": np.zeros((k, t, p, p))}
    if grad_o is not None:
        grad_o = _c64(grad_o)
        res.update(grad_wf=np.zeros_like(w_f), grad_in=np.zeros_like(img), grad_z=np.zeros((k, t, p, p)))
    _check(lib().wref_layer(m, c, h_i, w_i, k, _ptr(img), _ptr(w_f), _ptr(grad_o),
                            _ptr(res["o"]), _ptr(res["i_f"]), _ptr(res["z"]),
                            _ptr(res.get("grad_wf")), _ptr(res.get("grad_in")),
                            _ptr(res.get("grad_z"))))
    return res


def backward_input_without_grad_z(img, w_f, m=4):
    img, w_f = _c64(img), _c64(w_f)
    c, h_i, w_i = img.shape
    _check(lib().wref_backward_input_without_grad_z(m, c, h_i, w_i, w_f.shape[0], _ptr(img), _ptr(w_f)))


def compress_f32(w_f, zero_tol=0.0):
    """compress<float>: (row_ptr [pq][K+1] int64, col_idx list per slice, values list per slice)."""
    w_f = _c64(w_f)
    k, c, p, _ = w_f.shape
    counts = np.zeros(p * p, dtype=np.int64)
    _check(lib().wref_compress_f32(k, c, p, _ptr(w_f), C.c_double(zero_tol), _ptr(counts, _l),
                                   None, None, None))
    nnz = int(counts.sum())
    row_ptr = np.zeros((p * p, k + 1), dtype=np.int64)
    col = np.zeros(max(nnz, 1), dtype=np.int64)
    val = np.zeros(max(nnz, 1), dtype=np.float32)
    _check(lib().wref_compress_f32(k, c, p, _ptr(w_f), C.c_double(zero_tol), _ptr(counts, _l),
                                   _ptr(row_ptr, _l), _ptr(col, _l), _ptr(val, _f)))
    offs = np.concatenate([[0], np.cumsum(counts)])
    cols = [col[offs[s]:offs[s + 1]].copy() for s in range(p * p)]
    vals = [val[offs[s]:offs[s + 1]].copy() for s in range(p * p)]
    return row_ptr, cols, vals


def tiled_layout_f32(img, m=4):
    """build_tiled_layout<float>: (p*q) x C x T float32."""
    img = _c64(img)
    c, h_i, w_i = img.shape
    g = geometry(c, h_i, w_i, m)
    out = np.zeros((g["p"] * g["q"], c, g["t"]), dtype=np.float32)
    _check(lib().wref_tiled_layout_f32(m, c, h_i, w_i, _ptr(img), _ptr(out, _f)))
    return out


def sparse_forward(batch, w_f, m=4, workers=1, precision=32, return_mults=False):
    batch, w_f = _c64(batch), _c64(w_f)
    n, c, h_i, w_i = batch.shape
    k = w_f.shape[0]
    g = geometry(c, h_i, w_i, m)
    out = np.zeros((n, k, g["h_o"], g["w_o"]))
    mults = C.c_ulonglong(0)
    _check(lib().wref_sparse_forward(m, n, c, h_i, w_i, k, _ptr(batch), _ptr(w_f),
                                     C.c_uint(workers), precision, _ptr(out), C.byref(mults)))
    return (out, int(mults.value)) if return_mults else out


def direct_conv(img, w):
    img, w = _c64(img), _c64(w)
    c, h, wd = img.shape
    k, _, r, _ = w.shape
    out = np.zeros((k, h - r + 1, wd - r + 1))
    _check(lib().wref_direct_conv(c, h, wd, k, r, _ptr(img), _ptr(w), _ptr(out)))
    return out


def lift(w, m=4):
    w = _c64(w)
    k, c = w.shape[:2]
    p = m + 2
    out = np.zeros((k, c, p, p))
    _check(lib().wref_lift(m, k, c, _ptr(w), _ptr(out)))
    return out


def layer_fwd_bwd_batch(batch, w_f, grad_o, m=4, threads=None, n=None, want_outputs=True):
    """The reference's per-image dense f64 fwd+bwd over (the first n images of) a batch,
    images spread over `threads` host threads.  Returns (o, grad_in, sum_n grad_wf)."""
    batch, w_f, grad_o = _c64(batch), _c64(w_f), _c64(grad_o)
    nb, c, h_i, w_i = batch.shape
    n = nb if n is None else n
    k = w_f.shape[0]
    threads = threads or os.cpu_count() or 1
    g = geometry(c, h_i, w_i, m)
    o = np.zeros((nb, k, g["h_o"], g["w_o"])) if want_outputs else None
    gi = np.zeros_like(batch) if want_outputs else None
    gw = np.zeros_like(w_f)
    _check(lib().wref_layer_fwd_bwd_batch(m, n, c, h_i, w_i, k, _ptr(batch), _ptr(w_f), _ptr(grad_o),
                                          C.c_uint(threads), _ptr(o), _ptr(gi), _ptr(gw)))
    return o, gi, gw


def write_wgt1(path, arr, dtype="f64"):
    arr = _c64(arr)
    shape = np.array(arr.shape, dtype=np.int64)
    _check(lib().wref_write_wgt1(str(path).encode(), _ptr(shape, _l), arr.ndim, _ptr(arr),
                                 2 if dtype == "f32" else 1))


def uniform_stream(seed, name, n):
    out = np.zeros(n)
    _check(lib().wref_uniform_stream(C.c_ulonglong(seed), name.encode(), C.c_long(n), _ptr(out)))
    return out


def threshold_to_density(w, density):
    w = _c64(w).ravel().copy()
    _check(lib().wref_threshold_to_density(_ptr(w), C.c_long(w.size), C.c_double(density)))
    return w


def checkpoint_roundtrip(dir_in, dir_out):
    """The reference loads dir_in and saves what it loaded to dir_out."""
    _check(lib().wref_checkpoint_roundtrip(str(dir_in).encode(), str(dir_out).encode()))


def train_steps(seed, steps, batch, mode=0):
    """The reference trainer: losses of `steps` train_step calls on its toy Winograd network."""
    out = np.zeros(steps)
    _check(lib().wref_train_steps(C.c_ulonglong(seed), steps, batch, mode, _ptr(out)))
    return out
