"""Host-side mirror of the reference layer interface, over the C-ABI.

`WinogradLayer` is the batched, device-resident form of the reference's per-layer
state (TransformSet + TileGeometry + W_F, layer.hpp:28-43 / sparse.hpp:78-82);
`ForwardCache` is layer.hpp:19-25 on the device.  PyTorch is used only to own
device memory and to name the current CUDA stream.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import Geometry, LayerDesc, check, lib


def _stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _dptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def transforms(m: int, r: int = 3):
    """(A p×m, B p×p, G p×r) doubles, bit-identical to the reference (transforms.cpp:7-145)."""
    p = m + r - 1
    if p > 8 or m < 1 or r < 1:
        # let the library produce the reference's CapabilityError message
        a = np.zeros(64)
        check(lib().wino_transforms(m, r, a.ctypes.data_as(_lib._pd), a.ctypes.data_as(_lib._pd),
                                    a.ctypes.data_as(_lib._pd)))
    a, b, g = np.zeros((p, m)), np.zeros((p, p)), np.zeros((p, r))
    check(lib().wino_transforms(m, r, a.ctypes.data_as(_lib._pd), b.ctypes.data_as(_lib._pd),
                                g.ctypes.data_as(_lib._pd)))
    return a, b, g


def make_geometry(c, h_i, w_i, m=4, r=3) -> dict:
    g = Geometry()
    check(lib().wino_make_geometry(c, h_i, w_i, m, r, C.byref(g)))
    return g.as_dict()


@dataclass
class PointwiseCsr:
    """PointwiseCsr<float> (sparse.hpp:19-38): p·q K×C slices, (i,j) row-major."""

    k: int
    c: int
    p: int
    row_ptr: list = field(default_factory=list)   # p·q uint64 arrays of K+1
    col_idx: list = field(default_factory=list)   # p·q uint64 arrays
    values: list = field(default_factory=list)    # p·q float32 arrays

    def nnz_total(self) -> int:
        return int(sum(len(v) for v in self.values))

    def density(self) -> float:
        return self.nnz_total() / float(self.k * self.c * self.p * self.p)


def compress(w_f, zero_tol: float = 0.0) -> PointwiseCsr:
    """compress<float> (sparse.cpp:9-36) on the host: keep |v| > zero_tol (v != 0 at 0)."""
    w_f = np.asarray(w_f, dtype=np.float64)
    if w_f.ndim != 4 or w_f.shape[2] != w_f.shape[3]:
        raise _lib.ShapeError(f"compress: expected K x C x p x q weights, got {w_f.shape}")
    k, c, p, _ = w_f.shape
    csr = PointwiseCsr(k, c, p)
    for i in range(p):
        for j in range(p):
            sl = w_f[:, :, i, j]
            keep = (np.abs(sl) > zero_tol) | ((zero_tol == 0.0) & (sl != 0.0))
            rk, ck = np.nonzero(keep)
            rp = np.zeros(k + 1, dtype=np.uint64)
            rp[1:] = np.cumsum(np.bincount(rk, minlength=k)).astype(np.uint64)
            csr.row_ptr.append(rp)
            csr.col_idx.append(ck.astype(np.uint64))
            csr.values.append(sl[rk, ck].astype(np.float32))
    return csr


def reconstruct(csr: PointwiseCsr):
    """sparse.cpp:38-49: K×C×p×q f64 from the CSR."""
    w = np.zeros((csr.k, csr.c, csr.p, csr.p))
    for s in range(csr.p * csr.p):
        i, j = divmod(s, csr.p)
        rows = np.repeat(np.arange(csr.k), np.diff(csr.row_ptr[s].astype(np.int64)))
        w[rows, csr.col_idx[s].astype(np.int64), i, j] = csr.values[s].astype(np.float64)
    return w


class ForwardCache:
    """Device ForwardCache (layer.hpp:19-25): Ĩ_F and dL/dZ for up to n_max images."""

    def __init__(self, layer: "WinogradLayer", n_max: int):
        self.layer = layer
        self.n_max = n_max
        self._h = C.c_void_p()
        check(lib().wino_cache_create(layer._h, n_max, C.byref(self._h)))
        self.n = 0

    def close(self):
        if self._h:
            lib().wino_cache_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class WinogradLayer:
    """One Winograd layer on one GPU: F(m×m,3×3) with `pad` folded into φ."""

    def __init__(self, c: int, k: int, h: int, w: int, pad: int = 1, m: int = 4, r: int = 3,
                 device: int = 0, a=None, b=None):
        self.c, self.k, self.h, self.w, self.pad, self.m, self.r = c, k, h, w, pad, m, r
        self.device = device
        desc = LayerDesc(c, k, h, w, pad, m, r, None, None, device)
        if a is not None:
            self._a = np.ascontiguousarray(a, dtype=np.float64)
            self._b = np.ascontiguousarray(b, dtype=np.float64)
            desc.a = self._a.ctypes.data_as(_lib._pd)
            desc.b = self._b.ctypes.data_as(_lib._pd)
        self._h = C.c_void_p()
        check(lib().wino_plan_create(C.byref(desc), C.byref(self._h)))
        g = Geometry()
        check(lib().wino_plan_info(self._h, C.byref(g), None, None))
        self.geometry = g.as_dict()
        self.p = self.geometry["p"]
        self.ho, self.wo = self.geometry["h_o"], self.geometry["w_o"]

    # -- weights ------------------------------------------------------------------
    def set_weights(self, w_f, zero_tol: float = 0.0, dense: bool | str | None = None):
        """W_F (K×C×p×q).
        dense=False: CSR of the nonzeros (the sparse path).  dense=None: dense when no entry is
        dropped.  dense=True / 'tc': every coordinate is a weight; Z and dĨ_F run on the tensor
        cores (3xTF32 tcgen05, compensated fp32 fold per k-block — fp32-level accuracy).
        dense='exact': the reference-order SIMT kernels (bitwise forward).  dW_F is the exact
        int8 digit GEMM on every plan (to the reference's f64 accuracy)."""
        w_f = np.ascontiguousarray(w_f, dtype=np.float64)
        if w_f.shape != (self.k, self.c, self.p, self.p):
            raise _lib.ShapeError(f"weights {w_f.shape} do not match layer "
                                  f"{(self.k, self.c, self.p, self.p)}")
        if dense is None:
            kept = (np.abs(w_f) > zero_tol) | ((zero_tol == 0.0) & (w_f != 0.0))
            dense = bool(kept.all())
        mode = ({"tc": 2, "exact": 1}.get(dense, None) if isinstance(dense, str)
                else (2 if dense else 0))
        if mode is None:
            raise _lib.InvalidArgument(f"dense must be None, bool, 'tc' or 'exact', got {dense!r}")
        check(lib().wino_set_weights(self._h, w_f.ctypes.data_as(_lib._pd), zero_tol, mode))

    def set_weights_csr(self, csr: PointwiseCsr):
        n = self.p * self.p
        rps = [np.ascontiguousarray(x, dtype=np.uint64) for x in csr.row_ptr]
        cols = [np.ascontiguousarray(x, dtype=np.uint64) for x in csr.col_idx]
        vals = [np.ascontiguousarray(x, dtype=np.float32) for x in csr.values]
        if len(rps) != n or len(cols) != n or len(vals) != n:
            raise _lib.CorruptFormatError(f"expected {n} slices")
        self._keep = (rps, cols, vals)
        arr_rp = (_lib._pu64 * n)(*[x.ctypes.data_as(_lib._pu64) for x in rps])
        arr_c = (_lib._pu64 * n)(*[x.ctypes.data_as(_lib._pu64) for x in cols])
        arr_v = (_lib._pf * n)(*[x.ctypes.data_as(_lib._pf) for x in vals])
        nnz = np.array([len(v) for v in vals], dtype=np.uint64)
        check(lib().wino_set_weights_csr(self._h, arr_rp, arr_c, arr_v, nnz.ctypes.data_as(_lib._pu64)))

    @property
    def nnz(self) -> int:
        n = C.c_int64()
        check(lib().wino_plan_info(self._h, None, C.byref(n), None))
        return int(n.value)

    @property
    def is_dense(self) -> bool:
        d = C.c_int()
        check(lib().wino_plan_info(self._h, None, None, C.byref(d)))
        return bool(d.value)

    def get_csr(self) -> PointwiseCsr:
        n = self.p * self.p
        nnz = np.zeros(n, dtype=np.uint64)
        check(lib().wino_get_csr(self._h, nnz.ctypes.data_as(_lib._pu64), None, None, None))
        tot = int(nnz.sum())
        rp = np.zeros((n, self.k + 1), dtype=np.uint64)
        col = np.zeros(max(tot, 1), dtype=np.uint64)
        val = np.zeros(max(tot, 1), dtype=np.float32)
        check(lib().wino_get_csr(self._h, nnz.ctypes.data_as(_lib._pu64), rp.ctypes.data_as(_lib._pu64),
                                 col.ctypes.data_as(_lib._pu64), val.ctypes.data_as(_lib._pf)))
        offs = np.concatenate([[0], np.cumsum(nnz.astype(np.int64))])
        return PointwiseCsr(self.k, self.c, self.p, [rp[s].copy() for s in range(n)],
                            [col[offs[s]:offs[s + 1]].copy() for s in range(n)],
                            [val[offs[s]:offs[s + 1]].copy() for s in range(n)])

    def set_dw_mode(self, mode: str):
        """dW_F has one mode, 'exact': Ĩ_F and dZ recomputed in f64 from I and dO, split into five
        int8 digits and multiplied exactly on the int8 tensor cores (the reference's f64 dW_F
        within ~2^-35 of Σ|products|).  Any other name raises InvalidArgument."""
        check(lib().wino_set_option(self._h, _lib.WINO_OPT_DW_MODE, {"exact": 0}.get(mode, -1)))

    def set_contraction(self, mode: str):
        """Sparse plan contractions: 'csr' (default; the reference's order, forward bitwise equal
        to sparse_forward<float>), 'tc' (3xTF32 tcgen05 GEMM over the zero-filled W_F slices) or
        'auto' (tensor cores at density >= set_auto_density's value, else 'csr')."""
        check(lib().wino_set_option(self._h, _lib.WINO_OPT_CONTRACTION, {"csr": 0, "tc": 1, "auto": 2}[mode]))

    def set_spmm_operands(self, where: str):
        """CSR kernels' dense operand chunk: 'auto' (default; tensor memory where it is measured
        faster: 128 < rows <= 512, density >= 4%, enough work units — the hybrid split when its
        stream fits in shared memory), 'smem' (shared memory always), 'tmem' (tensor memory whenever
        128 < rows <= 512) or 'hybrid' (rows [0,128) in tensor memory, the rest in shared memory,
        whenever 128 < rows <= 256).  Bitwise the same results."""
        check(lib().wino_set_option(self._h, _lib.WINO_OPT_SPMM_OPERANDS, {"auto": 0, "smem": 1, "tmem": 2, "hybrid": 3}[where]))

    def set_auto_density(self, density: float):
        """Density from which contraction 'auto' uses the tensor cores (default: the measured
        crossover, 0.11 for 128 < C, K <= 256 and 0.08 otherwise)."""
        check(lib().wino_set_option(self._h, _lib.WINO_OPT_AUTO_DENSITY, int(round(density * 1000))))

    def weight_values(self):
        """Device pointer (int) of the live CSR values (nnz floats)."""
        ptr = C.c_void_p()
        check(lib().wino_weight_values(self._h, C.byref(ptr)))
        return ptr.value

    def values_updated(self, stream=None):
        """The values behind weight_values() were modified in place: refresh the derived
        operands (CSC copy, tensor-core splits)."""
        check(lib().wino_values_updated(self._h, _stream_ptr(stream)))

    # -- passes ---------------------------------------------------------------------
    def new_cache(self, n_max: int) -> ForwardCache:
        return ForwardCache(self, n_max)

    def _check_dev(self, t, shape, name):
        import torch

        if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
            raise _lib.ShapeError(f"{name}: expected a contiguous float32 CUDA tensor")
        if tuple(t.shape) != tuple(shape):
            raise _lib.ShapeError(f"{name}: shape {tuple(t.shape)} != {tuple(shape)}")

    def forward(self, x, cache: ForwardCache | None = None, relu: bool = False, out=None, stream=None):
        import torch

        n = x.shape[0]
        self._check_dev(x, (n, self.c, self.h, self.w), "input")
        if out is None:
            out = torch.empty((n, self.k, self.ho, self.wo), device=x.device, dtype=torch.float32)
        self._check_dev(out, (n, self.k, self.ho, self.wo), "output")
        check(lib().wino_forward(self._h, n, _dptr(x), _dptr(out), cache._h if cache else None,
                                 _lib.WINO_FWD_RELU if relu else 0, _stream_ptr(stream)))
        if cache is not None:
            cache.n = n
        return out

    def grad_w_shape(self):
        return (self.k, self.c, self.p, self.p) if self.is_dense else (self.nnz,)

    def backward_weights(self, grad_o, cache: ForwardCache, relu_out=None, out=None, stream=None):
        import torch

        n = cache.n
        self._check_dev(grad_o, (n, self.k, self.ho, self.wo), "grad_output")
        if relu_out is not None:
            self._check_dev(relu_out, (n, self.k, self.ho, self.wo), "relu_out")
        if out is None:
            out = torch.empty(self.grad_w_shape(), device=grad_o.device, dtype=torch.float32)
        check(lib().wino_backward_weights(self._h, _dptr(grad_o), _dptr(relu_out), cache._h, _dptr(out),
                                          _lib.WINO_BWD_RELU_MASK if relu_out is not None else 0,
                                          _stream_ptr(stream)))
        return out

    def set_dw_allreduce(self, comm=None):
        """Run the data-parallel dW_F exchange inside every backward (wino_set_dw_allreduce): right
        after the dW_F kernels, on their stream, overlapping the dI chain.  `comm`: an ncclComm_t
        address, a torch.distributed NCCL process group (its communicator), or None (off)."""
        if comm is not None and not isinstance(comm, int):
            from .dist import nccl_comm_ptr

            comm = nccl_comm_ptr(comm, self.device)
        check(lib().wino_set_dw_allreduce(self._h, C.c_void_p(comm or 0)))

    def allreduce_dw(self, grad_w, nccl_comm: int, count: int = -1, stream=None):
        """Sum grad_w in place over an NCCL communicator (an ncclComm_t address)."""
        check(lib().wino_allreduce_dw(self._h, C.c_void_p(nccl_comm), _dptr(grad_w), count, _stream_ptr(stream)))
        return grad_w

    def backward(self, grad_o, cache: ForwardCache, relu_out=None, out_w=None, out_i=None, stream=None,
                 want_input_grad: bool = True):
        """backward_weights + backward_input in one call, dW_F computed concurrently with dI
        (want_input_grad=False: dW_F only, as for the first layer of a stack)."""
        import torch

        n = cache.n
        self._check_dev(grad_o, (n, self.k, self.ho, self.wo), "grad_output")
        if relu_out is not None:
            self._check_dev(relu_out, (n, self.k, self.ho, self.wo), "relu_out")
        if out_w is None:
            out_w = torch.empty(self.grad_w_shape(), device=grad_o.device, dtype=torch.float32)
        if out_i is None and want_input_grad:
            out_i = torch.empty((max(n, 1), self.c, self.h, self.w), device=grad_o.device, dtype=torch.float32)
        check(lib().wino_backward(self._h, _dptr(grad_o), _dptr(relu_out), cache._h, _dptr(out_w), _dptr(out_i),
                                  _lib.WINO_BWD_RELU_MASK if relu_out is not None else 0, _stream_ptr(stream)))
        return out_w, out_i

    def forward_backward(self, x, grad_o, cache: ForwardCache, out=None, out_w=None, out_i=None, stream=None):
        """forward + backward (dW_F and dI) in one call, scheduled by data dependence: the dI chain
        and dW_F overlap the forward (wino_forward_backward; bitwise the two-call results)."""
        import torch

        n = x.shape[0]
        self._check_dev(x, (n, self.c, self.h, self.w), "input")
        self._check_dev(grad_o, (n, self.k, self.ho, self.wo), "grad_output")
        if out is None:
            out = torch.empty((n, self.k, self.ho, self.wo), device=x.device, dtype=torch.float32)
        if out_w is None:
            out_w = torch.empty(self.grad_w_shape(), device=x.device, dtype=torch.float32)
        if out_i is None:
            out_i = torch.empty((n, self.c, self.h, self.w), device=x.device, dtype=torch.float32)
        check(lib().wino_forward_backward(self._h, n, _dptr(x), _dptr(out), cache._h, _dptr(grad_o), _dptr(out_w),
                                          _dptr(out_i), _stream_ptr(stream)))
        cache.n = n
        return out, out_w, out_i

    # -- image ranges of one batch (pipelined host transfers, pipeline.PipelinedHostStep) --------
    def forward_range(self, x_part, n_total: int, n0: int, cache: ForwardCache, out_part, relu=False,
                      stream=None):
        """Images [n0, n0 + len(x_part)) of an n_total batch into `cache` (CSR plans only)."""
        n1 = n0 + x_part.shape[0]
        self._check_dev(x_part, (n1 - n0, self.c, self.h, self.w), "input")
        self._check_dev(out_part, (n1 - n0, self.k, self.ho, self.wo), "output")
        check(lib().wino_forward_range(self._h, n_total, n0, n1, _dptr(x_part), _dptr(out_part), cache._h,
                                       _lib.WINO_FWD_RELU if relu else 0, _stream_ptr(stream)))
        cache.n = n_total
        return out_part

    def backward_range(self, g_part, n0: int, cache: ForwardCache, out_part, relu_part=None, stream=None):
        """dL/dZ, dĨ_F and dI of images [n0, n0 + len(g_part)) (after their forward_range)."""
        n1 = n0 + g_part.shape[0]
        self._check_dev(g_part, (n1 - n0, self.k, self.ho, self.wo), "grad_output")
        self._check_dev(out_part, (n1 - n0, self.c, self.h, self.w), "grad_input")
        if relu_part is not None:
            self._check_dev(relu_part, (n1 - n0, self.k, self.ho, self.wo), "relu_out")
        check(lib().wino_backward_range(self._h, n0, n1, _dptr(g_part), _dptr(relu_part), cache._h,
                                        _dptr(out_part), _lib.WINO_BWD_RELU_MASK if relu_part is not None else 0,
                                        _stream_ptr(stream)))
        return out_part

    def backward_weights_cached(self, cache: ForwardCache, out=None, stream=None):
        """dW_F over the whole batch once every backward_range has run."""
        import torch

        if out is None:
            out = torch.empty(self.grad_w_shape(), device=f"cuda:{self.device}", dtype=torch.float32)
        check(lib().wino_backward_weights_cached(self._h, cache._h, _dptr(out), _stream_ptr(stream)))
        return out

    def backward_input(self, cache: ForwardCache, out=None, stream=None):
        import torch

        if out is None:
            out = torch.empty((max(cache.n, 1), self.c, self.h, self.w), device=f"cuda:{self.device}",
                              dtype=torch.float32)
        check(lib().wino_backward_input(self._h, cache._h, _dptr(out), _stream_ptr(stream)))
        return out

    def sgd_step(self, grad_w, lr: float, scale: float = 1.0, l2: float = 0.0, stream=None):
        """Masked SGD (fine-tune): update(norm=2, lmbda=l2)."""
        check(lib().wino_sgd_step(self._h, _dptr(grad_w), lr, scale, l2, _stream_ptr(stream)))

    def update(self, grad_w, lr: float, scale: float = 1.0, lmbda: float = 0.0, norm: int = 1,
               prune: bool = False, eps: float = 0.0, beta: float = 0.0, stream=None):
        """train_step's per-layer update (train.cpp:255-290): regulariser λ‖w‖_norm, SGD, and in
        prune mode the gradient threshold |v|·(|g|+β) < ε → 0.  Asynchronous; divergence is
        reported by check_finite()."""
        u = _lib.Update(lr, scale, lmbda, eps, beta, norm, int(bool(prune)))
        check(lib().wino_update_weights(self._h, _dptr(grad_w), C.byref(u), _stream_ptr(stream)))

    def check_finite(self, name: str = "winograd layer"):
        """Raise TrainingError if an update since the last check produced a non-finite weight."""
        n = C.c_int64()
        check(lib().wino_update_status(self._h, C.byref(n)))
        if n.value:
            raise _lib.TrainingError(f"train_step: divergence in {name} ({n.value} non-finite weights)")

    def recompress(self, zero_tol: float = 0.0):
        """Re-derive the CSR from the live weights (compress of them, on the device): after
        pruning steps the plan keeps only the surviving coordinates (set_masks_from_zeros)."""
        check(lib().wino_recompress(self._h, zero_tol))

    def weights(self) -> np.ndarray:
        """The live weights as K×C×p×q f64 (zeros off the CSR)."""
        return reconstruct(self.get_csr())

    # -- instrumentation ------------------------------------------------------------
    def launch_count(self) -> int:
        return int(lib().wino_launch_count(self._h))

    def reset_launch_count(self):
        lib().wino_reset_launch_count(self._h)

    def profile(self, enable: bool):
        check(lib().wino_profile_enable(self._h, int(enable)))

    def profile_read(self) -> dict:
        cap = 32
        names = (C.c_char_p * cap)()
        ms = np.zeros(cap)
        cnt = np.zeros(cap, dtype=np.int64)
        nk = C.c_int()
        check(lib().wino_profile_read(self._h, cap, names, ms.ctypes.data_as(_lib._pd),
                                      cnt.ctypes.data_as(_lib._pi64), C.byref(nk)))
        return {names[i].decode(): (float(ms[i]), int(cnt[i])) for i in range(nk.value) if cnt[i]}

    def close(self):
        if self._h:
            h, self._h = self._h, C.c_void_p()
            check(lib().wino_plan_destroy(h))

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def compact_to_dense(self, dw_compact: np.ndarray, csr: PointwiseCsr | None = None) -> np.ndarray:
        """Scatter an nnz-compact dW (CSR order) into K×C×p×q (zeros off the mask)."""
        csr = csr or self.get_csr()
        out = np.zeros((self.k, self.c, self.p, self.p))
        off = 0
        for s in range(self.p * self.p):
            i, j = divmod(s, self.p)
            n = len(csr.values[s])
            rows = np.repeat(np.arange(self.k), np.diff(csr.row_ptr[s].astype(np.int64)))
            out[rows, csr.col_idx[s].astype(np.int64), i, j] = dw_compact[off:off + n]
            off += n
        return out
