"""ctypes binding of the C-ABI in include/wino_cuda.h (libwino_b200.so, built in-tree).

There is no fallback: if the library is missing, or a compute entry point is called
without a CUDA device, the call raises.  Status codes map onto the reference's
exception classes as its pybind11 module maps them (bindings.cpp:201-204).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# WINO_LIB_PATH: load another build of the same C-ABI (A/B experiments); default in-tree
LIB_PATH = Path(os.environ.get("WINO_LIB_PATH", Path(__file__).resolve().parent / "libwino_b200.so"))
HEADER = Path(__file__).resolve().parent.parent / "include" / "wino_cuda.h"


class WinoError(RuntimeError):
    """Base class; `.code` is the wino_status."""

    code = -1


class ShapeError(WinoError, ValueError):
    """wino::ShapeError (tensor.hpp:12) -> ValueError, as bindings.cpp:201."""

    code = 1


class ConsistencyError(WinoError):
    """wino::ConsistencyError (layer.hpp:11)."""

    code = 2


class CorruptFormatError(WinoError):
    """wino::CorruptFormatError (sparse.hpp:12)."""

    code = 3


class CapabilityError(WinoError, ValueError):
    """wino::CapabilityError (transforms.hpp:10) -> ValueError, as bindings.cpp:203."""

    code = 4


class CudaError(WinoError):
    code = 5


class InvalidArgument(WinoError, ValueError):
    code = 6


class TrainingError(RuntimeError):
    """wino::train::TrainingError (train.hpp) — a non-finite update ("divergence")."""


_BY_CODE = {cls.code: cls for cls in (ShapeError, ConsistencyError, CorruptFormatError,
                                      CapabilityError, CudaError, InvalidArgument)}


class Geometry(C.Structure):
    """wino_geometry == wino::TileGeometry (transforms.hpp:39-53)."""

    _fields_ = [(n, C.c_int64) for n in ("c", "h_i", "w_i", "h_o", "w_o", "h_op", "w_op", "h_ip",
                                         "w_ip", "m", "r", "p", "tiles_y", "tiles_x", "t")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


class Update(C.Structure):
    """wino_update (include/wino_cuda.h)."""

    _fields_ = [("lr", C.c_double), ("scale", C.c_double), ("lmbda", C.c_double), ("eps", C.c_double),
                ("beta", C.c_double), ("norm", C.c_int), ("prune", C.c_int)]


class LayerDesc(C.Structure):
    _fields_ = [("c", C.c_int), ("k", C.c_int), ("h", C.c_int), ("w", C.c_int), ("pad", C.c_int),
                ("m", C.c_int), ("r", C.c_int), ("a", C.POINTER(C.c_double)),
                ("b", C.POINTER(C.c_double)), ("device", C.c_int)]


_vp = C.c_void_p
_i64 = C.c_int64
_pd = C.POINTER(C.c_double)
_pf = C.POINTER(C.c_float)
_pu64 = C.POINTER(C.c_uint64)
_pi64 = C.POINTER(C.c_int64)

# name -> (restype, argtypes); the full list of symbols include/wino_cuda.h declares
SIGNATURES = {
    "wino_make_geometry": (C.c_int, [_i64, _i64, _i64, C.c_int, C.c_int, C.POINTER(Geometry)]),
    "wino_phi": (C.c_int, [C.POINTER(Geometry), _i64, _i64, _i64, _pi64, _pi64]),
    "wino_psi": (C.c_int, [C.POINTER(Geometry), _i64, _i64, _pi64, _pi64, _pi64]),
    "wino_transforms": (C.c_int, [C.c_int, C.c_int, _pd, _pd, _pd]),
    "wino_plan_create": (C.c_int, [C.POINTER(LayerDesc), C.POINTER(_vp)]),
    "wino_plan_destroy": (C.c_int, [_vp]),
    "wino_plan_info": (C.c_int, [_vp, C.POINTER(Geometry), _pi64, C.POINTER(C.c_int)]),
    "wino_set_weights_csr": (C.c_int, [_vp, C.POINTER(_pu64), C.POINTER(_pu64), C.POINTER(_pf), _pu64]),
    "wino_set_weights": (C.c_int, [_vp, _pd, C.c_double, C.c_int]),
    "wino_get_csr": (C.c_int, [_vp, _pu64, _pu64, _pu64, _pf]),
    "wino_weight_values": (C.c_int, [_vp, C.POINTER(_vp)]),
    "wino_values_updated": (C.c_int, [_vp, _vp]),
    "wino_cache_create": (C.c_int, [_vp, C.c_int, C.POINTER(_vp)]),
    "wino_cache_destroy": (C.c_int, [_vp]),
    "wino_forward": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, C.c_int, _vp]),
    "wino_backward_weights": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_int, _vp]),
    "wino_backward_input": (C.c_int, [_vp, _vp, _vp, _vp]),
    "wino_backward": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, C.c_int, _vp]),
    "wino_forward_backward": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "wino_forward_range": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, C.c_int, _vp]),
    "wino_backward_range": (C.c_int, [_vp, C.c_int, C.c_int, _vp, _vp, _vp, _vp, C.c_int, _vp]),
    "wino_backward_weights_cached": (C.c_int, [_vp, _vp, _vp, _vp]),
    "wino_allreduce_dw": (C.c_int, [_vp, _vp, _vp, _i64, _vp]),
    "wino_set_dw_allreduce": (C.c_int, [_vp, _vp]),
    "wino_update_weights": (C.c_int, [_vp, _vp, C.POINTER(Update), _vp]),
    "wino_sgd_step": (C.c_int, [_vp, _vp, C.c_float, C.c_float, C.c_float, _vp]),
    "wino_update_status": (C.c_int, [_vp, _pi64]),
    "wino_recompress": (C.c_int, [_vp, C.c_double]),
    "wino_set_option": (C.c_int, [_vp, C.c_int, C.c_int]),
    "wino_launch_count": (C.c_int64, [_vp]),
    "wino_reset_launch_count": (None, [_vp]),
    "wino_profile_enable": (C.c_int, [_vp, C.c_int]),
    "wino_profile_read": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_char_p), _pd, _pi64, C.POINTER(C.c_int)]),
    "wino_last_error": (C.c_char_p, []),
    "wino_version": (C.c_char_p, []),
}

WINO_OPT_DW_MODE = 1
WINO_OPT_CONTRACTION = 2
WINO_OPT_AUTO_DENSITY = 3
WINO_OPT_SPMM_OPERANDS = 4
WINO_FWD_RELU = 1
WINO_BWD_RELU_MASK = 1

_lib = None


def lib():
    """Load the library (raises FileNotFoundError when it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise FileNotFoundError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        lib_ = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib_, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib_
    return _lib


def check(rc: int):
    if rc != 0:
        msg = lib().wino_last_error().decode(errors="replace")
        raise _BY_CODE.get(rc, WinoError)(msg)
