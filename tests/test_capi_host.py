"""C-ABI library: loads, exports every symbol include/wino_cuda.h declares, and its host-only
entry points (transforms, geometry, φ/ψ, errors) match the reference.  No GPU needed."""
from __future__ import annotations

import ctypes as C
import re

import numpy as np
import pytest

from helpers import GOLDEN
import paper_1702_08597_b200 as wb
from paper_1702_08597_b200 import _lib


def header_symbols():
    text = _lib.HEADER.read_text()
    return sorted(set(re.findall(r"WINO_API\s+[\w\s\*]*?\b(wino_\w+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 20
    lib = C.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(_lib.SIGNATURES), "ctypes signature table out of sync with the header"


def test_library_is_sm100a():
    data = _lib.LIB_PATH.read_bytes()
    assert b"sm_100a" in data


@pytest.mark.parametrize("m", [2, 3, 4, 6])
def test_transforms_bit_identical_to_reference(m):
    z = np.load(GOLDEN / "transforms.npz")
    a, b, g = wb.transforms(m)
    for mine, key in ((a, "A"), (b, "B"), (g, "G")):
        assert np.array_equal(mine.view(np.int64), z[f"{key}{m}"].view(np.int64))


def test_transforms_capability_error():
    with pytest.raises(wb.CapabilityError):
        wb.transforms(7, 3)
    with pytest.raises(ValueError):  # reference maps CapabilityError to ValueError
        wb.gen_transforms(m=7, r=3)


def test_gen_transforms_surface():
    # python/tests/test_smoke.py:11-18
    t = wb.gen_transforms(m=2, r=3)
    assert t["A1"].shape == (4, 2) and t["B1"].shape == (4, 4) and t["G1"].shape == (4, 3)
    np.testing.assert_array_equal(t["G1"], [[1, 0, 0], [0.5, 0.5, 0.5], [0.5, -0.5, 0.5], [0, 0, 1]])


def test_geometry_phi_psi_vs_golden():
    z = np.load(GOLDEN / "geometry.npz")
    lib = _lib.lib()
    for key in [k[5:] for k in z.files if k.startswith("geom_")]:
        c, h, w, m = (int(v) for v in key.split("_"))
        g = _lib.Geometry()
        _lib.check(lib.wino_make_geometry(c, h, w, m, 3, C.byref(g)))
        gd = g.as_dict()
        mine = [gd[f] for f in ("c", "h_i", "w_i", "h_o", "w_o", "h_op", "w_op", "h_ip", "w_ip", "p",
                                "p", "tiles_y", "tiles_x", "t")]
        assert mine == z["geom_" + key].tolist()
        y, x = C.c_int64(), C.c_int64()
        for t, i, j, yy, xx in z["phi_" + key][::7]:
            _lib.check(lib.wino_phi(C.byref(g), int(t), int(i), int(j), C.byref(y), C.byref(x)))
            assert (y.value, x.value) == (yy, xx)
        t_, i_, j_ = C.c_int64(), C.c_int64(), C.c_int64()
        for yy, xx, t, i, j in z["psi_" + key][::5]:
            _lib.check(lib.wino_psi(C.byref(g), int(yy), int(xx), C.byref(t_), C.byref(i_), C.byref(j_)))
            assert (t_.value, i_.value, j_.value) == (t, i, j)
        with pytest.raises(wb.ShapeError):
            _lib.check(lib.wino_phi(C.byref(g), g.t, 0, 0, C.byref(y), C.byref(x)))
        with pytest.raises(wb.ShapeError):
            _lib.check(lib.wino_psi(C.byref(g), g.h_op, 0, C.byref(t_), C.byref(i_), C.byref(j_)))


def test_geometry_shape_error():
    with pytest.raises(wb.ShapeError):
        wb.make_geometry(1, 2, 5, 2)


def test_plan_rejects_unbuilt_shapes():
    with pytest.raises(wb.CapabilityError):
        wb.WinogradLayer(4, 4, 8, 8, m=3)
    with pytest.raises(wb.ShapeError):
        wb.WinogradLayer(0, 4, 8, 8)


def test_host_compress_matches_reference_golden():
    from helpers import golden_csr_slices, load_layer

    for name in ("c0", "f63"):
        d = load_layer(name)
        csr = wb.compress(d["w_f"])
        rps, cols, vals = golden_csr_slices(d)
        for s in range(len(rps)):
            assert np.array_equal(csr.row_ptr[s].astype(np.int64), rps[s])
            assert np.array_equal(csr.col_idx[s].astype(np.int64), cols[s])
            assert np.array_equal(csr.values[s], vals[s])
        assert np.array_equal(wb.reconstruct(csr), d["w_f"])


def test_compress_zero_tolerance_rule():
    # test_sparse.cpp:40-46
    w = np.array([0.5, 1e-9, 0.0, -2.0]).reshape(1, 1, 2, 2)
    assert wb.compress(w).nnz_total() == 3
    assert wb.compress(w, 1e-6).nnz_total() == 2


def test_density():
    w = np.zeros((2, 2, 3, 3))
    w[0, 0, 0, 0] = 1
    assert wb.density(w) == 1 / 36


def test_compute_entry_points_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(wb.CudaError):
        wb.WinogradLayer(16, 16, 12, 12)


def test_builtin_coefficient_header_matches_reference():
    """csrc/builtin_coefs.h (compile-time coefficients of the specialised transform kernels)
    holds exactly the fp32 casts of the reference's TransformSet doubles."""
    import re

    text = (_lib.LIB_PATH.parent / "csrc" / "builtin_coefs.h").read_text()
    z = np.load(GOLDEN / "transforms.npz")
    for m in (2, 4, 6):
        blk = text[text.index(f"struct BuiltinCoefs<{m}, {m + 2}>"):]
        for key in ("a", "b"):
            body = re.search(rf"static constexpr float {key}\[\d+\] = \{{([^}}]*)\}}", blk).group(1)
            vals = np.array([float.fromhex(v.strip()[:-1]) if "0x" in v else float(v.strip()[:-1])
                             for v in body.split(",")], dtype=np.float32)
            ref = z[f"{key.upper()}{m}"].astype(np.float32).ravel()
            assert np.array_equal(vals.view(np.int32), ref.view(np.int32)), (m, key)
