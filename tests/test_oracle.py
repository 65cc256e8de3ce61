"""Pin the oracle (oracle/wino_oracle.py) before trusting it: against the golden vectors the
reference produced (tests/golden, always), and against the compiled reference itself
(oracle/_ref) on extra random cases when it is built.  CPU only."""
from __future__ import annotations

import numpy as np
import pytest

from helpers import GOLDEN, LAYER_CASES, assert_parity, golden_csr_slices, load_layer
from oracle import ref
from oracle import wino_oracle as wo

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("m", [2, 3, 4, 6])
def test_transforms_bit_exact_vs_golden(m):
    z = np.load(GOLDEN / "transforms.npz")
    a, b, g = wo.transforms(m)
    for mine, key in ((a, "A"), (b, "B"), (g, "G")):
        gold = z[f"{key}{m}"]
        assert mine.shape == gold.shape
        assert np.array_equal(mine.view(np.int64), gold.view(np.int64)), f"{key}{m} not bit-identical"


def test_f43_constants_match_survey_values():
    a, b, _ = wo.transforms(4)
    assert np.array_equal(a[3], [1, 2, 4, 8]) and np.array_equal(a[4], [1, -2, 4, -8])
    assert b[1, 5] == 4.0 and b[3, 5] == -5.0 and b[2, 0] == -1.25 and b[4, 0] == 0.25
    assert b[1, 1] == 2.0 / 3.0 and b[2, 3] == -1.0 / 24.0


def test_cook_toom_rejects_unsupported_sizes():
    # test_transforms.cpp:99-102
    with pytest.raises(ValueError):
        wo.cook_toom_1d(7, 3)
    with pytest.raises(ValueError):
        wo.cook_toom_1d(6, 5)


def test_geometry_phi_psi_vs_golden():
    z = np.load(GOLDEN / "geometry.npz")
    for key in [k[5:] for k in z.files if k.startswith("geom_")]:
        c, h, w, m = (int(v) for v in key.split("_"))
        g = wo.make_geometry(c, h, w, m)
        gold = z["geom_" + key]
        mine = [g.c, g.h_i, g.w_i, g.h_o, g.w_o, g.h_op, g.w_op, g.h_ip, g.w_ip, g.p, g.p, g.tiles_y,
                g.tiles_x, g.t]
        assert mine == gold.tolist(), key
        for t, i, j, y, x in z["phi_" + key]:
            assert wo.phi(g, t, i, j) == (y, x)
        for y, x, t, i, j in z["psi_" + key]:
            assert wo.psi(g, y, x) == (t, i, j)


def test_geometry_hand_values():
    # test_transforms.cpp:104-153
    g = wo.make_geometry(3, 6, 6, 2)
    assert (g.h_o, g.h_op, g.tiles_y, g.t) == (4, 4, 2, 4)
    g = wo.make_geometry(1, 7, 9, 2)
    assert (g.h_o, g.w_o, g.h_op, g.w_op, g.tiles_y, g.tiles_x, g.h_ip, g.w_ip) == (5, 7, 6, 8, 3, 4, 8, 10)
    g = wo.make_geometry(1, 12, 12, 2)
    assert g.tiles_x == 5
    assert wo.phi(g, 1, 0, 0) == (0, 2) and wo.phi(g, 3, 3, 3) == (3, 9) and wo.phi(g, 6, 1, 2) == (3, 4)
    assert wo.psi(g, 3, 2) == (6, 1, 0)
    with pytest.raises(ValueError):
        wo.make_geometry(1, 2, 5, 2)


@pytest.mark.parametrize("name", LAYER_CASES)
def test_f64_layer_vs_golden(name):
    d = load_layer(name)
    pad, m = d["pad"], d["m"]
    gw = np.zeros_like(d["w_f"])
    for i in range(d["n"]):
        imgp = np.pad(d["img"][i].astype(np.float64), ((0, 0), (pad, pad), (pad, pad)))
        o, cache = wo.forward_f64(imgp, d["w_f"], m)
        np.testing.assert_allclose(o, d["o_f64"][i], rtol=1e-11, atol=1e-11)
        gw += wo.backward_weights_f64(d["grad_o"][i].astype(np.float64), cache)
        gi = wo.backward_input_f64(cache, d["w_f"])[:, pad:pad + d["h"], pad:pad + d["w"]]
        np.testing.assert_allclose(gi, d["grad_in_f64"][i], rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(gw, d["grad_wf_f64"], rtol=1e-11, atol=1e-10)


@pytest.mark.parametrize("name", LAYER_CASES)
def test_compress_bit_exact_vs_golden(name):
    d = load_layer(name)
    csr = wo.compress(d["w_f"])
    rps, cols, vals = golden_csr_slices(d)
    for s in range(len(rps)):
        assert np.array_equal(csr.row_ptr[s], rps[s])
        assert np.array_equal(csr.col_idx[s], cols[s])
        assert np.array_equal(csr.values[s].view(np.int32), vals[s].view(np.int32))
    assert np.array_equal(wo.reconstruct(csr), d["w_f"])


@pytest.mark.parametrize("name", LAYER_CASES)
def test_f32_mirror_forward_bitwise_vs_reference_sparse_f32(name):
    """The f32 mirror reproduces the reference's own f32 sparse_forward bit for bit."""
    d = load_layer(name)
    res = wo.layer_f32(d["img"], wo.compress(d["w_f"]), None, m=d["m"], pad=d["pad"])
    assert np.array_equal(res["o"].astype(np.float64), d["o_sparse_f32"])


@pytest.mark.parametrize("name", LAYER_CASES)
def test_f32_mirror_backward_within_tolerance_of_f64_reference(name):
    d = load_layer(name)
    csr = wo.compress(d["w_f"])
    res = wo.layer_f32(d["img"], csr, d["grad_o"], m=d["m"], pad=d["pad"])
    assert_parity(res["di"], d["grad_in_f64"], "dI")
    dw = wo.reconstruct(wo.Csr(csr.k, csr.c, csr.p, csr.row_ptr, csr.col_idx,
                               [v.astype(np.float32) for v in res["dw"]]))
    mask = d["w_f"] != 0
    assert_parity(dw[mask], d["grad_wf_f64"][mask], "dW_F on the mask")


@needs_ref
@pytest.mark.parametrize("seed", range(6))
def test_f64_oracle_vs_compiled_reference_random(seed):
    rng = np.random.default_rng(seed)
    m = [2, 4, 6][seed % 3]
    c, k = rng.integers(1, 5, size=2)
    h, w = rng.integers(m + 2, 17, size=2)
    img = rng.uniform(-1, 1, (c, h, w))
    w_f = rng.uniform(-1, 1, (k, c, m + 2, m + 2))
    go = rng.uniform(-1, 1, (k, h - 2, w - 2))
    r = ref.layer(img, w_f, go, m=m)
    o, cache = wo.forward_f64(img, w_f, m)
    np.testing.assert_allclose(o, r["o"], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(cache["i_f"], r["i_f"], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(wo.backward_weights_f64(go, cache), r["grad_wf"], rtol=1e-10, atol=1e-9)
    np.testing.assert_allclose(cache["grad_z"], r["grad_z"], rtol=1e-10, atol=1e-9)
    np.testing.assert_allclose(wo.backward_input_f64(cache, w_f), r["grad_in"], rtol=1e-10, atol=1e-9)


@needs_ref
@pytest.mark.parametrize("seed", range(4))
def test_f32_mirror_vs_compiled_reference_random(seed):
    rng = np.random.default_rng(100 + seed)
    m = [2, 4, 6, 4][seed]
    n, c, k = 2, int(rng.integers(1, 6)), int(rng.integers(1, 6))
    h, w = (int(v) for v in rng.integers(m + 2, 19, size=2))
    batch = rng.standard_normal((n, c, h, w)).astype(np.float32).astype(np.float64)
    w_f = rng.standard_normal((k, c, m + 2, m + 2)).astype(np.float32).astype(np.float64)
    w_f[rng.uniform(size=w_f.shape) < 0.6] = 0.0
    out = ref.sparse_forward(batch, w_f, m=m, workers=3, precision=32)
    res = wo.layer_f32(batch, wo.compress(w_f), None, m=m, pad=0)
    assert np.array_equal(res["o"].astype(np.float64), out)
    assert np.array_equal(res["v"][:, :, : res["g"].t], ref.tiled_layout_f32(batch[0], m=m))


def test_direct_conv_equals_lifted_winograd():
    # test_layer.cpp:58-68 / acceptance criterion 1 on the oracle
    rng = np.random.default_rng(51)
    img = rng.uniform(-1, 1, (2, 10, 10))
    w = rng.uniform(-1, 1, (2, 2, 3, 3))
    o, _ = wo.forward_f64(img, wo.lift_f64(w, 4), 4)
    np.testing.assert_allclose(o, wo.direct_conv_f64(img, w), atol=1e-9)
