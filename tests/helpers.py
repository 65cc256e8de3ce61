"""Shared test helpers: golden fixtures and the parity tolerance of BASELINE.json:north_star."""
from __future__ import annotations

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"

# north_star: "within rel 1e-4 / abs 1e-5 for fp32 outputs and gradients", elementwise:
#     |got - ref| <= ATOL + RTOL * |ref|
RTOL = 1e-4
ATOL = 1e-5

LAYER_CASES = ["c0", "f23_odd", "f43_odd", "f63", "f43_dense", "f43_tiny"]


def load_layer(name):
    z = np.load(GOLDEN / f"layer_{name}.npz")
    d = {k: z[k] for k in z.files}
    m, n, c, k, h, w, pad, seed = (int(v) for v in d["meta"])
    d.update(m=m, n=n, c=c, k=k, h=h, w=w, pad=pad, seed=seed)
    return d


def golden_csr_slices(d):
    """(row_ptr list, col list, val list) of the reference's compress<float>."""
    offs = np.concatenate([[0], np.cumsum(d["csr_nnz"])])
    p2 = len(d["csr_nnz"])
    return ([d["csr_row_ptr"][s] for s in range(p2)],
            [d["csr_col"][offs[s]:offs[s + 1]] for s in range(p2)],
            [d["csr_val"][offs[s]:offs[s + 1]] for s in range(p2)])


def fail_fraction(got, ref, rtol=RTOL, atol=ATOL):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    bad = np.abs(got - ref) > atol + rtol * np.abs(ref)
    return float(bad.mean()) if bad.size else 0.0


def assert_parity(got, ref, what, rtol=RTOL, atol=ATOL):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, f"{what}: shape {got.shape} != {ref.shape}"
    bad = np.abs(got - ref) > atol + rtol * np.abs(ref)
    if bad.any():
        i = np.unravel_index(np.argmax(np.abs(got - ref) - rtol * np.abs(ref)), got.shape)
        raise AssertionError(f"{what}: {int(bad.sum())}/{bad.size} elements outside "
                             f"{atol}+{rtol}|ref|; worst at {i}: got {got[i]!r} ref {ref[i]!r}")
