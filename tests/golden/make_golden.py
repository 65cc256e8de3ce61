"""Generate tests/golden/*.npz from the REAL reference (oracle/_ref, built from
/root/reference by oracle/Makefile).  Run in the build container:

    make -C oracle && python tests/golden/make_golden.py

Everything numeric in the fixtures comes out of reference code (ref_shim.cpp only
marshals pointers).  Inputs come from the repo's portable seeded generator
(paper_1702_08597_b200.synth), so they are reproducible, and are stored too.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402
from paper_1702_08597_b200.synth import LayerConfig, make_inputs  # noqa: E402

OUT = Path(__file__).resolve().parent

# (name, m, N, C, K, H, W, pad, sparsity, seed); c0 is BASELINE.json configs[0]
LAYER_CASES = [
    ("c0", 4, 1, 16, 16, 12, 12, 1, 0.70, 0),
    ("f23_odd", 2, 2, 3, 4, 7, 9, 0, 0.60, 11),
    ("f43_odd", 4, 2, 5, 3, 10, 13, 1, 0.50, 12),
    ("f63", 6, 1, 4, 6, 14, 11, 1, 0.40, 13),
    ("f43_dense", 4, 1, 8, 8, 9, 9, 1, 0.0, 14),
    ("f43_tiny", 4, 1, 2, 3, 3, 3, 0, 0.30, 15),
]

GEOM_CASES = [(3, 6, 6, 2), (1, 7, 9, 2), (1, 12, 12, 2), (1, 9, 11, 2), (1, 5, 5, 2), (1, 7, 7, 2),
              (256, 15, 15, 4), (16, 14, 14, 4), (5, 12, 15, 4), (4, 16, 13, 6), (1, 3, 3, 4)]


def layer_case(name, m, n, c, k, h, w, pad, sparsity, seed):
    cfg = LayerConfig(name, n, c, k, h, sparsity, pad=pad, m=m, seed=seed)
    img, w_f, go = make_inputs(LayerConfig(name, n, c, k, h, sparsity, pad=pad, m=m, seed=seed))
    if w != h:  # make_inputs draws square images; redraw rectangular ones from the same streams
        from paper_1702_08597_b200.synth import Stream

        img = Stream(seed, f"{name}/L0/I").normal((n, c, h, w)).astype(np.float32)
        ho, wo = h + 2 * pad - 2, w + 2 * pad - 2
        go = Stream(seed, f"{name}/L0/dO").normal((n, k, ho, wo)).astype(np.float32)
    del cfg
    imgp = np.pad(img.astype(np.float64), ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    o = []
    gi = []
    gw = np.zeros_like(w_f)
    for i in range(n):
        r = ref.layer(imgp[i], w_f, go[i].astype(np.float64), m=m)
        o.append(r["o"])
        gi.append(r["grad_in"][:, pad:pad + h, pad:pad + w])
        gw += r["grad_wf"]
    o_sparse = ref.sparse_forward(imgp, w_f, m=m, workers=1, precision=32)
    o_sparse4 = ref.sparse_forward(imgp, w_f, m=m, workers=4, precision=32)
    assert np.array_equal(o_sparse, o_sparse4), "reference worker invariance"
    rp, cols, vals = ref.compress_f32(w_f)
    np.savez_compressed(
        OUT / f"layer_{name}.npz",
        meta=np.array([m, n, c, k, h, w, pad, seed], dtype=np.int64), sparsity=np.float64(sparsity),
        img=img, w_f=w_f, grad_o=go,
        o_f64=np.stack(o), grad_in_f64=np.stack(gi), grad_wf_f64=gw, o_sparse_f32=o_sparse,
        csr_row_ptr=rp, csr_col=np.concatenate(cols) if cols else np.zeros(0, np.int64),
        csr_val=np.concatenate(vals) if vals else np.zeros(0, np.float32),
        csr_nnz=np.array([len(x) for x in cols], dtype=np.int64))


# infer-bench layers (name, c, k, h, m); the first two are the reference's own CLI test config
# (tests/cli_smoke.cpp:127-128), the third exercises F(4x4,3x3)
BENCH_LAYERS = [("convA", 8, 8, 16, 2), ("convB", 4, 4, 12, 2), ("convC", 8, 16, 10, 4)]
BENCH_BATCH, BENCH_SEED, BENCH_DENSITIES = 2, 1, (0.25, 1.0)
STREAM_CASES = [(1, "bench/convA", 700), (0, "", 5), ((1 << 63) + 5, "init/conv1", 320)]


def io_and_bench():
    """WGT1 files written by the reference writer, its seeded uniform streams, its magnitude
    threshold, and infer-bench checksums of its f32 sparse_forward on its own inputs."""
    ref.write_wgt1(OUT / "ref_f64.wgt", np.array([[1.0, -2.5, 0.0], [1e300, -1e-300, 3.14159]]))
    ref.write_wgt1(OUT / "ref_f32.wgt", np.arange(8, dtype=np.float64).reshape(4, 1, 2) * 0.5 - 1.0,
                   dtype="f32")
    g = {}
    for seed, name, n in STREAM_CASES:
        g[f"stream_{seed}_{name.replace('/', '_')}"] = ref.uniform_stream(seed, name, n)
    tw = np.round(ref.uniform_stream(3, "ties", 60) * 4) / 4  # many equal magnitudes
    g["thr_in"] = tw
    for x in (0.0, 0.3, 0.5, 0.99, 1.0):
        g[f"thr_{x}"] = ref.threshold_to_density(tw, x)
    for name, c, k, h, m in BENCH_LAYERS:
        hi, p = h + 2, m + 2
        nb = BENCH_BATCH * c * hi * hi
        v = ref.uniform_stream(BENCH_SEED, "bench/" + name, nb + k * c * p * p)
        batch, w_f = v[:nb].reshape(BENCH_BATCH, c, hi, hi), v[nb:].reshape(k, c, p, p)
        for x in BENCH_DENSITIES:
            w = ref.threshold_to_density(w_f, x).reshape(w_f.shape)
            out = ref.sparse_forward(batch, w, m=m, workers=1, precision=32)
            cs = 0.0
            for val in out.ravel():  # the reference CLI's checksum loop
                cs += float(val)
            g[f"bench_{name}_{x}"] = np.float64(cs)
    np.savez_compressed(OUT / "io_bench.npz", **g)


def main():
    io_and_bench()
    tr = {}
    for m in (2, 3, 4, 6):
        a, b, g = ref.transforms(m)
        tr[f"A{m}"], tr[f"B{m}"], tr[f"G{m}"] = a, b, g
    np.savez_compressed(OUT / "transforms.npz", **tr)

    geo = {}
    for (c, h, w, m) in GEOM_CASES:
        key = f"{c}_{h}_{w}_{m}"
        g = ref.geometry(c, h, w, m)
        geo["geom_" + key] = np.array([g[f] for f in ref.GEOM_FIELDS], dtype=np.int64)
        phis = [(t, i, j) + ref.phi(c, h, w, m, t, i, j) for t in range(g["t"]) for i in range(g["p"])
                for j in range(g["p"])]
        geo["phi_" + key] = np.array(phis, dtype=np.int64)
        psis = [(y, x) + ref.psi(c, h, w, m, y, x) for y in range(g["h_op"]) for x in range(g["w_op"])]
        geo["psi_" + key] = np.array(psis, dtype=np.int64)
    np.savez_compressed(OUT / "geometry.npz", **geo)

    for case in LAYER_CASES:
        layer_case(*case)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
