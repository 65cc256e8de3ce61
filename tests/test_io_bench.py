"""WGT1 / config / checkpoint I/O and the infer-bench driver against fixtures the reference wrote
(tests/golden/make_golden.py: ref_f64.wgt, ref_f32.wgt, io_bench.npz).  Mirrors the reference's
test_tensor.cpp:67-110, test_harness.cpp:13-64,78+ and cli_smoke.cpp:126-185."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1702_08597_b200 import infer_bench as ib
from paper_1702_08597_b200 import io as wio

from helpers import GOLDEN
from oracle import ref

G = np.load(GOLDEN / "io_bench.npz")


# -- WGT1 -------------------------------------------------------------------------------------
def test_wgt1_reads_reference_files():
    a, dt = wio.read_wgt1(GOLDEN / "ref_f64.wgt", return_dtype=True)
    assert dt == "f64" and a.shape == (2, 3)
    assert np.array_equal(a, [[1.0, -2.5, 0.0], [1e300, -1e-300, 3.14159]])
    b, dt = wio.read_wgt1(GOLDEN / "ref_f32.wgt", return_dtype=True)
    assert dt == "f32" and b.shape == (4, 1, 2)
    assert np.array_equal(b, np.arange(8).reshape(4, 1, 2) * 0.5 - 1.0)


@pytest.mark.parametrize("name,dtype", [("ref_f64.wgt", "f64"), ("ref_f32.wgt", "f32")])
def test_wgt1_writer_is_byte_identical(tmp_path, name, dtype):
    a = wio.read_wgt1(GOLDEN / name)
    wio.write_wgt1(tmp_path / "x.wgt", a, dtype=dtype)
    assert (tmp_path / "x.wgt").read_bytes() == (GOLDEN / name).read_bytes()


def test_wgt1_round_trip_bits(tmp_path):
    t = np.array([[1.0, -2.5, 0.0], [1e300, -1e-300, 3.14159]])
    wio.write_wgt1(tmp_path / "t.wgt", t)
    back = wio.read_wgt1(tmp_path / "t.wgt")
    assert back.shape == t.shape and np.array_equal(back.view(np.uint64), t.view(np.uint64))


def test_wgt1_rejects_bad_files(tmp_path):
    p = tmp_path / "bad.wgt"
    p.write_bytes(b"NOPE")
    with pytest.raises(wio.IoError):
        wio.read_wgt1(p)
    wio.write_wgt1(p, np.zeros(8))
    data = p.read_bytes()
    p.write_bytes(data[:-5])  # chopped payload
    with pytest.raises(wio.IoError):
        wio.read_wgt1(p)
    p.write_bytes(data[:4] + bytes([7]) + data[5:])  # unknown dtype
    with pytest.raises(wio.IoError):
        wio.read_wgt1(p)
    p.write_bytes(b"WGT1\x01\x01\x00\x00\x00\x00")  # zero extent
    with pytest.raises(wio.IoError):
        wio.read_wgt1(p)
    p.write_bytes(b"WGT1\x01\x02\x01\x00")  # truncated extents
    with pytest.raises(wio.IoError):
        wio.read_wgt1(p)
    with pytest.raises(wio.IoError):
        wio.read_wgt1(tmp_path / "missing.wgt")


# -- config / csv / grid ------------------------------------------------------------------
def test_config_parses_sections_comments_whitespace():
    cfg = wio.Config.parse_string("top=1\n[dataset]\nseed = 7   # trailing comment\n"
                                  "# full-line comment\nchannels=2\n\n[prune]\nlambda = 0.004\n")
    assert cfg.get("", "top") == "1"
    assert cfg.get_int("dataset", "seed", 0) == 7
    assert cfg.get_int("dataset", "channels", 0) == 2
    assert cfg.get_double("prune", "lambda", 0.0) == 0.004
    assert cfg.get_or("prune", "missing", "dflt") == "dflt"
    assert cfg.get_int("prune", "missing", 9) == 9
    with pytest.raises(wio.ConfigError):
        cfg.get("prune", "missing")
    assert cfg.sections() == ["", "dataset", "prune"]


def test_config_rejects_malformed_lines():
    with pytest.raises(wio.ConfigError):
        wio.Config.parse_string("[unclosed\n")
    with pytest.raises(wio.ConfigError):
        wio.Config.parse_string("no equal sign\n")


def test_csv_quoting():
    assert ib.csv_field("plain") == "plain"
    assert ib.csv_field("a,b") == '"a,b"'
    assert ib.csv_field('say "hi"') == '"say ""hi"""'
    assert ib.csv_field("two\nlines") == '"two\nlines"'
    assert ib.csv_row(["a", "b,c", "d"]) == 'a,"b,c",d'


def test_density_grid():
    lin = ib.parse_density_grid("0.1:0.5:5")
    assert len(lin) == 5 and lin[0] == pytest.approx(0.1) and lin[-1] == pytest.approx(0.5)
    assert lin[1] == pytest.approx(0.2)
    lg = ib.parse_density_grid("0.01:1:log3")
    assert lg == pytest.approx([0.01, 0.1, 1.0])
    assert ib.parse_density_grid("1:1:1") == [1.0]
    assert len(ib.parse_density_grid("0.02:1.0:log")) == 20
    for bad in ("1:2", "0:1:4", "0.5:0.1:3", "0.1:1:0"):
        with pytest.raises(wio.ConfigError):
            ib.parse_density_grid(bad)


def test_effective_workers(monkeypatch):
    monkeypatch.delenv("WINO_THREADS", raising=False)
    assert ib.effective_workers(8) == 8 and ib.effective_workers(0) == 1
    monkeypatch.setenv("WINO_THREADS", "1")
    assert ib.effective_workers(8) == 1
    monkeypatch.setenv("WINO_THREADS", "16")
    assert ib.effective_workers(8) == 8


def test_layers_config(tmp_path):
    p = tmp_path / "layers.cfg"
    p.write_text("[convA]\nc=8\nk=8\nh=16\n[convB]\nc=4\nk=4\nh=12\nm=4\n")
    ls = ib.layers_from_config(p)
    assert [(d.name, d.c, d.k, d.h, d.r, d.m) for d in ls] == [("convA", 8, 8, 16, 3, 2),
                                                               ("convB", 4, 4, 12, 3, 4)]
    p.write_text("[bad]\nc=8\n")
    with pytest.raises(wio.ConfigError):
        ib.layers_from_config(p)
    p.write_text("x=1\n")
    with pytest.raises(wio.ConfigError):
        ib.layers_from_config(p)


# -- seeded inputs, thresholding ------------------------------------------------------------
@pytest.mark.parametrize("seed,name,n", [(1, "bench/convA", 700), (0, "", 5),
                                         ((1 << 63) + 5, "init/conv1", 320)])
def test_uniform_stream_matches_reference_bitwise(seed, name, n):
    want = G[f"stream_{seed}_{name.replace('/', '_')}"]
    got = ib.uniform_stream(seed, name, n)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_stream_continues_across_calls():
    rng = ib.MT19937_64(ib.stream_seed(1, "bench/convA"))
    parts = np.concatenate([ib.uniform(rng, k) for k in (1, 311, 2, 300, 86)])
    assert np.array_equal(parts, G["stream_1_bench_convA"])


@pytest.mark.parametrize("x", [0.0, 0.3, 0.5, 0.99, 1.0])
def test_threshold_to_density_matches_reference(x):
    got = ib.magnitude_threshold_to_density(G["thr_in"], x)
    assert np.array_equal(got, G[f"thr_{x}"])


def test_bench_inputs_shapes():
    d = ib.LayerDims("convB", 4, 4, 12)
    b, w = ib.bench_inputs(d, 2, 1)
    assert b.shape == (2, 4, 14, 14) and w.shape == (4, 4, 4, 4)
    assert b.min() >= -1.0 and b.max() < 1.0


def test_checksum_is_sequential():
    v = np.array([1e16, 1.0, -1e16, 1.0])
    assert ib.checksum(v) == ((1e16 + 1.0) + -1e16) + 1.0


def test_cli_usage_errors_exit_1(tmp_path, capsys):
    assert ib.main([]) == 1  # --layers is required
    assert ib.main(["--layers", str(tmp_path / "nope.cfg")]) == 1


# -- checkpoints ---------------------------------------------------------------------------
def _ck():
    rng = np.random.default_rng(0)
    w1 = rng.standard_normal((4, 2, 6, 6))
    mask = (np.abs(w1) < 0.3).astype(np.float64)
    convs = [wio.LayerRecord("conv1", w1 * (1 - mask), "winograd", 2, 4, 0.004, 1, mask, m=4),
             wio.LayerRecord("conv2", rng.standard_normal((3, 4, 3, 3)), "spatial", 4, 3, 0.0, 2, None, m=2)]
    return wio.Checkpoint(2, 8, 8, 3, convs, rng.standard_normal((3, 48)), rng.standard_normal(3))


def test_checkpoint_round_trip(tmp_path):
    ck = _ck()
    wio.save_checkpoint(tmp_path, ck)
    back = wio.load_checkpoint(tmp_path)
    assert (back.in_c, back.in_h, back.in_w, back.classes) == (2, 8, 8, 3)
    for a, b in zip(ck.convs, back.convs):
        assert (a.name, a.domain, a.in_c, a.out_c, a.lmbda, a.norm, a.m) == \
               (b.name, b.domain, b.in_c, b.out_c, b.lmbda, b.norm, b.m)
        assert np.array_equal(a.w, b.w)
        assert (a.mask is None) == (b.mask is None)
        if a.mask is not None:
            assert np.array_equal(a.mask, b.mask)
    assert np.array_equal(ck.dense_w, back.dense_w) and np.array_equal(ck.dense_b, back.dense_b)


def test_checkpoint_without_m_loads_as_f23(tmp_path):
    """A manifest the reference wrote has no m= key; it loads as F(2x2,3x3) like the reference."""
    ck = _ck()
    wio.save_checkpoint(tmp_path, ck)
    man = tmp_path / "manifest.cfg"
    man.write_text("\n".join(ln for ln in man.read_text().splitlines() if not ln.startswith("m=")) + "\n")
    assert [c.m for c in wio.load_checkpoint(tmp_path).convs] == [2, 2]


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_checkpoint_interoperates_with_reference(tmp_path):
    """Our checkpoint -> the reference's load_checkpoint/save_checkpoint -> our loader: every
    tensor survives bit for bit and the manifest is the reference's except for our m= lines (the
    reference drops them: it only knows F(2x2,3x3))."""
    ck = _ck()
    wio.save_checkpoint(tmp_path / "ours", ck)
    ref.checkpoint_roundtrip(tmp_path / "ours", tmp_path / "theirs")
    back = wio.load_checkpoint(tmp_path / "theirs")
    for a, b in zip(ck.convs, back.convs):
        assert (a.name, a.domain, a.in_c, a.out_c, a.lmbda, a.norm) == \
               (b.name, b.domain, b.in_c, b.out_c, b.lmbda, b.norm)
        assert b.m == 2 and np.array_equal(a.w, b.w)
        assert (a.mask is None) == (b.mask is None)
    for f in ("conv1.wgt", "conv1.mask.wgt", "conv2.wgt", "dense.wgt", "dense_bias.wgt"):
        assert (tmp_path / "ours" / f).read_bytes() == (tmp_path / "theirs" / f).read_bytes()
    # the manifest differs only by our m= lines
    ours = [ln for ln in (tmp_path / "ours" / "manifest.cfg").read_text().splitlines()
            if not ln.startswith("m=")]
    assert ours == (tmp_path / "theirs" / "manifest.cfg").read_text().splitlines()


def test_checkpoint_missing_manifest(tmp_path):
    with pytest.raises(wio.ConfigError):
        wio.load_checkpoint(tmp_path)


# -- the GPU driver --------------------------------------------------------------------------
BENCH_LAYERS = [("convA", 8, 8, 16, 2), ("convB", 4, 4, 12, 2), ("convC", 8, 16, 10, 4)]


@pytest.mark.gpu
def test_infer_bench_checksums_equal_reference():
    """The checksum column equals the reference CLI's f32 checksum bit for bit."""
    layers = [ib.LayerDims(n, c, k, h, 3, m) for n, c, k, h, m in BENCH_LAYERS]
    rows = ib.run(layers, [0.25, 1.0], batch=2, precision="f32", workers=2, seed=1)
    assert len(rows) == 6
    for name, x, wk, ns, gf, cs in rows:
        assert wk == 2 and ns > 0 and gf > 0
        want = float(G[f"bench_{name}_{x}"])
        assert cs == want, (name, x, cs, want)


@pytest.mark.gpu
def test_infer_bench_cli(tmp_path, monkeypatch):
    (tmp_path / "layers.cfg").write_text("[convA]\nc=8\nk=8\nh=16\n[convB]\nc=4\nk=4\nh=12\n")
    assert ib.main(["--batch", "2", "--layers", str(tmp_path / "layers.cfg"), "--density-sweep",
                    "0.25:1:2", "--precision", "f32", "--workers", "2", "--csv",
                    str(tmp_path / "ib.csv")]) == 0
    text = (tmp_path / "ib.csv").read_text()
    assert text.startswith("layer,density,workers,wall_ns,effective_gflops,checksum")
    assert "convA" in text and "convB" in text and len(text.splitlines()) == 5
    monkeypatch.setenv("WINO_THREADS", "1")
    assert ib.main(["--batch", "1", "--layers", str(tmp_path / "layers.cfg"), "--density-sweep",
                    "1:1:1", "--workers", "8", "--csv", str(tmp_path / "ib1.csv")]) == 0
    assert ",1," in (tmp_path / "ib1.csv").read_text()
    assert ib.main(["--layers", str(tmp_path / "layers.cfg"), "--precision", "f64"]) == 1
