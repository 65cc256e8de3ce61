"""Multi-process (world_size 2, gloo, CPU) tests of the data-parallel host logic: batch sharding
and the single bucketed all-reduce of nnz-compact dW_F.  The per-shard gradients come from the
oracle's f32 mirror (CPU) standing in for the kernels — what is under test is the sharding,
bucketing, reduction and 1/B scaling, which are identical on NCCL."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1702_08597_b200.dist import GradBucket, shard


def test_shard_covers_every_image_once():
    for n in (1, 7, 64, 512):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                s, c = shard(n, r, world)
                seen.extend(range(s, s + c))
            assert seen == list(range(n))
    with pytest.raises(ValueError):
        shard(8, 2, 2)


def test_bucket_views_alias_the_flat_buffer():
    b = GradBucket.allocate([3, 0, 5])
    b.views[0].fill_(1.0)
    b.views[2].fill_(2.0)
    assert b.flat.tolist() == [1, 1, 1, 2, 2, 2, 2, 2]
    assert b.offsets == [0, 3, 3, 8]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _layer_grads(img, w_f, go):
    """f32 mirror of one layer's fwd+bwd on a shard: (nnz-compact dW (f64 sums), O)."""
    from oracle import wino_oracle as wo

    res = wo.layer_f32(img, wo.compress(w_f), go, m=4, pad=1)
    return np.concatenate(res["dw"]), res["o"]


def _worker(rank, world, port, n_global, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1702_08597_b200.synth import CONFIGS, make_inputs

        cfg = CONFIGS["c0"]
        img, w_f, go = make_inputs(cfg, n=n_global)
        w_f2 = w_f[:, :, ::-1, ::-1].copy()  # a second layer's weights (same shapes, C=K)
        start, cnt = shard(n_global, rank, world)
        sizes = [int(np.count_nonzero(w_f)), int(np.count_nonzero(w_f2))]
        bucket = GradBucket.allocate(sizes, dtype=torch.float64)
        for i, w in enumerate((w_f, w_f2)):
            dw, _ = _layer_grads(img[start:start + cnt], w, go[start:start + cnt])
            bucket.views[i].copy_(torch.from_numpy(dw))
        bucket.allreduce()
        q.put((rank, bucket.flat.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_global", [4, 5])
def test_two_rank_allreduce_equals_full_batch_gradient(n_global):
    from paper_1702_08597_b200.synth import CONFIGS, make_inputs

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_global, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every rank holds the same reduced bucket ...
    assert np.array_equal(out[0], out[1])
    # ... equal to the single-process full-batch gradient (sum over images)
    cfg = CONFIGS["c0"]
    img, w_f, go = make_inputs(cfg, n=n_global)
    w_f2 = w_f[:, :, ::-1, ::-1].copy()
    full = np.concatenate([_layer_grads(img, w, go)[0] for w in (w_f, w_f2)])
    np.testing.assert_allclose(out[0], full, rtol=1e-12, atol=1e-9)


# ---- tile-axis split (bands of tile rows per rank; dist.py) ----
def test_tile_bands_cover_every_tile_row_once():
    from paper_1702_08597_b200.dist import band_rows, tile_bands

    for h in (4, 12, 13, 14, 56):
        for world in (1, 2, 3, 8):
            bands = tile_bands(h, world)
            rows = []
            for a, b in bands:
                _, _, o0, on = band_rows(h, a, b)
                rows.extend(range(o0, o0 + on))
            assert rows == list(range(h)), (h, world, bands)


def test_band_inputs_are_windows_of_the_padded_image():
    from paper_1702_08597_b200.dist import band_input, band_rows, tile_bands

    x = torch.arange(2 * 3 * 14 * 6, dtype=torch.float32).reshape(2, 3, 14, 6)
    xp = torch.nn.functional.pad(x, (1, 1, 1, 1))
    for world in (1, 2, 3):
        for a, b in tile_bands(14, world):
            y0, rows, _, _ = band_rows(14, a, b)
            assert torch.equal(band_input(x, a, b), xp[:, :, y0:y0 + rows, :])


def _tile_worker(rank, world, port, h, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import wino_oracle as wo
        from paper_1702_08597_b200.dist import band_input, band_rows, exchange_halo, tile_bands

        rng = np.random.default_rng(7)
        c, k, n = 5, 6, 2
        img = rng.standard_normal((n, c, h, h)).astype(np.float32)
        go = rng.standard_normal((n, k, h, h)).astype(np.float32)
        w_f = rng.standard_normal((k, c, 6, 6)) * (rng.random((k, c, 6, 6)) >= 0.5)
        bands = tile_bands(h, world)
        a, b = bands[rank]
        _, _, o0, on = band_rows(h, a, b)
        xb = band_input(torch.from_numpy(img), a, b).numpy()
        # the band through the f32 mirror with pad=0 (the kernels' stand-in on CPU)
        res = wo.layer_f32(xb, wo.compress(w_f), go[:, :, o0:o0 + on, :], m=4, pad=0)
        dw = torch.from_numpy(np.concatenate(res["dw"]))
        dist.all_reduce(dw)  # dW_F: the same sum all-reduce as the batch split
        di = exchange_halo(torch.from_numpy(res["di"]), rank, world, bands, h)
        q.put((rank, res["o"], dw.numpy(), di.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("h", [12, 14])
def test_two_rank_tile_split_equals_whole_image(h):
    """Tiles split over 2 ranks (gloo): O bands are bitwise the whole-image rows, the all-reduced
    dW_F and the halo-exchanged dI match the whole-image layer (f32 mirror on both sides)."""
    from oracle import wino_oracle as wo

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tile_worker, args=(r, 2, port, h, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        r, o, dw, di = q.get(timeout=300)
        got[r] = (o, dw, di)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(7)
    c, k, n = 5, 6, 2
    img = rng.standard_normal((n, c, h, h)).astype(np.float32)
    go = rng.standard_normal((n, k, h, h)).astype(np.float32)
    w_f = rng.standard_normal((k, c, 6, 6)) * (rng.random((k, c, 6, 6)) >= 0.5)
    whole = wo.layer_f32(img, wo.compress(w_f), go, m=4, pad=1)
    assert np.array_equal(np.concatenate([got[0][0], got[1][0]], axis=2), whole["o"])
    ref_dw = np.concatenate(whole["dw"])
    np.testing.assert_allclose(got[0][1], ref_dw, rtol=1e-9, atol=1e-9)
    assert np.array_equal(got[0][1], got[1][1])
    di = np.concatenate([got[0][2], got[1][2]], axis=2)
    np.testing.assert_allclose(di, whole["di"], rtol=1e-5, atol=1e-5)
