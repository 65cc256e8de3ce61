"""Data-parallel host logic: batch sharding and the one dW_F exchange.

The path shards by batch: every rank runs the layer kernels on its own images with W_F
replicated (the reference replicates weights per worker, sparse.cpp:237), and the only
exchange is a sum all-reduce of the nnz-compact dW_F, bucketed into ONE collective per step
(train.cpp:166,200 scale the summed per-sample gradients by 1/B).  Works with any
torch.distributed backend: NCCL over NVLink on the GPUs, gloo on CPU for the tests.
"""
from __future__ import annotations

from dataclasses import dataclass


def nccl_comm_ptr(group=None, device=None) -> int:
    """The ncclComm_t (as an int) behind a torch.distributed NCCL process group (default group
    if None) — what wino_set_dw_allreduce / WinogradLayer.set_dw_allreduce take to run the dW_F
    exchange inside the backward on the same communicator torch uses."""
    import torch
    import torch.distributed as dist

    pg = group if group is not None else dist.distributed_c10d._get_default_group()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    return int(pg._get_backend(dev)._comm_ptr())


def shard(n_global: int, rank: int, world: int) -> tuple[int, int]:
    """(start, count) of rank's contiguous slice of a batch of n_global images; the first
    n_global % world ranks take one extra image, so every image belongs to exactly one rank."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(n_global, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


@dataclass
class GradBucket:
    """One flat buffer holding every layer's nnz-compact dW_F, so a step needs a single
    all-reduce.  `views[i]` is layer i's slice (pass it as `out=` to backward_weights)."""

    flat: object            # torch.Tensor, 1-D
    views: list             # per-layer 1-D views
    offsets: list

    @staticmethod
    def allocate(sizes, device=None, dtype=None):
        import torch

        dtype = dtype or torch.float32
        offs = [0]
        for n in sizes:
            offs.append(offs[-1] + int(n))
        flat = torch.zeros(max(offs[-1], 1), device=device, dtype=dtype)
        views = [flat[offs[i]:offs[i + 1]] for i in range(len(sizes))]
        return GradBucket(flat, views, offs)

    def allreduce(self, group=None):
        """Sum over ranks in place (one collective); no-op when not distributed."""
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group)
        return self.flat


# ---------------------------------------------------------------------------------------------
# Tile-axis split (north_star: "partitioned ... by batch and tiles T"): when the batch is smaller
# than the number of GPUs, the T tiles of every image are split instead — contiguous bands of tile
# rows per rank.  Tiles are independent in the forward (sparse.cpp:204-246 splits the batch×tile
# columns over workers the same way), so a rank runs the unchanged layer kernels on its band of the
# zero-padded image ("pad 1" = the reference run on the padded image, tools/wino.cpp:337) and O is
# bitwise the whole-image O.  In the backward dW_F is a sum over tiles (the same all-reduce as the
# batch split) and dI needs one halo exchange: bands overlap by r-1 = 2 padded rows, the rows
# where the tiles of two neighbouring bands both contribute (layer.cpp:157-169).
# ---------------------------------------------------------------------------------------------
def tile_bands(h: int, world: int, m: int = 4) -> list:
    """Contiguous tile-row ranges [(a, b), ...] of an image of height h (pad 1, F(m×m,3×3)), one
    per rank; the first tiles_y % world ranks take one extra tile row (ranks beyond tiles_y get an
    empty band (a, a))."""
    if world <= 0:
        raise ValueError("world must be positive")
    tiles_y = -(-h // m)
    out = []
    for r in range(world):
        a, n = shard(tiles_y, r, world)
        out.append((a, a + n))
    return out


def band_rows(h: int, a: int, b: int, m: int = 4) -> tuple:
    """For the band of tile rows [a, b): (first padded input row, padded input rows, first output
    row, output rows).  Padded row Y = image row y + 1."""
    y0, y1 = m * a, min(m * b, h)
    return y0, (y1 - y0) + 2 if y1 > y0 else 0, y0, max(0, y1 - y0)


def band_input(x, a: int, b: int, m: int = 4):
    """The band's input: rows [m·a, m·b + 2) of the image zero-padded by 1 (N×C×(rows)×(W+2)),
    to be run through a layer built with pad=0 on that shape."""
    import torch.nn.functional as F

    h = x.shape[-2]
    y0, rows, _, _ = band_rows(h, a, b, m)
    # padded rows [y0, y0 + rows) = image rows [y0 - 1, y0 + rows - 1)
    lo, hi = y0 - 1, y0 + rows - 1
    top, bot = max(0, -lo), max(0, hi - h)
    return F.pad(x[..., max(lo, 0):min(hi, h), :], (1, 1, top, bot)).contiguous()


def merge_bands(parts, bands, h: int, m: int = 4):
    """Single-process form of the halo exchange: sum the bands' padded dI (each N×C×rows×(W+2),
    rows as band_rows) into the whole padded gradient — upper band first, the reference's
    ascending-tile order — and crop the padding: N×C×h×W."""
    import torch

    first = next(p for p in parts if p is not None)
    n, c, _, wp = first.shape
    full = torch.zeros((n, c, h + 2, wp), dtype=first.dtype, device=first.device)
    for p, (a, b) in zip(parts, bands):
        y0, rows, _, _ = band_rows(h, a, b, m)
        if rows:
            full[:, :, y0:y0 + rows, :] += p
    return full[:, :, 1:h + 1, 1:wp - 1]


def exchange_halo(di_band, rank: int, world: int, bands, h: int, m: int = 4, group=None):
    """The distributed halo exchange of a tile-split backward.  di_band: this rank's padded dI
    band (N×C×rows×(W+2)).  Neighbouring bands share r-1 = 2 padded rows; each rank sends the
    shared rows it does not own and adds what it receives (upper band's contribution first).
    Returns this rank's owned rows of dI, N×C×out_rows×W (image rows [m·a, min(m·b, h)))."""
    import torch
    import torch.distributed as dist

    a, b = bands[rank]
    y0, rows, _, out_rows = band_rows(h, a, b, m)
    if rows == 0:
        return di_band[:, :, :0, 1:-1]
    live = [r for r in range(world) if bands[r][1] > bands[r][0]]
    i = live.index(rank)
    up = live[i - 1] if i > 0 else None
    down = live[i + 1] if i + 1 < len(live) else None
    # local padded row j = Y - y0.  Shared with the upper band: j = 0 (owned by `up`: image row
    # y0 - 1) and j = 1 (owned here).  Shared with the lower band: j = rows - 2 (owned here) and
    # j = rows - 1 (owned by `down`).
    reqs = []
    recv_up = torch.empty_like(di_band[:, :, 0, :]) if up is not None else None
    recv_down = torch.empty_like(di_band[:, :, 0, :]) if down is not None else None
    send_up = di_band[:, :, 0, :].contiguous() if up is not None else None
    send_down = di_band[:, :, rows - 1, :].contiguous() if down is not None else None
    if up is not None:
        reqs += [dist.isend(send_up, up, group=group), dist.irecv(recv_up, up, group=group)]
    if down is not None:
        reqs += [dist.isend(send_down, down, group=group), dist.irecv(recv_down, down, group=group)]
    for q in reqs:
        q.wait()
    out = di_band.clone()
    if up is not None:  # the upper band's last row lands on local row 1
        out[:, :, 1, :] = recv_up + out[:, :, 1, :]
    if down is not None:  # the lower band's first row lands on local row rows - 2
        out[:, :, rows - 2, :] = out[:, :, rows - 2, :] + recv_down
    return out[:, :, 1:1 + out_rows, 1:-1]
