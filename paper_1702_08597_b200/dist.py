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
