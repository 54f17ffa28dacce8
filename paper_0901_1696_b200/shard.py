"""Data-parallel sharding of the batched path (BASELINE config 4).

Independent matrices shard with no data-path collective: rank r owns the
contiguous matrix range ``shard_range(total, r, world)``, factors and solves
it with the fused batched kernel on its own GPU, and the only collective is a
gather of the per-matrix results (info int32 + residual float64) to rank 0
after the compute.  Single matrices do not shard ("replicas
only").

The helpers here are backend-agnostic ``torch.distributed`` code: NCCL on the
GPU box (tensors on the rank's CUDA device), gloo in the CPU tests.
"""

from __future__ import annotations

import torch

__all__ = ["shard_range", "gather_results", "pack_results", "unpack_results"]


def shard_range(total: int, rank: int, world: int):
    """Contiguous [start, stop) of ``total`` items for ``rank`` of ``world``;
    the first ``total % world`` ranks get one extra item."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank/world {rank}/{world}")
    base, extra = divmod(int(total), world)
    start = rank * base + min(rank, extra)
    stop = start + base + (1 if rank < extra else 0)
    return start, stop


def pack_results(info: torch.Tensor, resid: torch.Tensor) -> torch.Tensor:
    """(count,) int32 info + (count,) float64 residual -> (count, 2) float64
    (info values are small integers, exact in float64) so one collective
    moves both."""
    return torch.stack([info.to(torch.float64), resid.to(torch.float64)], dim=1)


def unpack_results(packed: torch.Tensor):
    return packed[:, 0].to(torch.int32), packed[:, 1]


def gather_results(info: torch.Tensor, resid: torch.Tensor, total: int, group=None):
    """Gather every rank's (info, resid) shard to rank 0 in global matrix
    order.  Shards may differ by one item, so they are padded to the largest
    shard for a fixed-size all_gather_into_tensor (12 B per matrix: 768 KB at
    65,536 matrices) and trimmed afterwards.  Returns (info, resid) on rank 0
    and (None, None) elsewhere."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    local = pack_results(info, resid)
    width = -(-int(total) // world)  # ceil: the largest shard
    padded = torch.zeros((width, 2), dtype=torch.float64, device=local.device)
    padded[: local.shape[0]] = local
    out = torch.empty((world * width, 2), dtype=torch.float64, device=local.device)
    dist.all_gather_into_tensor(out, padded, group=group)
    if rank != 0:
        return None, None
    parts = []
    for r in range(world):
        s, e = shard_range(total, r, world)
        parts.append(out[r * width: r * width + (e - s)])
    return unpack_results(torch.cat(parts, dim=0))
