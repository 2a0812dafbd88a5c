"""Multi-GPU plumbing: one process per GPU, torch.distributed.

Partitioning of the hot path:
  * views / frames of a 3D batch are sharded round-robin across ranks
    (view v -> rank v mod world); each rank runs the whole rasterizer on its
    views; the per-primitive gradients of a SHARED parameter set are then
    summed across ranks with one all_reduce over a single flat bucket (NCCL
    over NVLink/NVSwitch on the GPU box; gloo in the CPU tests);
  * one large image: tile rows r = rank (mod world) per GPU, gradients summed
    the same way;
  * 6D frames with per-frame parameter rows are disjoint across ranks: no
    exchange;
  * independent 2D images (one primitive set each) need no exchange at all.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_views(B: int, rank: int, world: int) -> list[int]:
    """Round-robin view assignment (view v -> rank v mod world)."""
    return list(range(rank, B, world))


def tile_rows(GY: int, rank: int, world: int) -> list[int]:
    """Cyclic tile-row assignment for image-space sharding of one large image."""
    return list(range(rank, GY, world))


def reduce_flat(flat: torch.Tensor, group=None, deterministic: bool = False) -> torch.Tensor:
    """Sum a flat float32 gradient buffer across ranks in place on the current
    stream: one NCCL all_reduce, or (deterministic) an all_gather of every
    rank's partial summed in rank order (bitwise identical on every rank)."""
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return flat
    if deterministic:
        parts = [torch.empty_like(flat) for _ in range(dist.get_world_size(group))]
        dist.all_gather(parts, flat, group=group)
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p
        flat.copy_(acc)
    else:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return flat


class GradBucket:
    """Rebinds the tensors of `grads` (dict name -> tensor) to views of one flat
    float32 buffer so the cross-rank gradient sum is a single collective."""

    def __init__(self, grads: dict, group=None, deterministic: bool = False):
        self.keys = list(grads.keys())
        total = sum(grads[k].numel() for k in self.keys)
        dev = grads[self.keys[0]].device
        self.flat = torch.zeros(total, dtype=torch.float32, device=dev)
        off = 0
        for k in self.keys:
            n = grads[k].numel()
            view = self.flat[off:off + n].view(grads[k].shape)
            view.copy_(grads[k])  # keep current values
            grads[k] = view
            off += n
        self.group = group
        self.deterministic = deterministic

    def all_reduce(self):
        # SURVEY §8(e); deterministic option: gather every rank's partial and
        # sum in rank order (bitwise identical on every rank and run)
        return reduce_flat(self.flat, self.group, self.deterministic)
