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
        self.offs, self.rowlen = {}, {}
        for k in self.keys:
            n = grads[k].numel()
            view = self.flat[off:off + n].view(grads[k].shape)
            view.copy_(grads[k])  # keep current values
            grads[k] = view
            self.offs[k] = off
            self.rowlen[k] = n // max(1, grads[k].shape[0])
            off += n
        self.group = group
        self.deterministic = deterministic

    def all_reduce(self):
        # SURVEY §8(e); deterministic option: gather every rank's partial and
        # sum in rank order (bitwise identical on every rank and run)
        return reduce_flat(self.flat, self.group, self.deterministic)

    def row_views(self, r0: int, r1: int) -> list:
        """The flat-buffer slices holding parameter rows [r0, r1) of every group."""
        return [self.flat[self.offs[k] + r0 * self.rowlen[k]:self.offs[k] + r1 * self.rowlen[k]]
                for k in self.keys]

    def reduce_rows(self, r0: int, r1: int):
        """Sum rows [r0, r1) of every group across ranks on the current stream
        (the bucketed, overlapped exchange of DESIGN.md §9: called per
        preprocess-backward row chunk, Rasterizer.backward(on_rows=...)). NCCL:
        the groups' slices in one coalesced collective; deterministic: the
        rank-ordered all_gather sum of each slice."""
        views = self.row_views(r0, r1)
        if not (dist.is_initialized() and dist.get_world_size(self.group) > 1):
            return views
        if self.deterministic:
            for v in views:
                reduce_flat(v, self.group, True)
            return views
        if dist.get_backend(self.group) == "nccl":
            from torch.distributed.distributed_c10d import _coalescing_manager
            with _coalescing_manager(group=self.group, device=self.flat.device):
                for v in views:
                    dist.all_reduce(v, op=dist.ReduceOp.SUM, group=self.group)
        else:
            for v in views:
                dist.all_reduce(v, op=dist.ReduceOp.SUM, group=self.group)
        return views


class OverlappedReduce:
    """Bucketed gradient exchange overlapped with the preprocess backward
    (SURVEY §8(e) H9): pass `on_rows` to Rasterizer.backward(row_chunks=k,
    on_rows=...). Each row chunk's all-reduce is enqueued on a side stream as
    soon as the chunk's chain-rule launch is enqueued on the compute stream,
    so it runs while the next chunk computes; `finish()` makes the compute
    stream wait for the last one."""

    def __init__(self, bucket: GradBucket):
        self.bucket = bucket
        self.comm = torch.cuda.Stream(device=bucket.flat.device) if bucket.flat.is_cuda else None

    def on_rows(self, r0: int, r1: int):
        if self.comm is None:
            self.bucket.reduce_rows(r0, r1)
            return
        ev = torch.cuda.Event()
        ev.record()
        with torch.cuda.stream(self.comm):
            self.comm.wait_event(ev)
            self.bucket.reduce_rows(r0, r1)

    def finish(self):
        if self.comm is not None:
            torch.cuda.current_stream().wait_stream(self.comm)
