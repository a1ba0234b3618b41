"""Data-parallel exchange of the compressed step over torch.distributed.

The reference simulates N workers in one process and averages their parts
with compressors.aggregate (compressors.py:256-271) / aggregate_dense
(:274-285).  Here one process drives one GPU; the exchange is
  C1  all-gather of the fixed-size (u32 index, f32 value) payload -- every
      rank keeps exactly k entries (k depends only on M and the CF,
      compressors.py:79-83), so no size exchange is needed;
  K7  the shared-memory-tiled fp64 decompress-average over the gathered
      parts in rank order (bit-identical to aggregate() over the same parts);
  C3  dense fallback: all-gather + the fp64 rank-ordered mean
      (aggregate_dense), exact for any magnitudes.
The gain exchange (C2) lives in controller.run_iteration.
NCCL over NVLink on the GPU box; gloo works for the CPU tests of the
host-side packing logic.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _native as nat
from .compressors import SparseGradient, aggregate_packed
from .gradcore import GradientVector


def allgather_stats(flat: torch.Tensor, group=None) -> "np.ndarray":
    """C2: every rank's raw statistics bytes (selection result structs), rank order.

    The rows are gathered straight from device memory and read back once, so
    every rank forms the reference's worker-ordered mean (controller.py:284-288)
    from identical inputs and takes the identical epsilon decision.  An
    all-gather, not an all-reduce: the summation order must be the reference's.
    """
    world = dist.get_world_size(group)
    if flat.is_cuda:
        out = torch.empty((world, flat.numel()), dtype=flat.dtype, device=flat.device)
        dist.all_gather_into_tensor(out, flat, group=group)
        from . import _native as nat
        return np.frombuffer(nat.d2h_bytes(out), dtype=np.uint8).reshape(world, -1)
    out = [torch.empty_like(flat) for _ in range(world)]
    dist.all_gather(out, flat, group=group)
    return torch.stack(out).numpy()


class Payload:
    """Flat int32 wire buffer of one rank: [idx (kpad) | vals (kpad) | tile bounds (bpad)].

    kpad/bpad round to 4 words so every section stays 16-byte aligned.  The
    tile bounds (gvc_emit tile_bounds_dev) let K7 skip its boundary pass on the
    gathered parts; every rank uses the same layout (same kind, same k, n).
    """

    __slots__ = ("buf", "k", "kpad", "nb", "bpad", "idx", "vals", "bounds")

    def __init__(self, k: int, n: int, device, with_bounds: bool = True):
        self.k = k
        self.kpad = (k + 3) & ~3
        self.nb = (n + nat.AGG_TILE - 1) // nat.AGG_TILE + 1 if with_bounds else 0
        self.bpad = (self.nb + 3) & ~3
        self.buf = torch.empty(2 * self.kpad + self.bpad, dtype=torch.int32, device=device)
        self.idx = self.buf[:self.kpad].view(torch.uint32)
        self.vals = self.buf[self.kpad:2 * self.kpad].view(torch.float32)
        self.bounds = self.buf[2 * self.kpad:2 * self.kpad + self.nb].view(torch.uint32) if with_bounds else None

    @property
    def words(self) -> int:
        return self.buf.numel()


def new_payload(k: int, device, n: int | None = None) -> Payload:
    return Payload(k, n if n is not None else 0, device, with_bounds=n is not None)


def pack_payload(part: SparseGradient) -> Payload:
    pl = getattr(part, "_payload", None)
    if pl is not None:
        return pl
    pl = Payload(part.kept, part.original_length, part.vals.device, with_bounds=False)
    pl.idx[:part.kept].copy_(part.indices)
    pl.vals[:part.kept].copy_(part.vals)
    return pl


def allgather_payload(part: SparseGradient, group=None) -> tuple[torch.Tensor, torch.Tensor]:
    """C1: every rank's (indices, vals), concatenated in rank order."""
    world = dist.get_world_size(group)
    pl = pack_payload(part)
    out = torch.empty((world, pl.words), dtype=torch.int32, device=pl.buf.device)
    dist.all_gather_into_tensor(out, pl.buf, group=group)
    k = part.kept
    idx = out[:, :k].contiguous().view(torch.uint32).reshape(-1)
    vals = out[:, pl.kpad:pl.kpad + k].contiguous().view(torch.float32).reshape(-1)
    return idx, vals


def allgather_aggregate(part: SparseGradient, group=None, out: torch.Tensor | None = None) -> GradientVector:
    """C1 + K7: the rank-ordered fp64 mean of every rank's sparse part.

    The all-gathered (world, words) buffer is averaged in place: part r's
    indices start at r*words, its values kpad words later, its tile bounds
    (when the emit produced them) 2*kpad words later -- no repacking.
    """
    world = dist.get_world_size(group)
    pl = pack_payload(part)
    L = pl.words
    buf = torch.empty((world, L), dtype=torch.int32, device=pl.buf.device)
    dist.all_gather_into_tensor(buf, pl.buf, group=group)
    flat = buf.view(-1)
    bounds = flat[2 * pl.kpad:].view(torch.uint32) if pl.bounds is not None else None
    res = aggregate_packed(flat.view(torch.uint32), flat[pl.kpad:].view(torch.float32), [pl.k] * world,
                           part.original_length, out=out, offs=[r * L for r in range(world)],
                           bounds=bounds, bounds_stride=L)
    return GradientVector._wrap(res)


def allgather_dense_mean(g: GradientVector, group=None) -> GradientVector:
    """C3: dense fallback with the reference's fp64 rank-ordered mean."""
    from .compressors import aggregate_dense
    world = dist.get_world_size(group)
    out = torch.empty((world, g.length), dtype=torch.float32, device=g.values.device)
    dist.all_gather_into_tensor(out, g.values, group=group)
    return aggregate_dense([GradientVector._wrap(out[r]) for r in range(world)])
