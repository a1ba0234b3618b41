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


def payload_width(k: int) -> int:
    """Row length of the packed payload: k rounded up to 4 so both rows stay 16-byte aligned."""
    return (k + 3) & ~3


def new_payload(k: int, device) -> torch.Tensor:
    """(2, kpad) int32 wire buffer: row 0 index bits, row 1 value bits."""
    return torch.empty((2, payload_width(k)), dtype=torch.int32, device=device)


def pack_payload(part: SparseGradient) -> torch.Tensor:
    buf = getattr(part, "_payload", None)
    if buf is not None:
        return buf
    k = part.kept
    buf = new_payload(k, part.vals.device)
    buf[0, :k].copy_(part.indices.view(torch.int32))
    buf[1, :k].copy_(part.vals.view(torch.int32))
    return buf


def allgather_payload(part: SparseGradient, group=None) -> tuple[torch.Tensor, torch.Tensor]:
    """C1: every rank's (indices, vals), concatenated in rank order."""
    world = dist.get_world_size(group)
    payload = pack_payload(part)
    k, kp = part.kept, payload.shape[1]
    out = torch.empty((world, 2, kp), dtype=torch.int32, device=payload.device)
    dist.all_gather_into_tensor(out, payload, group=group)
    idx = out[:, 0, :k].contiguous().view(torch.uint32).reshape(-1)
    vals = out[:, 1, :k].contiguous().view(torch.float32).reshape(-1)
    return idx, vals


def allgather_aggregate(part: SparseGradient, group=None, out: torch.Tensor | None = None) -> GradientVector:
    """C1 + K7: the rank-ordered fp64 mean of every rank's sparse part.

    The all-gathered (world, 2, kpad) buffer is averaged in place: part r's
    indices start at r*2*kpad, its values kpad words later -- no repacking.
    """
    world = dist.get_world_size(group)
    payload = pack_payload(part)
    k, kp = part.kept, payload.shape[1]
    buf = torch.empty((world, 2, kp), dtype=torch.int32, device=payload.device)
    dist.all_gather_into_tensor(buf, payload, group=group)
    flat = buf.view(-1)
    res = aggregate_packed(flat.view(torch.uint32), flat[kp:].view(torch.float32), [k] * world,
                           part.original_length, out=out, offs=[r * 2 * kp for r in range(world)])
    return GradientVector._wrap(res)


def allgather_dense_mean(g: GradientVector, group=None) -> GradientVector:
    """C3: dense fallback with the reference's fp64 rank-ordered mean."""
    from .compressors import aggregate_dense
    world = dist.get_world_size(group)
    out = torch.empty((world, g.length), dtype=torch.float32, device=g.values.device)
    dist.all_gather_into_tensor(out, g.values, group=group)
    return aggregate_dense([GradientVector._wrap(out[r]) for r in range(world)])
