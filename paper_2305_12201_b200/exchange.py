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

import torch
import torch.distributed as dist

from .compressors import SparseGradient, aggregate_packed
from .gradcore import GradientVector


def allgather_gain_rows(row, group, device) -> list:
    """C2: (ef_norm, E_min, E_c, [extra...]) of every rank, in rank order.

    An all-gather (not an all-reduce) so every rank sums the ratios in the
    reference's worker order (controller.py:284-288) and takes the identical
    epsilon decision.
    """
    norm, e_min, e_c, extra = row
    t = torch.tensor([[norm, e_min, e_c, *extra]], dtype=torch.float64)
    if dist.get_backend(group) == "nccl":
        t = t.to(device)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    return [(r[0], r[1], r[2], list(r[3:])) for r in torch.cat(out).cpu().tolist()]


def pack_payload(part: SparseGradient) -> torch.Tensor:
    """(2, k) int32 view-compatible buffer: row 0 indices bits, row 1 value bits."""
    k = part.kept
    buf = torch.empty((2, k), dtype=torch.int32, device=part.vals.device)
    buf[0].copy_(part.indices.view(torch.int32))
    buf[1].copy_(part.vals.view(torch.int32))
    return buf


def allgather_payload(part: SparseGradient, group=None) -> tuple[torch.Tensor, torch.Tensor]:
    """C1: every rank's (indices, vals), concatenated in rank order."""
    world = dist.get_world_size(group)
    payload = pack_payload(part)
    k = part.kept
    out = torch.empty((world, 2, k), dtype=torch.int32, device=payload.device)
    dist.all_gather_into_tensor(out, payload, group=group)
    idx = out[:, 0, :].contiguous().view(torch.uint32).reshape(-1)
    vals = out[:, 1, :].contiguous().view(torch.float32).reshape(-1)
    return idx, vals


def allgather_aggregate(part: SparseGradient, group=None, out: torch.Tensor | None = None) -> GradientVector:
    """C1 + K7: the rank-ordered fp64 mean of every rank's sparse part."""
    world = dist.get_world_size(group)
    idx, vals = allgather_payload(part, group)
    res = aggregate_packed(idx, vals, [part.kept] * world, part.original_length, out=out)
    return GradientVector._wrap(res)


def allgather_dense_mean(g: GradientVector, group=None) -> GradientVector:
    """C3: dense fallback with the reference's fp64 rank-ordered mean."""
    from .compressors import aggregate_dense
    world = dist.get_world_size(group)
    out = torch.empty((world, g.length), dtype=torch.float32, device=g.values.device)
    dist.all_gather_into_tensor(out, g.values, group=group)
    return aggregate_dense([GradientVector._wrap(out[r]) for r in range(world)])
