"""Sparsifying compressors on the GPU behind the reference's (indices, values) API.

Drop-in for ``gravac.compressors`` (/root/reference/pkg/src/gravac/compressors.py).
Every selection -- Top-k, Redsync, Random-k and DGC -- runs as the sm_100a
pipeline in csrc/gvc_select.cu: one streaming pass that compacts a
candidate superset, radix refinement over candidates only, and an
index-ordered emit.  ``SparseGradient.indices``/``.vals`` are CUDA tensors
(uint32 / float32); the selection rule, the exact keep count, the tie order
(lower index wins) and the value substitution are the reference's.

Random-k positions and DGC's threshold sample come from a counter-based
Philox4x32-10 position hash (k smallest hashes, ties to the lower index)
instead of numpy's sequential Generator.choice; see DESIGN.md.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np
import torch

from . import _native as nat
from .gradcore import GradientVector, SeededRng, as_f32_tensor

TOPK = "topk"
DGC = "dgc"
REDSYNC = "redsync"
RANDOMK = "randomk"
KIND_NAMES = (TOPK, DGC, REDSYNC, RANDOMK)

# (kind, input_length, kept) -> modeled seconds (compressors.py:27-28)
LatencyFn = Callable[["CompressorKind", int, int], float]


@dataclass(frozen=True)
class CompressorKind:
    """Compressor selector plus per-kind knobs (compressors.py:31-45)."""

    name: str
    dgc_sample_fraction: float = 0.01
    redsync_max_rounds: int = 20

    def __post_init__(self):
        if self.name not in KIND_NAMES:
            raise ValueError(f"unknown compressor {self.name!r}, expected one of {KIND_NAMES}")
        if not (0.0 < self.dgc_sample_fraction <= 1.0):
            raise ValueError(f"dgc_sample_fraction must be in (0, 1], got {self.dgc_sample_fraction}")
        if self.redsync_max_rounds < 1:
            raise ValueError(f"redsync_max_rounds must be >= 1, got {self.redsync_max_rounds}")

    @property
    def kind_id(self) -> int:
        return nat.KIND_IDS[self.name]


class SparseGradient:
    """(index, value) encoding of a compressed gradient (compressors.py:48-76).

    ``indices`` strictly increasing uint32 positions into the dense vector of
    ``original_length`` entries, ``vals`` float32; ``achieved_cf`` =
    original_length / kept.  Host inputs are validated like the reference;
    tensors produced by the kernels are trusted (the parity suite checks them).
    """

    __slots__ = ("indices", "vals", "original_length", "achieved_cf", "_payload", "_bounds")

    def __init__(self, indices, vals, original_length: int, achieved_cf: float, device=None):
        if isinstance(indices, torch.Tensor) and indices.is_cuda:
            idx_h = indices.cpu().numpy().astype(np.int64)
        else:
            idx_h = np.asarray(indices).astype(np.int64)
        vals_t = as_f32_tensor(vals, device)
        if idx_h.ndim != 1 or tuple(vals_t.shape) != idx_h.shape:
            raise ValueError("indices and vals must be 1-D and equally sized")
        if idx_h.size == 0:
            raise ValueError("sparse gradient must keep at least one entry")
        if np.any(np.diff(idx_h) <= 0):
            raise ValueError("indices must be strictly increasing")
        if idx_h[0] < 0 or int(idx_h[-1]) >= original_length:
            raise ValueError("index beyond original length")
        self.indices = torch.from_numpy(idx_h.astype(np.uint32)).to(vals_t.device)
        self.vals = vals_t
        self.original_length = int(original_length)
        self.achieved_cf = float(achieved_cf)
        self._payload = None
        self._bounds = None

    @classmethod
    def _wrap(cls, indices: torch.Tensor, vals: torch.Tensor, original_length: int,
              achieved_cf: float) -> "SparseGradient":
        s = cls.__new__(cls)
        s.indices = indices
        s.vals = vals
        s.original_length = int(original_length)
        s.achieved_cf = float(achieved_cf)
        s._payload = None
        s._bounds = None
        return s

    @property
    def kept(self) -> int:
        return self.vals.numel()

    def __repr__(self) -> str:
        return f"SparseGradient(kept={self.kept}, original_length={self.original_length}, achieved_cf={self.achieved_cf})"


def keep_count(length: int, cf: float) -> int:
    """max(1, floor(length / cf)) with Python float division (compressors.py:79-83)."""
    if cf < 1.0:
        raise ValueError(f"compression factor must be >= 1, got {cf}")
    return max(1, math.floor(length / cf))


# --------------------------------------------------------------- selection
class Selection:
    """One gvc_select over n values for a ladder of keep counts.

    EF mode (``g`` and ``resid``): values = fl32(g + resid), written over
    ``resid`` (feedback.py:32-36 fused into the pass).  Plain mode: ``values``.
    Results stay on the device until :meth:`result` is called.
    """

    def __init__(self, kind: CompressorKind, ks: Sequence[int], *, values: torch.Tensor | None = None,
                 g: torch.Tensor | None = None, resid: torch.Tensor | None = None,
                 rng: SeededRng | None = None, pos_base: int = 0, slot: str = "sel0",
                 force_exact: int = 0, pending=None, key_est: torch.Tensor | None = None,
                 allow_short: bool = False, persist_res: bool = False,
                 dgc_thr: torch.Tensor | None = None, dgc_bits: torch.Tensor | None = None,
                 equal_magnitudes: bool = False, res_dev: torch.Tensor | None = None):
        src = values if values is not None else g
        nat.require_cuda(src)
        self.kind = kind
        self.n = src.numel()
        self.ks = [int(k) for k in ks]
        self.device = src.device
        lib = nat.load()
        self.ws = nat.select_workspace(self.device, slot, kind.kind_id, self.n)
        # persist_res: the slot's result buffer is reused (the controller reads
        # it back within the step), so an unchanged plan needs no graph update
        # (res_dev: a caller's buffer, e.g. one of two adjacent records read back together)
        self.res_dev = (res_dev if res_dev is not None else
                        nat.Workspace.get(self.device, slot + "/res", nat.RESULT_BYTES)[:nat.RESULT_BYTES]
                        if persist_res else torch.empty(nat.RESULT_BYTES, dtype=torch.uint8, device=self.device))
        a = nat.SelectArgs()
        a.kind = kind.kind_id
        a.n_ks = len(self.ks)
        a.n = self.n
        a.values_dev = values.data_ptr() if values is not None else None
        a.g_dev = g.data_ptr() if g is not None else None
        a.resid_dev = resid.data_ptr() if resid is not None else None
        for j, k in enumerate(self.ks):
            a.ks[j] = k
        a.seed = rng.seed if rng is not None else 0
        a.rng_stream = rng.stream if rng is not None else 0
        a.pos_base = pos_base
        a.dgc_sample_fraction = kind.dgc_sample_fraction
        a.force_exact = int(force_exact)
        a.equal_magnitudes = 1 if equal_magnitudes else 0  # every nonzero |v| equal: position order
        if key_est is not None:  # forced candidate threshold (DGC), a device u32/i32 scalar
            a.key_est_dev = key_est.data_ptr()
            a.allow_short = 1 if allow_short else 0
        if dgc_thr is not None:  # DGC in one selection: composite keys (gvc_select_args.dgc_thr_dev)
            a.dgc_thr_dev = dgc_thr.data_ptr()
            a.dgc_sampled_dev = dgc_bits.data_ptr()
        self._keep = (key_est, dgc_thr, dgc_bits)  # device inputs stay alive until the stream consumed them
        if pending is not None:  # (mask, m, mode): deferred residual update of the previous step
            a.pending_mask_dev = pending[0].data_ptr()
            a.pending_m_dev = pending[1].data_ptr()
            a.pending_mode = int(pending[2])
        nat.check(lib.gvc_select(ctypes.byref(a), nat.ptr(self.ws), self.ws.numel(), nat.ptr(self.res_dev),
                                 nat.stream_ptr(self.device)), "gvc_select")
        self._result = None

    def emit(self, j: int = 0, idx_map: torch.Tensor | None = None, resid: torch.Tensor | None = None,
             stats: torch.Tensor | None = None, sent_mask: torch.Tensor | None = None,
             sent_m: torch.Tensor | None = None, count: int | None = None,
             payload=None, tile_bounds: torch.Tensor | None = None):
        """Index-ascending (indices, values) of ladder entry j; optionally the
        residual update, either direct (``resid``) or deferred (``sent_mask``).
        ``count`` overrides the entry count (a DGC overshoot keeps fewer)."""
        k = self.ks[j] if count is None else int(count)
        mirrors = None
        if payload is not None:  # write straight into the packed wire buffer (exchange.Payload)
            out_idx, out_val = payload.idx[:k], payload.vals[:k]
            tile_bounds = payload.bounds if payload.bounds is not None else tile_bounds
            mirrors = payload.mirrors
        else:
            out_idx = torch.empty(k, dtype=torch.uint32, device=self.device)
            out_val = torch.empty(k, dtype=torch.float32, device=self.device)
        lib = nat.load()
        if mirrors is not None:  # push exchange: the peers' receive slots get the same stores
            nat.check(lib.gvc_emit_mirrored(nat.ptr(self.ws), self.ws.numel(), j, nat.ptr(idx_map), nat.ptr(out_idx),
                                            nat.ptr(out_val), nat.ptr(resid), nat.ptr(sent_mask), nat.ptr(sent_m),
                                            nat.ptr(tile_bounds), nat.ptr(stats), ctypes.byref(mirrors),
                                            nat.stream_ptr(self.device)), "gvc_emit")
            payload.pushed = mirrors.count > 0 and tile_bounds is not None and count is None
            payload.wire16 = bool(mirrors.off16_dev) and count is None
        else:
            nat.check(lib.gvc_emit(nat.ptr(self.ws), self.ws.numel(), j, nat.ptr(idx_map), nat.ptr(out_idx),
                                   nat.ptr(out_val), nat.ptr(resid), nat.ptr(sent_mask), nat.ptr(sent_m),
                                   nat.ptr(tile_bounds), nat.ptr(stats), nat.stream_ptr(self.device)), "gvc_emit")
        return out_idx, out_val

    def result(self) -> nat.SelectResult:
        if self._result is None:
            self._result = nat.read_result(self.res_dev)
            if self._result.status == nat.GVC_ERR_NAN:
                raise ValueError("NaN in gradient: compression order undefined")
            if self._result.status != nat.GVC_OK:
                raise RuntimeError(f"selection consistency failure (status {self._result.status})")
        return self._result


def _iota(n: int, device) -> torch.Tensor:
    out = torch.empty(n, dtype=torch.uint32, device=device)
    nat.check(nat.load().gvc_iota(nat.ptr(out), n, nat.stream_ptr(device)), "iota")
    return out


def _select(kind: CompressorKind, values: torch.Tensor, k: int, rng: SeededRng | None,
            pos_base: int = 0, idx_map: torch.Tensor | None = None, check: bool = True):
    """compressors.py:164-190 on the GPU -> (ascending indices, values to send)."""
    n = values.numel()
    if k >= n:  # identity passthrough for every kind (compressors.py:172-173)
        idx = _iota(n, values.device) if idx_map is None else idx_map.clone()
        return idx, values.clone()
    if kind.name in (RANDOMK, DGC) and rng is None:
        raise ValueError(f"{kind.name} compression requires an rng")
    if kind.name == DGC:
        from .dgc import dgc_select
        return dgc_select(kind, values, k, rng, pos_base=pos_base, idx_map=idx_map, check=check)
    sel = Selection(kind, [k], values=values, rng=rng, pos_base=pos_base)
    out = sel.emit(0, idx_map=idx_map)
    if check:
        sel.result()  # raises ValueError on NaN
    return out


_LAYOUTS: dict = {}


def _layerwise(kind: CompressorKind, values: torch.Tensor, g: GradientVector, cf: float, rng):
    """compressors.py:204-217: per segment keep_count(len, cf) by the kind's
    rule, indices offset by the segment start, concatenated in order.  Top-k
    and Random-k: one segmented selection over every segment
    (gvc_segmented_select); Redsync: the same segmented Top-k support (F1)
    then each segment's mean substitution (gvc_segmented_redsync_values);
    DGC: every segment's sample, threshold and composite-key selection at
    once (gvc_segmented_dgc_select).  Non-contiguous layouts: one selection
    per segment, enqueued back to back, statuses read once at the end."""
    n = values.numel()
    if kind.name in (RANDOMK, DGC) and rng is None:
        raise ValueError(f"{kind.name} compression requires an rng")
    dev = values.device
    lib = nat.load()
    # the layout's segment table (bounds, keep counts, the C arrays): built once
    # per (offsets, length, cf) -- a training loop passes the same layout every step
    key = (g.layer_offsets, n, float(cf))
    lay = _LAYOUTS.get(key)
    if lay is None:
        bounds = [sl for sl in g.layer_slices() if sl.stop > sl.start]
        ks = [keep_count(sl.stop - sl.start, cf) for sl in bounds]
        total = sum(min(k, sl.stop - sl.start) for k, sl in zip(ks, bounds))
        offs = (ctypes.c_uint64 * (len(bounds) + 1))(*[sl.start for sl in bounds], bounds[-1].stop)
        kk = (ctypes.c_uint64 * len(bounds))(*ks)
        # (segments are contiguous in GradientVector: each starts where the previous ended)
        contiguous = all(bounds[q].stop == bounds[q + 1].start for q in range(len(bounds) - 1))
        # per-segment output offsets and lengths (layerwise Redsync; host arrays)
        cnt = [min(k, sl.stop - sl.start) for k, sl in zip(ks, bounds)]
        out_off = (ctypes.c_uint64 * (len(bounds) + 1))(0, *[int(c) for c in np.cumsum(cnt)])
        seg_len = (ctypes.c_uint64 * len(bounds))(*[sl.stop - sl.start for sl in bounds])
        # (segment starts and kept counts on the device: the per-segment path's index offsets)
        starts_dev = torch.tensor([sl.start for sl in bounds], dtype=torch.int64).to(dev)
        out_off_dev = torch.tensor(list(out_off), dtype=torch.int64).to(dev)
        lay = _LAYOUTS[key] = (bounds, ks, total, offs, kk, contiguous, out_off, seg_len, starts_dev, out_off_dev)
        if len(_LAYOUTS) > 64:
            _LAYOUTS.pop(next(iter(_LAYOUTS)))
    bounds, ks, total, offs, kk, contiguous, out_off, seg_len, starts_dev, out_off_dev = lay
    if kind.name in (TOPK, RANDOMK, "redsync"):
        if contiguous:
            idx = torch.empty(total, dtype=torch.int32, device=dev).view(torch.uint32)
            vals = torch.empty(total, dtype=torch.float32, device=dev)
            ws = nat.Workspace.get(dev, "segsel", int(lib.gvc_segmented_select_workspace_bytes(n, len(bounds))))
            status = torch.zeros(1, dtype=torch.int32, device=dev)
            sel_kind = kind.kind_id if kind.name != "redsync" else CompressorKind(TOPK).kind_id
            nat.check(lib.gvc_segmented_select(sel_kind, nat.ptr(values), n, offs, kk, len(bounds),
                                               rng.seed if rng is not None else 0, rng.stream if rng is not None else 0,
                                               nat.ptr(idx), nat.ptr(vals), nat.ptr(ws), ws.numel(), nat.ptr(status),
                                               nat.stream_ptr(dev)), "segmented_select")
            if kind.name == "redsync":
                rws = nat.Workspace.get(dev, "segrs", int(lib.gvc_segmented_redsync_workspace_bytes(total, len(bounds))))
                nat.check(lib.gvc_segmented_redsync_values(nat.ptr(vals), out_off, seg_len, len(bounds), nat.ptr(rws),
                                                           rws.numel(), nat.stream_ptr(dev)), "segmented_redsync")
            if nat.d2h_bytes(status)[0] & 1:  # (event spin: no scheduler-quantum wake-up)
                raise ValueError("NaN in gradient: compression order undefined")
            return idx, vals
    if kind.name == DGC and contiguous:
        # every segment's sample, threshold and composite-key selection at once
        idx = torch.empty(total, dtype=torch.int32, device=dev).view(torch.uint32)
        vals = torch.empty(total, dtype=torch.float32, device=dev)
        frac = float(kind.dgc_sample_fraction)
        ws = nat.Workspace.get(dev, "segdgc", int(lib.gvc_segmented_dgc_workspace_bytes(n, len(bounds), frac)))
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        nat.check(lib.gvc_segmented_dgc_select(nat.ptr(values), n, offs, kk, len(bounds), frac, rng.seed, rng.stream,
                                               nat.ptr(idx), nat.ptr(vals), nat.ptr(ws), ws.numel(), nat.ptr(status),
                                               nat.stream_ptr(dev)), "segmented_dgc_select")
        if nat.d2h_bytes(status)[0] & 1:
            raise ValueError("NaN in gradient: compression order undefined")
        return idx, vals
    idx_parts, val_parts = [], []
    # every segment's result record in one buffer: ONE read-back at the end
    rb = nat.RESULT_BYTES
    recs = nat.Workspace.get(dev, "lw/res", rb * len(bounds))
    nrec = 0
    for sl, k in zip(bounds, ks):
        seg = values[sl.start:sl.stop]
        if seg.data_ptr() % 16:
            seg = seg.clone()
        m = sl.stop - sl.start
        if k >= m:
            i, v = _iota(m, dev), seg.clone()
        elif kind.name == DGC:
            from .dgc import dgc_select
            i, v, sel = dgc_select(kind, seg, k, rng, pos_base=sl.start, check=False, want_result=True,
                                   res_dev=recs[nrec * rb:(nrec + 1) * rb])
            nrec += 1
        else:
            sel = Selection(kind, [k], values=seg, rng=rng, pos_base=sl.start,
                            res_dev=recs[nrec * rb:(nrec + 1) * rb])
            i, v = sel.emit(0)
            nrec += 1
        idx_parts.append(i)  # segment-local positions
        val_parts.append(v)
    if nrec:
        raw = nat.d2h_bytes(recs[:nrec * rb])
        for q in range(nrec):
            r = nat.SelectResult.from_buffer_copy(raw[q * rb:(q + 1) * rb])
            if r.status == nat.GVC_ERR_NAN:
                raise ValueError("NaN in gradient: compression order undefined")
            if r.status != nat.GVC_OK:
                raise RuntimeError(f"selection consistency failure (status {r.status})")
    # global indices in three launches for all segments (two small torch ops
    # per segment cost ~10 us of host time each; the layout's starts and counts
    # live on the device -- a pageable upload here would synchronise the stream)
    # segment-local -> global indices, every segment in one launch
    if len(bounds) > 3000:  # (the kernel stages the offsets in 48 KB of shared memory)
        idx = torch.cat([t.to(torch.int64) + sl.start for t, sl in zip(idx_parts, bounds)]).to(torch.uint32)
        return idx, torch.cat(val_parts)
    idx = torch.cat([t.view(torch.int32) for t in idx_parts]).view(torch.uint32)
    nat.check(lib.gvc_add_segment_offsets(nat.ptr(idx), total, nat.ptr(out_off_dev), nat.ptr(starts_dev), len(bounds),
                                          nat.stream_ptr(dev)), "add_segment_offsets")
    return idx, torch.cat(val_parts)


def compress(kind: CompressorKind, g: GradientVector, cf: float, rng: SeededRng | None = None,
             latency: LatencyFn | None = None, layerwise: bool = False) -> tuple[SparseGradient, float]:
    """Compress a dense gradient to factor cf (compressors.py:193-223).

    Keeps exactly max(1, floor(M / cf)) entries (per layer segment when
    ``layerwise``).  The seconds come from the modeled latency hook, 0.0 when
    absent -- never from a clock, as in the reference.
    """
    values = g.values
    nat.require_cuda(values)
    n = values.numel()
    if layerwise and len(g.layer_offsets) > 1:
        indices, vals = _layerwise(kind, values, g, cf, rng)
        kept = vals.numel()
    else:
        kept = keep_count(n, cf)
        indices, vals = _select(kind, values, kept, rng)
    seconds = latency(kind, n, kept) if latency is not None else 0.0
    return SparseGradient._wrap(indices, vals, n, n / kept), seconds


def compress_further(kind: CompressorKind, s: SparseGradient, step: float, rng: SeededRng | None = None,
                     latency: LatencyFn | None = None) -> tuple[SparseGradient, float]:
    """Second-level compression over the kept entries only (compressors.py:226-246)."""
    if step < 1.0:
        raise ValueError(f"step factor must be >= 1, got {step}")
    k1 = s.kept
    k2 = keep_count(k1, step)
    if k2 >= k1:
        out = SparseGradient._wrap(s.indices.clone(), s.vals.clone(), s.original_length, s.achieved_cf)
    else:
        vals = s.vals if s.vals.data_ptr() % 16 == 0 else s.vals.clone()
        idx, v = _select(kind, vals, k2, rng, idx_map=s.indices)
        out = SparseGradient._wrap(idx, v, s.original_length, s.original_length / k2)
    seconds = latency(kind, k1, k2) if latency is not None else 0.0
    return out, seconds


def decompress(s: SparseGradient, layer_offsets: Sequence[int] | None = None) -> GradientVector:
    """Zeros with the kept values scattered in place (compressors.py:249-253)."""
    dev = s.vals.device
    nat.require_cuda(s.vals)
    lib = nat.load()
    n = s.original_length
    out = torch.empty(n, dtype=torch.float32, device=dev)
    ws = nat.Workspace.get(dev, "agg", int(lib.gvc_aggregate_workspace_bytes(1, n)))
    nat.check(lib.gvc_decompress(nat.ptr(s.indices), nat.ptr(s.vals), s.kept, n, nat.ptr(out), nat.ptr(ws),
                                 ws.numel(), nat.stream_ptr(dev)), "decompress")
    return GradientVector._wrap(out, layer_offsets)


def aggregate_packed(idx: torch.Tensor, vals: torch.Tensor, counts: Sequence[int], n: int,
                     out: torch.Tensor | None = None, offs: Sequence[int] | None = None,
                     bounds: torch.Tensor | None = None, bounds_stride: int = 0) -> torch.Tensor:
    """fp64 worker-ordered mean of parts in (idx, vals); part p starts at offs[p]
    (default: back to back).  ``bounds``: precomputed tile boundaries of every
    part (gvc_emit tile_bounds_dev), part p's at bounds + p * bounds_stride."""
    dev = vals.device
    lib = nat.load()
    nparts = len(counts)
    if offs is None:
        offs, acc = [], 0
        for c in counts:
            offs.append(acc)
            acc += int(c)
    offs_c = (ctypes.c_uint64 * nparts)(*[int(o) for o in offs])
    cnts_c = (ctypes.c_uint64 * nparts)(*[int(c) for c in counts])
    if out is None:
        out = torch.empty(n, dtype=torch.float32, device=dev)
    if bounds is None:  # the boundary pass needs scratch
        ws = nat.Workspace.get(dev, "agg", int(lib.gvc_aggregate_workspace_bytes(nparts, n)))
        ws_p, ws_n = nat.ptr(ws), ws.numel()
    else:
        ws_p, ws_n = None, 0
    nat.check(lib.gvc_aggregate(nat.ptr(idx), nat.ptr(vals), offs_c, cnts_c, nparts, n, nat.ptr(out), ws_p,
                                ws_n, nat.ptr(bounds), bounds_stride, nat.stream_ptr(dev)), "aggregate")
    return out


def aggregate(parts: Sequence[SparseGradient]) -> GradientVector:
    """Element-wise mean of densified parts, fp64 in the order given (compressors.py:256-271)."""
    if not parts:
        raise ValueError("aggregate of zero parts")
    m = parts[0].original_length
    for p in parts:
        if p.original_length != m:
            raise ValueError(f"length mismatch in aggregate: {p.original_length} != {m}")
    idx = torch.cat([p.indices for p in parts]) if len(parts) > 1 else parts[0].indices
    vals = torch.cat([p.vals for p in parts]) if len(parts) > 1 else parts[0].vals
    return GradientVector._wrap(aggregate_packed(idx, vals, [p.kept for p in parts], m))


def aggregate_dense(parts: Sequence[GradientVector]) -> GradientVector:
    """Element-wise fp64 mean of dense gradients (compressors.py:274-285)."""
    if not parts:
        raise ValueError("aggregate of zero parts")
    m = parts[0].length
    for p in parts:
        if p.length != m:
            raise ValueError(f"length mismatch in aggregate: {p.length} != {m}")
    stacked = torch.stack([p.values for p in parts]).contiguous()
    out = torch.empty(m, dtype=torch.float32, device=stacked.device)
    nat.check(nat.load().gvc_aggregate_dense(nat.ptr(stacked), len(parts), m, nat.ptr(out),
                                             nat.stream_ptr(stacked.device)), "aggregate_dense")
    return GradientVector._wrap(out, parts[0].layer_offsets)
