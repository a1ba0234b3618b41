"""DGC sampled-threshold selection on the GPU (compressors.py:110-137).

The reference:
  s   = min(n, max(256, round(f * n)))                       :112
  s >= n -> exact top-k                                       :113-115
  sample = s positions drawn without replacement              :118  (numpy choice)
  thr = rank-th largest sampled |v|, rank = round(k s / n)    :119-121
  chosen = {|v| >= thr};  if |chosen| >= k: top-k of chosen   :123-125
  else: chosen + largest sampled below thr (ties -> lower index) + global top-up  :126-137

This build composes it from the sm_100a primitives:
  * the sample is one counter-based (Philox) position per stratum of n / s
    positions (gvc_dgc_sample; see DESIGN.md for why it replaces numpy's
    choice);
  * g_ef at the sampled positions is gathered (EF applied on the fly);
  * thr is the exact rank-th largest sampled key (a Top-k select on s values);
  * ONE fused collect pass with the candidate threshold forced to thr yields
    exactly `chosen` (and writes g_ef, in EF mode).  If |chosen| >= k the exact
    top-k of chosen is the usual radix select on those candidates, which equals
    the global top-k;
  * overshoot: every chosen entry is kept; the pads and the top-up are Top-k
    selects over "below-threshold" keys (gvc_below_keys), and the union is
    re-ordered by an ordered bit-mask compaction.
"""

from __future__ import annotations

import ctypes

import numpy as np

import torch

from . import _native as nat


def _mask_for(n: int, device) -> torch.Tensor:
    return torch.zeros((n + 31) // 32, dtype=torch.int32, device=device).view(torch.uint32)


def _mark(idx: torch.Tensor, mask: torch.Tensor) -> None:
    nat.check(nat.load().gvc_mark_sent(nat.ptr(idx), idx.numel(), nat.ptr(mask), nat.stream_ptr(idx.device)),
              "mark_sent")


def _below_keys(v: torch.Tensor, thr_ptr: torch.Tensor, excl: torch.Tensor | None = None):
    out = torch.empty_like(v)
    cnt = torch.zeros(1, dtype=torch.int64, device=v.device)
    nat.check(nat.load().gvc_below_keys(nat.ptr(v), None, v.numel(), nat.ptr(thr_ptr), nat.ptr(excl), nat.ptr(out),
                                        nat.ptr(cnt), nat.stream_ptr(v.device)), "below_keys")
    return out, cnt


def _gather(pos: torch.Tensor, values=None, g=None, resid=None, pending=None) -> torch.Tensor:
    dev = pos.device
    out = torch.empty(pos.numel(), dtype=torch.float32, device=dev)
    pm, pmk, mode = (None, None, 0) if pending is None else (pending[0], pending[1], int(pending[2]))
    nat.check(nat.load().gvc_gather_ef(nat.ptr(pos), pos.numel(), nat.ptr(values), nat.ptr(g), nat.ptr(resid),
                                       nat.ptr(pm), nat.ptr(pmk), mode, nat.ptr(out), nat.stream_ptr(dev)),
              "gather_ef")
    return out


def _take_u32(src: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
    """src[pos] for uint32 tensors (bit-exact gather through the float path)."""
    return _gather(pos, values=src.view(torch.float32)).view(torch.uint32)


def _compact(mask: torch.Tensor, n: int, count: int) -> torch.Tensor:
    dev = mask.device
    lib = nat.load()
    out = torch.empty(count, dtype=torch.uint32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = nat.Workspace.get(dev, "compact", int(lib.gvc_compact_workspace_bytes(n)))
    nat.check(lib.gvc_compact_mask(nat.ptr(mask), n, nat.ptr(out), nat.ptr(cnt), nat.ptr(ws), ws.numel(),
                                   nat.stream_ptr(dev)), "compact_mask")
    return out


def _largest(keys: torch.Tensor, kk: int, slot: str) -> torch.Tensor:
    """Positions of the kk largest keys (ties -> lower index), ascending."""
    from .compressors import CompressorKind, Selection, _iota
    n = keys.numel()
    if kk >= n:
        return _iota(n, keys.device)
    sel = Selection(CompressorKind("topk"), [kk], values=keys, slot=slot)
    idx, _ = sel.emit(0)
    return idx


def dgc_select(kind, values: torch.Tensor | None, k: int, rng, pos_base: int = 0,
               idx_map: torch.Tensor | None = None, check: bool = True, *, g: torch.Tensor | None = None,
               resid: torch.Tensor | None = None, pending=None, slot: str = "dgc", want_result: bool = False,
               sent_mask: torch.Tensor | None = None):
    """(ascending indices, values) of the DGC selection of k entries.

    Plain mode: ``values``.  EF mode: ``g`` + ``resid`` (+ ``pending``): g_ef is
    computed in the fused pass and written over ``resid``.  With ``want_result``
    also returns the gvc_select_result of the fused pass (its ef_norm_sq is
    ||g_ef||^2).  ``sent_mask`` (level 1, no idx_map): also write the bit mask
    of the selected positions there, every word of it.
    """
    from .compressors import CompressorKind, Selection
    src = values if values is not None else g
    n = src.numel()
    dev = src.device
    topk = CompressorKind("topk")
    s = min(n, max(256, int(round(kind.dgc_sample_fraction * n))))
    if s >= n:  # full sample: threshold estimation degenerates to exact selection (:113-115)
        sel = Selection(topk, [k], values=values, g=g, resid=resid, pending=pending, slot=slot + "c")
        idx, vals = sel.emit(0, idx_map=idx_map, sent_mask=sent_mask)
        res = sel.result() if (check or want_result) else None
        return (idx, vals, res) if want_result else (idx, vals)

    # sample positions: one per stratum of n / s positions (gvc_dgc_sample)
    P = torch.empty(s, dtype=torch.int32, device=dev).view(torch.uint32)
    nat.check(nat.load().gvc_dgc_sample(n, s, rng.seed if rng is not None else 0, rng.stream if rng is not None else 0,
                                        pos_base, nat.ptr(P), nat.stream_ptr(dev)), "dgc_sample")
    vP = _gather(P, values=values, g=g, resid=resid, pending=pending)
    rank = min(s, max(1, int(round(k * s / n))))
    if rank < s:
        sel_t = Selection(topk, [rank], values=vP, slot=slot + "t")
        off = nat.SelectResult.threshold_key.offset
        thr = sel_t.res_dev[off:off + 4].view(torch.int32)
    else:  # the threshold is the smallest sampled magnitude
        thr = (vP.view(torch.int32) & 0x7FFFFFFF).min().reshape(1)
    thr_u = thr.view(torch.int32)

    sel_c = Selection(topk, [k], values=values, g=g, resid=resid, pending=pending, slot=slot + "c",
                      key_est=thr_u, allow_short=True)
    res = sel_c.result()  # host decision point: did the threshold overshoot?
    short = int(res.shortfall)
    if short == 0:
        idx, vals = sel_c.emit(0, idx_map=idx_map, sent_mask=sent_mask)
        return (idx, vals, res) if want_result else (idx, vals)

    # overshoot (:126-137): keep all of `chosen`, pad from the sample below thr,
    # then top up globally; re-order the union by position
    e = values if values is not None else resid  # g_ef now lives in resid (EF mode)
    nchosen = k - short
    if nchosen and idx_map is None:
        # `chosen` straight into a complete mask (every word written by the emit)
        # (past ~4.6e8 values the emit ORs bits in global memory: start from zero)
        mask = (_mask_for(n, dev) if n > 400_000_000 else
                torch.empty((n + 31) // 32, dtype=torch.int32, device=dev).view(torch.uint32))
        sel_c.emit(0, count=nchosen, sent_mask=mask)
    else:
        mask = _mask_for(n, dev)
        if nchosen:
            ci, _ = sel_c.emit(0, count=nchosen)
            _mark(ci, mask)
    keysP, cntP = _below_keys(vP, thr_u)
    nb = int(np.frombuffer(nat.d2h_bytes(cntP), dtype=np.int64)[0])
    take = min(short, nb)
    if take:
        _mark(_take_u32(P, _largest(keysP, take, slot + "p")), mask)
    rest = short - take
    if rest:
        excl = _mask_for(n, dev)
        _mark(P, excl)  # sampled positions are not part of the top-up pool
        keysE, _ = _below_keys(e, thr_u, excl)
        _mark(_largest(keysE, rest, slot + "u"), mask)
    idx = _compact(mask, n, k)
    vals = _gather(idx, values=e)
    if sent_mask is not None:
        sent_mask.copy_(mask)
    if idx_map is not None:
        idx = _take_u32(idx_map, idx)
    return (idx, vals, res) if want_result else (idx, vals)
