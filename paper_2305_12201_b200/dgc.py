"""DGC sampled-threshold selection on the GPU (compressors.py:110-137).

The reference:
  s   = min(n, max(256, round(f * n)))                       :112
  s >= n -> exact top-k                                       :113-115
  sample = s positions drawn without replacement              :118  (numpy choice)
  thr = rank-th largest sampled |v|, rank = round(k s / n)    :119-121
  chosen = {|v| >= thr};  if |chosen| >= k: top-k of chosen   :123-125
  else: chosen + largest sampled below thr (ties -> lower index) + global top-up  :126-137

This build runs it with no host decision:
  * the sample is one counter-based (Philox) position per stratum of n / s
    positions (see DESIGN.md for why it replaces numpy's choice); one pass
    (gvc_dgc_sample_gather) gathers g_ef there (EF applied on the fly) and
    marks the positions in a bitmap;
  * thr is the exact rank-th largest sampled key (a Top-k select on s
    values, threshold left on the device);
  * ONE fused selection over the composite key
        (|v| >= thr or sampled) ? 0x80000000 | |v| : |v|
    whose top-k is the DGC pick in both branches: when k entries reach thr,
    the k largest of them (they sit on top); otherwise all of them, then the
    largest sampled values below thr, then the largest of the rest -- the
    global top-up -- ties to the lower index.  The fused pass also writes g_ef
    (EF mode), and nothing about the branch is read back.
"""

from __future__ import annotations

import torch

from . import _native as nat


def dgc_select(kind, values: torch.Tensor | None, k: int, rng, pos_base: int = 0,
               idx_map: torch.Tensor | None = None, check: bool = True, *, g: torch.Tensor | None = None,
               resid: torch.Tensor | None = None, pending=None, slot: str = "dgc", want_result: bool = False,
               sent_mask: torch.Tensor | None = None, tile_bounds: torch.Tensor | None = None,
               res_dev: torch.Tensor | None = None):
    """(ascending indices, values) of the DGC selection of k entries.

    Plain mode: ``values``.  EF mode: ``g`` + ``resid`` (+ ``pending``): g_ef is
    computed in the fused pass and written over ``resid``.  ``want_result``:
    also return the fused pass's Selection (its ``res_dev`` holds ||g_ef||^2
    and the status on the device).  ``sent_mask`` (level 1, no idx_map): also
    write the bit mask of the selected positions there, every word of it.
    ``tile_bounds``: also write the aggregate's tile boundaries of the
    selection (gvc_emit tile_bounds_dev), sparing the decompress its own pass.
    ``check``: read the status back (raises on NaN); the fused controller step
    leaves it on the device.
    """
    from .compressors import CompressorKind, Selection
    src = values if values is not None else g
    n = src.numel()
    dev = src.device
    topk = CompressorKind("topk")
    s = min(n, max(256, int(round(kind.dgc_sample_fraction * n))))
    if s >= n:  # full sample: threshold estimation degenerates to exact selection (:113-115)
        sel = Selection(topk, [k], values=values, g=g, resid=resid, pending=pending, slot=slot + "c",
                        res_dev=res_dev)
    else:
        # the sample's values and position bitmap in one pass (gvc_dgc_sample_gather)
        vP = torch.empty(s, dtype=torch.float32, device=dev)
        words = (n + 31) // 32
        bits = nat.Workspace.get(dev, slot + "/bits", words * 4)[:words * 4].view(torch.int32).view(torch.uint32)
        pm, pmk, mode = (None, None, 0) if pending is None else (pending[0], pending[1], int(pending[2]))
        nat.check(nat.load().gvc_dgc_sample_gather(n, s, rng.seed if rng is not None else 0,
                                                   rng.stream if rng is not None else 0, pos_base,
                                                   nat.ptr(values), nat.ptr(g), nat.ptr(resid), nat.ptr(pm),
                                                   nat.ptr(pmk), mode, nat.ptr(vP), nat.ptr(bits),
                                                   nat.stream_ptr(dev)), "dgc_sample_gather")
        rank = min(s, max(1, int(round(k * s / n))))
        if rank < s:
            sel_t = Selection(topk, [rank], values=vP, slot=slot + "t")
            off = nat.SelectResult.threshold_key.offset
            thr = sel_t.res_dev[off:off + 4].view(torch.int32)
        else:  # the threshold is the smallest sampled magnitude
            thr = (vP.view(torch.int32) & 0x7FFFFFFF).min().reshape(1)
        sel = Selection(topk, [k], values=values, g=g, resid=resid, pending=pending, slot=slot + "c",
                        dgc_thr=thr, dgc_bits=bits, res_dev=res_dev)
    idx, vals = sel.emit(0, idx_map=idx_map, sent_mask=sent_mask, tile_bounds=tile_bounds)
    if check:
        sel.result()  # raises ValueError on NaN
    return (idx, vals, sel) if want_result else (idx, vals)
