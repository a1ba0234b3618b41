"""DGC sampled-threshold selection (compressors.py:110-137) -- see csrc/gvc_dgc.cu."""

from __future__ import annotations


def dgc_select(kind, values, k, rng, pos_base=0, idx_map=None, check=True):
    raise NotImplementedError("dgc selection kernel not built yet")
