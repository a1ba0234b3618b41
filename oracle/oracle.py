"""Python face of the CPU oracle (TEST INFRASTRUCTURE -- never product code).

Wraps ``libgravac_oracle.so`` (gravac_oracle.c) with numpy in/out and
restates the small host-side rules the hot path needs (keep_count,
SeededRng.split stream derivation, compress / compress_further framing).
Each function cites the reference function it restates
(/root/reference/pkg/src/gravac/...).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module; the product package never does (and a test asserts it).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgravac_oracle.so")

TOPK, DGC, REDSYNC, RANDOMK = 0, 1, 2, 3
KIND_IDS = {"topk": TOPK, "dgc": DGC, "redsync": REDSYNC, "randomk": RANDOMK}
_MASK64 = (1 << 64) - 1

_lib = None


def build() -> str:
    """Compile the oracle with its own Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        u64, i32, dbl, vp = ctypes.c_uint64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
        L.orc_philox4x32_10.argtypes = [vp, vp, vp]
        L.orc_position_hash.argtypes = [u64, u64, u64]
        L.orc_position_hash.restype = ctypes.c_uint32
        L.orc_randomk_hash.argtypes = [u64, u64, u64]
        L.orc_randomk_hash.restype = ctypes.c_uint32
        L.orc_ef_add.argtypes = [vp, vp, vp, u64]
        L.orc_sq_norm.argtypes = [vp, u64]
        L.orc_sq_norm.restype = dbl
        L.orc_pairwise_sum_f64.argtypes = [vp, u64]
        L.orc_pairwise_sum_f64.restype = dbl
        L.orc_topk_indices.argtypes = [vp, u64, u64, vp]
        L.orc_select_keys.argtypes = [vp, u64, u64, vp]
        L.orc_select.argtypes = [i32, vp, u64, u64, u64, u64, u64, dbl, vp, vp]
        L.orc_aggregate.argtypes = [vp, vp, vp, i32, u64, vp]
        L.orc_aggregate_dense.argtypes = [vp, i32, u64, vp]
        L.orc_update_residual.argtypes = [vp, vp, vp, u64, u64, vp]
        L.orc_dgc_sample_positions.argtypes = [u64, u64, u64, u64, u64, vp]
        L.orc_set_threads.argtypes = [i32]
        L.orc_get_threads.restype = i32
        _lib = L
    return _lib


def set_threads(t: int) -> int:
    """OpenMP threads of the oracle's O(n) passes (1: the checker's exact
    sequential semantics; bench.py's CPU legs use the host's cores).  Returns
    the previous count."""
    L = lib()
    prev = int(L.orc_get_threads())
    L.orc_set_threads(int(t))
    return prev


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(rc: int):
    if rc == -1:
        raise ValueError("NaN in gradient: selection order undefined")
    if rc != 0:
        raise ValueError(f"oracle error {rc}")


# ---------------------------------------------------------------- host rules
def keep_count(length: int, cf: float) -> int:
    """compressors.py:79-83."""
    if cf < 1.0:
        raise ValueError(f"compression factor must be >= 1, got {cf}")
    return max(1, math.floor(length / cf))


def splitmix64(x: int) -> int:
    """gradcore.py:122-126."""
    x = (x + 0x9E3779B97F4A7C15) & _MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _MASK64
    return x ^ (x >> 31)


def split_stream(stream: int, *path: int) -> int:
    """gradcore.py:151-155: stream of SeededRng(seed, stream).split(*path)."""
    s = stream & _MASK64
    for p in path:
        s = splitmix64(s ^ splitmix64(int(p) & _MASK64))
    return s


def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def position_hash(seed: int, stream: int, i: int) -> int:
    """Philox4x32-10 word 0 at counter (i, stream): the DGC sample's draw."""
    return int(lib().orc_position_hash(seed & _MASK64, stream & _MASK64, i))


def randomk_hash(seed: int, stream: int, i: int) -> int:
    """Random-k's hash of position i: word (i & 3) of Philox4x32-10 at counter (i >> 2, stream)."""
    return int(lib().orc_randomk_hash(seed & _MASK64, stream & _MASK64, i))


# ------------------------------------------------------------------- dense
def ef_add(g: np.ndarray, r: np.ndarray) -> np.ndarray:
    """feedback.py:32-36."""
    g = np.ascontiguousarray(g, dtype=np.float32)
    r = np.ascontiguousarray(r, dtype=np.float32)
    out = np.empty_like(g)
    lib().orc_ef_add(_p(g), _p(r), _p(out), g.size)
    return out


def sq_norm(x: np.ndarray) -> float:
    """gradcore.py:61-70 (sequential fp64; numpy's ddot differs only in order)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    return float(lib().orc_sq_norm(_p(x), x.size))


def pairwise_sum(a: np.ndarray) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().orc_pairwise_sum_f64(_p(a), a.size))


def gain_raw(vals: np.ndarray, ef_norm_sq: float) -> float:
    """metrics.py:18-32."""
    if ef_norm_sq <= 0.0:
        raise ValueError("zero-norm reference gradient: compression gain undefined")
    return sq_norm(vals) / ef_norm_sq


# ---------------------------------------------------------------- selection
def select(kind, values: np.ndarray, k: int, seed: int = 0, stream: int = 0,
           pos_base: int = 0, dgc_sample_fraction: float = 0.01):
    """compressors.py:164-190 (with the counter-based sampler for RandomK/DGC)."""
    kind = KIND_IDS[kind] if isinstance(kind, str) else int(kind)
    values = np.ascontiguousarray(values, dtype=np.float32)
    n = values.size
    kk = min(k, n)
    idx = np.empty(kk, dtype=np.uint32)
    vals = np.empty(kk, dtype=np.float32)
    _check(lib().orc_select(kind, _p(values), n, k, seed & _MASK64, stream & _MASK64,
                            pos_base, dgc_sample_fraction, _p(idx), _p(vals)))
    return idx, vals


def dgc_sample_positions(n: int, s: int, seed: int, stream: int, pos_base: int = 0) -> np.ndarray:
    """The s stratified sample positions of the DGC threshold estimate (gravac_oracle.c)."""
    out = np.empty(s, dtype=np.uint32)
    lib().orc_dgc_sample_positions(n, s, seed & _MASK64, stream & _MASK64, pos_base, _p(out))
    return out


def dgc_overshoots(values: np.ndarray, k: int, seed: int, stream: int, frac: float = 0.01) -> bool:
    """Which branch compressors.py:123-137 takes: True when fewer than k entries
    reach the sampled threshold (the pad + top-up branch)."""
    values = np.ascontiguousarray(values, dtype=np.float32)
    n = values.size
    s = min(n, max(256, round(frac * n)))
    if s >= n:
        return False
    mk = values.view(np.uint32) & np.uint32(0x7FFFFFFF)
    sk = np.sort(mk[dgc_sample_positions(n, s, seed, stream).astype(np.int64)])[::-1]
    rank = min(s, max(1, round(k * s / n)))
    thr = sk[rank - 1]
    return int(np.count_nonzero(mk >= thr)) < k


def topk_indices(values: np.ndarray, k: int) -> np.ndarray:
    values = np.ascontiguousarray(values, dtype=np.float32)
    out = np.empty(min(k, values.size), dtype=np.uint32)
    _check(lib().orc_topk_indices(_p(values), values.size, k, _p(out)))
    return out


def compress(kind, x: np.ndarray, cf: float, seed: int = 0, stream: int = 0,
             layer_offsets=None, layerwise: bool = False, dgc_sample_fraction: float = 0.01):
    """compressors.py:193-223 -> (indices u32, vals f32, achieved_cf)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    n = x.size
    if layerwise and layer_offsets is not None and len(layer_offsets) > 1:
        bounds = list(layer_offsets) + [n]
        parts_i, parts_v = [], []
        for a, b in zip(bounds[:-1], bounds[1:]):
            if b <= a:
                continue
            i, v = select(kind, x[a:b], keep_count(b - a, cf), seed, stream, pos_base=a,
                          dgc_sample_fraction=dgc_sample_fraction)
            parts_i.append(i.astype(np.int64) + a)
            parts_v.append(v)
        idx = np.concatenate(parts_i).astype(np.uint32)
        vals = np.concatenate(parts_v)
    else:
        idx, vals = select(kind, x, keep_count(n, cf), seed, stream,
                           dgc_sample_fraction=dgc_sample_fraction)
    return idx, vals, n / vals.size


def compress_further(kind, idx: np.ndarray, vals: np.ndarray, original_length: int,
                     step: float, seed: int = 0, stream: int = 0,
                     dgc_sample_fraction: float = 0.01):
    """compressors.py:226-246 -> (indices, vals, achieved_cf)."""
    if step < 1.0:
        raise ValueError(f"step factor must be >= 1, got {step}")
    k1 = vals.size
    k2 = keep_count(k1, step)
    if k2 >= k1:
        return idx.copy(), vals.copy(), original_length / k1
    local, v2 = select(kind, vals, k2, seed, stream, dgc_sample_fraction=dgc_sample_fraction)
    return idx[local.astype(np.int64)], v2, original_length / k2


def update_residual(ef: np.ndarray, idx: np.ndarray, vals: np.ndarray) -> np.ndarray:
    """feedback.py:39-51."""
    ef = np.ascontiguousarray(ef, dtype=np.float32)
    idx = np.ascontiguousarray(idx, dtype=np.uint32)
    vals = np.ascontiguousarray(vals, dtype=np.float32)
    out = np.empty_like(ef)
    lib().orc_update_residual(_p(ef), _p(idx), _p(vals), vals.size, ef.size, _p(out))
    return out


def decompress(idx: np.ndarray, vals: np.ndarray, n: int) -> np.ndarray:
    """compressors.py:249-253."""
    out = np.zeros(n, dtype=np.float32)
    out[np.asarray(idx, dtype=np.int64)] = vals
    return out


def aggregate(parts, n: int) -> np.ndarray:
    """compressors.py:256-271; parts = [(idx, vals), ...] in worker order."""
    idx = np.ascontiguousarray(np.concatenate([np.asarray(p[0], dtype=np.uint32) for p in parts]))
    vals = np.ascontiguousarray(np.concatenate([np.asarray(p[1], dtype=np.float32) for p in parts]))
    counts = np.array([len(p[1]) for p in parts], dtype=np.uint64)
    out = np.empty(n, dtype=np.float32)
    _check(lib().orc_aggregate(_p(idx), _p(vals), _p(counts), len(parts), n, _p(out)))
    return out


def aggregate_dense(xs) -> np.ndarray:
    """compressors.py:274-285."""
    arr = np.ascontiguousarray(np.stack([np.asarray(x, dtype=np.float32) for x in xs]))
    out = np.empty(arr.shape[1], dtype=np.float32)
    _check(lib().orc_aggregate_dense(_p(arr), arr.shape[0], arr.shape[1], _p(out)))
    return out
