"""ctypes binding of libgravac_b200.so (include/gravac_b200.h).

The product path has exactly one backend: the sm_100a kernels in this
library.  There is no CPU fallback -- if the library is missing or no CUDA
device is present, every compute call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgravac_b200.so")

GVC_OK, GVC_ERR_ARG, GVC_ERR_NAN, GVC_ERR_WORKSPACE, GVC_ERR_CUDA, GVC_ERR_STATE = 0, -1, -2, -3, -4, -5
GVC_TOPK, GVC_DGC, GVC_REDSYNC, GVC_RANDOMK = 0, 1, 2, 3
KIND_IDS = {"topk": GVC_TOPK, "dgc": GVC_DGC, "redsync": GVC_REDSYNC, "randomk": GVC_RANDOMK}
MAX_LADDER = 16
AGG_TILE = 4096  # GVC_AGG_TILE: outputs per CTA of the decompress-average

# every symbol include/gravac_b200.h declares (tests assert the .so exports them)
EXPORTS = (
    "gvc_last_error", "gvc_abi_version", "gvc_select_workspace_bytes", "gvc_select", "gvc_emit",
    "gvc_ef_add", "gvc_sq_norm_workspace_bytes", "gvc_sq_norm", "gvc_update_residual",
    "gvc_decompress", "gvc_aggregate", "gvc_aggregate_workspace_bytes", "gvc_aggregate_dense",
    "gvc_iota", "gvc_prof_enable", "gvc_prof_min_n", "gvc_prof_read", "gvc_launch_count", "gvc_mark_sent", "gvc_apply_pending",
    "gvc_gather_ef", "gvc_below_keys", "gvc_compact_workspace_bytes", "gvc_compact_mask",
    "gvc_peer_signal", "gvc_aggregate_peers", "gvc_tile_bounds", "gvc_emit_mirrored",
    "gvc_aggregate_peers_staged", "gvc_dgc_sample", "gvc_dgc_sample_gather", "gvc_select_phase_times", "gvc_dense_mean_peers",
    "gvc_dense_collect", "gvc_segmented_select_workspace_bytes", "gvc_segmented_select", "gvc_segmented_dgc_workspace_bytes", "gvc_segmented_dgc_select", "gvc_workspace_forget", "gvc_segmented_redsync_values", "gvc_segmented_redsync_workspace_bytes", "gvc_add_segment_offsets", "gvc_read_async", "gvc_event_done", "gvc_event_record", "gvc_stream_wait_event", "gvc_copy_async",
)
MAX_PEERS = 8  # GVC_MAX_PEERS

_u64, _i32, _f64, _vp, _sz = ctypes.c_uint64, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t


class SelectArgs(ctypes.Structure):
    _fields_ = [
        ("kind", _i32), ("n_ks", _i32), ("n", _u64),
        ("values_dev", _vp), ("g_dev", _vp), ("resid_dev", _vp),
        ("ks", _u64 * MAX_LADDER),
        ("seed", _u64), ("rng_stream", _u64), ("pos_base", _u64),
        ("dgc_sample_fraction", _f64),
        ("force_exact", _i32), ("pending_mode", _i32),
        ("pending_mask_dev", _vp), ("pending_m_dev", _vp),
        ("key_est_dev", _vp), ("allow_short", _i32), ("equal_magnitudes", _i32),
        ("dgc_thr_dev", _vp), ("dgc_sampled_dev", _vp),
    ]


class SelectResult(ctypes.Structure):
    _fields_ = [
        ("ef_norm_sq", _f64),
        ("kept_sq", _f64 * MAX_LADDER),
        ("kept_abs", _f64 * MAX_LADDER),
        ("threshold_key", ctypes.c_uint32 * MAX_LADDER),
        ("pad0", ctypes.c_uint32 * MAX_LADDER),
        ("tie_quota", _u64 * MAX_LADDER),
        ("redsync_mean", ctypes.c_float * MAX_LADDER),
        ("candidates", _u64),
        ("status", _i32),
        ("fallback_used", _i32),
        ("kept_count", _u64 * MAX_LADDER),
        ("kept_nonzero", _u64 * MAX_LADDER),
        ("shortfall", _u64),
    ]


RESULT_BYTES = ctypes.sizeof(SelectResult)


class PeerStaging(ctypes.Structure):
    """gvc_peer_staging: the staged-pull exchange (copier CTAs + merge tiles)."""
    _fields_ = [("self_rank", _i32), ("copy_blocks", _i32), ("chunk_entries", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32), ("ready_dev", _vp), ("src_idx_dev", _vp * 8),
                ("src_vals_dev", _vp * 8), ("src_bounds_dev", _vp * 8), ("src_off16_dev", _vp * 8),
                ("off16_dev", _vp * 8)]


class EmitMirrors(ctypes.Structure):
    """gvc_emit_mirrors: peer destinations the emit also writes (push exchange),
    and the staged exchange's 16-bit wire indices (off16_dev)."""
    _fields_ = [("count", _i32), ("reserved", _i32), ("idx_dev", _vp * 8), ("vals_dev", _vp * 8),
                ("bounds_dev", _vp * 8), ("off16_dev", _vp)]

_lib = None
_lock = threading.Lock()


def load(build_if_missing: bool = False):
    """Load the native library; raises ImportError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            if build_if_missing:
                from . import build_ext
                build_ext.build()
            else:
                raise ImportError(
                    f"{LIB_PATH} is missing: build the sm_100a extension first "
                    "(python -m paper_2305_12201_b200.build_ext); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        L.gvc_last_error.restype = ctypes.c_char_p
        L.gvc_abi_version.restype = ctypes.c_int
        L.gvc_select_workspace_bytes.argtypes = [ctypes.c_int, _u64]
        L.gvc_select_workspace_bytes.restype = _sz
        L.gvc_select.argtypes = [ctypes.POINTER(SelectArgs), _vp, _sz, _vp, _vp]
        L.gvc_emit.argtypes = [_vp, _sz, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
        L.gvc_mark_sent.argtypes = [_vp, _u64, _vp, _vp]
        L.gvc_apply_pending.argtypes = [_vp, _vp, _u64, ctypes.c_int, _vp, _vp]
        L.gvc_ef_add.argtypes = [_vp, _vp, _vp, _u64, _vp]
        L.gvc_sq_norm_workspace_bytes.argtypes = [_u64]
        L.gvc_sq_norm_workspace_bytes.restype = _sz
        L.gvc_sq_norm.argtypes = [_vp, _u64, _vp, _vp, _sz, _vp]
        L.gvc_update_residual.argtypes = [_vp, _vp, _vp, _u64, _u64, _vp, _vp]
        L.gvc_decompress.argtypes = [_vp, _vp, _u64, _u64, _vp, _vp, _sz, _vp]
        L.gvc_aggregate.argtypes = [_vp, _vp, _vp, _vp, ctypes.c_int, _u64, _vp, _vp, _sz, _vp, _u64, _vp]
        L.gvc_aggregate_workspace_bytes.argtypes = [ctypes.c_int, _u64]
        L.gvc_aggregate_workspace_bytes.restype = _sz
        L.gvc_aggregate_dense.argtypes = [_vp, ctypes.c_int, _u64, _vp, _vp]
        L.gvc_iota.argtypes = [_vp, _u64, _vp]
        L.gvc_gather_ef.argtypes = [_vp, _u64, _vp, _vp, _vp, _vp, _vp, ctypes.c_int, _vp, _vp]
        L.gvc_below_keys.argtypes = [_vp, _vp, _u64, _vp, _vp, _vp, _vp, _vp]
        L.gvc_compact_workspace_bytes.argtypes = [_u64]
        L.gvc_compact_workspace_bytes.restype = _sz
        L.gvc_compact_mask.argtypes = [_vp, _u64, _vp, _vp, _vp, _sz, _vp]
        L.gvc_peer_signal.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_uint32, _vp]
        L.gvc_aggregate_peers.argtypes = [_vp, _vp, _vp, _vp, ctypes.c_int, _u64, _vp, ctypes.c_uint32, _vp, _vp]
        L.gvc_tile_bounds.argtypes = [_vp, _u64, _u64, _vp, _vp]
        L.gvc_dgc_sample.argtypes = [_u64, _u64, _u64, _u64, _u64, _vp, _vp]
        L.gvc_dgc_sample_gather.argtypes = [_u64, _u64, _u64, _u64, _u64, _vp, _vp, _vp, _vp, _vp, ctypes.c_int,
                                            _vp, _vp, _vp]
        L.gvc_dense_mean_peers.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _u64, _vp, ctypes.c_uint32, _vp, _vp]
        L.gvc_dense_collect.argtypes = [_vp, _vp, _u64, _vp, ctypes.c_int, ctypes.c_uint32, _vp, _vp]
        L.gvc_segmented_select_workspace_bytes.argtypes = [_u64, ctypes.c_int]
        L.gvc_segmented_select_workspace_bytes.restype = _sz
        L.gvc_workspace_forget.argtypes = [_vp]
        L.gvc_add_segment_offsets.argtypes = [_vp, _u64, _vp, _vp, ctypes.c_int, _vp]
        L.gvc_segmented_redsync_values.argtypes = [_vp, _vp, _vp, ctypes.c_int, _vp, _sz, _vp]
        L.gvc_segmented_redsync_workspace_bytes.argtypes = [_u64, ctypes.c_int]
        L.gvc_segmented_redsync_workspace_bytes.restype = _sz
        L.gvc_read_async.argtypes = [_vp, _vp, _sz, _vp, _vp, _vp]
        L.gvc_event_done.argtypes = [_vp]
        L.gvc_event_record.argtypes = [_vp, _vp]
        L.gvc_stream_wait_event.argtypes = [_vp, _vp]
        L.gvc_copy_async.argtypes = [_vp, _vp, _sz, _vp]
        L.gvc_segmented_dgc_workspace_bytes.argtypes = [_u64, ctypes.c_int, ctypes.c_double]
        L.gvc_segmented_dgc_workspace_bytes.restype = _sz
        L.gvc_segmented_dgc_select.argtypes = [_vp, _u64, _vp, _vp, ctypes.c_int, ctypes.c_double, _u64, _u64, _vp,
                                               _vp, _vp, _sz, _vp, _vp]
        L.gvc_segmented_select.argtypes = [ctypes.c_int, _vp, _u64, _vp, _vp, ctypes.c_int, _u64, _u64, _vp, _vp,
                                           _vp, _sz, _vp, _vp]
        L.gvc_aggregate_peers_staged.argtypes = [_vp, _vp, _vp, _vp, ctypes.c_int, _u64, _vp, ctypes.c_uint32,
                                                 ctypes.POINTER(PeerStaging), _vp, _vp]
        L.gvc_emit_mirrored.argtypes = [_vp, _sz, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                        ctypes.POINTER(EmitMirrors), _vp]
        L.gvc_prof_enable.argtypes = [ctypes.c_int]
        L.gvc_prof_enable.restype = None
        L.gvc_prof_min_n.argtypes = [_u64]
        L.gvc_prof_min_n.restype = None
        L.gvc_prof_read.argtypes = [_vp, _vp, ctypes.c_int]
        L.gvc_launch_count.restype = ctypes.c_ulonglong
        if hasattr(L, "gvc_select_phase_times"):  # diagnostic
            L.gvc_select_phase_times.argtypes = [_vp, _vp, ctypes.c_int]
        if L.gvc_abi_version() != 2:
            raise ImportError("libgravac_b200 ABI version mismatch")
        _lib = L
        return L


def check(rc: int, what: str = "") -> None:
    if rc == GVC_OK:
        return
    msg = load().gvc_last_error().decode(errors="replace")
    if rc in (GVC_ERR_ARG, GVC_ERR_NAN):
        raise ValueError(msg or what)
    raise RuntimeError(f"{what}: {msg} (status {rc})")


def require_cuda(t: torch.Tensor) -> None:
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor (the compression path runs on the GPU only)")


def ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _dev_index(device) -> int:
    if device is None:
        return torch.cuda.current_device()
    if isinstance(device, int):
        return device
    idx = device.index
    return torch.cuda.current_device() if idx is None else idx


def stream_ptr(device=None):
    """The current CUDA stream of ``device`` as a raw cudaStream_t (the fast
    accessor: torch.cuda.current_stream() costs tens of microseconds of host
    time per call in this torch build)."""
    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(_dev_index(device)))


class Workspace:
    """Grow-only device scratch buffers, one per (device, slot)."""

    _bufs: dict = {}

    @classmethod
    def get(cls, device: torch.device, slot: str, nbytes: int) -> torch.Tensor:
        key = (device.index if device.index is not None else torch.cuda.current_device(), slot)
        buf = cls._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            if buf is not None:  # the library's per-workspace caches name the old address
                load().gvc_workspace_forget(ctypes.c_void_p(buf.data_ptr()))
            buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
            cls._bufs[key] = buf
        return buf


_ws_bytes: dict = {}


def select_workspace(device, slot: str, kind: int, n: int) -> torch.Tensor:
    nb = _ws_bytes.get((kind, n))
    if nb is None:
        nb = _ws_bytes[(kind, n)] = int(load().gvc_select_workspace_bytes(kind, n))
    return Workspace.get(device, slot, nb)


PROF_CATS = ("collect", "select", "emit", "aggregate")


def prof_enable(on: bool) -> None:
    load().gvc_prof_enable(1 if on else 0)


def prof_read() -> dict:
    """{category: (total_ms, launches)} since the last read (synchronises on the events)."""
    ms = (ctypes.c_double * len(PROF_CATS))()
    cnt = (ctypes.c_ulonglong * len(PROF_CATS))()
    load().gvc_prof_read(ms, cnt, len(PROF_CATS))
    return {c: (ms[i], cnt[i]) for i, c in enumerate(PROF_CATS)}


def launch_count() -> int:
    return int(load().gvc_launch_count())


_pinned: dict = {}


def d2h_bytes(t: torch.Tensor) -> bytes:
    """Device -> host copy of a small tensor with a low-latency wait.

    The copy goes to a cached pinned buffer and the host spins on a CUDA event
    instead of a blocking synchronise, so the controller's single read-back per
    step costs microseconds of wake-up, not a scheduler quantum."""
    nb = t.numel() * t.element_size()
    key = (t.device.index, nb)
    buf = _pinned.get(key)
    if buf is None:
        buf = (torch.empty(nb, dtype=torch.uint8, pin_memory=True), (ctypes.c_void_p * 2)())
        _pinned[key] = buf
    host, evs = buf
    if not t.is_contiguous():
        t = t.contiguous()
    s = stream_ptr(t.device)  # copied on the current stream itself
    check(load().gvc_read_async(ctypes.c_void_p(host.data_ptr()), ctypes.c_void_p(t.data_ptr()), nb, s, s, evs),
          "read")
    return PendingRead(host, ctypes.c_void_p(evs[1]), t).wait()


_side: dict = {}
_events: dict = {}


def event_slot(device, name: str):
    """A per-(device, name) slot holding a library-created cudaEvent_t
    (gvc_event_record creates it on first use)."""
    idx = device.index if device.index is not None else torch.cuda.current_device()
    slot = _events.get((idx, name))
    if slot is None:
        slot = _events[(idx, name)] = (ctypes.c_void_p * 1)()
    return slot


def side_stream(device) -> torch.cuda.Stream:
    """A per-device side stream for read-backs and small collectives that
    must not queue behind the main stream's later work."""
    idx = device.index if device.index is not None else torch.cuda.current_device()
    s = _side.get(idx)
    if s is None:
        s = torch.cuda.Stream(device=device)
        _side[idx] = s
    return s


class PendingRead:
    """A device->host copy started on the side stream; ``wait()`` spins on its event."""

    __slots__ = ("host", "ev", "src")

    def __init__(self, host, ev, src):
        self.host, self.ev, self.src = host, ev, src

    def wait(self) -> bytes:
        done = load().gvc_event_done
        while True:
            r = done(self.ev)
            if r:
                break
        check(r if r < 0 else 0, "read-back")
        self.src = None
        return self.host.numpy().tobytes()


def d2h_start(t: torch.Tensor, ready: "torch.cuda.Event | None" = None) -> PendingRead:
    """Start the read-back of a small tensor once the current stream reaches
    this point (or ``ready``), on the side stream: work enqueued afterwards on
    the current stream is not delayed by the copy, and the host can wait for
    this result while that work runs."""
    nb = t.numel() * t.element_size()
    key = ("async", t.device.index, nb)
    buf = _pinned.get(key)
    if buf is None:
        # (ready, done) events, created by the library on first use
        buf = (torch.empty(nb, dtype=torch.uint8, pin_memory=True), (ctypes.c_void_p * 2)())
        _pinned[key] = buf
    host, evs = buf
    if not t.is_contiguous():
        t = t.contiguous()
    side = side_stream(t.device)
    if ready is not None:
        side.wait_event(ready)
    # one C call: no torch stream bookkeeping (tens of microseconds of host time
    # per torch stream / event call in this build)
    check(load().gvc_read_async(ctypes.c_void_p(host.data_ptr()), ctypes.c_void_p(t.data_ptr()), nb,
                                stream_ptr(t.device), ctypes.c_void_p(side.cuda_stream), evs), "read_async")
    return PendingRead(host, ctypes.c_void_p(evs[1]), t)


def read_result(res_dev: torch.Tensor) -> SelectResult:
    """Device -> host copy of a gvc_select_result (waits for the stream)."""
    return SelectResult.from_buffer_copy(d2h_bytes(res_dev)[:RESULT_BYTES])
