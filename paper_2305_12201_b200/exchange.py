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

import ctypes

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
    """Flat int32 wire buffer of one rank:
    [idx (kpad) | vals (kpad) | tile bounds (bpad) | 16-bit wire indices (opad, optional)].

    kpad/bpad/opad round to 4 words so every section stays 16-byte aligned.  The
    tile bounds (gvc_emit tile_bounds_dev) let K7 skip its boundary pass on the
    gathered parts; every rank uses the same layout (same kind, same k, n).
    The 16-bit wire indices (idx mod GVC_AGG_TILE, written by the emit beside
    idx) are what the staged exchange moves over NVLink instead of idx: 6
    bytes per entry instead of 8.
    """

    __slots__ = ("buf", "k", "kpad", "nb", "bpad", "opad", "idx", "vals", "bounds", "bounds_area", "peer",
                 "mirrors", "pushed", "off_word", "wire16")

    def __init__(self, k: int, n: int, device, with_bounds: bool = True, buf: torch.Tensor | None = None,
                 off16: bool = False):
        self.k = k
        self.kpad = (k + 3) & ~3
        self.nb = (n + nat.AGG_TILE - 1) // nat.AGG_TILE + 1 if (with_bounds or buf is not None) else 0
        self.bpad = (self.nb + 3) & ~3
        self.opad = ((self.kpad + 7) & ~7) // 2 if off16 else 0  # u16 entries padded to 8 (int4 granules)
        self.off_word = 2 * self.kpad + self.bpad
        self.wire16 = False  # set by the emit once it wrote the 16-bit wire indices
        if buf is None:
            buf = torch.empty(2 * self.kpad + self.bpad + self.opad, dtype=torch.int32, device=device)
        self.buf = buf
        self.idx = self.buf[:self.kpad].view(torch.uint32)
        self.vals = self.buf[self.kpad:2 * self.kpad].view(torch.float32)
        self.bounds_area = self.buf[2 * self.kpad:2 * self.kpad + self.nb].view(torch.uint32) if self.nb else None
        # bounds: set when the emit writes them (level-1 Top-k emits do)
        self.bounds = self.bounds_area if with_bounds else None
        self.peer = None
        self.mirrors = None  # nat.EmitMirrors: the peers' receive slots (push exchange)
        self.pushed = False  # set by the emit once the mirrors hold the full payload

    @staticmethod
    def words_for(k: int, n: int, off16: bool = False) -> int:
        nb = (n + nat.AGG_TILE - 1) // nat.AGG_TILE + 1
        kpad = (k + 3) & ~3
        return 2 * kpad + ((nb + 3) & ~3) + (((kpad + 7) & ~7) // 2 if off16 else 0)

    @property
    def off16_ptr(self) -> int:
        return self.buf.data_ptr() + 4 * self.off_word

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


class PeerExchange:
    """C1 + K7 fused over NVLink peer memory (one node, NCCL process group).

    Every rank owns one symmetric (peer-mapped) buffer:
        [flags: 64 u32 | parity 0: slot[0..W-1] | parity 1: slot[0..W-1]]
    Exchange number e uses parity e % 2; slot[r] holds rank r's payload
    (idx | vals | tile bounds, exchange.Payload layout).

    Push (Top-k level-1 emits, the hot path): the emit writes rank r's payload
    into slot[r] of its OWN buffer and, through gvc_emit_mirrored, into
    slot[r] of every peer's buffer while it runs (ordinary stores over
    NVLink, then a system fence).  gvc_peer_signal posts e into every rank's
    flags[r]; gvc_aggregate_peers waits for flags[p] >= e and merges the W
    slots of its own buffer -- local HBM reads only.
    Pull (any other payload): only the own slot is written; the merge reads
    slot[p] of rank p's buffer over NVLink.

    Reuse of parity e % 2 by exchange e + 2 needs no second barrier: a rank
    starts exchange e + 2 only after its merge of e + 1 saw every flag e + 1,
    and each rank posts e + 1 after its merge of e completed (same stream).
    All ranks run the same sequence of exchanges because they take identical
    decisions (C2).
    """

    FLAG_WORDS = 64
    CHUNK = 4096  # entries per staged-pull chunk (power of two)
    _cache: dict = {}

    def __init__(self, group, device):
        self.group, self.device = group, device
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if self.world > nat.MAX_PEERS:
            raise ValueError(f"peer exchange supports at most {nat.MAX_PEERS} ranks on one node")
        self.cap = 0
        self.epoch = 0
        self.buf = None
        self.handle = None
        self.staged = True  # pull payloads through the staged (copier + trailing merge) kernel
        self.ok = True
        import os
        sms = torch.cuda.get_device_properties(device).multi_processor_count
        # measured on B200 (scripts/stage_sweep.sh): 4096-entry chunks with one
        # copier CTA per 2 SMs beat 2048 x 148, 8192 x 148 and 1024 x 148
        self.copy_blocks = int(os.environ.get("GVC_STAGE_COPIERS", max(1, sms // 2)))
        self.chunk = int(os.environ.get("GVC_STAGE_CHUNK", self.CHUNK))

    @classmethod
    def get(cls, group, device) -> "PeerExchange":
        key = (id(group), device.index)
        px = cls._cache.get(key)
        if px is None:
            px = cls(group, device)
            px.ok = px._probe()
            cls._cache[key] = px
        return px

    def _probe(self) -> bool:
        """Can every rank map the others' memory?  A first (small) symmetric
        buffer is allocated and exchanged; the ranks agree on the outcome, so
        a node without peer access falls back to the NCCL exchange everywhere."""
        ok = 1
        try:
            self._ensure(4096)
        except Exception:  # no symmetric-memory backend / peer access on this node
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device=self.device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
        return bool(flag.item())

    def _slot_word(self, parity: int, src: int) -> int:
        return self.FLAG_WORDS + (parity * self.world + src) * self.cap

    def _ensure(self, words: int) -> None:
        if words <= self.cap:
            return
        import torch.distributed._symmetric_memory as symm
        # the step's C2 all-gather may still be in flight on the side stream:
        # finish it before this rank issues the collectives below
        torch.cuda.synchronize(self.device)
        cap = (words + 1023) & ~1023
        buf = symm.empty(self.FLAG_WORDS + 2 * self.world * cap, dtype=torch.int32, device=self.device)
        buf[:self.FLAG_WORDS].zero_()
        handle = symm.rendezvous(buf, self.group)  # collective: every rank grows together
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)  # every flag array is zero before anyone signals
        self.buf, self.handle, self.cap, self.epoch = buf, handle, cap, 0
        self._err_check = None
        self.bases = [int(p) for p in handle.buffer_ptrs]
        self._flag_ptrs = (ctypes.c_void_p * self.world)(*self.bases)
        # staged pull: per-chunk ready epochs (local); epochs restart with the buffer
        self.ready = torch.zeros(self.copy_blocks + cap // self.chunk + 2, dtype=torch.int32, device=self.device)

    ERR_WORD = 63  # GVC_FLAG_ERR_WORD: set by a bounded peer wait that timed out
    ERR_EVERY = 64

    def _check_err(self, e: int) -> None:
        """Every ERR_EVERY exchanges, read the flag area's error word back
        asynchronously (no stream sync); a timed-out wait of an earlier exchange
        -- a rank died or diverged -- raises here."""
        pend = self._err_check
        if pend is not None and pend[1].query():
            if int(pend[0][0]):
                raise RuntimeError("peer exchange: a wait for another rank timed out (a rank died or diverged); "
                                   "the exchanged averages since then are invalid")
            self._err_check = pend = None
        if pend is None and e % self.ERR_EVERY == 1:
            host = torch.empty(1, dtype=torch.int32, pin_memory=True)
            host.copy_(self.buf[self.ERR_WORD:self.ERR_WORD + 1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            self._err_check = (host, ev)

    def slot(self, k: int, n: int, push: bool = True, bounds: bool | None = None, off16: bool = False) -> Payload:
        """This rank's payload slot of the next exchange.  With ``push`` (a
        level-1 Top-k emit, which writes the tile bounds) the emit also writes
        the same slot of every peer; otherwise the peers pull.  ``bounds``
        (default: ``push``): the emit writes the tile bounds into the slot
        (a level-1 Top-k emit), else the exchange computes them.  ``off16``
        (staged pull): the emit also writes the 16-bit wire indices, which the
        copiers move instead of the u32 indices."""
        words = Payload.words_for(k, n, off16)
        self._ensure(words)
        e = self.epoch + 1
        base = self._slot_word(e % 2, self.rank)
        pl = Payload(k, n, self.device, with_bounds=push if bounds is None else bounds,
                     buf=self.buf[base:base + words], off16=off16)
        pl.peer = (self, e, base)
        if off16 and not push:
            m = nat.EmitMirrors()
            m.count = 0
            m.off16_dev = pl.off16_ptr
            pl.mirrors = m
        if push and self.world > 1:
            m = nat.EmitMirrors()
            m.count = self.world - 1
            for i, q in enumerate(r for r in range(self.world) if r != self.rank):
                b = self.bases[q] + 4 * base
                m.idx_dev[i] = b
                m.vals_dev[i] = b + 4 * pl.kpad
                m.bounds_dev[i] = b + 8 * pl.kpad
            pl.mirrors = m
        return pl

    def aggregate(self, part: SparseGradient, out: torch.Tensor | None = None, staged: bool = True) -> torch.Tensor:
        """The rank-ordered fp64 mean of every rank's part (aggregate() semantics).

        Pull payloads are merged either ``staged`` (copier CTAs stream the
        peers' payloads into this rank's own slots chunk by chunk while the
        merge tiles trail them) or directly (the tiles read the peers' slots
        over NVLink)."""
        n = part.original_length
        pl = getattr(part, "_payload", None)
        if pl is None or pl.peer is None or pl.peer[0] is not self or pl.peer[1] != self.epoch + 1 \
                or pl.vals.data_ptr() != part.vals.data_ptr():
            pl = self.slot(part.kept, n, push=False)
            pl.idx[:part.kept].copy_(part.indices)
            pl.vals[:part.kept].copy_(part.vals)
            pl.bounds = None
        _, e, _ = pl.peer
        self._check_err(e)
        lib = nat.load()
        stream = nat.stream_ptr(self.device)
        pushed = pl.pushed
        if not pushed and pl.bounds is None:  # the emit did not write them (level-2 / non-Top-k views)
            nat.check(lib.gvc_tile_bounds(nat.ptr(pl.idx), part.kept, n, nat.ptr(pl.bounds_area), stream),
                      "tile_bounds")
        self.epoch = e
        nat.check(lib.gvc_peer_signal(self._flag_ptrs, self.world, self.rank, e, stream), "peer_signal")
        W = self.world
        own = self.bases[self.rank]
        if out is None:
            out = torch.empty(n, dtype=torch.float32, device=self.device)
        counts = (ctypes.c_uint64 * W)(*([part.kept] * W))
        peer_slot = [self.bases[p] + 4 * self._slot_word(e % 2, p) for p in range(W)]  # slot p in rank p's buffer
        own_slot = [own + 4 * self._slot_word(e % 2, p) for p in range(W)]  # slot p in this rank's buffer
        if not pushed and staged and W > 1:
            # staged pull: local staging = own_slot[p] (payload and tile bounds); sources = peer_slot[p]
            sg = nat.PeerStaging()
            sg.self_rank = self.rank
            sg.copy_blocks = self.copy_blocks
            sg.chunk_entries = self.chunk
            sg.ready_dev = self.ready.data_ptr()
            for p in range(W):
                sg.src_idx_dev[p] = peer_slot[p]
                sg.src_vals_dev[p] = peer_slot[p] + 4 * pl.kpad
                sg.src_bounds_dev[p] = peer_slot[p] + 8 * pl.kpad
                if pl.wire16:  # every rank's emit wrote them (identical decisions, identical path)
                    sg.src_off16_dev[p] = peer_slot[p] + 4 * pl.off_word
                    sg.off16_dev[p] = own_slot[p] + 4 * pl.off_word
            idx = (ctypes.c_void_p * W)(*own_slot)
            vals = (ctypes.c_void_p * W)(*[b + 4 * pl.kpad for b in own_slot])
            bnd = (ctypes.c_void_p * W)(*[b + 8 * pl.kpad for b in own_slot])
            nat.check(lib.gvc_aggregate_peers_staged(idx, vals, bnd, counts, W, n, nat.ptr(self.buf), e,
                                                     ctypes.byref(sg), nat.ptr(out), stream), "aggregate_peers")
            return out
        # push: every slot is in this rank's buffer; pull: slot p lives in rank p's buffer
        bases = own_slot if pushed else peer_slot
        idx = (ctypes.c_void_p * W)(*bases)
        vals = (ctypes.c_void_p * W)(*[b + 4 * pl.kpad for b in bases])
        bnd = (ctypes.c_void_p * W)(*[b + 8 * pl.kpad for b in bases])
        nat.check(lib.gvc_aggregate_peers(idx, vals, bnd, counts, W, n, nat.ptr(self.buf), e, nat.ptr(out),
                                          stream), "aggregate_peers")
        return out


def exchange_mode(group) -> str:
    """"staged" / "pull" / "push" (the NVLink peer-memory exchange) or "nccl"
    (all-gather + K7).  Peer memory needs an NCCL group of at most 8 ranks on one node.
    GVC_EXCHANGE overrides; the default is the staged pull (measured on B200,
    ms/step: 2 ranks staged 0.350, pull 0.367, push 0.389, nccl 0.397; 4 ranks
    staged 0.454, pull 0.533, nccl 0.598, push 0.638)."""
    import os
    if group is None or dist.get_backend(group) != "nccl" or dist.get_world_size(group) > nat.MAX_PEERS:
        return "nccl"
    mode = os.environ.get("GVC_EXCHANGE", "auto")
    if mode == "auto":
        mode = "staged"
    if mode not in ("push", "pull", "staged", "nccl"):
        raise ValueError(f"GVC_EXCHANGE={mode!r}: expected push, pull, staged, nccl or auto")
    return mode


class DenseExchange:
    """C3 -- the dense fallback's exchange + mean -- fused over NVLink peer memory.

    Every rank owns one symmetric buffer [flags: 64 u32 | parity 0: n | parity 1: n]
    (floats).  Exchange x: each rank copies its dense message into its own
    parity-x%2 region and posts 2x - 1; gvc_dense_mean_peers makes it the owner
    of 1/W of the positions: it sums the W inputs there in fp64 in rank order
    (aggregate_dense's arithmetic, compressors.py:274-285) and writes the mean
    into that range of every rank's region; after everyone posted 2x, the full
    mean is copied out.  Per rank 2 (W - 1) / W of the vector crosses NVLink
    (the all-gather fallback receives W - 1 whole vectors).  A region is reused
    two exchanges later, after every rank posted 2x + 1 -- which it does only
    after its own copy-out of x.
    """

    FLAG_WORDS = 64
    _cache: dict = {}

    def __init__(self, group, device):
        self.group, self.device = group, device
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.cap = 0
        self.x = 0
        self.err = torch.zeros(1, dtype=torch.int32, device=device)

    @classmethod
    def get(cls, group, device) -> "DenseExchange":
        key = (id(group), device.index)
        dx = cls._cache.get(key)
        if dx is None:
            dx = cls._cache[key] = cls(group, device)
        return dx

    def _ensure(self, n: int) -> None:
        if n <= self.cap:
            return
        import torch.distributed._symmetric_memory as symm
        torch.cuda.synchronize(self.device)
        cap = (n + 1023) & ~1023
        buf = symm.empty(self.FLAG_WORDS + 2 * cap, dtype=torch.int32, device=self.device)
        buf[:self.FLAG_WORDS].zero_()
        handle = symm.rendezvous(buf, self.group)  # collective: every rank grows together
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        self.buf, self.handle, self.cap, self.x = buf, handle, cap, 0
        self.bases = [int(p) for p in handle.buffer_ptrs]
        self._flag_ptrs = (ctypes.c_void_p * self.world)(*self.bases)

    def mean(self, g: GradientVector, out: torch.Tensor | None = None) -> torch.Tensor:
        n = g.length
        self._ensure(n)
        x = self.x + 1
        base = self.FLAG_WORDS + (x % 2) * self.cap  # words
        own = self.buf[base:base + n].view(torch.float32)
        own.copy_(g.values)
        lib = nat.load()
        stream = nat.stream_ptr(self.device)
        W = self.world
        nat.check(lib.gvc_peer_signal(self._flag_ptrs, W, self.rank, 2 * x - 1, stream), "peer_signal")
        regions = (ctypes.c_void_p * W)(*[b + 4 * base for b in self.bases])
        nat.check(lib.gvc_dense_mean_peers(regions, W, self.rank, n, nat.ptr(self.buf), 2 * x - 1,
                                           nat.ptr(self.err), stream), "dense_mean_peers")
        nat.check(lib.gvc_peer_signal(self._flag_ptrs, W, self.rank, 2 * x, stream), "peer_signal")
        if out is None:
            out = torch.empty(n, dtype=torch.float32, device=self.device)
        nat.check(lib.gvc_dense_collect(nat.ptr(own), nat.ptr(out), n, nat.ptr(self.buf), W, 2 * x,
                                        nat.ptr(self.err), stream), "dense_collect")
        self.x = x
        return out


def dense_mean(g: GradientVector, group=None) -> GradientVector:
    """C3 with the reference's fp64 rank-ordered mean: fused over peer memory
    (DenseExchange) on an NCCL group of one node, else all-gather + mean."""
    if (group is not None and dist.get_backend(group) == "nccl" and dist.get_world_size(group) <= nat.MAX_PEERS
            and exchange_mode(group) != "nccl"):
        px = PeerExchange.get(group, g.values.device)
        if px.ok:  # symmetric memory works on this node (probed once, agreed by every rank)
            return GradientVector._wrap(DenseExchange.get(group, g.values.device).mean(g), g.layer_offsets)
    return allgather_dense_mean(g, group)


def allgather_dense_mean(g: GradientVector, group=None) -> GradientVector:
    """C3: dense fallback with the reference's fp64 rank-ordered mean."""
    from .compressors import aggregate_dense
    world = dist.get_world_size(group)
    out = torch.empty((world, g.length), dtype=torch.float32, device=g.values.device)
    dist.all_gather_into_tensor(out, g.values, group=group)
    return aggregate_dense([GradientVector._wrap(out[r]) for r in range(world)])
