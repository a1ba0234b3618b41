"""GraVAC adaptive-CF controller with the fused GPU compression step.

Drop-in for ``gravac.controller`` (/root/reference/pkg/src/gravac/controller.py).
The scalar state machine (select_cf, scaling_policy, check_gravac, EWMA
observation order) is host logic kept arithmetic-identical to the reference,
so the chosen CF is bit-exact.  The data plane of ``run_iteration`` is the
hot path: per worker ONE fused selection pass computes g_ef = g + r (written
over the residual), ||g_ef||^2 and the kept energy of every CF in the ladder;
the host reads back 3 doubles per worker, decides, and a single emit kernel
writes the chosen (index, value) list and leaves g_ef - sent in the residual.
"""

from __future__ import annotations

import ctypes

from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

from . import _native as nat
from .compressors import (TOPK, CompressorKind, Selection, SparseGradient, _iota, compress,
                          compress_further, keep_count)
from .costmodel import (CostModelParams, allreduce_time, dense_message_words, iteration_time,
                        sparse_message_words)
from .feedback import ResidualStore
from .gradcore import GradientVector, SeededRng, ewma_lambda_from_workers
from .metrics import GainTracker, ThroughputTable, update_step

EXPONENTIAL = "exponential"
GEOMETRIC = "geometric"
POLICIES = (EXPONENTIAL, GEOMETRIC)

CANDIDATE = "candidate"
MINIMUM = "minimum"
DENSE = "dense"

# observability counters (bench.py reports them): exact-path re-scans after a
# missed threshold estimate, and speculative emits that had to be redone
STATS = {"fallbacks": 0, "spec_misses": 0, "steps": 0}

_STAGE_MIN = 0   # rng substream tags (controller.py:33-35)
_STAGE_STEP = 1


@dataclass(frozen=True)
class ControllerConfig:
    theta_min: float = 10.0
    theta_max: float = 1000.0
    epsilon: float = 0.7
    omega: float = 0.01
    window: int = 500
    policy: str = EXPONENTIAL
    compressor: CompressorKind = CompressorKind("topk")

    def __post_init__(self):
        if self.theta_min < 1.0:
            raise ValueError(f"theta_min must be >= 1, got {self.theta_min}")
        if self.theta_max < self.theta_min:
            raise ValueError(f"theta_max must be >= theta_min, got {self.theta_max}")
        if not (0.0 < self.epsilon < 1.0):
            raise ValueError(f"epsilon out of (0,1): {self.epsilon}")
        if not (0.0 < self.omega < 1.0):
            raise ValueError(f"omega out of (0,1): {self.omega}")
        if self.window < 1:
            raise ValueError(f"window must be >= 1, got {self.window}")
        if self.policy not in POLICIES:
            raise ValueError(f"unknown policy {self.policy!r}, expected one of {POLICIES}")


@dataclass
class CfDecision:
    choice: str
    cf: float
    gain: float
    delta_min: float
    delta_c: float


def select_cf(delta_c: float, delta_min: float, epsilon: float,
              candidate_cf: float | None = None, minimum_cf: float | None = None) -> CfDecision:
    """Candidate if its smoothed gain clears epsilon, else minimum, else dense (controller.py:74-82)."""
    if delta_c >= epsilon:
        return CfDecision(CANDIDATE, candidate_cf, delta_c, delta_min, delta_c)
    if delta_min >= epsilon:
        return CfDecision(MINIMUM, minimum_cf, delta_min, delta_min, delta_c)
    return CfDecision(DENSE, 1.0, 1.0, delta_min, delta_c)


def scaling_policy(policy: str, step: int, theta_min_initial: float, theta_max: float,
                   theta_min_current: float | None = None) -> float:
    """Step factor at policy step `step`, capped at theta_max / theta_min (controller.py:85-105).

    Step 0 evaluates theta_min itself (factor 1).  Exponential: 2^(2^(step-1));
    geometric: 2^step.
    """
    if step < 0:
        raise ValueError(f"policy step must be >= 0, got {step}")
    if policy not in POLICIES:
        raise ValueError(f"unknown policy {policy!r}")
    base = theta_min_initial if theta_min_current is None else theta_min_current
    cap = theta_max / base
    if step == 0:
        return min(1.0, cap)
    exponent = step if policy == GEOMETRIC else 2 ** (step - 1)
    if exponent >= 1024:  # 2.0**exponent would overflow; the cap wins anyway
        return cap
    return min(2.0 ** exponent, cap)


@dataclass
class ControllerState:
    config: ControllerConfig
    gains: GainTracker
    table: ThroughputTable
    theta_min: float
    theta_min_initial: float
    theta_s: float = 1.0
    step: int = 0
    iteration: int = 0
    frozen: bool = False
    theta_ideal: float | None = None
    saturation_picked_higher_cf: bool = False

    @classmethod
    def fresh(cls, config: ControllerConfig, workers: int) -> "ControllerState":
        return cls(config=config, gains=GainTracker(ewma_lambda_from_workers(workers)),
                   table=ThroughputTable(), theta_min=config.theta_min,
                   theta_min_initial=config.theta_min)

    @property
    def candidate_cf(self) -> float:
        return self.theta_s * self.theta_min


def check_gravac(state: ControllerState, iteration: int, delta_min: float | None,
                 delta_c: float | None) -> ControllerState:
    """Window-boundary escalation / step advance / saturation freeze (controller.py:137-171)."""
    cfg = state.config
    if state.frozen or iteration % cfg.window != 0:
        return state
    if delta_min is not None and delta_c is not None and delta_min > 0:
        if cfg.omega >= abs(delta_min - delta_c) / delta_min:
            state.theta_min = min(cfg.theta_max, state.theta_s * state.theta_min)
    state.step += 1
    state.theta_s = scaling_policy(cfg.policy, state.step, state.theta_min_initial, cfg.theta_max,
                                   state.theta_min)
    top = state.table.top_two()
    if top is not None:
        (cf_first, v_first), (cf_second, v_second) = top
        if v_second > 0 and abs(v_first - v_second) / v_second <= cfg.omega:
            state.theta_ideal = cf_second
            state.frozen = True
            if cf_second > cf_first:
                state.saturation_picked_higher_cf = True
            state.theta_s = max(1.0, state.theta_ideal / state.theta_min)
    return state


@dataclass
class IterationResult:
    sent: Sequence[SparseGradient] | Sequence[GradientVector]
    decision: CfDecision
    t_compute: float
    t_compress: float
    t_sync: float
    t_iter: float
    floats_sent: int
    words_sent: int
    gain_min_raw: float
    gain_c_raw: float
    candidate_cf: float
    theta_min: float
    # beyond the reference: raw mean gain of every CF evaluated in the fused sweep
    ladder_gains: dict = field(default_factory=dict)
    # run_iteration(average=True): the exchanged, averaged gradient of this step
    averaged: GradientVector | None = None


# ------------------------------------------------------------ fused step
class _WorkerStep:
    """Device-side work of one worker for one iteration (level 1 + level 2).

    Top-k evaluates every keep count of the step -- k1 (theta_min), k2 (the
    candidate) and the extra CFs' counts -- as ONE descending, de-duplicated
    ladder; ``slot[k]`` is the ladder entry holding keep count k.  Counts >= n
    keep everything (gain 1, no ladder entry)."""

    def __init__(self, kind: CompressorKind, g: torch.Tensor, store: ResidualStore, k1: int, k2: int,
                 extra_ks: Sequence[int], rng: SeededRng, i: int, w: int):
        self.kind, self.k1, self.k2 = kind, k1, k2
        self.extra_ks = list(extra_ks)
        self.store = store
        if k1 >= g.numel():
            resid = store.residual  # materialise any deferred update first
            pending = None
        else:
            pending = store._take_pending()
            resid = store._resid
        self.resid = resid
        self.n = g.numel()
        self.g_min: SparseGradient | None = None
        self.sel2: Selection | None = None
        self.identity1 = k1 >= self.n
        # the per-stage streams only feed Random-k (Top-k and Redsync draw nothing)
        needs_rng = kind.name not in (TOPK, "redsync")
        rng0 = rng.split(i, w, _STAGE_MIN) if needs_rng else None
        rng1 = rng.split(i, w, _STAGE_STEP) if needs_rng else None
        slot = f"step{w}"
        if kind.name == TOPK:
            self.ladder = sorted({k for k in [k1, k2, *self.extra_ks] if k < self.n}, reverse=True)
        else:
            self.ladder = [k1] if k1 < self.n else []
        self.slot = {k: j for j, k in enumerate(self.ladder)}
        if self.identity1:
            # theta_min == 1: level 1 keeps everything; g_ef by the EF kernel
            nat.check(nat.load().gvc_ef_add(nat.ptr(g), nat.ptr(resid), nat.ptr(resid), self.n,
                                            nat.stream_ptr(g.device)), "apply_feedback")
            self.g_min = SparseGradient._wrap(_iota(self.n, g.device), resid.clone(), self.n, 1.0)
            self.sel1 = None
            from .gradcore import squared_l2_norm_dev
            self._norm_dev = squared_l2_norm_dev(resid)
            if kind.name == TOPK:
                self.sel2 = Selection(kind, self.ladder, values=resid, slot=slot + "b") if self.ladder else None
            else:
                self.sel2 = (Selection(kind, [k2], values=self.g_min.vals, rng=rng1, slot=slot + "b")
                             if k2 < self.n else None)
            return
        if kind.name == TOPK:
            # F2: nested Top-k == exact top-k2 of the whole vector -> one sweep
            self.sel1 = Selection(kind, self.ladder, g=g, resid=resid, rng=rng0, slot=slot + "a",
                                  pending=pending, persist_res=True)
        else:
            self.ladder = [k1]
            # both levels' result records side by side: one read-back, no concatenation
            rb = nat.RESULT_BYTES
            self._res12 = nat.Workspace.get(g.device, slot + "/res12", 2 * rb)[:2 * rb]
            self.sel1 = Selection(kind, [k1], g=g, resid=resid, rng=rng0, slot=slot + "a", pending=pending,
                                  res_dev=self._res12[:rb])
            # the level-1 emit also builds its sent mask (every word, in the spare
            # buffer), the Redsync mean and the K7 tile bounds; taken if level 1 is sent
            self._mask1 = store._spare_buf()
            if self.n > 400_000_000:
                self._mask1.zero_()  # the emit ORs bits in global memory there
            bounds = torch.empty((self.n + nat.AGG_TILE - 1) // nat.AGG_TILE + 1, dtype=torch.int32,
                                 device=g.device).view(torch.uint32)
            idx, vals = self.sel1.emit(0, sent_mask=self._mask1, sent_m=store._pm, tile_bounds=bounds)
            self.g_min = SparseGradient._wrap(idx, vals, self.n, self.n / k1)
            self._bounds1 = bounds
            if k2 < k1:
                # a Redsync level 1 sends sign(v) * m: every nonzero level-1 value
                # has magnitude m, so level 2 (compressors.py:226-246) orders by
                # position alone -- equal_magnitudes skips the all-ties path
                # (152 us of k_pass1 + 86 us of tie handling at 66M, measured)
                self.sel2 = Selection(kind, [k2], values=vals, rng=rng1, slot=slot + "b",
                                      equal_magnitudes=kind.name == "redsync", res_dev=self._res12[rb:])

    def stats_dev(self) -> list[torch.Tensor]:
        """Device tensors whose bytes the host reads once per iteration."""
        out = [self._norm_dev.reshape(1)] if self.identity1 else []
        if self.sel1 is not None and self.sel2 is not None and getattr(self, "_res12", None) is not None:
            return out + [self._res12]  # the two records, adjacent
        if self.sel1 is not None:
            out.append(self.sel1.res_dev)
        if self.sel2 is not None:
            out.append(self.sel2.res_dev)
        return out

    def gains_from(self, raw: list[bytes], norm_host: float | None):
        """(ef_norm, E_min, E_c, extra energies) from the read-back results."""
        if self.identity1:
            import numpy as np
            norm_host = float(np.frombuffer(raw[0], dtype=np.float64)[0])
            raw = raw[1:]
        rb = nat.RESULT_BYTES
        results = [nat.SelectResult.from_buffer_copy(b[o:o + rb]) for b in raw for o in range(0, len(b), rb)]
        STATS["fallbacks"] += sum(int(r.fallback_used) for r in results)
        r1 = results[0] if self.sel1 is not None else None
        r2 = results[-1] if self.sel2 is not None else None
        for r in results:
            if r.status == nat.GVC_ERR_NAN:
                raise ValueError("NaN in gradient: compression order undefined")
            if r.status != nat.GVC_OK:
                raise RuntimeError(f"selection consistency failure (status {r.status})")
        norm = norm_host if self.identity1 else r1.ef_norm_sq
        if self.kind.name == TOPK:
            res = r2 if self.identity1 else r1

            def energy(k):  # a count >= n keeps everything: E = ||g_ef||^2
                return res.kept_sq[self.slot[k]] if k in self.slot else norm
            return norm, energy(self.k1), energy(self.k2), [energy(k) for k in self.extra_ks]
        if self.identity1:
            return norm, norm, (r2.kept_sq[0] if r2 is not None else norm), []
        e_min = r1.kept_sq[0]
        e_c = r2.kept_sq[0] if r2 is not None else e_min
        return norm, e_min, e_c, []

    def chosen_count(self, candidate: bool) -> int:
        if self.kind.name == TOPK:
            k = self.k2 if candidate else self.k1
            return k if k in self.slot else self.n
        return self.k2 if (candidate and self.sel2 is not None) else self.g_min.kept

    def emit(self, candidate: bool, payload=None, bounds: bool = False) -> SparseGradient:
        """Materialise the chosen view (into ``payload`` when given, with the
        K7 tile bounds when ``bounds``); the residual update g_ef - sent is
        deferred into the store's sent-mask (applied by the next fused pass)."""
        self._tile_bounds = None
        if bounds and payload is None and self.kind.name == TOPK and not self.identity1:
            self._tile_bounds = torch.empty((self.n + nat.AGG_TILE - 1) // nat.AGG_TILE + 1, dtype=torch.int32,
                                            device=self.resid.device).view(torch.uint32)
        part = self._emit(candidate, payload)
        if payload is not None and part.vals.data_ptr() == payload.vals.data_ptr():
            part._payload = payload
        if self._tile_bounds is not None:
            part._bounds = self._tile_bounds
        return part

    def _emit(self, candidate: bool, payload: torch.Tensor | None) -> SparseGradient:
        lib = nat.load()
        store = self.store
        mode = 2 if self.kind.name == "redsync" else 1
        if self.identity1:
            # theta_min == 1 (level 1 keeps everything): direct update, no mask
            if candidate and self.sel2 is not None and (self.kind.name != TOPK or self.k2 in self.slot):
                j = self.slot[self.k2] if self.kind.name == TOPK else 0
                idx, vals = self.sel2.emit(j, idx_map=self.g_min.indices, resid=self.resid)
                return SparseGradient._wrap(idx, vals, self.n, self.n / self.k2)
            # theta_s == 1 too (k2 >= n): the whole g_ef is sent, as compress_further copies
            part = self.g_min
            nat.check(lib.gvc_update_residual(nat.ptr(self.resid), nat.ptr(part.indices), nat.ptr(part.vals),
                                              part.kept, self.n, nat.ptr(self.resid),
                                              nat.stream_ptr(self.resid.device)), "update_residual")
            return part
        mask = store._mask_buf()
        if self.kind.name == TOPK:
            k = self.k2 if candidate else self.k1
            idx, vals = self.sel1.emit(self.slot[k], sent_mask=mask, sent_m=store._pm, payload=payload,
                                       tile_bounds=self._tile_bounds)
            part = SparseGradient._wrap(idx, vals, self.n, self.n / k)
        elif candidate and self.sel2 is not None:
            idx, vals = self.sel2.emit(0, idx_map=self.g_min.indices, sent_mask=mask, sent_m=store._pm,
                                       payload=payload)
            part = SparseGradient._wrap(idx, vals, self.n, self.n / self.k2)
        else:
            part = self.g_min
            part._bounds = self._bounds1
            # mask, Redsync mean (in store._pm) and bounds came with the level-1 emit
            store._adopt_mask(self._mask1, mode)
            return part
        store._pmode = mode
        return part


class _DgcStep:
    """DGC worker step: level 1 over g_ef (fused EF pass with the sampled
    threshold), level 2 over the level-1 values (compressors.py:226-246).
    Both levels are device-only (dgc.py): the norms, kept energies and the
    selects' statuses travel in the controller's one read-back."""

    def __init__(self, kind: CompressorKind, g: torch.Tensor, store: ResidualStore, k1: int, k2: int,
                 rng: SeededRng, i: int, w: int):
        from .dgc import dgc_select
        from .gradcore import squared_l2_norm_dev
        self.kind, self.k1, self.k2, self.store = kind, k1, k2, store
        self.n = g.numel()
        self.identity1 = False
        self._res = []
        self._res12 = None
        rng0 = rng.split(i, w, _STAGE_MIN)
        rng1 = rng.split(i, w, _STAGE_STEP)
        slot = f"dgc{w}"
        if k1 >= self.n:
            resid = store.residual
            nat.check(nat.load().gvc_ef_add(nat.ptr(g), nat.ptr(resid), nat.ptr(resid), self.n,
                                            nat.stream_ptr(g.device)), "apply_feedback")
            self.g_min = SparseGradient._wrap(_iota(self.n, g.device), resid.clone(), self.n, 1.0)
            self.norm = None
            self.identity_level1 = True
        else:
            self.identity_level1 = False
            pending = store._take_pending()
            # the level-1 emit also builds its sent mask (taken if level 1 is sent)
            self._mask1 = store._spare_buf()
            if self.n > 400_000_000:
                # past ~4.6e8 values the emit ORs mask bits in global memory
                # instead of writing every word from shared memory
                self._mask1.zero_()
            # (+ the decompress-average's tile boundaries of level 1, its emit's by-product)
            nb = (self.n + nat.AGG_TILE - 1) // nat.AGG_TILE + 1
            bounds = torch.empty(nb, dtype=torch.int32, device=g.device)  # owned by the sent part
            # both levels' result records side by side: one read-back, no concatenation
            rb = nat.RESULT_BYTES
            self._res12 = nat.Workspace.get(g.device, slot + "/res12", 2 * rb)[:2 * rb]
            idx, vals, sel1 = dgc_select(kind, None, k1, rng0, g=g, resid=store._resid, pending=pending,
                                         slot=slot + "a", want_result=True, sent_mask=self._mask1, check=False,
                                         tile_bounds=bounds, res_dev=self._res12[:rb])
            self.g_min = SparseGradient._wrap(idx, vals, self.n, self.n / k1)
            self.g_min._bounds = bounds
            self.norm = sel1.res_dev[:8].view(torch.float64)  # ||g_ef||^2 of the fused pass, on the device
            self._res.append(sel1.res_dev)
        if k2 < self.g_min.kept:
            res2 = self._res12[nat.RESULT_BYTES:] if self._res12 is not None else None
            idx2, vals2, sel2 = dgc_select(kind, self.g_min.vals, k2, rng1, idx_map=self.g_min.indices,
                                           slot=slot + "b", want_result=True, check=False, res_dev=res2)
            self.g_c = SparseGradient._wrap(idx2, vals2, self.n, self.n / k2)
            self._res.append(sel2.res_dev)
        else:
            self.g_c = self.g_min
        self.stats = None
        if self.identity_level1:
            # ||g_ef||^2 as a device scalar (every rank's row travels the same way in C2)
            self.stats = squared_l2_norm_dev(store._resid).reshape(1)
        # otherwise every number is in the selects' result records: ||g_ef||^2
        # of the fused pass and each level's kept energy -- the fp64 sums of
        # exactly the values sent (no separate norm kernels)

    def stats_dev(self) -> list[torch.Tensor]:
        if self.stats is None and len(self._res) == 2 and self._res12 is not None:
            return [self._res12]  # the two levels' records, adjacent
        return ([self.stats] if self.stats is not None else []) + self._res

    def gains_from(self, raw: list[bytes], norm_host=None):
        import numpy as np
        recs = []
        rb = nat.RESULT_BYTES
        chunks = [b[o:o + rb] for b in raw[1 if self.stats is not None else 0:] for o in range(0, len(b), rb)]
        for b in chunks:  # the DGC selects' records
            r = nat.SelectResult.from_buffer_copy(b)
            if r.status == nat.GVC_ERR_NAN:
                raise ValueError("NaN in gradient: compression order undefined")
            if r.status != nat.GVC_OK:
                raise RuntimeError(f"selection consistency failure (status {r.status})")
            recs.append(r)
        if self.identity_level1:  # theta_min == 1: the level-1 gain is exactly 1 (same sum)
            norm = float(np.frombuffer(raw[0], dtype=np.float64)[0])
            e_c = float(recs[0].kept_sq[0]) if recs else norm
            return norm, norm, e_c, []
        norm, e_min = float(recs[0].ef_norm_sq), float(recs[0].kept_sq[0])
        e_c = float(recs[1].kept_sq[0]) if len(recs) > 1 else e_min
        return norm, e_min, e_c, []

    def chosen_count(self, candidate: bool) -> int:
        return (self.g_c if candidate else self.g_min).kept

    def emit(self, candidate: bool, payload=None, bounds: bool = False) -> SparseGradient:
        part = self.g_c if candidate else self.g_min
        store = self.store
        if self.norm is None:  # identity level 1: direct residual update
            nat.check(nat.load().gvc_update_residual(nat.ptr(store._resid), nat.ptr(part.indices),
                                                     nat.ptr(part.vals), part.kept, self.n, nat.ptr(store._resid),
                                                     nat.stream_ptr(store._resid.device)), "update_residual")
            return part
        if not candidate or self.g_c is self.g_min:
            store._adopt_mask(self._mask1)  # built by the level-1 emit
            return part
        mask = store._mask_buf()
        nat.check(nat.load().gvc_mark_sent(nat.ptr(part.indices), part.kept, nat.ptr(mask),
                                           nat.stream_ptr(mask.device)), "mark_sent")
        store._pmode = 1
        return part


TIMELINE = None  # development aid (scripts/timeline.py): a list receiving (name, event, host time)


def _mark(name: str, stream=None) -> None:
    if TIMELINE is not None:
        import time
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        TIMELINE.append((name, ev, time.perf_counter()))


def _mean_raw_gain(energies: Sequence[float], ef_norms: Sequence[float]) -> float:
    """Mean over non-zero-norm workers of min(1, E/||g_ef||^2), worker order (controller.py:284-288)."""
    gains = [min(1.0, e / n) for e, n in zip(energies, ef_norms) if n > 0.0]
    return sum(gains) / len(gains)


def _average(sent, group, out: torch.Tensor | None, peer=None):
    """The step's exchange + mean of the sent views: worker parts on this GPU
    (compressors.aggregate / aggregate_dense) or, with a process group, C1 + K7
    (sparse; fused over peer memory when ``peer``) / C3 (dense) across the ranks."""
    from .compressors import aggregate_packed, aggregate_dense
    if isinstance(sent[0], SparseGradient):
        if peer is not None:
            return GradientVector._wrap(peer.aggregate(sent[0], out=out, staged=peer.staged))
        if group is not None:
            from .exchange import allgather_aggregate
            return allgather_aggregate(sent[0], group, out=out)
        if len(sent) == 1:
            p0 = sent[0]
            return GradientVector._wrap(aggregate_packed(p0.indices, p0.vals, [p0.kept], p0.original_length, out=out,
                                                         bounds=p0._bounds))
        from .compressors import aggregate
        return aggregate(sent)
    if group is not None:  # C3: the dense fallback, fused over peer memory where the node allows
        from .exchange import dense_mean
        return dense_mean(sent[0], group)
    return aggregate_dense(sent)


def run_iteration(state: ControllerState, gradients, residuals, cost: CostModelParams, rng: SeededRng,
                  batch_size: int = 1, *, extra_cfs: Sequence[float] = (), group=None,
                  average: bool = False, average_out: torch.Tensor | None = None) -> IterationResult:
    """One adaptive GraVAC step (controller.py:192-281) on the GPU.

    ``gradients``/``residuals``: one object (one worker) or worker-ascending
    sequences (workers simulated on this GPU), exactly as in the reference.
    With ``group`` (a torch.distributed process group), this process is ONE
    worker -- worker index = rank -- and the per-worker gain ratios are
    all-gathered so every rank takes the same decision in the reference's
    worker order.  ``extra_cfs``: more CFs whose gains the Top-k sweep
    evaluates in the same pass (any order, any value >= 1: a CF >= theta_min
    is nested under level 1 like compress_further, a smaller one is a plain
    compress); reported in ``ladder_gains`` but never fed to the EWMA
    trackers.  ``average=True`` also performs the
    step's exchange and mean (what the reference's simworkers does after
    run_iteration, simworkers.py:242-245) into ``IterationResult.averaged``;
    it is enqueued behind the speculative emit, so the device never waits for
    the host's decision.
    """
    _mark("start")
    cfg = state.config
    grads = [gradients] if isinstance(gradients, GradientVector) else list(gradients)
    stores = [residuals] if isinstance(residuals, ResidualStore) else list(residuals)
    if len(grads) != len(stores):
        raise ValueError(f"{len(grads)} gradients for {len(stores)} residual stores")
    if group is not None and len(grads) != 1:
        raise ValueError("with a process group each rank passes exactly one gradient")
    kind = cfg.compressor
    state.iteration += 1
    i = state.iteration
    theta_min = state.theta_min
    candidate_cf = state.candidate_cf
    length = grads[0].length
    rank = 0
    if group is not None:
        import torch.distributed as dist
        rank = dist.get_rank(group)
    k1 = keep_count(length, theta_min)
    k2 = keep_count(k1, state.theta_s)
    extra = [float(c) for c in extra_cfs if kind.name == TOPK]
    # an extra CF >= theta_min nests under level 1 (compress_further from k1);
    # one below theta_min is a plain compress of the whole gradient (larger k)
    extra_ks = [keep_count(k1, c / theta_min) if c >= theta_min else keep_count(length, c) for c in extra]

    steps = []
    for w, (g, store) in enumerate(zip(grads, stores)):
        if g.length != store.length:
            raise ValueError(f"length mismatch: gradient {g.length}, residual {store.length}")
        nat.require_cuda(g.values)
        if kind.name == "dgc":
            steps.append(_DgcStep(kind, g.values, store, k1, k2, rng, i, rank + w))
        else:
            steps.append(_WorkerStep(kind, g.values, store, k1, k2, extra_ks, rng, i, rank + w))

    _mark("selected")
    dev = grads[0].values.device
    peer = None
    if group is not None:
        from .exchange import PeerExchange, exchange_mode
        xmode = exchange_mode(group)
        if xmode != "nccl":
            peer = PeerExchange.get(group, dev)
            if peer.ok:
                peer.staged = xmode == "staged"
            else:  # no peer access: the all-gather exchange
                peer, xmode = None, "nccl"

    # ---- one device->host read per iteration: every worker's norms and
    # energies (with a process group: C2, all-gathered first).  Started on the
    # side stream BEFORE the speculative emit is enqueued, so the host decides
    # while the GPU emits and exchanges.
    stats = [t for s in steps for t in s.stats_dev()]
    sizes = [t.numel() * t.element_size() for t in stats]
    flat = stats[0].reshape(-1).view(torch.uint8) if len(stats) == 1 else \
        torch.cat([t.reshape(-1).view(torch.uint8) for t in stats])
    pending = rows = None
    c2_ready = None
    if group is not None:
        import torch.distributed as dist
        if dist.get_backend(group) == "nccl" and peer is not None:
            # C2 on a side stream (the peer-memory exchange issues no other NCCL
            # work this step, so the collective cannot be reordered against
            # one), ordered after the select by an event recorded here; its host
            # setup (~0.1 ms of torch / NCCL calls) is done after the speculative
            # emit and exchange are enqueued, so the GPU never waits for it
            c2_ready = nat.event_slot(dev, "c2_ready")
            nat.check(nat.load().gvc_event_record(c2_ready, nat.stream_ptr(dev)), "event_record")
        elif dist.get_backend(group) == "nccl":
            # NCCL exchange: every collective of this communicator on one stream
            # (collectives on two streams may execute in different orders on
            # different ranks and deadlock)
            gathered = torch.empty((dist.get_world_size(group), flat.numel()), dtype=torch.uint8, device=dev)
            dist.all_gather_into_tensor(gathered, flat, group=group)
            pending = nat.d2h_start(gathered)
        else:
            from .exchange import allgather_stats
            rows = allgather_stats(flat.cpu(), group)
    else:
        pending = nat.d2h_start(flat)
    _mark("stats_started")

    # ---- speculative emit: enqueue the previous step's choice right behind the
    # select so the GPU keeps working while the host reads the gains back; a
    # misprediction is re-emitted below (the sent mask is rebuilt from zero)
    spec = getattr(state, "_spec_choice", CANDIDATE)
    spec_parts = None

    def wire(s, c, bnd):
        if peer is not None:
            # staged pull: the emit writes the tile bounds (level-1 Top-k) and the
            # 16-bit wire indices into the slot, so the exchange launches no
            # bounds pass and moves 6 bytes per entry over NVLink
            return peer.slot(s.chosen_count(c), length, push=bnd and xmode == "push", bounds=bnd,
                             off16=xmode == "staged")
        from .exchange import new_payload
        return new_payload(s.chosen_count(c), dev, n=length if bnd else None)

    if kind.name == TOPK and not steps[0].identity1 and spec in (CANDIDATE, MINIMUM):
        c = spec == CANDIDATE
        if group is not None:
            spec_parts = [s.emit(c, wire(s, c, True)) for s in steps]
        else:
            spec_parts = [s.emit(c, bounds=average) for s in steps]
    _mark("spec_emitted")
    spec_avg = _average(spec_parts, group, average_out, peer) if (average and spec_parts is not None) else None
    _mark("spec_averaged")
    if c2_ready is not None:
        side = nat.side_stream(dev)
        nat.check(nat.load().gvc_stream_wait_event(ctypes.c_void_p(side.cuda_stream), c2_ready[0]), "stream_wait")
        with torch.cuda.stream(side):
            gathered = torch.empty((dist.get_world_size(group), flat.numel()), dtype=torch.uint8, device=dev)
            dist.all_gather_into_tensor(gathered, flat, group=group)
            pending = nat.d2h_start(gathered)
            _mark("c2_read", side)

    if pending is not None:
        raw_all = pending.wait()
        _mark("host_has_stats")
        if group is not None:
            rows = np.frombuffer(raw_all, dtype=np.uint8).reshape(-1, flat.numel())
    if group is not None:
        local = []
        for row in rows:
            raw, pos = [], 0
            for nb in sizes:
                raw.append(row[pos:pos + nb].tobytes())
                pos += nb
            local.append(steps[0].gains_from(raw, None))
    else:
        local, pos, t = [], 0, 0
        for s in steps:
            raw = []
            for _ in range(len(s.stats_dev())):
                raw.append(raw_all[pos:pos + sizes[t]])
                pos += sizes[t]
                t += 1
            local.append(s.gains_from(raw, None))
    ef_norms = [x[0] for x in local]

    def drop_speculation():
        for store in stores:
            if store._mask is not None:
                store._mask.zero_()
            store._pmode = 0

    if all(nv == 0.0 for nv in ef_norms):
        # vanished gradient: dense no-op (controller.py:217-230)
        if spec_parts is not None:
            drop_speculation()
        sent = []
        for store in stores:
            sent.append(GradientVector._wrap(store._resid, grads[0].layer_offsets))
            store._resid = torch.zeros_like(store._resid)
        t_sync = allreduce_time(dense_message_words(length), cost)
        decision = CfDecision(DENSE, 1.0, 1.0, 1.0, 1.0)
        t_iter = iteration_time(decision, cost.t_compute, 0.0, t_sync)
        update_step(state.table, 1.0, 1.0, t_iter, cost.workers, batch_size)
        d_min = state.gains.value(theta_min) if state.gains.has(theta_min) else None
        d_c = state.gains.value(candidate_cf) if state.gains.has(candidate_cf) else None
        check_gravac(state, i, d_min, d_c)
        out = IterationResult(sent, decision, cost.t_compute, 0.0, t_sync, t_iter, length,
                              dense_message_words(length), 1.0, 1.0, candidate_cf, theta_min)
        if average:
            out.averaged = _average(sent, group, None, peer)
        return out

    raw_min = _mean_raw_gain([x[1] for x in local], ef_norms)
    delta_min = state.gains.observe(theta_min, raw_min)
    raw_c = _mean_raw_gain([x[2] for x in local], ef_norms)
    delta_c = state.gains.observe(candidate_cf, raw_c)
    ladder = {theta_min: raw_min, candidate_cf: raw_c}
    for j, c in enumerate(extra):
        ladder[c] = _mean_raw_gain([x[3][j] for x in local], ef_norms)
    t_min = cost.compression_latency(kind, length, k1)
    t_step = cost.compression_latency(kind, k1, k2)
    t_compress = t_min + t_step

    decision = select_cf(delta_c, delta_min, cfg.epsilon, candidate_cf=candidate_cf, minimum_cf=theta_min)
    if decision.choice != DENSE:
        state._spec_choice = decision.choice
    STATS["steps"] += 1
    if spec_parts is not None and decision.choice != spec:
        STATS["spec_misses"] += 1
        drop_speculation()
        spec_parts = None
    if decision.choice == DENSE:
        sent = []
        for store in stores:
            # the residual buffer holds g_ef (the pending mask was consumed by the
            # fused pass): hand it over as the dense message, restart from zero
            sent.append(GradientVector._wrap(store._resid, grads[0].layer_offsets))
            store._resid = torch.zeros_like(store._resid)
        floats = length
        words = dense_message_words(length)
    else:
        cand = decision.choice == CANDIDATE
        if spec_parts is not None:
            sent = spec_parts
        elif group is not None:  # emit straight into the wire buffer (peer slot / all-gather payload)
            bnd = kind.name == TOPK and not steps[0].identity1
            sent = [s.emit(cand, wire(s, cand, bnd)) for s in steps]
        else:
            sent = [s.emit(cand, bounds=average) for s in steps]
        floats = sent[0].kept
        words = sparse_message_words(sent[0])

    t_sync = allreduce_time(words, cost)
    t_iter = iteration_time(decision, cost.t_compute, t_compress, t_sync)
    update_step(state.table, decision.cf, decision.gain, t_iter, cost.workers, batch_size)
    check_gravac(state, i, delta_min, delta_c)
    out = IterationResult(sent, decision, cost.t_compute, 0.0 if decision.choice == DENSE else t_compress,
                          t_sync, t_iter, floats, words, raw_min, raw_c, candidate_cf, theta_min, ladder)
    if average:
        out.averaged = spec_avg if (spec_parts is not None and sent is spec_parts) else \
            _average(sent, group, average_out if decision.choice != DENSE else None, peer)
    _mark("end")
    return out
