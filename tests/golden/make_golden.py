"""Generate golden input/output vectors from the UNMODIFIED reference.

Run in the build container only (the reference lives at /root/reference and
does not travel to the GPU box):

    python tests/golden/make_golden.py

It imports ``gravac`` from /root/reference/pkg/src, drives the hot-path
functions on seeded synthetic inputs and writes ``tests/golden/*.npz``.  The
fixtures are committed; the oracle (oracle/) and the CUDA path are both
checked against them by the test-suite, so neither needs the reference at
run time.

Fixture families (every case stores its inputs next to the reference's
outputs; float arrays are stored as float32 so bit patterns survive):

* ``topk.npz`` / ``redsync.npz`` -- compressors.compress(kind, g, cf)
  (compressors.py:193-223) over six input distributions incl. heavy ties,
  exact zeros with -0.0, +-inf and layer-scaled magnitudes.
* ``further.npz`` -- compress_further on a level-1 result (compressors.py:226-246).
* ``feedback.npz`` -- apply_feedback / update_residual (feedback.py:32-51).
* ``gain.npz`` -- squared_l2_norm + compression_gain_raw (gradcore.py:61-70,
  metrics.py:18-32).
* ``aggregate.npz`` -- aggregate / aggregate_dense / decompress
  (compressors.py:249-285).
* ``dgc_small.npz`` -- DGC where the sample is the whole vector (n <= 256,
  compressors.py:112-115): position-exact.
* ``run_iteration.npz`` -- controller.run_iteration traces (controller.py:192-281)
  for Top-k and Redsync with 1 and 3 workers: chosen CF, raw gains, theta_min.
* ``training.npz`` -- simworkers.run_training in every mode (simworkers.py:174-304)
  on tests/fixture_tasks.NoisyBowl: trace columns, final weights, JSON lines.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    if not os.path.isdir(REF):
        raise SystemExit("reference not present; golden vectors are generated in the build container only")
    sys.path.insert(0, REF)
    import gravac  # noqa: F401
    return gravac


def dist_vector(kind: str, n: int, rng: np.random.Generator) -> np.ndarray:
    """The six synthetic input distributions of SURVEY.md section 8(d)."""
    g = rng.standard_normal(n).astype(np.float32)
    if kind == "gauss":
        return g
    if kind == "ties":
        return (np.round(8 * g) / 8).astype(np.float32)
    if kind == "zeros":
        z = g.copy()
        mask = rng.random(n) < 0.5
        z[mask] = 0.0
        neg = mask & (rng.random(n) < 0.5)
        z[neg] = -0.0
        return z
    if kind == "layered":
        out = g.copy()
        cuts = rng.integers(1, n, size=max(1, n // 500)) if n > 1 else np.zeros(0, dtype=np.int64)
        bounds = np.unique(np.concatenate([[0], cuts, [n]]))
        for a, b in zip(bounds[:-1], bounds[1:]):
            out[a:b] *= np.float32(10.0 ** rng.uniform(-3, 0))
        return out
    if kind == "inf":
        x = g.copy()
        pos = rng.choice(n, size=max(1, n // 1000), replace=False)
        x[pos] = np.where(rng.random(pos.size) < 0.5, np.inf, -np.inf).astype(np.float32)
        return x
    if kind == "const":
        return np.full(n, np.float32(rng.choice([-1.0, 1.0]) * 0.5), dtype=np.float32) * \
            np.where(rng.random(n) < 0.5, 1, -1).astype(np.float32)
    raise ValueError(kind)


DISTS = ("gauss", "ties", "zeros", "layered", "inf", "const")


def _cases_compress(gravac, kind_name, seed):
    from gravac.compressors import CompressorKind, compress
    from gravac.gradcore import GradientVector
    kind = CompressorKind(kind_name)
    rng = np.random.default_rng(seed)
    out = {}
    sizes = [1, 2, 3, 7, 64, 257, 1000, 4099, 20_000, 65_537]
    i = 0
    for n in sizes:
        for d in DISTS:
            if kind_name == "redsync" and d == "inf":
                continue  # inf - inf in the mean makes values nan; not a valid fixture
            x = dist_vector(d, n, rng)
            cfs = [1.5, 10.0, 100.0, float(rng.uniform(1, max(1.0, n)))]
            if n <= 4099:
                cfs.append(1.0)
            out[f"{i}/x"] = x
            out[f"{i}/cfs"] = np.array(cfs, dtype=np.float64)
            out[f"{i}/dist"] = np.array(d)
            for j, cf in enumerate(cfs):
                s, _ = compress(kind, GradientVector(x), cf)
                out[f"{i}/{j}/idx"] = s.indices.astype(np.uint32)
                out[f"{i}/{j}/vals"] = s.vals.astype(np.float32)
            i += 1
    out["n_cases"] = np.int64(i)
    return out


def _cases_further(gravac):
    from gravac.compressors import CompressorKind, compress, compress_further
    from gravac.gradcore import GradientVector
    rng = np.random.default_rng(7)
    out = {}
    i = 0
    for kind_name in ("topk", "redsync"):
        kind = CompressorKind(kind_name)
        for n in (10, 1000, 20_000):
            for d in ("gauss", "ties", "zeros", "layered"):
                x = dist_vector(d, n, rng)
                pairs = ((10.0, 10.0), (10.0, 100.0), (4.0, 2.0), (2.0, 1.0), (3.0, 7.5))
                out[f"{i}/kind"] = np.array(kind_name)
                out[f"{i}/x"] = x
                out[f"{i}/pairs"] = np.array(pairs)
                for j, (cf1, step) in enumerate(pairs):
                    s1, _ = compress(kind, GradientVector(x), cf1)
                    s2, _ = compress_further(kind, s1, step)
                    out[f"{i}/{j}/idx1"] = s1.indices
                    out[f"{i}/{j}/vals1"] = s1.vals
                    out[f"{i}/{j}/idx2"] = s2.indices
                    out[f"{i}/{j}/vals2"] = s2.vals
                    out[f"{i}/{j}/cf2"] = np.float64(s2.achieved_cf)
                i += 1
    out["n_cases"] = np.int64(i)
    return out


def _cases_feedback(gravac):
    from gravac.compressors import CompressorKind, compress
    from gravac.feedback import ResidualStore, apply_feedback, update_residual
    from gravac.gradcore import GradientVector
    rng = np.random.default_rng(11)
    out = {}
    i = 0
    for kind_name in ("topk", "redsync"):
        kind = CompressorKind(kind_name)
        for n in (5, 300, 10_000, 30_011):
            for d in ("gauss", "ties", "zeros", "layered"):
                store = ResidualStore(n)
                # three chained iterations so the residual is non-trivial
                for it in range(3):
                    g = dist_vector(d, n, rng)
                    ef = apply_feedback(GradientVector(g), store)
                    s, _ = compress(kind, ef, 10.0)
                    update_residual(ef, s, store)
                    out[f"{i}/kind"] = np.array(kind_name)
                    out[f"{i}/g"] = g
                    out[f"{i}/chain"] = np.int64(it)
                    if n <= 300:
                        out[f"{i}/ef"] = ef.values
                    out[f"{i}/idx"] = s.indices
                    out[f"{i}/vals"] = s.vals
                    out[f"{i}/r_after"] = store.residual.copy()
                    i += 1
    out["n_cases"] = np.int64(i)
    return out


def _cases_gain(gravac):
    from gravac.compressors import CompressorKind, compress
    from gravac.gradcore import GradientVector, squared_l2_norm
    from gravac.metrics import compression_gain_raw
    rng = np.random.default_rng(13)
    out = {}
    i = 0
    for kind_name in ("topk", "redsync"):
        kind = CompressorKind(kind_name)
        for n in (2, 100, 5000, 50_000):
            for d in ("gauss", "ties", "zeros", "layered"):
                x = dist_vector(d, n, rng)
                if not np.any(x):
                    x[0] = 1.0
                g = GradientVector(x)
                cfs = (1.0, 10.0, 100.0, 1000.0)
                out[f"{i}/kind"] = np.array(kind_name)
                out[f"{i}/x"] = x
                out[f"{i}/cfs"] = np.array(cfs)
                out[f"{i}/norm"] = np.float64(squared_l2_norm(g))
                out[f"{i}/gain_raw"] = np.array([compression_gain_raw(compress(kind, g, cf)[0], g)
                                                 for cf in cfs])
                i += 1
    out["n_cases"] = np.int64(i)
    return out


def _cases_aggregate(gravac):
    from gravac.compressors import (CompressorKind, aggregate, aggregate_dense,
                                    compress, decompress)
    from gravac.gradcore import GradientVector
    rng = np.random.default_rng(17)
    topk = CompressorKind("topk")
    out = {}
    i = 0
    for n in (4, 1000, 20_011):
        for nparts in (1, 2, 3, 4, 8):
            for cf in ((1.0, 2.0, 10.0, 100.0) if n <= 1000 else (2.0, 10.0, 100.0)):
                xs = [dist_vector("gauss" if p % 2 == 0 else "layered", n, rng) for p in range(nparts)]
                parts = [compress(topk, GradientVector(x), cf)[0] for x in xs]
                out[f"{i}/n"] = np.int64(n)
                out[f"{i}/nparts"] = np.int64(nparts)
                for p, s in enumerate(parts):
                    out[f"{i}/idx{p}"] = s.indices
                    out[f"{i}/vals{p}"] = s.vals
                out[f"{i}/agg"] = aggregate(parts).values
                if nparts <= 3 and cf == 10.0:
                    for p in range(nparts):
                        out[f"{i}/x{p}"] = xs[p]
                    out[f"{i}/agg_dense"] = aggregate_dense([GradientVector(x) for x in xs]).values
                out[f"{i}/dec0"] = decompress(parts[0]).values
                i += 1
    out["n_cases"] = np.int64(i)
    return out


def _cases_dgc_small(gravac):
    from gravac.compressors import CompressorKind, compress
    from gravac.gradcore import GradientVector, SeededRng
    rng = np.random.default_rng(19)
    dgc = CompressorKind("dgc")
    out = {}
    i = 0
    for n in (1, 5, 64, 200, 256):
        for d in ("gauss", "ties", "zeros"):
            x = dist_vector(d, n, rng)
            for cf in (1.0, 2.0, 4.0, 16.0):
                s, _ = compress(dgc, GradientVector(x), cf, SeededRng(i))
                out[f"{i}/x"] = x
                out[f"{i}/cf"] = np.float64(cf)
                out[f"{i}/idx"] = s.indices
                out[f"{i}/vals"] = s.vals
                i += 1
    out["n_cases"] = np.int64(i)
    return out


def _cases_dgc_stats(gravac):
    """Distribution of DGC's overlap with exact top-k over 300 rng seeds
    (the reference's test_compressors.py:88-96 case, n=1e4, cf=100).  The
    sample positions themselves are parity-unpinned; their statistics are not."""
    from gravac.compressors import CompressorKind, compress
    from gravac.gradcore import GradientVector, SeededRng
    x = SeededRng(11).generator.standard_normal(10_000).astype(np.float32)
    order = np.lexsort((np.arange(x.size), -np.abs(x)))
    top = set(order[:100].tolist())
    overlaps = []
    for s in range(300):
        sp, _ = compress(CompressorKind("dgc"), GradientVector(x), 100, SeededRng(s))
        overlaps.append(len(set(sp.indices.tolist()) & top) / 100)
    return {"x": x, "overlaps": np.array(overlaps), "n_cases": np.int64(1)}


def _cases_run_iteration(gravac):
    from gravac.compressors import CompressorKind
    from gravac.controller import ControllerConfig, ControllerState, run_iteration
    from gravac.costmodel import CostModelParams
    from gravac.feedback import ResidualStore
    from gravac.gradcore import GradientVector, SeededRng
    out = {}
    i = 0
    configs = [
        # (kind, workers, length, theta_min, theta_max, eps, window, policy, iters)
        ("topk", 1, 4096, 10.0, 1000.0, 0.4, 3, "exponential", 14),
        ("topk", 3, 2048, 4.0, 256.0, 0.5, 2, "geometric", 12),
        ("topk", 2, 1000, 2.0, 64.0, 0.7, 2, "exponential", 12),
        ("redsync", 1, 4096, 10.0, 1000.0, 0.3, 3, "exponential", 12),
        ("redsync", 3, 2048, 4.0, 256.0, 0.2, 2, "geometric", 12),
    ]
    for (kind_name, workers, length, tmin, tmax, eps, window, policy, iters) in configs:
        cfg = ControllerConfig(theta_min=tmin, theta_max=tmax, epsilon=eps, omega=0.05,
                               window=window, policy=policy, compressor=CompressorKind(kind_name))
        state = ControllerState.fresh(cfg, workers)
        cost = CostModelParams(workers=workers)
        rng = SeededRng(3)
        data = SeededRng(1234)
        stores = [ResidualStore(length) for _ in range(workers)]
        grads_all, rec = [], []
        for it in range(1, iters + 1):
            grads = [data.split(1, 0, w, it).generator.standard_normal(length, dtype=np.float32)
                     * np.float32(1.0 + 0.5 * w) for w in range(workers)]
            grads_all.append(np.stack(grads))
            res = run_iteration(state, [GradientVector(g) for g in grads], stores, cost, rng)
            rec.append([it, {"candidate": 0, "minimum": 1, "dense": 2}[res.decision.choice],
                        res.decision.cf, res.gain_min_raw, res.gain_c_raw, res.candidate_cf,
                        res.theta_min, res.floats_sent, res.decision.delta_min, res.decision.delta_c])
        out[f"{i}/kind"] = np.array(kind_name)
        out[f"{i}/cfg"] = np.array([workers, length, tmin, tmax, eps, window, iters], dtype=np.float64)
        out[f"{i}/policy"] = np.array(policy)
        out[f"{i}/grads"] = np.stack(grads_all)
        out[f"{i}/trace"] = np.array(rec, dtype=np.float64)
        out[f"{i}/resid_final"] = np.stack([s.residual for s in stores])
        i += 1
    out["n_cases"] = np.int64(i)
    return out


def _cases_training(gravac):
    """simworkers.run_training (simworkers.py:174-304) in every mode on the
    tests' NoisyBowl task (tests/fixture_tasks.py)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from tests.fixture_tasks import CHOICES, TRACE_COLUMNS, TRAINING_CASES, NoisyBowl
    from gravac.compressors import CompressorKind
    from gravac.controller import ControllerConfig
    from gravac.costmodel import CostModelParams
    from gravac.gradcore import GradientVector
    from gravac.simworkers import OptimizerState, run_training
    out = {}
    for i, (mode, kind, cf, tmin, eps, workers, size, iters, lr, mom) in enumerate(TRAINING_CASES):
        task = NoisyBowl(size, GradientVector, seed=i)
        cfg = (ControllerConfig(theta_min=tmin, theta_max=256.0, epsilon=eps, omega=0.05, window=3,
                                compressor=CompressorKind(kind)) if mode == "gravac" else None)
        opt = OptimizerState(np.zeros(size), lr=lr, momentum=mom, weight_decay=1e-4, lr_decay_iters=(iters - 2,))
        res = run_training(task, opt, CostModelParams(workers=workers), mode, iters, seed=100 + i,
                           controller_config=cfg, compressor=CompressorKind(kind) if kind else None, static_cf=cf)
        out[f"{i}/trace"] = np.array([[getattr(r, c) for c in TRACE_COLUMNS] for r in res.trace], dtype=np.float64)
        out[f"{i}/choice"] = np.array([CHOICES[r.choice] for r in res.trace], dtype=np.int64)
        out[f"{i}/weights"] = res.weights
        out[f"{i}/metric"] = np.float64(res.metric_value)
        out[f"{i}/jsonl"] = np.array(res.trace.to_jsonl())
    out["n_cases"] = np.int64(len(TRAINING_CASES))
    return out


def main():
    gravac = _import_reference()
    families = {
        "topk": lambda: _cases_compress(gravac, "topk", 1),
        "redsync": lambda: _cases_compress(gravac, "redsync", 2),
        "further": lambda: _cases_further(gravac),
        "feedback": lambda: _cases_feedback(gravac),
        "gain": lambda: _cases_gain(gravac),
        "aggregate": lambda: _cases_aggregate(gravac),
        "dgc_small": lambda: _cases_dgc_small(gravac),
        "dgc_stats": lambda: _cases_dgc_stats(gravac),
        "run_iteration": lambda: _cases_run_iteration(gravac),
        "training": lambda: _cases_training(gravac),
    }
    only = set(sys.argv[1:])
    for name, fn in families.items():
        if only and name not in only:
            continue
        data = fn()
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **data)
        print(f"{name}: {int(data['n_cases'])} cases -> {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
