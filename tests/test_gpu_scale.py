"""GPU parity at the sizes the benchmark measures, and the adaptive controller
with an extra-CF ladder.

BASELINE configs: C2 (ResNet101, 44.5M, Top-k CF search {10,100,1000}), C4
(LSTM, 66M, Redsync and Random-k, CF {10,100}), C3 / north star (VGG16, 138M,
Top-k ladder and DGC in both of its branches).  Each step runs through the
drop-in ``run_iteration`` (EF, fused select, decision, emit, deferred residual,
decompress-average) and is replayed on the C oracle: indices, chosen CF,
averaged gradient and residual bit-exact; gains within 1e-6 (fp64 summation
order only); Redsync values within 1e-6 (their fp64 mean is summed in a
different order, compressors.py:188).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from tests.conftest import bits  # noqa: E402

RTOL = 1e-6


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2305_12201_b200 as G
    from paper_2305_12201_b200 import _native
    _native.load()
    return G


def host(t):
    return t.cpu().numpy()


def _gauss(n, seed):
    return np.random.default_rng(seed).standard_normal(n, dtype=np.float32)


def _ladder_k(n, k1, theta_min, c):
    """Keep count of an extra CF (controller.run_iteration's nesting rule)."""
    return O.keep_count(k1, c / theta_min) if c >= theta_min else O.keep_count(n, c)


def _replay_step(kind, ef, k1, theta_s, it, w, rng):
    """(i1, v1), (i2, v2): level 1 and the nested candidate of one worker (controller.py:232-250)."""
    n = ef.size
    s0, s1 = rng.split(it, w, 0), rng.split(it, w, 1)
    if kind == "topk":
        i1 = O.topk_indices(ef, k1)
        v1 = ef[i1.astype(np.int64)]
    else:
        i1, v1 = O.select(kind, ef, k1, seed=s0.seed, stream=s0.stream)
    i2, v2, _ = O.compress_further(kind, i1, v1, n, theta_s, seed=s1.seed, stream=s1.stream)
    return (i1, v1), (i2, v2)


def _run_chain(G, kind, n, steps, *, theta_min=10.0, theta_s=10.0, extra=(), epsilon=0.35, seed0=0):
    """`steps` chained run_iteration steps of one worker vs the oracle replay."""
    cfg = G.ControllerConfig(theta_min=theta_min, theta_max=1000.0, epsilon=epsilon, window=1 << 30,
                             compressor=G.CompressorKind(kind))
    state = G.ControllerState.fresh(cfg, 1)
    state.theta_s = theta_s
    store = G.ResidualStore(n)
    cost = G.CostModelParams(workers=1)
    rng = G.SeededRng(7)
    r_host = np.zeros(n, dtype=np.float32)
    seen = []
    for it in range(1, steps + 1):
        g = _gauss(n, seed0 + it)
        k1 = O.keep_count(n, state.theta_min)
        ts = state.theta_s
        res = G.run_iteration(state, G.GradientVector(g), store, cost, rng, extra_cfs=extra, average=True)
        ef = O.ef_add(g, r_host)
        norm = O.sq_norm(ef)
        (i1, v1), (i2, v2) = _replay_step(kind, ef, k1, ts, it, 0, rng)
        assert res.gain_min_raw == pytest.approx(min(1.0, O.sq_norm(v1) / norm), rel=RTOL)
        assert res.gain_c_raw == pytest.approx(min(1.0, O.sq_norm(v2) / norm), rel=RTOL)
        for c in extra:
            kc = _ladder_k(n, k1, theta_min, c)
            want = min(1.0, O.sq_norm(ef[O.topk_indices(ef, kc).astype(np.int64)]) / norm)
            assert res.ladder_gains[c] == pytest.approx(want, rel=RTOL), (it, c)
        seen.append(res.decision.choice)
        assert res.decision.choice != "dense", (it, res.decision)
        ci, cv = (i2, v2) if res.decision.choice == "candidate" else (i1, v1)
        part = res.sent[0]
        assert np.array_equal(host(part.indices), ci), it
        if kind == "redsync":
            np.testing.assert_allclose(host(part.vals), cv, rtol=RTOL)
        else:
            assert np.array_equal(bits(host(part.vals)), bits(cv)), it
        # the step's average (one worker: fp64 sum / 1 -> fp32, simworkers.py:242-245)
        want_avg = O.aggregate([(host(part.indices), host(part.vals))], n)
        assert np.array_equal(bits(host(res.averaged.values)), bits(want_avg)), it
        r_host = O.update_residual(ef, ci, host(part.vals))
        assert np.array_equal(bits(host(store.residual)), bits(r_host)), it
    return seen


@pytest.mark.slow
def test_resnet101_topk_ladder_44M(G):
    """C2: 44.5M, Top-k with the CF search {10, 100, 1000} in one sweep, EF, 3 chained steps."""
    seen = _run_chain(G, "topk", 44_500_000, 3, extra=(1000.0,))
    assert seen


@pytest.mark.slow
@pytest.mark.parametrize("kind,eps", [("redsync", 0.25), ("randomk", 0.05)])
def test_lstm_66M(G, kind, eps):
    """C4: 66M, Redsync and Random-k at CF {10, 100}, EF, 2 chained steps."""
    _run_chain(G, kind, 66_000_000, 2, epsilon=eps)


@pytest.mark.slow
def test_vgg16_topk_ladder_138M(G):
    """North star: 138M, Top-k ladder {10, 100, 1000} + EF, 2 chained steps."""
    _run_chain(G, "topk", 138_000_000, 2, extra=(1000.0,), seed0=20)


@pytest.mark.slow
def test_vgg16_dgc_138M_both_branches(G):
    """C3: DGC at 138M in both branches of compressors.py:123-137 (seeds chosen
    with the oracle so that one takes the exact branch and one the overshoot
    pad + top-up branch), bit-exact against the oracle."""
    n = 138_000_000
    x = _gauss(n, 0)
    g = G.GradientVector(x)
    K = G.CompressorKind("dgc")
    branches = set()
    for cf, seed in ((10.0, 0), (10.0, 1), (100.0, 0), (100.0, 1)):
        k = O.keep_count(n, cf)
        rng = G.SeededRng(seed)
        branches.add(O.dgc_overshoots(x, k, rng.seed, rng.stream))
        s, _ = G.compress(K, g, cf, rng)
        oi, ov = O.select("dgc", x, k, seed=rng.seed, stream=rng.stream)
        assert np.array_equal(host(s.indices), oi), (cf, seed)
        assert np.array_equal(bits(host(s.vals)), bits(ov)), (cf, seed)
    assert branches == {True, False}


@pytest.mark.slow
def test_vgg16_dgc_run_iteration_138M(G):
    """C3 through run_iteration: DGC level 1 over g_ef + level 2, EF, 2 chained steps."""
    _run_chain(G, "dgc", 138_000_000, 2, seed0=40)


# ------------------------------------------------- adaptive run + extra CFs
@pytest.mark.parametrize("workers", [1, 2])
def test_adaptive_run_with_extra_cfs(G, workers):
    """The exponential policy with window 2 escalates theta_min and grows
    theta_s while extra CFs on both sides of theta_min ride in the same sweep
    (controller.py:85-105, 137-171): no error, and every ladder gain, the
    chosen CF, the sent entries and the residual match the oracle."""
    n = 400_003
    extra = (20.0, 100.0, 160.0, 1000.0)
    cfg = G.ControllerConfig(theta_min=10.0, theta_max=1000.0, epsilon=0.2, omega=0.9, window=2,
                             policy="exponential", compressor=G.CompressorKind("topk"))
    state = G.ControllerState.fresh(cfg, workers)
    cost = G.CostModelParams(workers=workers)
    rng = G.SeededRng(5)
    stores = [G.ResidualStore(n) for _ in range(workers)]
    r_host = [np.zeros(n, dtype=np.float32) for _ in range(workers)]
    tmins = set()
    for it in range(1, 15):
        gs = [_gauss(n, 1000 * w + it) for w in range(workers)]
        tmin, ts = state.theta_min, state.theta_s
        tmins.add(tmin)
        k1 = O.keep_count(n, tmin)
        res = G.run_iteration(state, [G.GradientVector(x) for x in gs], stores, cost, rng, extra_cfs=extra)
        efs = [O.ef_add(gs[w], r_host[w]) for w in range(workers)]
        norms = [O.sq_norm(e) for e in efs]
        want = {}
        for c in (tmin, tmin * ts, *extra):
            kc = k1 if c == tmin else (O.keep_count(k1, ts) if c == tmin * ts else _ladder_k(n, k1, tmin, c))
            gains = [min(1.0, O.sq_norm(e[O.topk_indices(e, kc).astype(np.int64)]) / nv) if kc < n else 1.0
                     for e, nv in zip(efs, norms)]
            want[c] = sum(gains) / workers
        for c in extra:
            assert res.ladder_gains[c] == pytest.approx(want[c], rel=RTOL), (it, c)
        assert res.gain_min_raw == pytest.approx(want[tmin], rel=RTOL)
        assert res.gain_c_raw == pytest.approx(want[tmin * ts], rel=RTOL)
        for w in range(workers):
            if res.decision.choice == "dense":
                r_host[w] = np.zeros(n, dtype=np.float32)
                continue
            kc = k1 if res.decision.choice == "minimum" else O.keep_count(k1, ts)
            ci = O.topk_indices(efs[w], kc)
            cv = efs[w][ci.astype(np.int64)]
            assert np.array_equal(host(res.sent[w].indices), ci), (it, w)
            assert np.array_equal(bits(host(res.sent[w].vals)), bits(cv)), (it, w)
            r_host[w] = O.update_residual(efs[w], ci, cv)
            assert np.array_equal(bits(host(stores[w].residual)), bits(r_host[w])), (it, w)
    assert len(tmins) > 1, tmins  # theta_min escalated at least once


def test_identity_level1_with_extra_cfs(G):
    """theta_min == 1 with extra CFs: at policy step 0 the candidate is CF 1 too
    (k2 == n), so the candidate sends all of g_ef (compress_further copies,
    compressors.py:239-240) and the residual becomes zero; the extra CFs' gains
    are still reported."""
    n = 200_001
    cfg = G.ControllerConfig(theta_min=1.0, theta_max=1000.0, epsilon=0.5, window=1 << 30,
                             compressor=G.CompressorKind("topk"))
    state = G.ControllerState.fresh(cfg, 1)
    store = G.ResidualStore(n)
    cost = G.CostModelParams(workers=1)
    g = _gauss(n, 3)
    res = G.run_iteration(state, G.GradientVector(g), store, cost, G.SeededRng(1), extra_cfs=(10.0, 100.0))
    assert res.decision.choice == "candidate" and res.decision.cf == 1.0
    assert res.floats_sent == n and res.sent[0].kept == n
    assert np.array_equal(bits(host(res.sent[0].vals)), bits(g))
    assert not host(store.residual).any()
    for c in (10.0, 100.0):
        k = O.keep_count(n, c)
        want = O.sq_norm(g[O.topk_indices(g, k).astype(np.int64)]) / O.sq_norm(g)
        assert res.ladder_gains[c] == pytest.approx(want, rel=RTOL)


# ------------------------------------------------------------- layerwise
def _resnet101_offsets():
    """Parameter tensor sizes of ResNet-101 (torchvision layout: conv, BN weight
    and bias, downsample, fc), as GradientVector layer offsets: ~314 segments,
    44.5M values."""
    sizes = [64 * 3 * 7 * 7, 64, 64]
    inplanes = 64
    for planes, blocks in ((64, 3), (128, 4), (256, 23), (512, 3)):
        for b in range(blocks):
            sizes += [inplanes * planes, planes, planes, planes * planes * 9, planes, planes,
                      planes * planes * 4, planes * 4, planes * 4]
            if b == 0:
                sizes += [inplanes * planes * 4, planes * 4, planes * 4]
            inplanes = planes * 4
    sizes += [2048 * 1000, 1000]
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    return offs, int(np.sum(sizes))


@pytest.mark.parametrize("kind", ["topk", "randomk", "redsync", "dgc"])
def test_layerwise_resnet101_segments(G, kind):
    """compressors.py:204-217 on ResNet-101's ~314 layer segments (44.5M values)
    as one segmented selection: every segment's keep count, order and values
    bit-exact against the oracle's per-segment compress."""
    offs, n = _resnet101_offsets()
    assert len(offs) > 300 and abs(n - 44_500_000) < 200_000
    x = _gauss(n, 11)
    for a, b in zip(offs[:40:3], offs[1:41:3]):  # layer-scaled segments, heavy ties in some
        x[a:b] *= np.float32(10.0 ** (-(a % 7) / 3))
    x[offs[5]:offs[6]] = np.round(x[offs[5]:offs[6]] * 2) / 2
    rng = G.SeededRng(9)
    g = G.GradientVector(x, tuple(int(o) for o in offs))
    for cf in (10.0, 100.0):
        s, _ = G.compress(G.CompressorKind(kind), g, cf, rng, layerwise=True)
        oi, ov, _ = O.compress(kind, x, cf, seed=rng.seed, stream=rng.stream, layer_offsets=offs, layerwise=True)
        assert np.array_equal(host(s.indices), oi), cf
        if kind == "redsync":  # each segment's mean: an fp64 sum in another order
            np.testing.assert_allclose(host(s.vals), ov, rtol=RTOL)
        else:
            assert np.array_equal(bits(host(s.vals)), bits(ov)), cf


@pytest.mark.parametrize("kind", ["topk", "randomk", "redsync", "dgc"])
def test_layerwise_edge_segments(G, kind):
    """Segments of length 1, segments where keep_count keeps everything
    (cf 1), tie-only segments and -0.0, for every compressor."""
    x = _gauss(70_001, 3)
    x[100:400] = 0.5
    x[400:410] = -0.0
    offs = (0, 1, 2, 100, 400, 410, 5000, 5001, 69_000)
    g = G.GradientVector(x, offs)
    rng = G.SeededRng(4).split(2)
    for cf in (1.0, 3.0, 10.0):
        s, _ = G.compress(G.CompressorKind(kind), g, cf, rng, layerwise=True)
        oi, ov, _ = O.compress(kind, x, cf, seed=rng.seed, stream=rng.stream, layer_offsets=offs, layerwise=True)
        assert np.array_equal(host(s.indices), oi), (kind, cf)
        if kind == "redsync":
            np.testing.assert_allclose(host(s.vals), ov, rtol=RTOL)
        else:
            assert np.array_equal(bits(host(s.vals)), bits(ov)), (kind, cf)


@pytest.mark.parametrize("frac", [0.003, 0.01, 0.05, 1.0])
def test_layerwise_dgc_sample_fractions(G, frac):
    """Layerwise DGC (gvc_segmented_dgc_select) at several sample fractions:
    segments sampled at 256 (the floor), at f * len, in full (exact top-k),
    a rank that reaches the whole sample (cf ~ 1: the minimum sampled |v|),
    tie-only and scaled segments -- bit-exact against the oracle's
    per-segment DGC."""
    x = _gauss(400_003, 8)
    x[1000:3000] = 0.25
    x[3000:90_000] *= np.float32(1e-3)
    x[90_000:90_600] = np.round(x[90_000:90_600])
    offs = (0, 1000, 3000, 90_000, 90_600, 91_600, 300_000)
    K = G.CompressorKind("dgc", dgc_sample_fraction=frac)
    rng = G.SeededRng(31).split(3)
    for cf in (1.001, 2.0, 10.0, 300.0):
        g = G.GradientVector(x, offs)
        s, _ = G.compress(K, g, cf, rng, layerwise=True)
        oi, ov, _ = O.compress("dgc", x, cf, seed=rng.seed, stream=rng.stream, layer_offsets=offs, layerwise=True,
                               dgc_sample_fraction=frac)
        assert np.array_equal(host(s.indices), oi), (frac, cf)
        assert np.array_equal(bits(host(s.vals)), bits(ov)), (frac, cf)


def test_layerwise_layout_changes_on_one_workspace(G):
    """The segmented select caches a layout's work tables per workspace: a
    different layout of the same length and segment count, then the first one
    again, then a workspace forgotten (gvc_workspace_forget) -- every call
    bit-exact against the oracle."""
    from paper_2305_12201_b200 import _native as nat
    x = _gauss(300_007, 21)
    layouts = [(0, 1000, 50_000, 200_000), (0, 7, 150_000, 250_000), (0, 1000, 50_000, 200_000)]
    rng = G.SeededRng(2)
    for q, offs in enumerate(layouts + layouts[:1]):
        if q == 3:
            ws = nat.Workspace.get(torch.device("cuda", 0), "segsel", 1)
            nat.check(nat.load().gvc_workspace_forget(nat.ptr(ws)))
        g = G.GradientVector(x, offs)
        for kind in ("topk", "randomk", "dgc"):
            s, _ = G.compress(G.CompressorKind(kind), g, 10.0, rng, layerwise=True)
            oi, ov, _ = O.compress(kind, x, 10.0, seed=rng.seed, stream=rng.stream, layer_offsets=offs,
                                   layerwise=True)
            assert np.array_equal(host(s.indices), oi), (q, kind)
            assert np.array_equal(bits(host(s.vals)), bits(ov)), (q, kind)


def test_select_after_workspace_forget(G):
    """gvc_workspace_forget drops the select graphs and plan of a workspace;
    the next select on it captures afresh and stays exact."""
    from paper_2305_12201_b200 import _native as nat
    from paper_2305_12201_b200.compressors import Selection
    x = _gauss(1_000_003, 5)
    xd = torch.from_numpy(x).cuda()
    K = G.CompressorKind("topk")
    for rep in range(3):
        sel = Selection(K, [100_000, 10_000], values=xd, slot="forget")
        for j, k in enumerate((100_000, 10_000)):
            idx, vals = sel.emit(j)
            oi = O.topk_indices(x, k)
            assert np.array_equal(host(idx), oi), (rep, j)
        nat.check(nat.load().gvc_workspace_forget(nat.ptr(sel.ws)))
