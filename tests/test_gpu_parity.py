"""GPU parity: the sm_100a path against the reference's golden vectors and the
CPU oracle.  Bar (BASELINE.json north_star): indices, chosen CF and residuals
bit-exact; fp64 gains within 1e-6 relative (observed ~1e-15: only the fp64
summation order differs).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from tests.conftest import bits  # noqa: E402

GAIN_RTOL = 1e-6


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


def gv(G, x):
    return G.GradientVector(np.asarray(x, dtype=np.float32))


# ------------------------------------------------------------ golden vectors
@pytest.mark.parametrize("family,kind", [("topk", "topk"), ("redsync", "redsync")])
def test_compress_golden(G, golden, family, kind):
    d = golden(family)
    K = G.CompressorKind(kind)
    for i in range(int(d["n_cases"])):
        x = d[f"{i}/x"]
        g = gv(G, x)
        for j, cf in enumerate(d[f"{i}/cfs"]):
            s, secs = G.compress(K, g, float(cf))
            assert secs == 0.0
            assert np.array_equal(host(s.indices), d[f"{i}/{j}/idx"]), (i, j, x.size, cf)
            assert np.array_equal(bits(host(s.vals)), bits(d[f"{i}/{j}/vals"])), (i, j)
            assert s.achieved_cf == x.size / s.kept


def test_compress_further_golden(G, golden):
    d = golden("further")
    for i in range(int(d["n_cases"])):
        K = G.CompressorKind(str(d[f"{i}/kind"]))
        g = gv(G, d[f"{i}/x"])
        for j, (cf1, step) in enumerate(d[f"{i}/pairs"]):
            s1, _ = G.compress(K, g, float(cf1))
            s2, _ = G.compress_further(K, s1, float(step))
            assert np.array_equal(host(s2.indices), d[f"{i}/{j}/idx2"]), (i, j)
            assert np.array_equal(bits(host(s2.vals)), bits(d[f"{i}/{j}/vals2"])), (i, j)
            assert s2.achieved_cf == float(d[f"{i}/{j}/cf2"])


def test_feedback_golden_api(G, golden):
    """apply_feedback -> compress -> update_residual through the drop-in API."""
    d = golden("feedback")
    store = None
    for i in range(int(d["n_cases"])):
        K = G.CompressorKind(str(d[f"{i}/kind"]))
        g = d[f"{i}/g"]
        if int(d[f"{i}/chain"]) == 0:
            store = G.ResidualStore(g.size)
        ef = G.apply_feedback(gv(G, g), store)
        if f"{i}/ef" in d:
            assert np.array_equal(bits(host(ef.values)), bits(d[f"{i}/ef"]))
        s, _ = G.compress(K, ef, 10.0)
        assert np.array_equal(host(s.indices), d[f"{i}/idx"])
        assert np.array_equal(bits(host(s.vals)), bits(d[f"{i}/vals"]))
        G.update_residual(ef, s, store)
        assert np.array_equal(bits(host(store.residual)), bits(d[f"{i}/r_after"])), i


def test_feedback_golden_fused(G, golden):
    """The fused EF select + emit(resid) must leave the same residual bits."""
    from paper_2305_12201_b200.compressors import Selection
    d = golden("feedback")
    r = None
    for i in range(int(d["n_cases"])):
        K = G.CompressorKind(str(d[f"{i}/kind"]))
        g = torch.from_numpy(d[f"{i}/g"]).cuda()
        if int(d[f"{i}/chain"]) == 0:
            r = torch.zeros_like(g)
        k = G.keep_count(g.numel(), 10.0)
        if k >= g.numel():
            continue
        sel = Selection(K, [k], g=g, resid=r)
        idx, vals = sel.emit(0, resid=r)
        assert np.array_equal(host(idx), d[f"{i}/idx"]), i
        assert np.array_equal(bits(host(vals)), bits(d[f"{i}/vals"])), i
        assert np.array_equal(bits(host(r)), bits(d[f"{i}/r_after"])), i


def test_gain_golden(G, golden):
    d = golden("gain")
    for i in range(int(d["n_cases"])):
        K = G.CompressorKind(str(d[f"{i}/kind"]))
        g = gv(G, d[f"{i}/x"])
        norm = G.squared_l2_norm(g)
        assert norm == pytest.approx(float(d[f"{i}/norm"]), rel=1e-12)
        for cf, want in zip(d[f"{i}/cfs"], d[f"{i}/gain_raw"]):
            s, _ = G.compress(K, g, float(cf))
            assert G.compression_gain_raw(s, g) == pytest.approx(float(want), rel=GAIN_RTOL)


def test_aggregate_golden(G, golden):
    d = golden("aggregate")
    for i in range(int(d["n_cases"])):
        n = int(d[f"{i}/n"])
        parts = [G.SparseGradient(d[f"{i}/idx{p}"], d[f"{i}/vals{p}"], n, 1.0)
                 for p in range(int(d[f"{i}/nparts"]))]
        assert np.array_equal(bits(host(G.aggregate(parts).values)), bits(d[f"{i}/agg"])), i
        assert np.array_equal(bits(host(G.decompress(parts[0]).values)), bits(d[f"{i}/dec0"])), i
        if f"{i}/agg_dense" in d:
            xs = [gv(G, d[f"{i}/x{p}"]) for p in range(len(parts))]
            assert np.array_equal(bits(host(G.aggregate_dense(xs).values)), bits(d[f"{i}/agg_dense"]))


def test_run_iteration_golden(G, golden):
    """Controller traces of the unmodified reference: chosen CF bit-exact."""
    d = golden("run_iteration")
    codes = {"candidate": 0, "minimum": 1, "dense": 2}
    for c in range(int(d["n_cases"])):
        workers, length, tmin, tmax, eps, window, iters = d[f"{c}/cfg"]
        workers, length, window, iters = int(workers), int(length), int(window), int(iters)
        cfg = G.ControllerConfig(theta_min=tmin, theta_max=tmax, epsilon=eps, omega=0.05, window=window,
                                 policy=str(d[f"{c}/policy"]), compressor=G.CompressorKind(str(d[f"{c}/kind"])))
        state = G.ControllerState.fresh(cfg, workers)
        cost = G.CostModelParams(workers=workers)
        rng = G.SeededRng(3)
        stores = [G.ResidualStore(length) for _ in range(workers)]
        grads_all = d[f"{c}/grads"]
        for it in range(iters):
            grads = [gv(G, grads_all[it, w]) for w in range(workers)]
            res = G.run_iteration(state, grads, stores, cost, rng)
            want = d[f"{c}/trace"][it]
            assert codes[res.decision.choice] == int(want[1]), (c, it)
            assert res.decision.cf == want[2], (c, it)
            assert res.gain_min_raw == pytest.approx(want[3], rel=GAIN_RTOL)
            assert res.gain_c_raw == pytest.approx(want[4], rel=GAIN_RTOL)
            assert res.candidate_cf == want[5] and res.theta_min == want[6]
            assert res.floats_sent == int(want[7])
        for w in range(workers):
            assert np.array_equal(bits(host(stores[w].residual)), bits(d[f"{c}/resid_final"][w])), (c, w)


# -------------------------------------------------- oracle at larger sizes
def _vec(kind, n, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n).astype(np.float32)
    if kind == "ties":
        x = (np.round(8 * x) / 8).astype(np.float32)
    elif kind == "zeros":
        x[rng.random(n) < 0.5] = -0.0
    elif kind == "layered":
        for a in range(0, n, max(1, n // 37)):
            x[a:a + n // 37] *= np.float32(10.0 ** rng.uniform(-3, 0))
    return x


@pytest.mark.parametrize("n", [1_000_003, 11_700_000])
@pytest.mark.parametrize("dist", ["gauss", "ties", "layered", "zeros"])
def test_topk_ladder_ef_vs_oracle(G, n, dist):
    """Fused EF + 3-CF ladder over 3 chained iterations vs the oracle (C1/C2 configs)."""
    from paper_2305_12201_b200.compressors import Selection
    if n > 2_000_000 and dist not in ("gauss", "ties"):
        pytest.skip("large size covered by gauss/ties")
    K = G.CompressorKind("topk")
    r_host = np.zeros(n, dtype=np.float32)
    r = torch.zeros(n, dtype=torch.float32, device="cuda")
    for it in range(3):
        g_host = _vec(dist, n, 100 * it + 7)
        g = torch.from_numpy(g_host).cuda()
        k1 = G.keep_count(n, 10.0)
        ks = [k1, G.keep_count(k1, 10.0), G.keep_count(k1, 100.0)]
        sel = Selection(K, ks, g=g, resid=r)
        res = sel.result()
        ef = O.ef_add(g_host, r_host)
        norm = O.sq_norm(ef)
        # oracle sums sequentially (error ~n*eps); the GPU tree is closer to exact
        assert res.ef_norm_sq == pytest.approx(norm, rel=1e-9)
        assert res.fallback_used == 0
        for j, k in enumerate(ks):
            oi = O.topk_indices(ef, k)
            assert res.kept_sq[j] == pytest.approx(O.sq_norm(ef[oi]), rel=1e-9)
        choose = it % 3
        idx, vals = sel.emit(choose, resid=r)
        oi = O.topk_indices(ef, ks[choose])
        assert np.array_equal(host(idx), oi)
        assert np.array_equal(bits(host(vals)), bits(ef[oi]))
        r_host = O.update_residual(ef, oi, ef[oi])
        assert np.array_equal(bits(host(r)), bits(r_host))


@pytest.mark.parametrize("kind", ["topk", "redsync", "randomk"])
def test_exact_and_fallback_paths_equal_estimate_path(G, kind):
    from paper_2305_12201_b200.compressors import Selection
    K = G.CompressorKind(kind)
    x = torch.from_numpy(_vec("ties", 3_000_000, 5)).cuda()
    ks = [300_000, 30_000, 3_000]
    rng = G.SeededRng(4)
    a = Selection(K, ks, values=x, slot="x1", rng=rng)
    b = Selection(K, ks, values=x, slot="x2", rng=rng, force_exact=1)
    c = Selection(K, ks, values=x, slot="x3", rng=rng, force_exact=2)
    ra, rb, rc = a.result(), b.result(), c.result()
    assert rb.candidates == x.numel() and ra.candidates < x.numel() // 5
    assert rc.fallback_used == 1 and rc.candidates == x.numel() and ra.fallback_used == 0
    for j in range(3):
        assert ra.kept_sq[j] == rb.kept_sq[j] == rc.kept_sq[j]
        ia, va = a.emit(j)
        ib, vb = b.emit(j)
        ic, vc = c.emit(j)
        assert torch.equal(ia, ib) and torch.equal(va, vb) and torch.equal(ia, ic) and torch.equal(va, vc)
    oi, ov = O.select(kind, host(x), ks[0], seed=rng.seed, stream=rng.stream)
    ia, va = a.emit(0)
    assert np.array_equal(host(ia), oi)


@pytest.mark.parametrize("n,cf", [(1000, 3.0), (65_536, 10.0), (1_000_000, 10.0), (4_000_037, 100.0)])
def test_randomk_vs_oracle(G, n, cf):
    K = G.CompressorKind("randomk")
    x = _vec("gauss", n, 3)
    rng = G.SeededRng(77).split(1, 2, 3)
    s, _ = G.compress(K, gv(G, x), cf, rng)
    oi, ov = O.select("randomk", x, G.keep_count(n, cf), seed=rng.seed, stream=rng.stream)
    assert np.array_equal(host(s.indices), oi)
    assert np.array_equal(bits(host(s.vals)), bits(ov))


@pytest.mark.parametrize("n,cf", [(4_000_000, 10.0), (2_000_000, 1000.0)])
def test_redsync_vs_oracle_large(G, n, cf):
    K = G.CompressorKind("redsync")
    x = _vec("layered", n, 9)
    s, _ = G.compress(K, gv(G, x), cf)
    oi, ov = O.select("redsync", x, G.keep_count(n, cf))
    assert np.array_equal(host(s.indices), oi)
    np.testing.assert_allclose(host(s.vals), ov, rtol=GAIN_RTOL)


def test_nan_rejected_and_inf_kept(G):
    K = G.CompressorKind("topk")
    with pytest.raises(ValueError):
        G.compress(K, gv(G, [1.0, float("nan"), 3.0, 2.0]), 2)
    s, _ = G.compress(K, gv(G, [1.0, float("-inf"), 3.0, 2.0]), 2)
    assert host(s.indices).tolist() == [1, 2]


def test_reference_known_answers(G):
    """The reference's own hand examples (test_compressors.py, test_feedback.py, test_metrics.py)."""
    T, R = G.CompressorKind("topk"), G.CompressorKind("redsync")
    s, _ = G.compress(T, gv(G, [3, -1, 0.5, 2]), 2)
    assert host(s.indices).tolist() == [0, 3] and host(s.vals).tolist() == [3.0, 2.0] and s.achieved_cf == 2.0
    s, _ = G.compress(T, gv(G, [5.0, -5.0, 5.0, 1.0]), 2)
    assert host(s.indices).tolist() == [0, 1]
    s, _ = G.compress(R, gv(G, [4.0, 4.0, -4.0, 1.0]), 2)
    assert host(s.indices).tolist() == [0, 1] and host(s.vals).tolist() == [4.0, 4.0]
    s, _ = G.compress(R, gv(G, [8.0, -2.0, 0.1, 0.05]), 2)
    assert host(s.indices).tolist() == [0, 1]
    np.testing.assert_allclose(host(s.vals), [5.0, -5.0])
    store = G.ResidualStore(3)
    g = gv(G, [3.0, 2.0, 1.0])
    sent, _ = G.compress(T, g, 3)
    G.update_residual(g, sent, store)
    assert host(store.residual).tolist() == [0.0, 2.0, 1.0]
    s = G.SparseGradient(np.array([1]), np.array([4.0]), 2, 2.0)
    assert G.compression_gain(s, gv(G, [3.0, 4.0])) == pytest.approx(16.0 / 25.0)
    a = G.SparseGradient(np.array([0]), np.array([3.0]), 2, 2.0)
    b = G.SparseGradient(np.array([1]), np.array([5.0]), 2, 2.0)
    assert host(G.aggregate([a, b]).values).tolist() == [1.5, 2.5]
    assert host(G.decompress(G.SparseGradient(np.array([0, 3]), np.array([3.0, 2.0]), 4, 2.0)).values).tolist() \
        == [3.0, 0.0, 0.0, 2.0]


def test_layerwise(G):
    T = G.CompressorKind("topk")
    g = G.GradientVector(np.arange(1, 21, dtype=np.float32), layer_offsets=(0, 8))
    s, _ = G.compress(T, g, 4, layerwise=True)
    assert s.kept == 5
    assert len([i for i in host(s.indices).tolist() if i < 8]) == 2
    x = _vec("gauss", 50_000, 4)
    offs = (0, 1000, 1003, 30_000)
    K = G.CompressorKind("randomk")
    rng = G.SeededRng(5)
    s, _ = G.compress(K, G.GradientVector(x, offs), 10, rng, layerwise=True)
    oi, ov, _ = O.compress("randomk", x, 10, seed=5, stream=rng.stream, layer_offsets=offs, layerwise=True)
    assert np.array_equal(host(s.indices), oi) and np.array_equal(bits(host(s.vals)), bits(ov))


def test_determinism(G):
    from paper_2305_12201_b200.compressors import Selection
    K = G.CompressorKind("topk")
    x = torch.from_numpy(_vec("layered", 2_000_000, 8)).cuda()
    outs = []
    for _ in range(2):
        sel = Selection(K, [200_000, 2_000], values=x)
        r = sel.result()
        outs.append((r.ef_norm_sq, r.kept_sq[0], r.kept_sq[1], host(sel.emit(0)[0]).tobytes()))
    assert outs[0] == outs[1]


@pytest.mark.parametrize("kind", ["topk", "redsync", "randomk", "dgc"])
@pytest.mark.parametrize("workers", [1, 2])
def test_run_iteration_vs_oracle(G, kind, workers):
    """Fused step (deferred residual mask included) vs an oracle replay of
    controller.py:192-281's data plane, every kind, 8 chained iterations."""
    n = 300_007
    cfg = G.ControllerConfig(theta_min=10.0, theta_max=1000.0, epsilon=0.05 if kind == "randomk" else 0.3,
                             omega=0.05, window=3, compressor=G.CompressorKind(kind))
    state = G.ControllerState.fresh(cfg, workers)
    cost = G.CostModelParams(workers=workers)
    rng = G.SeededRng(11)
    stores = [G.ResidualStore(n) for _ in range(workers)]
    r_host = [np.zeros(n, dtype=np.float32) for _ in range(workers)]
    seen = set()
    for it in range(1, 9):
        gs = [_vec("gauss" if w == 0 else "layered", n, 31 * it + w) for w in range(workers)]
        tmin, ts = state.theta_min, state.theta_s
        res = G.run_iteration(state, [gv(G, g) for g in gs], stores, cost, rng, average=True)
        seen.add(res.decision.choice)
        k1 = O.keep_count(n, tmin)
        gmin_raw, gc_raw = [], []
        for w in range(workers):
            ef = O.ef_add(gs[w], r_host[w])
            norm = O.sq_norm(ef)
            s0 = rng.split(it, w, 0)
            s1 = rng.split(it, w, 1)
            i1, v1 = O.select(kind, ef, k1, seed=s0.seed, stream=s0.stream)
            i2, v2, _ = O.compress_further(kind, i1, v1, n, ts, seed=s1.seed, stream=s1.stream)
            gmin_raw.append(min(1.0, O.sq_norm(v1) / norm))
            gc_raw.append(min(1.0, O.sq_norm(v2) / norm))
            if res.decision.choice == "dense":
                r_host[w] = np.zeros(n, dtype=np.float32)
                continue
            ci, cv = (i2, v2) if res.decision.choice == "candidate" else (i1, v1)
            part = res.sent[w]
            assert np.array_equal(host(part.indices), ci), (it, w)
            np.testing.assert_allclose(host(part.vals), cv, rtol=GAIN_RTOL)
            r_host[w] = O.update_residual(ef, ci, cv)
        if res.decision.choice != "dense":  # the step's average (simworkers.py:242-245)
            want = O.aggregate([(host(p.indices), host(p.vals)) for p in res.sent], n)
            assert np.array_equal(bits(host(res.averaged.values)), bits(want)), it
        assert res.gain_min_raw == pytest.approx(sum(gmin_raw) / workers, rel=GAIN_RTOL)
        assert res.gain_c_raw == pytest.approx(sum(gc_raw) / workers, rel=GAIN_RTOL)
        if kind != "redsync":  # Redsync values carry the 1e-6 mean tolerance into r
            for w in range(workers):
                assert np.array_equal(bits(host(stores[w].residual)), bits(r_host[w])), (it, w)
        else:
            for w in range(workers):
                np.testing.assert_allclose(host(stores[w].residual), r_host[w], rtol=1e-5, atol=1e-6)
    assert seen - {"dense"}, seen


# ------------------------------------------------------------------- DGC
def test_dgc_degenerate_golden(G, golden):
    """n <= 256: the sample is the whole vector, DGC == exact top-k (compressors.py:112-115)."""
    d = golden("dgc_small")
    K = G.CompressorKind("dgc")
    for i in range(int(d["n_cases"])):
        s, _ = G.compress(K, gv(G, d[f"{i}/x"]), float(d[f"{i}/cf"]), G.SeededRng(i))
        assert np.array_equal(host(s.indices), d[f"{i}/idx"]), i
        assert np.array_equal(bits(host(s.vals)), bits(d[f"{i}/vals"])), i


@pytest.mark.parametrize("n", [300, 5_000, 20_000, 300_001, 4_000_000])
def test_dgc_vs_oracle(G, n):
    """Both DGC branches (exact top-k of `chosen`, and the overshoot pad/top-up)
    bit-exact against the oracle's restatement over many seeds and CFs."""
    K = G.CompressorKind("dgc")
    for t, dist in enumerate(["gauss", "ties", "layered", "zeros"]):
        x = _vec(dist, n, 70 + t)
        g = gv(G, x)
        for cf in (2.0, 10.0, 100.0, 1000.0):
            if G.keep_count(n, cf) >= n:
                continue
            for seed in range(3 if n > 1_000_000 else 6):
                rng = G.SeededRng(seed).split(t, int(cf))
                s, _ = G.compress(K, g, cf, rng)
                oi, ov = O.select("dgc", x, G.keep_count(n, cf), seed=rng.seed, stream=rng.stream)
                assert np.array_equal(host(s.indices), oi), (dist, cf, seed)
                assert np.array_equal(bits(host(s.vals)), bits(ov)), (dist, cf, seed)


@pytest.mark.parametrize("n,s", [(1000, 256), (300_001, 3_000), (138_000_000, 1_380_000), (4_000_000_000, 5_000)])
def test_dgc_sample_gather_vs_oracle(G, n, s):
    """gvc_dgc_sample_gather: the stratified sample positions (the oracle's
    restatement), the values there (plain and EF with a deferred mask) and the
    position bitmap, bit-exact; the large n exercise the fp64 stratum bounds."""
    from paper_2305_12201_b200 import _native as nat
    lib = nat.load()
    want = O.dgc_sample_positions(n, s, 11, 22, 5).astype(np.int64)
    pos = torch.empty(s, dtype=torch.int32, device="cuda")
    nat.check(lib.gvc_dgc_sample(n, s, 11, 22, 5, nat.ptr(pos), None))
    assert np.array_equal(host(pos).view(np.uint32).astype(np.int64), want)
    if n > 200_000_000:
        return  # positions only: no n-sized buffers
    gen = torch.Generator(device="cuda").manual_seed(n)
    g = torch.randn(n, device="cuda", generator=gen)
    r = torch.randn(n, device="cuda", generator=gen)
    words = (n + 31) // 32
    mask = torch.randint(0, 2**31, (words,), device="cuda", generator=gen, dtype=torch.int64).to(torch.int32)
    out = torch.empty(s, device="cuda")
    bm = torch.full((words,), -1, dtype=torch.int32, device="cuda")
    for mode, args in (("plain", (g, None, None, None, None, 0)), ("ef", (None, g, r, mask, None, 1))):
        v, gg, rr, mk, pm, pmode = args
        nat.check(lib.gvc_dgc_sample_gather(n, s, 11, 22, 5, nat.ptr(v), nat.ptr(gg), nat.ptr(rr), nat.ptr(mk),
                                            nat.ptr(pm), pmode, nat.ptr(out), nat.ptr(bm), None))
        gh = host(g)
        if mode == "plain":
            exp = gh[want]
        else:
            rh = host(r)[want].copy()
            hit = (host(mask).view(np.uint32)[want >> 5] >> (want & 31).astype(np.uint32)) & 1
            rh[hit == 1] = rh[hit == 1] - rh[hit == 1]  # pending mode 1: the sent entry's residual is zero
            exp = (gh[want] + rh).astype(np.float32)
        assert np.array_equal(bits(host(out)), bits(exp)), mode
        b = np.zeros(words, dtype=np.uint32)
        np.bitwise_or.at(b, want >> 5, (np.uint32(1) << (want & 31).astype(np.uint32)))
        assert np.array_equal(host(bm).view(np.uint32), b), mode


def test_dgc_overlap_distribution(G, golden):
    """Reference's test_compressors.py:88-96 as a distribution over 300 seeds."""
    d = golden("dgc_stats")
    x = d["x"]
    top = set(np.lexsort((np.arange(x.size), -np.abs(x)))[:100].tolist())
    g = gv(G, x)
    ours = []
    for s in range(300):
        sp, _ = G.compress(G.CompressorKind("dgc"), g, 100, G.SeededRng(s))
        ours.append(len(set(host(sp.indices).tolist()) & top) / 100)
    ours, ref = np.array(ours), d["overlaps"]
    assert abs(ours.mean() - ref.mean()) < 0.03


def test_dgc_compress_further_vs_oracle(G):
    K = G.CompressorKind("dgc")
    x = _vec("gauss", 200_003, 5)
    for step in (2.0, 10.0, 100.0):
        r1, r2 = G.SeededRng(1), G.SeededRng(2)
        s1, _ = G.compress(K, gv(G, x), 10.0, r1)
        s2, _ = G.compress_further(K, s1, step, r2)
        i1, v1, _ = O.compress("dgc", x, 10.0, seed=1, stream=r1.stream)
        i2, v2, _ = O.compress_further("dgc", i1, v1, x.size, step, seed=2, stream=r2.stream)
        assert np.array_equal(host(s2.indices), i2) and np.array_equal(bits(host(s2.vals)), bits(v2))


def test_graph_and_direct_launch_paths_agree(G):
    """The captured CUDA-graph select and the probed direct-launch select
    (bench.py's measurement pass) must produce identical results."""
    from paper_2305_12201_b200 import _native as nat
    from paper_2305_12201_b200.compressors import Selection
    K = G.CompressorKind("topk")
    x = torch.from_numpy(_vec("layered", 2_000_003, 12)).cuda()
    outs = []
    for probed in (False, True, False):
        nat.prof_enable(probed)
        try:
            sel = Selection(K, [200_000, 20_000, 2_000], values=x, slot="gp")
            r = sel.result()
            i, v = sel.emit(1)
            outs.append((r.ef_norm_sq, tuple(r.kept_sq[:3]), host(i).tobytes(), host(v).tobytes()))
        finally:
            nat.prof_enable(False)
            nat.prof_read()
    assert outs[0] == outs[1] == outs[2]


@pytest.mark.parametrize("n,k", [(10, 3), (4096, 1), (4097, 4096), (100_000, 7), (1_000_003, 100_000),
                                 (3_000_000, 30)])
def test_emit_tile_bounds(G, n, k):
    """gvc_emit's tile bounds == searchsorted of the output indices at every
    4096-boundary, and the K7 average that consumes them is unchanged."""
    from paper_2305_12201_b200 import _native as nat
    from paper_2305_12201_b200.compressors import Selection, aggregate_packed
    x = torch.from_numpy(_vec("layered", n, n % 97)).cuda()
    if k >= n:
        pytest.skip("identity")
    sel = Selection(G.CompressorKind("topk"), [k], values=x, slot="tb")
    ntiles = (n + nat.AGG_TILE - 1) // nat.AGG_TILE
    tb = torch.full((ntiles + 1,), -1, dtype=torch.int32, device="cuda").view(torch.uint32)
    idx, vals = sel.emit(0, tile_bounds=tb)
    hidx = host(idx).astype(np.int64)
    want = np.searchsorted(hidx, np.arange(ntiles + 1, dtype=np.int64) * nat.AGG_TILE, side="left")
    assert np.array_equal(host(tb).astype(np.int64), want)
    a = aggregate_packed(idx, vals, [k], n)
    b = aggregate_packed(idx, vals, [k], n, bounds=tb)
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))


@pytest.mark.parametrize("nparts", [1, 2, 3, 4, 5, 8])
def test_aggregate_adversarial(G, nparts):
    """K7 fast paths vs the fp64 oracle on values built to break them: exact
    cancellation, exponent gaps > 29, sums that overflow fp32 but not fp64,
    subnormal sums, -0.0, +-inf, and 3+ parts at one position."""
    rs = np.random.default_rng(77 + nparts)
    n = 3 * 4096 + 123
    specials = np.array([0.0, -0.0, 3.0e38, -3.0e38, 1e-40, -1e-40, 1.5e-45, 2.0 ** -126, np.inf, -np.inf,
                         1.0, 1.0 + 2.0 ** -23, 2.0 ** -30, -1.0, 6.0e37], dtype=np.float32)
    parts = []
    for p in range(nparts):
        k = int(rs.integers(n // 4, n // 2))
        idx = np.sort(rs.choice(n, k, replace=False)).astype(np.uint32)
        vals = rs.standard_normal(k).astype(np.float32)
        pick = rs.random(k) < 0.5
        vals[pick] = specials[rs.integers(0, len(specials), pick.sum())]
        parts.append((idx, vals))
    # a block of positions every part hits: the same special pattern in every
    # part (3e38 + 3e38 overflows fp32 only, 1 + -1 cancels, ...)
    common = np.arange(100, 100 + len(specials), dtype=np.uint32)
    full = []
    for p, (i, v) in enumerate(parts):
        keep = ~np.isin(i, common)
        i2 = np.concatenate([i[keep], common])
        v2 = np.concatenate([v[keep], np.roll(specials, p % 2)])
        o = np.argsort(i2, kind="stable")
        full.append((i2[o].astype(np.uint32), v2[o].astype(np.float32)))
    parts = full
    ref = O.aggregate(parts, n)
    sg = [G.SparseGradient(i, v, n, 1.0) for i, v in parts]
    out = host(G.aggregate(sg).values)
    fin = np.isfinite(ref) | np.isinf(ref)
    assert np.array_equal(bits(out)[fin], bits(ref)[fin])
    assert np.array_equal(np.isnan(out), np.isnan(ref))


def test_integration_ctypes_stub(G):
    """The reference-side binding of INTEGRATION.md §2 (raw C-ABI through
    ctypes: gvc_select + gvc_emit) equals the oracle's Top-k."""
    import ctypes
    from paper_2305_12201_b200 import _native as nat
    lib = nat.load()
    x_np = np.random.default_rng(5).standard_normal(300_001).astype(np.float32)
    k = 3_000
    x = torch.from_numpy(x_np).cuda()
    n = x.numel()
    ws = torch.empty(lib.gvc_select_workspace_bytes(0, n), dtype=torch.uint8, device="cuda")
    res = torch.empty(nat.RESULT_BYTES, dtype=torch.uint8, device="cuda")
    a = nat.SelectArgs(kind=0, n_ks=1, n=n, values_dev=x.data_ptr())
    a.ks[0] = k
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    nat.check(lib.gvc_select(ctypes.byref(a), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                             ctypes.c_void_p(res.data_ptr()), stream))
    idx = torch.empty(k, dtype=torch.int32, device="cuda").view(torch.uint32)
    val = torch.empty(k, dtype=torch.float32, device="cuda")
    nat.check(lib.gvc_emit(ctypes.c_void_p(ws.data_ptr()), ws.numel(), 0, None,
                           ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(val.data_ptr()),
                           None, None, None, None, None, stream))
    oi = O.topk_indices(x_np, k)
    assert np.array_equal(host(idx).astype(np.int64), np.asarray(oi, dtype=np.int64))
    assert np.array_equal(bits(host(val)), bits(x_np[oi]))


@pytest.mark.parametrize("kind", ["topk", "randomk"])
@pytest.mark.parametrize("dist", ["gauss", "ties", "layered"])
@pytest.mark.parametrize("ladder", [(10.0,), (10.0, 10.0), (10.0, 100.0), (2.0, 2.0, 2.0),
                                    (10.0, 100.0, 1000.0, 1.001), (1.5, 3.0, 10.0, 30.0, 100.0, 300.0),
                                    (10.0, 10.5, 11.0, 12.0, 20.0, 40.0, 80.0, 160.0, 320.0)])
def test_ladder_shapes_vs_oracle(G, kind, dist, ladder):
    """Every entry of ladders of 1-9 CFs (coinciding, adjacent and far-apart
    thresholds: k_pass1's register band windows, its slow queue and the member
    path of every NB instantiation) against the oracle's exact selection."""
    from paper_2305_12201_b200.compressors import Selection
    K = G.CompressorKind(kind)
    n = 1_500_007
    x = _vec(dist, n, 11)
    ks = [G.keep_count(n, ladder[0])]
    for cf in ladder[1:]:
        ks.append(G.keep_count(ks[-1], cf))
    rng = G.SeededRng(5).split(0, 1, 2)
    sel = Selection(K, ks, values=torch.from_numpy(x).cuda(), rng=rng, slot="lad")
    res = sel.result()
    assert res.fallback_used == 0
    for j, k in enumerate(ks):
        oi, ov = O.select(kind, x, k, seed=rng.seed, stream=rng.stream)
        idx, vals = sel.emit(j)
        assert np.array_equal(host(idx), oi), (j, k)
        assert np.array_equal(bits(host(vals)), bits(x[oi]))
        assert res.kept_sq[j] == pytest.approx(O.sq_norm(x[oi]), rel=1e-9)
        assert res.kept_count[j] == k


@pytest.mark.parametrize("dist", ["gauss", "ties"])
@pytest.mark.parametrize("ladder", [(10.0, 10.0), (10.0, 100.0, 1000.0), (1.5, 3.0, 10.0, 30.0, 100.0)])
def test_redsync_ladder_vs_oracle(G, dist, ladder):
    """Redsync over multi-CF ladders: k_pass1's |v| band sums (the mean) for
    every entry -- support bit-exact, substituted values within 1e-6."""
    from paper_2305_12201_b200.compressors import Selection
    K = G.CompressorKind("redsync")
    n = 1_500_007
    x = _vec(dist, n, 13)
    ks = [G.keep_count(n, ladder[0])]
    for cf in ladder[1:]:
        ks.append(G.keep_count(ks[-1], cf))
    sel = Selection(K, ks, values=torch.from_numpy(x).cuda(), slot="lrs")
    assert sel.result().fallback_used == 0
    for j, k in enumerate(ks):
        oi, ov = O.select("redsync", x, k)
        idx, vals = sel.emit(j)
        assert np.array_equal(host(idx), oi), (j, k)
        np.testing.assert_allclose(host(vals), ov, rtol=1e-6, atol=0)


@pytest.mark.parametrize("n", [1000, 300_007, 6_600_000])
def test_equal_magnitudes_select_vs_oracle(G, n):
    """gvc_select_args.equal_magnitudes (the level-2 pick over a Redsync level-1
    output, +-m or 0): the same entries, values and gains as the magnitude
    select, with zeros kept when fewer than k values are nonzero."""
    from paper_2305_12201_b200.compressors import Selection
    rs = np.random.default_rng(n)
    m = np.float32(0.8125)
    for zeros in (0.0, 0.3, 0.95):
        x = np.where(rs.random(n) < 0.5, m, -m).astype(np.float32)
        x[rs.random(n) < zeros] = 0.0
        xd = torch.from_numpy(x).cuda()
        for kind in ("redsync", "topk"):
            for cf in (2.0, 10.0, 100.0):
                k = G.keep_count(n, cf)
                sel = Selection(G.CompressorKind(kind), [k], values=xd, slot="eqm", equal_magnitudes=True)
                res = sel.result()
                idx, vals = sel.emit(0)
                oi, ov = O.select(kind, x, k)
                assert np.array_equal(host(idx), oi), (kind, zeros, cf)
                if kind == "redsync":
                    np.testing.assert_allclose(host(vals), ov, rtol=GAIN_RTOL)
                else:
                    assert np.array_equal(bits(host(vals)), bits(ov)), (zeros, cf)
                want_e = O.sq_norm(ov)
                assert res.kept_sq[0] == pytest.approx(want_e, rel=GAIN_RTOL, abs=1e-30), (kind, zeros, cf)
                assert res.kept_nonzero[0] == int(np.count_nonzero(ov)), (kind, zeros, cf)
