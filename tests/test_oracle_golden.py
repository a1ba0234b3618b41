"""Pin the CPU oracle (oracle/) against the reference's own outputs.

The golden vectors were produced by the unmodified reference
(tests/golden/make_golden.py).  Every family here must match bit-exactly
except fp64 norms/gains (summation order: numpy's BLAS ddot vs the oracle's
sequential sum), which carry an explicit 1e-12 relative tolerance.
"""
import numpy as np
import pytest

from oracle import oracle as O
from tests.conftest import bits


def test_philox_known_answers():
    # Random123 kat_vectors for philox4x32_10
    assert [hex(v) for v in O.philox4x32_10([0, 0, 0, 0], [0, 0])] == \
        ["0x6627e8d5", "0xe169c58d", "0xbc57ac4c", "0x9b00dbd8"]
    assert [hex(v) for v in O.philox4x32_10([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2)] == \
        ["0x408f276d", "0x41c83b0e", "0xa20bc7c6", "0x6d5451fd"]
    assert [hex(v) for v in O.philox4x32_10([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344],
                                            [0xA4093822, 0x299F31D0])] == \
        ["0xd16cfe09", "0x94fdcceb", "0x5001e420", "0x24126ea1"]


def test_pairwise_sum_matches_numpy():
    rng = np.random.default_rng(0)
    for n in list(range(1, 200)) + [1000, 4097, 100_000]:
        a = np.abs(rng.standard_normal(n)).astype(np.float64) * rng.uniform(0.1, 1e3)
        assert np.add.reduce(a) == O.pairwise_sum(a)


def test_split_stream_matches_reference_rule():
    # gradcore.py:151-155 applied by hand for path (1, 2)
    s = O.splitmix64(0 ^ O.splitmix64(1))
    s = O.splitmix64(s ^ O.splitmix64(2))
    assert O.split_stream(0, 1, 2) == s


@pytest.mark.parametrize("family,kind", [("topk", "topk"), ("redsync", "redsync")])
def test_compress_golden(golden, family, kind):
    d = golden(family)
    for i in range(int(d["n_cases"])):
        x = d[f"{i}/x"]
        for j, cf in enumerate(d[f"{i}/cfs"]):
            idx, vals, acf = O.compress(kind, x, float(cf))
            assert np.array_equal(idx, d[f"{i}/{j}/idx"]), (i, j)
            assert np.array_equal(bits(vals), bits(d[f"{i}/{j}/vals"])), (i, j)
            assert acf == x.size / idx.size


def test_compress_further_golden(golden):
    d = golden("further")
    for i in range(int(d["n_cases"])):
        kind = str(d[f"{i}/kind"])
        x = d[f"{i}/x"]
        for j, (cf1, step) in enumerate(d[f"{i}/pairs"]):
            i1, v1, _ = O.compress(kind, x, float(cf1))
            assert np.array_equal(i1, d[f"{i}/{j}/idx1"])
            assert np.array_equal(bits(v1), bits(d[f"{i}/{j}/vals1"]))
            i2, v2, cf2 = O.compress_further(kind, i1, v1, x.size, float(step))
            assert np.array_equal(i2, d[f"{i}/{j}/idx2"]), (i, j)
            assert np.array_equal(bits(v2), bits(d[f"{i}/{j}/vals2"])), (i, j)
            assert cf2 == float(d[f"{i}/{j}/cf2"])


def test_feedback_golden(golden):
    d = golden("feedback")
    r = None
    for i in range(int(d["n_cases"])):
        kind = str(d[f"{i}/kind"])
        g = d[f"{i}/g"]
        if int(d[f"{i}/chain"]) == 0:
            r = np.zeros_like(g)
        ef = O.ef_add(g, r)
        if f"{i}/ef" in d:
            assert np.array_equal(bits(ef), bits(d[f"{i}/ef"]))
        idx, vals, _ = O.compress(kind, ef, 10.0)
        assert np.array_equal(idx, d[f"{i}/idx"])
        assert np.array_equal(bits(vals), bits(d[f"{i}/vals"]))
        r = O.update_residual(ef, idx, vals)
        assert np.array_equal(bits(r), bits(d[f"{i}/r_after"])), i


def test_gain_golden(golden):
    d = golden("gain")
    for i in range(int(d["n_cases"])):
        kind = str(d[f"{i}/kind"])
        x = d[f"{i}/x"]
        norm = O.sq_norm(x)
        assert norm == pytest.approx(float(d[f"{i}/norm"]), rel=1e-12)
        for cf, want in zip(d[f"{i}/cfs"], d[f"{i}/gain_raw"]):
            _, vals, _ = O.compress(kind, x, float(cf))
            assert O.gain_raw(vals, norm) == pytest.approx(float(want), rel=1e-12)


def test_aggregate_golden(golden):
    d = golden("aggregate")
    for i in range(int(d["n_cases"])):
        n = int(d[f"{i}/n"])
        parts = [(d[f"{i}/idx{p}"], d[f"{i}/vals{p}"]) for p in range(int(d[f"{i}/nparts"]))]
        assert np.array_equal(bits(O.aggregate(parts, n)), bits(d[f"{i}/agg"])), i
        assert np.array_equal(bits(O.decompress(*parts[0], n)), bits(d[f"{i}/dec0"]))
        if f"{i}/agg_dense" in d:
            xs = [d[f"{i}/x{p}"] for p in range(len(parts))]
            assert np.array_equal(bits(O.aggregate_dense(xs)), bits(d[f"{i}/agg_dense"]))


def test_dgc_degenerate_golden(golden):
    # n <= 256: the sample is the whole vector, DGC == exact top-k (compressors.py:112-115)
    d = golden("dgc_small")
    for i in range(int(d["n_cases"])):
        idx, vals, _ = O.compress("dgc", d[f"{i}/x"], float(d[f"{i}/cf"]), seed=i)
        assert np.array_equal(idx, d[f"{i}/idx"])
        assert np.array_equal(bits(vals), bits(d[f"{i}/vals"]))


def _exact_topk_support(values, k):
    mag = np.abs(values)
    order = np.lexsort((np.arange(len(values)), -mag))
    return set(order[:k].tolist())


def test_dgc_properties(golden):
    # test_compressors.py:88-96 asserts >= 95% overlap with exact top-k for ONE
    # numpy sample (seed 21).  Positions are parity-unpinned, so compare the
    # overlap DISTRIBUTION over 300 seeds with the reference's own (golden).
    d = golden("dgc_stats")
    x = d["x"]
    top = _exact_topk_support(x, 100)
    ours = []
    for s in range(300):
        idx, vals, _ = O.compress("dgc", x, 100, seed=s)
        assert idx.size == 100
        assert np.all(np.diff(idx.astype(np.int64)) > 0)
        assert np.array_equal(vals, x[idx])
        ours.append(len(set(idx.tolist()) & top) / 100)
    ours, ref = np.array(ours), d["overlaps"]
    assert abs(ours.mean() - ref.mean()) < 0.03
    assert abs((ours >= 0.95).mean() - (ref >= 0.95).mean()) < 0.1


def test_randomk_properties():
    # test_compressors.py:68-85
    x = np.random.default_rng(1).standard_normal(1000).astype(np.float32)
    a, va, _ = O.compress("randomk", x, 10, seed=5)
    b, _, _ = O.compress("randomk", x, 10, seed=5)
    c, _, _ = O.compress("randomk", x, 10, seed=6)
    assert a.size == 100 and np.array_equal(a, b) and not np.array_equal(a, c)
    assert np.array_equal(va, x[a])
    # the sampler is exactly "k smallest position hashes, ties to the lower index"
    h = np.array([O.randomk_hash(5, 0, i) for i in range(1000)], dtype=np.uint64)
    order = np.lexsort((np.arange(1000), h))[:100]
    assert np.array_equal(np.sort(order).astype(np.uint32), a)


def test_randomk_uniformity():
    # every position equally likely: chi-square over 2000 draws of k=50 from n=200
    x = np.ones(200, dtype=np.float32)
    counts = np.zeros(200)
    for s in range(2000):
        idx, _, _ = O.compress("randomk", x, 4, seed=s)
        counts[idx] += 1
    expected = 2000 * 50 / 200
    chi2 = float(((counts - expected) ** 2 / expected).sum())
    assert chi2 < 300  # 199 dof: mean 199, sd ~20


def test_nan_rejected():
    with pytest.raises(ValueError):
        O.compress("topk", np.array([1, np.nan, 3, 2], dtype=np.float32), 2)


def test_support_size_exactness_all_kinds():
    # test_compressors.py:223-232 / acceptance criterion 1
    rng = np.random.default_rng(14)
    for i in range(200):
        kind = ("topk", "dgc", "redsync", "randomk")[i % 4]
        n = int(rng.integers(1, 3000))
        x = rng.standard_normal(n).astype(np.float32)
        cf = float(rng.uniform(1, max(1.0, n)))
        idx, _, _ = O.compress(kind, x, cf, seed=i)
        assert idx.size == O.keep_count(n, cf)
        if kind == "topk":
            assert set(idx.tolist()) == _exact_topk_support(x, idx.size)
