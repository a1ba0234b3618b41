"""The oracle's multi-threaded O(n) passes (bench.py's CPU legs) against its
single-threaded checker path: identical selections, residuals and aggregates,
the fp64 norm within summation-order rounding."""
import numpy as np
import pytest

from oracle import oracle as O


@pytest.fixture
def threads():
    prev = O.set_threads(1)
    yield
    O.set_threads(prev)


@pytest.mark.parametrize("n", [1_048_577, 3_000_001])
def test_threaded_passes_match_checker(threads, n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n).astype(np.float32)
    x[::7] = x[::7].round(1)  # heavy ties at the threshold
    r = rng.standard_normal(n).astype(np.float32)
    k = n // 10
    want = {}
    for t in (1, 4):
        O.set_threads(t)
        ef = O.ef_add(x, r)
        idx = O.topk_indices(ef, k)
        i2, v2, _ = O.compress_further("topk", idx, ef[idx.astype(np.int64)], n, 10.0)
        res = O.update_residual(ef, idx, ef[idx.astype(np.int64)])
        agg = O.aggregate([(idx, ef[idx.astype(np.int64)]), (i2, v2)], n)
        got = (ef.view(np.uint32), idx, i2, res.view(np.uint32), agg.view(np.uint32))
        if t == 1:
            want = got
            norm1 = O.sq_norm(ef)
        else:
            for a, b in zip(want, got):
                assert np.array_equal(a, b)
            assert O.sq_norm(ef) == pytest.approx(norm1, rel=1e-12)
