"""CPU tests of the drop-in's host-side logic (no GPU): the controller state
machine, trackers, cost model and RNG streams replay the reference's own
test expectations (test_controller.py, test_metrics.py, test_gradcore.py,
test_costmodel.py); the exchange's gain all-gather runs on gloo, world 2."""
import math
import os

import numpy as np
import pytest
import torch

import paper_2305_12201_b200 as G
from paper_2305_12201_b200 import controller as C
from oracle import oracle as O


def make_state(theta_min=10.0, theta_max=1000.0, epsilon=0.7, omega=0.01, window=500,
               policy="exponential", workers=4):
    cfg = G.ControllerConfig(theta_min=theta_min, theta_max=theta_max, epsilon=epsilon, omega=omega,
                             window=window, policy=policy)
    return G.ControllerState.fresh(cfg, workers)


def test_keep_count():
    assert G.keep_count(100, 10) == 10 and G.keep_count(101, 10) == 10 and G.keep_count(10, 3) == 3
    assert G.keep_count(5, 100) == 1
    with pytest.raises(ValueError):
        G.keep_count(10, 0.5)
    rng = np.random.default_rng(0)
    for _ in range(1000):
        n = int(rng.integers(1, 10**9))
        cf = float(rng.uniform(1, 5000))
        assert G.keep_count(n, cf) == O.keep_count(n, cf)


def test_select_cf():
    d = G.select_cf(0.95, 0.99, 0.9, candidate_cf=20.0, minimum_cf=10.0)
    assert (d.choice, d.cf, d.gain) == ("candidate", 20.0, 0.95)
    d = G.select_cf(0.6, 0.8, 0.7, candidate_cf=20.0, minimum_cf=10.0)
    assert (d.choice, d.cf, d.gain) == ("minimum", 10.0, 0.8)
    d = G.select_cf(0.5, 0.6, 0.7, candidate_cf=20.0, minimum_cf=10.0)
    assert (d.choice, d.cf, d.gain) == ("dense", 1.0, 1.0)


def test_scaling_policy_ladders():
    assert [10.0 * G.scaling_policy("exponential", k, 10.0, 1000.0) for k in range(5)] == \
        [10.0, 20.0, 40.0, 160.0, 1000.0]
    assert [10.0 * G.scaling_policy("geometric", k, 10.0, 2000.0) for k in range(9)] == \
        [10.0, 20.0, 40.0, 80.0, 160.0, 320.0, 640.0, 1280.0, 2000.0]
    for k in (5, 20, 200):
        assert G.scaling_policy("exponential", k, 10.0, 1000.0) == 100.0
        assert G.scaling_policy("geometric", k + 8, 10.0, 2000.0) == 200.0
    assert G.scaling_policy("geometric", 3, 10.0, 1000.0, theta_min_current=500.0) == 2.0
    with pytest.raises(ValueError):
        G.scaling_policy("exponential", -1, 10.0, 1000.0)


def test_check_gravac_schedule():
    state = make_state(window=500)
    G.check_gravac(state, 499, 0.9, 0.5)
    assert state.step == 0 and state.theta_s == 1.0
    G.check_gravac(state, 500, 0.9, 0.5)
    assert state.step == 1 and state.theta_s == 2.0
    state = make_state(window=10)
    G.check_gravac(state, 10, 0.90, 0.895)
    assert state.theta_min == 10.0
    G.check_gravac(state, 20, 0.90, 0.895)
    assert state.theta_min == 20.0
    state = make_state(window=10, theta_min=10.0, theta_max=1000.0)
    for boundary, want in enumerate([(10.0, 2.0), (20.0, 4.0), (80.0, 12.5), (1000.0, 1.0), (1000.0, 1.0)], 1):
        G.check_gravac(state, boundary * 10, 1.0, 1.0)
        assert (state.theta_min, state.theta_s) == want


def test_saturation_freeze_published_numbers():
    # T_compress 1029.9 (1280x) vs 1035.4 (2000x) -> freeze 1280x
    state = make_state(window=10, theta_min=10.0, theta_max=2000.0, policy="geometric")
    state.table.t_compress = {1280.0: 1029.9, 2000.0: 1035.4}
    G.check_gravac(state, 10, 0.9, 0.5)
    assert state.frozen and state.theta_ideal == 1280.0 and state.theta_s == 128.0
    assert state.candidate_cf == 1280.0 and not state.saturation_picked_higher_cf
    state = make_state(window=10)
    state.table.t_compress = {40.0: 100.0, 10.0: 100.5}
    G.check_gravac(state, 10, 0.9, 0.5)
    assert state.frozen and state.theta_ideal == 40.0 and state.saturation_picked_higher_cf


def test_trackers_and_tables():
    t = G.GainTracker(0.5)
    assert t.observe(1.0, 0.3) == 1.0 and t.value(1.0) == 1.0
    t.observe(10.0, 0.8)
    t.observe(20.0, 0.4)
    t.observe(10.0, 0.6)
    assert t.value(10.0) == pytest.approx(0.7) and t.value(20.0) == pytest.approx(0.4)
    table = G.update_step(G.ThroughputTable(), 10.0, 1.0, 1.0, 32, 32)
    assert table.t_sys[10.0] == 1024.0 and table.t_compress[10.0] == 1024.0
    table = G.ThroughputTable()
    table.t_compress = {10.0: 100.0, 40.0: 300.0, 160.0: 250.0}
    assert table.top_two() == ((40.0, 300.0), (160.0, 250.0))
    table.t_compress = {10.0: 5.0, 40.0: 5.0, 7.0: 1.0}
    assert table.top_two() == ((40.0, 5.0), (10.0, 5.0))
    for bad in ((10.0, 1.0, 0.0), (10.0, 1.5, 1.0), (0.5, 1.0, 1.0)):
        with pytest.raises(ValueError):
            G.update_step(G.ThroughputTable(), bad[0], bad[1], bad[2], 4, 32)
    assert G.scaling_efficiency(300.0, 100.0, 4) == 0.75


def test_ewma_and_lambda():
    e = G.EwmaTracker(0.5)
    assert e.update(1.0) == 1.0 and e.update(0.0) == 0.5
    lam, xs = 0.32, [0.9, 0.8, 0.95]
    s = xs[0]
    for x in xs[1:]:
        s = lam * x + (1 - lam) * s
    e = G.EwmaTracker(lam)
    for x in xs:
        G.ewma_update(e, x)
    assert e.value == s
    with pytest.raises(ValueError):
        e.update(float("nan"))
    with pytest.raises(ValueError):
        _ = G.EwmaTracker(0.5).value
    assert G.ewma_lambda_from_workers(32) == pytest.approx(0.32)
    assert G.ewma_lambda_from_workers(200) == 1.0 and G.ewma_lambda_from_workers(1) == 0.01


def test_seeded_rng_streams_match_reference_rule():
    r = G.SeededRng(99)
    assert r.split(3, 4).stream == O.split_stream(0, 3, 4)
    assert r.split(3, 4).stream != r.split(4, 3).stream
    a = G.SeededRng(1234).generator.random(1000)
    b = np.random.Generator(np.random.Philox(key=[1234, 0])).random(1000)
    assert np.array_equal(a, b)


def test_costmodel():
    p = G.CostModelParams(workers=4, alpha=1e-5, beta=1e-9)
    assert G.allreduce_time(1000, p) == pytest.approx(2 * 3 * 1e-5 + 2 * 1000 * 1e-9 * 3 / 4)
    q = G.CostModelParams(workers=8, alpha=1e-5, beta=1e-9, topology="tree")
    assert G.allreduce_time(10, q) == pytest.approx(2 * 1e-5 * 3 + 2 * 10 * 3 * 1e-9)
    assert G.allreduce_time(5, G.CostModelParams(workers=1)) == 0.0
    assert G.iteration_time("dense", 1.0, 2.0, 3.0) == 4.0
    assert G.iteration_time("minimum", 1.0, 2.0, 3.0) == 6.0
    c = G.LatencyCoeffs(5e-6, 2e-9, 2e-9)
    assert c.seconds(100, 10) == 5e-6 + 2e-9 * 100 + 2e-9 * 10 * math.log2(10)


def test_config_validation():
    with pytest.raises(ValueError, match=r"epsilon out of \(0,1\)"):
        G.ControllerConfig(epsilon=1.5)
    with pytest.raises(ValueError):
        G.ControllerConfig(theta_min=100.0, theta_max=10.0)
    with pytest.raises(ValueError):
        G.ControllerConfig(policy="linear")
    with pytest.raises(ValueError):
        G.CompressorKind("qsgd")


def test_gradient_vector_validation_cpu():
    g = G.GradientVector([1.0, 2.0, 3.0], layer_offsets=(0, 2), device="cpu")
    assert g.length == 3 and g.layer_slices() == [slice(0, 2), slice(2, 3)]
    for offs in ((1, 2), (0, 2, 2), (0, 5)):
        with pytest.raises(ValueError):
            G.GradientVector([1, 2, 3], layer_offsets=offs, device="cpu")
    with pytest.raises(ValueError):
        G.GradientVector([], device="cpu")


def test_compute_refuses_cpu_tensors():
    g = G.GradientVector([3.0, 1.0], device="cpu")
    with pytest.raises((ValueError, ImportError, RuntimeError)):
        G.compress(G.CompressorKind("topk"), g, 2)


def test_mean_raw_gain_worker_order():
    assert C._mean_raw_gain([1.0, 3.0, 0.5], [2.0, 0.0, 1.0]) == (0.5 + 0.5) / 2
    assert C._mean_raw_gain([4.0], [1.0]) == 1.0


def test_product_never_imports_oracle():
    pkg = os.path.dirname(G.__file__)
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(root, f)).read()
                assert "oracle" not in src.replace("oracle/", ""), f


def _gain_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2305_12201_b200.exchange import allgather_stats
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    row = torch.tensor([10.0 + rank, 4.0 + rank, 1.0 + rank, 0.5 * rank], dtype=torch.float64)
    rows = allgather_stats(row.view(torch.uint8), None)
    vals = [np.frombuffer(r.tobytes(), dtype=np.float64).tolist() for r in rows]
    q.put((rank, vals, C._mean_raw_gain([v[1] for v in vals], [v[0] for v in vals])))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gain_exchange_gloo(world):
    """C2 on gloo: every rank gets every rank's row in rank order and forms the
    same worker-ordered mean (controller.py:284-288)."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gain_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(60)
    want_rows = [[10.0 + r, 4.0 + r, 1.0 + r, 0.5 * r] for r in range(world)]
    want_mean = sum(min(1.0, (4.0 + r) / (10.0 + r)) for r in range(world)) / world
    for r in range(world):
        assert out[r][1] == want_rows
        assert out[r][2] == want_mean


def test_wire_payload_layout():
    """exchange.Payload with the 16-bit wire indices (staged exchange): every
    section 16-byte aligned, the offset area holds k entries padded to the
    copier's 8-entry granules, and words_for matches the buffer the slot carves."""
    from paper_2305_12201_b200 import _native as nat
    from paper_2305_12201_b200.exchange import Payload
    for k in (1, 3, 4, 5, 7, 8, 9, 4095, 4096, 4097, 4_450_000):
        for n in (k, 44_500_000):
            pl = Payload(k, n, "cpu", with_bounds=True, off16=True)
            assert pl.buf.numel() == Payload.words_for(k, n, True)
            assert pl.kpad % 4 == 0 and pl.bpad % 4 == 0 and pl.opad % 4 == 0 and pl.off_word % 4 == 0
            assert 2 * pl.opad >= ((k + 7) & ~7)  # u16 entries, padded to int4 granules
            assert pl.off_word == 2 * pl.kpad + pl.bpad
            assert pl.nb == (n + nat.AGG_TILE - 1) // nat.AGG_TILE + 1
            plain = Payload(k, n, "cpu", with_bounds=True)
            assert plain.opad == 0 and plain.buf.numel() == Payload.words_for(k, n)
            assert not pl.wire16  # set only by the emit that writes the offsets
