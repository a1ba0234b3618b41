"""Multi-GPU path (one process per GPU, NCCL): the C2 gain exchange gives every
rank the reference's worker-ordered decision, and C1 + K7 -- fused over NVLink
peer memory (GVC_EXCHANGE=staged / pull / push) or all-gather + K7 (nccl) -- equals
aggregate() over the same parts, bit for bit.  Skipped with fewer than 2 GPUs."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _worker(rank, world, port, kind, q, exchange="auto"):
    os.environ["GVC_EXCHANGE"] = exchange
    import torch.distributed as dist
    import paper_2305_12201_b200 as G
    from paper_2305_12201_b200.exchange import allgather_aggregate, allgather_payload
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    n = 200_003
    cfg = G.ControllerConfig(theta_min=10.0, theta_max=1000.0, epsilon=0.3, omega=0.05, window=3,
                             compressor=G.CompressorKind(kind))
    state = G.ControllerState.fresh(cfg, world)
    cost = G.CostModelParams(workers=world)
    store = G.ResidualStore(n)
    rng = G.SeededRng(5)
    out = []
    for it in range(1, 6):
        g = np.random.default_rng(100 * it + rank).standard_normal(n).astype(np.float32) * (1 + rank)
        res = G.run_iteration(state, G.GradientVector(g), store, cost, rng, group=dist.group.WORLD,
                              average=True)
        part = res.sent[0]
        avg = res.averaged
        assert torch.equal(avg.values, allgather_aggregate(part, dist.group.WORLD).values)
        idx, vals = allgather_payload(part, dist.group.WORLD)
        parts = [G.SparseGradient._wrap(idx[r * part.kept:(r + 1) * part.kept],
                                        vals[r * part.kept:(r + 1) * part.kept], n, part.achieved_cf)
                 for r in range(world)]
        ref = G.aggregate(parts)
        wire16 = bool(getattr(getattr(part, "_payload", None), "wire16", False))
        out.append((res.decision.choice, res.decision.cf, res.gain_min_raw, res.gain_c_raw,
                    bool(torch.equal(avg.values.view(torch.int32), ref.values.view(torch.int32))), wire16))
    q.put((rank, out))
    dist.destroy_process_group()


def _spawn(target, world, *args, attempts=3):
    """Run target on `world` ranks; a rendezvous port taken between choosing it
    and binding it (EADDRINUSE) is retried on a fresh port."""
    import queue

    import torch.multiprocessing as mp
    for attempt in range(attempts):
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        procs = [ctx.Process(target=target, args=(r, world, port) + args + (q,)) for r in range(world)]
        for p in procs:
            p.start()
        try:
            res = dict(q.get(timeout=300) for _ in procs)
        except queue.Empty:
            for p in procs:
                p.join(30)
                if p.is_alive():
                    p.kill()
            if attempt + 1 < attempts:
                continue
            raise
        for p in procs:
            p.join(60)
            assert p.exitcode == 0
        return res


def _world():
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs 2 GPUs")
    return min(n, 4)


@pytest.mark.parametrize("exchange", ["staged", "push", "pull", "nccl"])
@pytest.mark.parametrize("kind", ["topk", "dgc", "redsync"])
def test_multi_rank_step(kind, exchange):
    world = _world()
    res = _spawn(_step_worker, world, kind, exchange)
    for r in range(1, world):
        assert res[r] == res[0]  # identical decisions and gains on every rank
    assert all(r[4] for r in res[0])  # exchange == aggregate() bit for bit
    if exchange == "staged" and kind == "topk":
        # the emitted payloads carried the 16-bit wire indices (6 bytes per entry over NVLink)
        assert all(r[5] for r in res[0] if r[0] != "dense")


def _step_worker(rank, world, port, kind, exchange, q):
    _worker(rank, world, port, kind, q, exchange)


def _peer_worker(rank, world, port, q):
    """Many exchanges through the two peer slots (growing k re-allocates the
    symmetric buffer), each against the fp64 rank-ordered oracle mean."""
    import torch.distributed as dist
    from oracle import oracle as O
    import paper_2305_12201_b200 as G
    from paper_2305_12201_b200.exchange import PeerExchange
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            device_id=dev)
    px = PeerExchange.get(dist.group.WORLD, dev)
    ok = []
    n = 300_007
    for e, k in enumerate([1, 5000, 5000, 30_001, 30_001, 30_001, 4096, 120_000, 7]):
        parts = []
        for r in range(world):
            rs = np.random.default_rng(1000 * e + r)
            idx = np.sort(rs.choice(n, k, replace=False)).astype(np.uint32)
            vals = (rs.standard_normal(k) * (1 + r)).astype(np.float32)
            if e == 3:
                vals[::7] = -0.0
            parts.append((idx, vals))
        staged = e % 2 == 0
        pl = px.slot(k, n, push=False, off16=staged)
        pl.idx[:k].copy_(torch.from_numpy(parts[rank][0].view(np.int32)).to(dev).view(torch.uint32))
        if staged:  # the 16-bit wire indices (what an emit writes beside idx): idx mod GVC_AGG_TILE
            wire = (parts[rank][0] % 4096).astype(np.int16)
            pl.buf[pl.off_word:pl.off_word + pl.opad].view(torch.int16)[:k].copy_(torch.from_numpy(wire).to(dev))
            pl.wire16 = True
        pl.vals[:k].copy_(torch.from_numpy(parts[rank][1]).to(dev))
        pl.bounds = None  # not written by an emit: the exchange computes them
        part = G.SparseGradient._wrap(pl.idx[:k], pl.vals[:k], n, n / k)
        part._payload = pl
        out = px.aggregate(part, staged=staged).cpu().numpy()
        ref = O.aggregate(parts, n)
        ok.append(bool(np.array_equal(out.view(np.int32), ref.view(np.int32))))
    q.put((rank, ok))
    dist.destroy_process_group()


def test_peer_exchange_epochs():
    world = _world()
    res = _spawn(_peer_worker, world)
    for r in range(world):
        assert all(res[r]), res[r]


def _dense_worker(rank, world, port, exchange, q):
    """The dense fallback (every decision DENSE at epsilon 0.99) through
    run_iteration: the averaged gradient equals aggregate_dense over every
    rank's g_ef, bit for bit; then DenseExchange alone on odd lengths (float4
    tails, buffer growth, both parities) against the oracle's fp64 mean."""
    os.environ["GVC_EXCHANGE"] = exchange
    import torch.distributed as dist
    from oracle import oracle as O
    import paper_2305_12201_b200 as G
    from paper_2305_12201_b200.exchange import DenseExchange, allgather_dense_mean
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            device_id=dev)
    n = 300_007
    cfg = G.ControllerConfig(theta_min=10.0, theta_max=1000.0, epsilon=0.99, window=1 << 30,
                             compressor=G.CompressorKind("topk"))
    state = G.ControllerState.fresh(cfg, world)
    store = G.ResidualStore(n)
    ok = []
    for it in range(1, 4):
        g = np.random.default_rng(10 * it + rank).standard_normal(n).astype(np.float32) * (1 + rank)
        r_before = store.residual.clone()
        res = G.run_iteration(state, G.GradientVector(g), store, G.CostModelParams(workers=world), G.SeededRng(1),
                              group=dist.group.WORLD, average=True)
        ef = G.apply_feedback(G.GradientVector(g), G.ResidualStore(n)).values + r_before
        ref = allgather_dense_mean(G.GradientVector._wrap(ef), dist.group.WORLD).values
        ok.append(res.decision.choice == "dense" and bool(torch.equal(res.averaged.values.view(torch.int32),
                                                                     ref.view(torch.int32))))
    if exchange != "nccl":
        dx = DenseExchange.get(dist.group.WORLD, dev)
        for e, m in enumerate([1, 5, 4099, 300_007, 1_000_001, 17]):
            xs = [np.random.default_rng(100 * e + r).standard_normal(m).astype(np.float32) * (1 + r)
                  for r in range(world)]
            if e == 2:
                xs[0][::3] = -0.0
            out = dx.mean(G.GradientVector(xs[rank])).cpu().numpy()
            ok.append(bool(np.array_equal(out.view(np.int32), O.aggregate_dense(xs).view(np.int32))))
        ok.append(int(dx.err.item()) == 0)
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["staged", "nccl"])
def test_dense_fallback_multi_rank(exchange):
    world = _world()
    res = _spawn(_dense_worker, world, exchange)
    for r in range(world):
        assert all(res[r]), res[r]
