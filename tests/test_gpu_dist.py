"""Multi-GPU path (one process per GPU, NCCL): the C2 gain exchange gives every
rank the reference's worker-ordered decision, and C1 + K7 (all-gather of the
(idx, val) payload + fp64 rank-ordered average) equals aggregate() over the
same parts, bit for bit.  Skipped with fewer than 2 GPUs."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _worker(rank, world, port, kind, q):
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
        out.append((res.decision.choice, res.decision.cf, res.gain_min_raw, res.gain_c_raw,
                    bool(torch.equal(avg.values.view(torch.int32), ref.values.view(torch.int32)))))
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["topk", "dgc"])
def test_two_rank_step(kind):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert res[0] == res[1]  # identical decisions and gains on both ranks
    assert all(r[4] for r in res[0])  # fused exchange == aggregate() bit for bit
