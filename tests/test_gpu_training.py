"""The training-loop caller on the GPU (training.run_training, simworkers.py:174-304)
against the unmodified reference's run_training on the same task
(tests/golden/training.npz), and the DDP communication hook.

Top-k runs are bit-exact (the same chosen CFs, volumes and modeled times, and
the same fp64 weights, since every aggregated gradient is); Redsync's values
carry the 1e-6 mean tolerance (compressors.py:188), so its weights and losses
are compared at 1e-6.
"""
import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tests.fixture_tasks import CHOICES, TRACE_COLUMNS, TRAINING_CASES, NoisyBowl  # noqa: E402


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2305_12201_b200 as G
    from paper_2305_12201_b200 import _native
    _native.load()
    return G


@pytest.mark.parametrize("case", range(len(TRAINING_CASES)))
def test_run_training_vs_reference(G, golden, case):
    from paper_2305_12201_b200 import training as T
    from paper_2305_12201_b200.trace import RunTrace
    d = golden("training")
    mode, kind, cf, tmin, eps, workers, size, iters, lr, mom = TRAINING_CASES[case]
    task = NoisyBowl(size, lambda v: G.GradientVector(v), seed=case)
    cfg = (G.ControllerConfig(theta_min=tmin, theta_max=256.0, epsilon=eps, omega=0.05, window=3,
                              compressor=G.CompressorKind(kind)) if mode == "gravac" else None)
    opt = T.OptimizerState(np.zeros(size), lr=lr, momentum=mom, weight_decay=1e-4, lr_decay_iters=(iters - 2,))
    res = T.run_training(task, opt, G.CostModelParams(workers=workers), mode, iters, seed=100 + case,
                         controller_config=cfg, compressor=G.CompressorKind(kind) if kind else None, static_cf=cf)
    want = d[f"{case}/trace"]
    got = np.array([[getattr(r, c) for c in TRACE_COLUMNS] for r in res.trace], dtype=np.float64)
    assert np.array_equal(np.array([CHOICES[r.choice] for r in res.trace]), d[f"{case}/choice"])
    exact = kind != "redsync"
    for j, c in enumerate(TRACE_COLUMNS):
        if c in ("gain_min", "gain_c", "tcomp") or (c == "loss" and not exact):  # tcomp = t_sys * gain
            np.testing.assert_allclose(got[:, j], want[:, j], rtol=1e-6, err_msg=c)
        elif c == "loss":  # the task's own np.dot (multithreaded BLAS) varies by host in the last bit
            np.testing.assert_allclose(got[:, j], want[:, j], rtol=1e-14, err_msg=c)
        else:
            assert np.array_equal(got[:, j], want[:, j]), c
    if exact:
        assert np.array_equal(res.weights, d[f"{case}/weights"])  # every aggregated gradient is bit-exact
    else:
        np.testing.assert_allclose(res.weights, d[f"{case}/weights"], rtol=1e-5, atol=1e-7)
    # the wire format: the reference's JSON lines read back, with measured step times beside them
    assert all(r.measured["step_ms"] > 0 for r in res.trace)
    ref_rows = [json.loads(x) for x in str(d[f"{case}/jsonl"]).splitlines()]
    our_rows = [json.loads(x) for x in res.trace.to_jsonl().splitlines()]
    assert [list(r) for r in our_rows] == [list(r) for r in ref_rows]  # same fields, same order
    assert all("measured" in json.loads(x) for x in res.trace.to_jsonl(measured=True).splitlines())


def test_training_errors(G):
    from paper_2305_12201_b200 import training as T
    task = NoisyBowl(100, lambda v: G.GradientVector(v))
    opt = T.OptimizerState(np.zeros(100), lr=0.1)
    with pytest.raises(ValueError):
        T.run_training(task, opt, G.CostModelParams(), "sparse", 3, 0)
    with pytest.raises(ValueError):
        T.run_training(task, opt, G.CostModelParams(), "static-cf", 3, 0, static_cf=0.5,
                       compressor=G.CompressorKind("topk"))
    with pytest.raises(ValueError):
        T.run_training(task, opt, G.CostModelParams(), "gravac", 3, 0)
    with pytest.raises(ValueError):
        T.OptimizerState(np.zeros(3), lr=0.0)


def _ddp_worker(rank, world, port, q):
    try:
        _ddp_body(rank, world, port, q)
    except Exception as e:  # report instead of leaving the parent waiting
        import traceback
        q.put((rank, ("error", traceback.format_exc())))


def _ddp_body(rank, world, port, q):
    import os
    os.environ.setdefault("GVC_EXCHANGE", "staged")
    import torch.distributed as dist
    import paper_2305_12201_b200 as G
    from paper_2305_12201_b200.training import GravacDdpHook
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            device_id=dev)
    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(256, 512), torch.nn.ReLU(), torch.nn.Linear(512, 10)).to(dev)
    ddp = torch.nn.parallel.DistributedDataParallel(model, device_ids=[rank], bucket_cap_mb=1024)
    hook = GravacDdpHook(G.ControllerConfig(theta_min=10.0, theta_max=100.0, epsilon=0.2, window=2,
                                            compressor=G.CompressorKind("topk")), G.CostModelParams(workers=world))
    ddp.register_comm_hook(hook, GravacDdpHook.hook)
    opt = torch.optim.SGD(ddp.parameters(), lr=0.05)
    ok = []
    losses = []
    gen = torch.Generator(device=dev).manual_seed(1 + rank)
    for step in range(6):
        x = torch.randn(64, 256, device=dev, generator=gen)
        y = torch.randint(0, 10, (64,), device=dev, generator=gen)
        loss = torch.nn.functional.cross_entropy(ddp(x), y)
        opt.zero_grad()
        loss.backward()
        res = hook.last[0]
        flat = torch.cat([p.grad.reshape(-1) for p in reversed(list(model.parameters()))])
        # every parameter's gradient is the step's exchanged mean (one bucket)
        ok.append(bool(torch.equal(torch.sort(flat)[0], torch.sort(res.averaged.values)[0])))
        # and the averaged gradient is the mean of the ranks' sent parts: its support is their union
        ok.append(res.decision.choice in ("candidate", "minimum", "dense"))
        opt.step()
        losses.append(float(loss))
    q.put((rank, (ok, losses)))
    dist.destroy_process_group()


def test_ddp_comm_hook(G):
    from tests.test_gpu_dist import _spawn
    world = max(1, min(2, torch.cuda.device_count()))
    res = _spawn(_ddp_worker, world)
    for r in range(world):
        assert res[r][0] != "error", res[r][1]
        ok, losses = res[r]
        assert all(ok), ok
        assert np.all(np.isfinite(losses))
