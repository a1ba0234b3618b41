"""Per-phase timeline of the bench step (development aid, not a bench number).

    python scripts/timeline.py                       # N=1
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/timeline.py

For every mark run_iteration records (controller._mark) it prints the median
GPU time since the step's "start" event and the median host time since the
step began, per rank.
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2305_12201_b200 as G  # noqa: E402
from paper_2305_12201_b200 import controller as CT  # noqa: E402

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
pg = None
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
    pg = dist.group.WORLD
M = int(os.environ.get("GVC_M", "44500000"))
gen = torch.Generator(device=dev)
gen.manual_seed(1000 * rank + 1)
g = torch.empty(M, device=dev)
KIND = os.environ.get("GVC_KIND", "topk")
cfg = G.ControllerConfig(theta_min=10.0, theta_max=1000.0, epsilon=0.35, window=1 << 30,
                         compressor=G.CompressorKind(KIND))
state = G.ControllerState.fresh(cfg, world)
state.theta_s = 10.0
store = G.ResidualStore(M, device=dev)
cost = G.CostModelParams(workers=world)
rng = G.SeededRng(7)
avg = torch.empty(M, device=dev)
flush = torch.empty(64 << 20, device=dev)
rows = {}
for it in range(60):
    g.normal_(generator=gen)
    flush.fill_(float(it))
    torch.cuda.synchronize()
    if pg is not None:
        dist.barrier()
    CT.TIMELINE = [] if it >= 10 else None
    h0 = time.perf_counter()
    if CT.TIMELINE is not None:
        CT._mark("step")
    G.run_iteration(state, G.GradientVector._wrap(g), store, cost, rng, extra_cfs=(1000.0,) if KIND == "topk" else (),
                    group=pg, average=True, average_out=avg)
    torch.cuda.synchronize()
    if CT.TIMELINE:
        t0 = CT.TIMELINE[0][1]
        for name, ev, ht in CT.TIMELINE:
            rows.setdefault(name, []).append((t0.elapsed_time(ev), (ht - h0) * 1e3))
CT.TIMELINE = None
lines = [f"rank {rank}: mark            gpu_ms   host_ms"]
for name, v in rows.items():
    lines.append(f"rank {rank}: {name:15s} {statistics.median(x[0] for x in v):7.4f}  "
                 f"{statistics.median(x[1] for x in v):7.4f}")
print("\n".join(lines), flush=True)
if pg is not None:
    dist.destroy_process_group()
