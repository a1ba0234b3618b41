"""Host-side profile of the bench step (cProfile) -- development aid."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_12201_b200 as G  # noqa: E402
from paper_2305_12201_b200.compressors import aggregate_packed  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 44_500_000
dev = torch.device("cuda", 0)
pool = [torch.randn(M, device=dev) for _ in range(3)]
cfg = G.ControllerConfig(theta_min=10.0, epsilon=0.4, window=1 << 30)
state = G.ControllerState.fresh(cfg, 1)
state.theta_s = 10.0
store = G.ResidualStore(M, device=dev)
cost = G.CostModelParams()
rng = G.SeededRng(7)
avg = torch.empty(M, device=dev)


def step(g):
    res = G.run_iteration(state, G.GradientVector._wrap(g), store, cost, rng, extra_cfs=(1000.0,))
    p = res.sent[0]
    aggregate_packed(p.indices, p.vals, [p.kept], M, out=avg)


for i in range(5):
    step(pool[i % 3])
torch.cuda.synchronize()
import time  # noqa: E402
t0 = time.perf_counter()
for i in range(20):
    step(pool[i % 3])
torch.cuda.synchronize()
print("wall ms/step", (time.perf_counter() - t0) / 20 * 1e3)
pr = cProfile.Profile()
pr.enable()
for i in range(20):
    step(pool[i % 3])
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
