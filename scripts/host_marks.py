"""Host-side phase timing of one fused step (development aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_12201_b200 as G  # noqa: E402
from paper_2305_12201_b200 import compressors as C, controller as CT  # noqa: E402

M = 44_500_000
dev = torch.device("cuda", 0)
g = torch.randn(M, device=dev)
cfg = G.ControllerConfig(theta_min=10.0, epsilon=0.35, window=1 << 30)
state = G.ControllerState.fresh(cfg, 1)
state.theta_s = 10.0
store = G.ResidualStore(M, device=dev)
cost = G.CostModelParams()
rng = G.SeededRng(7)
avg = torch.empty(M, device=dev)
marks = []
orig_init = C.Selection.__init__
orig_read = CT._read_results


def sel_init(self, *a, **k):
    marks.append(("sel_in", time.perf_counter()))
    orig_init(self, *a, **k)
    marks.append(("sel_out", time.perf_counter()))


def read(t):
    marks.append(("read_in", time.perf_counter()))
    r = orig_read(t)
    marks.append(("read_out", time.perf_counter()))
    return r


C.Selection.__init__ = sel_init
CT._read_results = read
for it in range(30):
    g.normal_()
    torch.cuda.synchronize()
    marks.clear()
    t0 = time.perf_counter()
    res = G.run_iteration(state, G.GradientVector._wrap(g), store, cost, rng, extra_cfs=(1000.0,),
                          average=True, average_out=avg)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    if it >= 25:
        print(" ".join(f"{n}={1e6 * (t - t0):.0f}" for n, t in marks), f"ret={1e6 * (t1 - t0):.0f}",
              f"gpu_done={1e6 * (t2 - t0):.0f}")
