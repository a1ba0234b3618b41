import os, sys, time, statistics
sys.path.insert(0, "/root/repo")
import torch
import paper_2305_12201_b200 as G
from paper_2305_12201_b200 import controller as CT, compressors as C, gradcore as GC
M = 44_500_000
dev = torch.device("cuda", 0)
g = torch.randn(M, device=dev)
cfg = G.ControllerConfig(theta_min=10.0, theta_max=1000.0, epsilon=0.2, window=1 << 30)
state = G.ControllerState.fresh(cfg, 1); state.theta_s = 10.0
store = G.ResidualStore(M, device=dev); cost = G.CostModelParams(); rng = G.SeededRng(7)
avg = torch.empty(M, device=dev)
T = {}
def wrap(obj, name, label):
    f = getattr(obj, name)
    def w(*a, **k):
        t = time.perf_counter(); r = f(*a, **k); T.setdefault(label, []).append(time.perf_counter() - t); return r
    setattr(obj, name, w)
wrap(C.Selection, "__init__", "Selection.__init__")
wrap(CT._WorkerStep, "__init__", "_WorkerStep.__init__")
wrap(GC.SeededRng, "split", "rng.split")
wrap(C.Selection, "emit", "Selection.emit")
wrap(CT, "_average", "_average")
for it in range(60):
    if it == 10: T.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    G.run_iteration(state, G.GradientVector._wrap(g), store, cost, rng, extra_cfs=(1000.0,), average=True, average_out=avg)
    T.setdefault("run_iteration (host, incl. wait)", []).append(time.perf_counter() - t0)
for k, v in T.items():
    print(f"{k:36s} n/step={len(v)/50:.1f}  median {statistics.median(v)*1e6:7.1f} us")
