"""cProfile of the host side of run_iteration (development aid)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_12201_b200 as G  # noqa: E402

M = int(os.environ.get("GVC_M", "44500000"))
dev = torch.device("cuda", 0)
g = torch.randn(M, device=dev)
TMIN = float(os.environ.get("GVC_TMIN", "10"))
TS = float(os.environ.get("GVC_TS", "10"))
EXTRA = tuple(float(x) for x in os.environ.get("GVC_EXTRA", "1000").split(",") if x)
cfg = G.ControllerConfig(theta_min=TMIN, theta_max=1000.0, epsilon=float(os.environ.get("GVC_EPS", "0.2")),
                         window=1 << 30, compressor=G.CompressorKind("topk"))
state = G.ControllerState.fresh(cfg, 1)
state.theta_s = TS
store = G.ResidualStore(M, device=dev)
cost = G.CostModelParams()
rng = G.SeededRng(7)
avg = torch.empty(M, device=dev)


def run(n):
    for _ in range(n):
        G.run_iteration(state, G.GradientVector._wrap(g), store, cost, rng, extra_cfs=EXTRA, average=True,
                        average_out=avg)
    torch.cuda.synchronize()


run(10)
import time  # noqa: E402
t0 = time.perf_counter()
run(100)
print(f"wall per iteration: {(time.perf_counter() - t0) * 10:.3f} ms")
pr = cProfile.Profile()
pr.enable()
run(100)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats(os.environ.get("GVC_SORT", "tottime")).print_stats(int(os.environ.get("GVC_TOP", "25")))
