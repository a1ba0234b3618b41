"""key_est / shift0 / max_key / candidates of the controller's select over a few bench-like steps."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_12201_b200 as G  # noqa: E402
from paper_2305_12201_b200 import _native as nat  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 44_500_000
cfg = G.ControllerConfig(theta_min=10.0, theta_max=1000.0, epsilon=0.35, window=1 << 30)
state = G.ControllerState.fresh(cfg, 1)
state.theta_s = 10.0
store = G.ResidualStore(M)
g = torch.empty(M, device="cuda")
for it in range(5):
    g.normal_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    G.run_iteration(state, G.GradientVector._wrap(g), store, G.CostModelParams(), G.SeededRng(7), extra_cfs=(1000.0,))
    b.record()
    torch.cuda.synchronize()
    ws = nat.Workspace._bufs[(0, "step0a")]
    out = (ctypes.c_ulonglong * 32)()
    nat.check(nat.load().gvc_select_phase_times(nat.ptr(ws), out, 32))
    t = list(out)
    print(f"step {it}: {a.elapsed_time(b) * 1000:.0f} us key_est {t[0]:#x} shift0 {t[1]} max_key {t[2]:#x} cands {t[3]}",
          flush=True)
