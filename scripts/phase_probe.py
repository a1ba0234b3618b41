"""Phase timestamps of the cooperative collect (gvc_select_phase_times) at one size.

    python scripts/phase_probe.py [n]
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_12201_b200 as G  # noqa: E402
from paper_2305_12201_b200 import _native as nat  # noqa: E402
from paper_2305_12201_b200.compressors import Selection  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 44_500_000
g = torch.randn(n, device="cuda")
r = torch.zeros(n, device="cuda")
flush = torch.zeros(64 << 20, device="cuda")
K = G.CompressorKind("topk")
k0 = n // 10
names = ["start", "b1 last arrives", "b1 resolved", "b2 last arrives", "b2 resolved", "b3 last arrives",
         "b3 resolved", "cta0 pass end", "post start", "pass1 done", "thresholds", "members done", "finish", "b1 loads", "b1 prefix", "-", "L1 crossed", "L1 refined", "L2 crossed",
         "L2 refined", "L3 crossed", "L3 refined", "fin loaded", "fin tie cut", "fin phase2", "-", "fin partial", "bar1", "bar2", "bar3"]
for it in range(6):
    flush.sum()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    sel = Selection(K, [k0, k0 // 10, k0 // 100], g=g, resid=r, slot="probe", persist_res=True)
    b.record()
    torch.cuda.synchronize()
    out = (ctypes.c_ulonglong * 32)()
    nat.check(nat.load().gvc_select_phase_times(nat.ptr(sel.ws), out, 32))
    t = list(out)
    rel = {nm: round((t[i] - t[0]) / 1000, 2) for i, nm in enumerate(names) if t[i]}
    print(f"select {a.elapsed_time(b) * 1000:.1f} us", rel, "fallback", sel.result().fallback_used,
          "cands", sel.result().candidates, flush=True)
