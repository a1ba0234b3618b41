"""Per-kernel timeline of one select (gvc_select_phase_times) at one size, from a
library built with -DGVC_PHASE_STAMPS=1 (scripts/build_variant.py).

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
names = ["sample", "collect", "resolve0", "pass1", "resolve1", "members", "finish_j", "s:zero|loads", "s:merge|fin",
         "s:resolve"]
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
    t0 = t[0]
    rel = {nm: (round((t[2 * k] - t0) / 1000, 1), round((t[2 * k + 1] - t0) / 1000, 1)) for k, nm in enumerate(names)}
    try:
        extra = f"fallback {sel.result().fallback_used} cands {sel.result().candidates}"
    except Exception as e:  # ablation variants (scripts/ab_phase.sh) break the downstream kernels
        extra = f"result: {str(e)[:60]}"
    print(f"select {a.elapsed_time(b) * 1000:.1f} us", rel, extra, flush=True)
