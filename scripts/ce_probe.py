"""Copy-engine peer bandwidth (cudaMemcpyPeerAsync through torch's cross-device copy),
GPU p -> GPU 0, for exchange-sized payloads (development probe)."""
import sys

import torch

W = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for mb in (35.6, 107.0):
    n = int(mb * 1e6 / 4)
    dst = [torch.empty(n, device="cuda:0") for _ in range(1, W)]
    src = [torch.randn(n, device=f"cuda:{p}") for p in range(1, W)]
    streams = [torch.cuda.Stream(device="cuda:0") for _ in range(1, W)]
    for it in range(6):
        torch.cuda.synchronize()
        for d in range(W):
            torch.cuda.synchronize(d)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for q in range(W - 1):
            streams[q].wait_event(a)
            with torch.cuda.stream(streams[q]):
                dst[q].copy_(src[q], non_blocking=True)
        for q in range(W - 1):
            torch.cuda.current_stream().wait_stream(streams[q])
        b.record()
        torch.cuda.synchronize()
        if it >= 2:
            t = a.elapsed_time(b)
            print(f"W={W} {mb} MB from each of {W - 1} peers: {t * 1e3:.1f} us, "
                  f"{(W - 1) * mb * 1e6 / (t * 1e-3) / 1e9:.0f} GB/s into GPU 0", flush=True)
