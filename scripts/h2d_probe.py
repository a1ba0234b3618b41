"""Host->device bandwidth probe for the e2e leg (development aid)."""
import torch
M = 44_500_000
h = torch.randn(M).pin_memory()
d = torch.empty(M, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]


def run(nchunks, nstreams):
    ts = []
    for _ in range(8):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        cur = torch.cuda.current_stream()
        step = (M + nchunks - 1) // nchunks
        for c in range(nchunks):
            s = streams[c % nstreams]
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                d[c * step:(c + 1) * step].copy_(h[c * step:(c + 1) * step], non_blocking=True)
        for s in streams[:nstreams]:
            cur.wait_stream(s)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts[2:])[len(ts[2:]) // 2]
    return f"{ms:.3f} ms {4 * M / ms / 1e6:.1f} GB/s"


for nc, ns in [(1, 1), (2, 2), (4, 2), (4, 4), (8, 2), (16, 4)]:
    print(f"chunks={nc} streams={ns}: {run(nc, ns)}", flush=True)
