"""HBM probe for the collect access pattern (development aid): read g, read r,
write r (12 B/value) with torch's vectorized add, vs a plain copy (8 B/value)."""
import torch
M = 44_500_000
g = torch.randn(M, device="cuda")
r = torch.randn(M, device="cuda")
flush = torch.empty(64 << 20, device="cuda")


def t(fn, nbytes):
    ts = []
    for i in range(20):
        flush.fill_(float(i))
        torch.cuda._sleep(100_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts[3:])[len(ts[3:]) // 2]
    return f"{ms * 1e3:.1f} us, {nbytes / ms / 1e6:.0f} GB/s"


print("add g+r -> r (12 B/value):", t(lambda: torch.add(g, r, out=r), 12 * M))
print("copy g -> r  (8 B/value):", t(lambda: r.copy_(g), 8 * M))
print("fill r       (4 B/value):", t(lambda: r.fill_(1.0), 4 * M))
print("sum g        (4 B/value):", t(lambda: g.sum(), 4 * M))
