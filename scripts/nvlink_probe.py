"""The fused exchange + decompress-average kernel pulling a peer GPU's payload
over NVLink, in ONE process (so ncu can replay it; a multi-rank job cannot be
profiled).  GPU 0 merges its own part with the parts of GPUs 1..W-1, read
through peer mappings; the peers' flags are pre-posted, so no kernel waits.

    python scripts/nvlink_probe.py [W] [n] [cf] [G]   (W parts on G GPUs, default G = W;
                                                       parts 1.. round-robin over GPUs 1..G-1)

Prints CUDA-event times of the direct pull and the staged pull (copier CTAs
+ trailing merge) and checks both against the C oracle's aggregate().
"""
import ctypes
import os
import sys

import numpy as np
import torch
from cuda import cudart

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2305_12201_b200 import _native as nat  # noqa: E402
from paper_2305_12201_b200.exchange import Payload  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 44_500_000
cf = float(sys.argv[3]) if len(sys.argv) > 3 else 10.0
NG = int(sys.argv[4]) if len(sys.argv) > 4 else W
k = int(n // cf)
lib = nat.load()


def gpu_of(r):
    return 0 if r == 0 else 1 + (r - 1) % (NG - 1)


for d in range(1, NG):
    cudart.cudaSetDevice(0)
    cudart.cudaDeviceEnablePeerAccess(d, 0)
torch.cuda.set_device(0)
parts, pls = [], []
for r in range(W):
    rs = np.random.default_rng(r)
    idx = np.sort(rs.choice(n, k, replace=False)).astype(np.uint32)
    vals = rs.standard_normal(k).astype(np.float32)
    parts.append((idx, vals))
    dev = torch.device("cuda", gpu_of(r))
    pl = Payload(k, n, dev, with_bounds=True, off16=True)
    pl.idx[:k].copy_(torch.from_numpy(idx.view(np.int32)).to(dev).view(torch.uint32))
    # the 16-bit wire indices an emit writes beside idx (idx mod GVC_AGG_TILE)
    pl.buf[pl.off_word:pl.off_word + pl.opad].view(torch.int16)[:k].copy_(
        torch.from_numpy((idx % 4096).astype(np.int16)).to(dev))
    pl.vals[:k].copy_(torch.from_numpy(vals).to(dev))
    with torch.cuda.device(dev):
        nat.check(lib.gvc_tile_bounds(nat.ptr(pl.idx), k, n, nat.ptr(pl.bounds_area), nat.stream_ptr(dev)))
        torch.cuda.synchronize(dev)
    pls.append(pl)
dev0 = torch.device("cuda", 0)
flags = torch.zeros(64, dtype=torch.int32, device=dev0)
flags[:W] = 1  # every part posted epoch 1
out = torch.empty(n, dtype=torch.float32, device=dev0)
counts = (ctypes.c_uint64 * W)(*([k] * W))
ref = O.aggregate(parts, n)


def ptrs(attr):
    return (ctypes.c_void_p * W)(*[getattr(p, attr).data_ptr() for p in pls])


def direct():
    nat.check(lib.gvc_aggregate_peers(ptrs("idx"), ptrs("vals"), ptrs("bounds_area"), counts, W, n,
                                      nat.ptr(flags), 1, nat.ptr(out), nat.stream_ptr(dev0)), "aggregate_peers")


# staged: local copies of the remote parts on GPU 0 are the merge's inputs; the copiers fill them
local = [pls[0]] + [Payload(k, n, dev0, with_bounds=True, off16=True) for _ in range(1, W)]
ready = torch.zeros(74 + (k + 4095) // 4096 + 2, dtype=torch.int32, device=dev0)
epoch = [1]


def staged(wire16=False):
    sg = nat.PeerStaging()
    sg.self_rank = 0
    sg.copy_blocks = 74
    sg.chunk_entries = 4096
    sg.ready_dev = ready.data_ptr()
    for p in range(W):
        sg.src_idx_dev[p] = pls[p].idx.data_ptr()
        sg.src_vals_dev[p] = pls[p].vals.data_ptr()
        sg.src_bounds_dev[p] = pls[p].bounds_area.data_ptr()
        if wire16:
            sg.src_off16_dev[p] = pls[p].off16_ptr
            sg.off16_dev[p] = local[p].off16_ptr
    li = (ctypes.c_void_p * W)(*[p.idx.data_ptr() for p in local])
    lv = (ctypes.c_void_p * W)(*[p.vals.data_ptr() for p in local])
    lb = (ctypes.c_void_p * W)(*[p.bounds_area.data_ptr() for p in local])
    nat.check(lib.gvc_aggregate_peers_staged(li, lv, lb, counts, W, n, nat.ptr(flags), epoch[0], ctypes.byref(sg),
                                             nat.ptr(out), nat.stream_ptr(dev0)), "aggregate_peers_staged")


for name, fn in (("direct pull", direct), ("staged pull", staged), ("staged pull 16-bit wire", lambda: staged(True))):
    ms = []
    for it in range(8):
        if name.startswith("staged pull"):  # every run is a new exchange for the readiness epochs
            epoch[0] = it + 1
            flags[:W] = epoch[0]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    ok = np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    recv = (W - 1) * (6 if "16-bit" in name else 8) * k
    t = float(np.median(ms[2:]))
    print(f"{name}: W={W} n={n} k={k} {t * 1e3:.1f} us, {recv / (t * 1e-3) / 1e9:.0f} GB/s received "
          f"({recv / 1e6:.1f} MB over NVLink), oracle {'ok' if ok else 'MISMATCH'}", flush=True)
