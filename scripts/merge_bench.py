"""Exchange + decompress-average alone (development aid, not a bench number).

    python scripts/merge_bench.py                                   # local K7, 1/2/4 parts
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/merge_bench.py

Fixed payloads of k = M / CF sorted random positions per rank.  Every timed
iteration starts after a device sync + barrier, so rank skew is excluded;
times are CUDA events on the current stream, median of 30.
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2305_12201_b200 as G  # noqa: E402
from paper_2305_12201_b200 import exchange as X  # noqa: E402
from paper_2305_12201_b200.compressors import aggregate_packed  # noqa: E402

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
M = int(os.environ.get("GVC_M", "44500000"))
CF = float(os.environ.get("GVC_CF", "10"))
k = int(M // CF)
pg = None
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
    pg = dist.group.WORLD


def payload(seed):
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    idx = torch.sort(torch.randperm(M, device=dev, generator=gen)[:k]).values.to(torch.int32).view(torch.uint32)
    vals = torch.randn(k, device=dev, generator=gen)
    return idx, vals


def timeit(fn, reps=30):
    ts = []
    for _ in range(reps + 3):
        torch.cuda.synchronize()
        if pg is not None:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(400_000)  # the GPU stays busy while the host enqueues fn()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts[3:])


out = torch.empty(M, device=dev)
idx, vals = payload(100 + rank)
nb = (M + G._native.AGG_TILE - 1) // G._native.AGG_TILE + 1
res = {}
if pg is None:
    for parts in (1, 2, 4):
        pl = [X.Payload(k, M, dev) for _ in range(parts)]
        for p in pl:
            p.idx[:k].copy_(idx)
            p.vals[:k].copy_(vals)
            G._native.check(G._native.load().gvc_tile_bounds(G._native.ptr(p.idx), k, M, G._native.ptr(p.bounds),
                                                             G._native.stream_ptr(dev)))
        flat = torch.cat([p.buf for p in pl])
        L = pl[0].words
        res[f"k7_local_{parts}parts"] = timeit(lambda: aggregate_packed(
            flat.view(torch.uint32), flat[pl[0].kpad:].view(torch.float32), [k] * parts, M, out=out,
            offs=[r * L for r in range(parts)], bounds=flat[2 * pl[0].kpad:].view(torch.uint32), bounds_stride=L))
else:
    px = X.PeerExchange.get(pg, dev)

    def peer():
        pl = px.slot(k, M, push=False)
        pl.idx[:k].copy_(idx)
        pl.vals[:k].copy_(vals)
        pl.bounds = None
        part = G.SparseGradient._wrap(pl.idx[:k], pl.vals[:k], M, M / k)
        part._payload = pl
        px.aggregate(part, out=out)

    def nccl():
        pl = X.Payload(k, M, dev)
        pl.idx[:k].copy_(idx)
        pl.vals[:k].copy_(vals)
        G._native.check(G._native.load().gvc_tile_bounds(G._native.ptr(pl.idx), k, M, G._native.ptr(pl.bounds),
                                                         G._native.stream_ptr(dev)))
        part = G.SparseGradient._wrap(pl.idx[:k], pl.vals[:k], M, M / k)
        part._payload = pl
        X.allgather_aggregate(part, pg, out=out)

    def copies():
        pl = X.Payload(k, M, dev)
        pl.idx[:k].copy_(idx)
        pl.vals[:k].copy_(vals)
        G._native.check(G._native.load().gvc_tile_bounds(G._native.ptr(pl.idx), k, M, G._native.ptr(pl.bounds),
                                                         G._native.stream_ptr(dev)))

    res["payload_fill_only"] = timeit(copies)
    # raw SM pull over NVLink: an elementwise kernel reading the peer's slot
    px._ensure(X.Payload.words_for(k, M))
    peer_rank = (rank + 1) % world
    remote = px.handle.get_buffer(peer_rank, (2 * k,), torch.float32, px.FLAG_WORDS)
    sink = torch.empty(2 * k, device=dev)
    res["sm_pull_8k_bytes"] = timeit(lambda: torch.add(remote, 0.0, out=sink))
    res["local_copy_4k_bytes"] = timeit(lambda: torch.add(sink[:k], 0.0, out=sink[k:]))
    res["peer_signal_merge"] = timeit(peer)
    res["nccl_allgather_k7"] = timeit(nccl)
print(f"rank {rank} M={M} k={k} world={world}: " + ", ".join(f"{a}={b * 1e3:.1f}us" for a, b in res.items()),
      flush=True)
if pg is not None:
    dist.destroy_process_group()
