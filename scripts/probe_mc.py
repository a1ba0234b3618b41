"""Probe: NVSwitch multicast through torch symmetric memory (development aid).

torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/probe_mc.py
Writes an iota through the multicast address on rank 0 (plain stores from
gvc_iota) and checks every rank's local buffer received it; times a 35.6 MB
multicast write against a unicast peer write.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.distributed._symmetric_memory as symm  # noqa: E402

from paper_2305_12201_b200 import _native as nat  # noqa: E402

rank = int(os.environ["RANK"])
world = int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
n = 8_900_000  # 35.6 MB of u32
buf = symm.empty(2 * n, dtype=torch.int32, device=dev)
buf.zero_()
h = symm.rendezvous(buf, dist.group.WORLD)
mc = h.has_multicast_support and h.multicast_ptr
print(f"rank {rank}: multicast_support={h.has_multicast_support} mc_ptr={h.multicast_ptr:#x} "
      f"ptrs={[hex(p) for p in h.buffer_ptrs]}", flush=True)
torch.cuda.synchronize()
dist.barrier()
lib = nat.load()
if mc:
    if rank == 0:
        nat.check(lib.gvc_iota(ctypes.c_void_p(h.multicast_ptr), n, nat.stream_ptr(dev)))
        torch.cuda.synchronize()
    dist.barrier()
    ok = torch.equal(buf[:n].cpu(), torch.arange(n, dtype=torch.int32))
    print(f"rank {rank}: multicast iota received: {ok}", flush=True)
    dist.barrier()

    def t(fn):
        ts = []
        for _ in range(12):
            torch.cuda.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(200_000)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return sorted(ts[2:])[len(ts[2:]) // 2] * 1e3
    peer = h.buffer_ptrs[(rank + 1) % world]
    us_mc = t(lambda: lib.gvc_iota(ctypes.c_void_p(h.multicast_ptr + 4 * n), n, nat.stream_ptr(dev)))
    us_uc = t(lambda: lib.gvc_iota(ctypes.c_void_p(peer + 4 * n), n, nat.stream_ptr(dev)))
    us_lo = t(lambda: lib.gvc_iota(ctypes.c_void_p(h.buffer_ptrs[rank] + 4 * n), n, nat.stream_ptr(dev)))
    print(f"rank {rank}: 35.6MB write: multicast {us_mc:.1f}us, unicast peer {us_uc:.1f}us, local {us_lo:.1f}us",
          flush=True)
    remote = h.get_buffer((rank + 1) % world, (n,), torch.float32, n)
    src = torch.randn(n, device=dev)
    us_ce = t(lambda: remote.copy_(src))
    us_sm = t(lambda: torch.add(src, 0.0, out=remote))
    print(f"rank {rank}: remote tensor device {remote.device}; copy_ {us_ce:.1f}us, add-out (SM v4) {us_sm:.1f}us",
          flush=True)
dist.destroy_process_group()
