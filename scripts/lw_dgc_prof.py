import cProfile, pstats, sys, time, os
sys.path.insert(0, "/root/repo")
import torch
import bench
import paper_2305_12201_b200 as G
offs, M = bench.resnet101_offsets()
x = torch.randn(M, device="cuda")
g = G.GradientVector._wrap(x, offs)
K = G.CompressorKind("dgc")
rng = G.SeededRng(1)
for _ in range(3):
    G.compress(K, g, 10.0, rng, layerwise=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    G.compress(K, g, 10.0, rng, layerwise=True)
torch.cuda.synchronize()
print("wall ms", (time.perf_counter() - t0) / 5 * 1e3)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
pr = cProfile.Profile(); pr.enable()
G.compress(K, g, 10.0, rng, layerwise=True)
pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(15)
