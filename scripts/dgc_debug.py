import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2305_12201_b200 as G
from paper_2305_12201_b200 import dgc as D
K = G.CompressorKind("dgc")
for n in (64, 300, 5000, 30000, 300001):
    for cf in (2.0, 10.0, 100.0):
        x = np.random.default_rng(n).standard_normal(n).astype(np.float32)
        k = G.keep_count(n, cf)
        try:
            s, _ = G.compress(K, G.GradientVector(x), cf, G.SeededRng(3))
            torch.cuda.synchronize()
            print("ok", n, cf, s.kept, flush=True)
        except Exception as e:
            print("FAIL", n, cf, repr(e)[:300], flush=True)
            raise
