"""Build a libgravac_b200.so variant with extra -D flags into scripts/probes/lib_<name>.so (A/B experiments).

    python scripts/build_variant.py NAME [-DFOO=1 ...]
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_12201_b200 import build_ext as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(B.ROOT, "scripts", "probes", f"lib_{name}.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
objs = []
for src in B.SOURCES:
    obj = f"/tmp/{name}_{src}.o"
    subprocess.run([B.NVCC, *B.FLAGS, *defs, "-c", os.path.join(B.CSRC, src), "-o", obj], check=True)
    objs.append(obj)
subprocess.run([B.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static", *objs, "-o", out],
               check=True)
print(out)
