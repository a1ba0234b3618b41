#!/bin/bash
# N=4 exchange-mode A/B (ResNet101 44.5M): step-time distribution per mode
for X in ${MODES:-staged pull nccl}; do
  P=$((29500 + RANDOM % 1000))
  GVC_EXCHANGE=$X timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${N:-4} --master-addr 127.0.0.1 --master-port $P \
    bench.py --gpus ${N:-4} --steps 20 --warmup 5 --no-north-star > gpurun_out/x4_$X.log 2>&1
  python - <<PY
import json
d=json.loads(open("gpurun_out/x4_$X.log").read().strip().splitlines()[-1])
print("$X", round(d["ms_per_step"],4), {k: round(v,3) if isinstance(v,float) else v for k,v in d["step_ms"].items()}, round(d["breakdown_ms"]["aggregate"],4))
PY
done
