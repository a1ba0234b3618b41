#!/bin/bash
# staged-exchange copier count / chunk sweep at N GPUs (ResNet101 44.5M and VGG16 138M)
for cfg in "74 4096" "148 4096" "37 4096" "74 8192" "148 8192" "74 2048"; do
  set -- $cfg
  for W in resnet101 vgg16; do
    P=$((29500 + RANDOM % 1000))
    GVC_STAGE_COPIERS=$1 GVC_STAGE_CHUNK=$2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${N:-4} \
      --master-addr 127.0.0.1 --master-port $P bench.py --gpus ${N:-4} --steps 20 --warmup 5 --workload $W --no-north-star > gpurun_out/ss_$W.log 2>&1
    python - <<PY
import json
d=json.loads(open("gpurun_out/ss_$W.log").read().strip().splitlines()[-1])
print("copiers $1 chunk $2 $W", round(d["ms_per_step"],4), "median", round(d["step_ms"]["median"],4), "agg", round(d["breakdown_ms"]["aggregate"],4), "nvl", round(d["nvlink"]["frac"],3))
PY
  done
done
