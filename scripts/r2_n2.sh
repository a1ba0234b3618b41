#!/bin/bash
# 2-GPU check: every multi-rank test, then the N = 2 bench lines (ResNet101, VGG16).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/n2_tests.log 2>&1; tail -2 gpurun_out/n2_tests.log
for W in ${WORKLOADS:-resnet101 vgg16}; do
  P=$((29500 + RANDOM % 1000))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P \
    bench.py --gpus 2 --steps 20 --warmup 5 --workload $W --no-north-star > gpurun_out/n2_$W.log 2>&1
  echo "$W rc=$?"
done
python scripts/bench_summary.py gpurun_out/n2_resnet101.log gpurun_out/n2_vgg16.log
