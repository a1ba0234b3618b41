#!/bin/bash
# Multi-GPU evidence on a 4-GPU box: bench lines at N = 2 and 4 (ResNet101,
# VGG16), the reference arm under torchrun at N = 4, and every multi-rank test.
mkdir -p gpurun_out
for N in 2 4; do
  for W in resnet101 vgg16; do
    P=$((29500 + RANDOM % 1000))
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P \
      bench.py --gpus $N --steps 20 --warmup 5 --workload $W --no-north-star > gpurun_out/s${N}_$W.log 2>&1
  done
  python scripts/bench_summary.py gpurun_out/s${N}_resnet101.log gpurun_out/s${N}_vgg16.log
done
P=$((29500 + RANDOM % 1000))
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P \
  bench.py --gpus 4 --steps 20 --warmup 5 --impl reference > gpurun_out/s4_reference.log 2>&1; echo "reference rc=$?"
timeout 1500 python -m pytest tests/test_gpu_dist.py -q > gpurun_out/s4_tests.log 2>&1; tail -2 gpurun_out/s4_tests.log
