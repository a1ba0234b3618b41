#!/bin/bash
# 1-GPU check after a select change: the GPU suite, the default line (with the
# north star) and the VGG16 / DGC / Redsync lines.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/c_pytest.log 2>&1; tail -1 gpurun_out/c_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/c_default.log 2>&1; echo "default rc=$?"
for W in ${WORKLOADS:-vgg16 vgg16-dgc lstm-redsync}; do
  timeout 400 python bench.py --workload $W --steps 20 --warmup 5 --no-cpu-baseline --no-north-star > gpurun_out/c_$W.log 2>&1
done
python scripts/bench_summary.py gpurun_out/c_default.log gpurun_out/c_vgg16.log gpurun_out/c_vgg16-dgc.log gpurun_out/c_lstm-redsync.log
