#!/bin/bash
# Quick dev loop: parity suite (no multi-rank), default + VGG16 bench summaries.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x ${PYTEST_ARGS} > gpurun_out/q_tests.log 2>&1; tail -3 gpurun_out/q_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/q_bench.log 2>&1; tail -3 gpurun_out/q_bench.log | cut -c1-400
timeout 300 python bench.py --workload vgg16 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/q_vgg.log 2>&1
python scripts/bench_summary.py gpurun_out/q_bench.log gpurun_out/q_vgg.log
