#!/bin/bash
timeout 300 python scripts/phase_probe.py 2>&1 | tail -3
timeout 300 python scripts/phase_probe.py 138000000 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x > gpurun_out/q_tests.log 2>&1; tail -3 gpurun_out/q_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/q_bench.log 2>&1; tail -3 gpurun_out/q_bench.log | cut -c1-300
timeout 300 python bench.py --workload vgg16 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/q_vgg.log 2>&1
python scripts/bench_summary.py gpurun_out/q_bench.log gpurun_out/q_vgg.log
