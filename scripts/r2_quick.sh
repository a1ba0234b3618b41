#!/bin/bash
# Quick dev loop: parity suite (no multi-rank), default + VGG16 bench summaries, VGG16 launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x ${PYTEST_ARGS} > gpurun_out/q_tests.log 2>&1; tail -3 gpurun_out/q_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/q_bench.log 2>&1
timeout 300 python bench.py --workload vgg16 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/q_vgg.log 2>&1
python scripts/bench_summary.py gpurun_out/q_bench.log gpurun_out/q_vgg.log
GVC_BENCH_NOPROF=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 40 --csv --log-file gpurun_out/q_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
GVC_BENCH_NOPROF=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 40 --csv --log-file gpurun_out/q_vgg_launches.csv python bench.py --workload vgg16 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
