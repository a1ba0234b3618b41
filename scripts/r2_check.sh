#!/bin/bash
# Round-2 dev loop: GPU suite (incl. the measured-size parity tests), default + VGG16 bench, launch list.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/r2_tests.log 2>&1; tail -3 gpurun_out/r2_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench.log 2>&1; tail -1 gpurun_out/r2_bench.log | cut -c1-300
timeout 300 python bench.py --workload vgg16 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_vgg.log 2>&1
python scripts/bench_summary.py gpurun_out/r2_bench.log gpurun_out/r2_vgg.log
GVC_BENCH_NOPROF=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 40 --csv --log-file gpurun_out/r2_vgg_launches.csv python bench.py --workload vgg16 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
