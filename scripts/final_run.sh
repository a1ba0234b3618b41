#!/bin/bash
# Round-end evidence: GPU parity suite, smoke, default bench (+ CPU baseline), VGG16 bench,
# reference arm, and the ncu launch lists of the default and VGG16 benches.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/f_tests.log 2>&1; tail -2 gpurun_out/f_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
python bench.py > gpurun_out/f_bench.log 2>&1; tail -1 gpurun_out/f_bench.log
python bench.py --workload vgg16 --no-cpu-baseline > gpurun_out/f_vgg.log 2>&1
python scripts/bench_summary.py gpurun_out/f_bench.log gpurun_out/f_vgg.log
python bench.py --impl reference > gpurun_out/f_ref.log 2>&1; tail -1 gpurun_out/f_ref.log | cut -c1-200
GVC_BENCH_NOPROF=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 40 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
GVC_BENCH_NOPROF=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 40 --csv --log-file gpurun_out/f_vgg_launches.csv python bench.py --workload vgg16 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
