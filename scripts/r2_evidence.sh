#!/bin/bash
# Round-2 evidence on 1 GPU: bench lines of every workload, launch lists, one full ncu capture
# of k_collect and k_pass1 (default workload).
mkdir -p gpurun_out
for W in resnet101 vgg16 resnet18 vgg16-dgc lstm-redsync lstm-randomk; do
  timeout 400 python bench.py --workload $W --steps 20 --warmup 5 --no-cpu-baseline --no-north-star > gpurun_out/e_$W.log 2>&1
done
python scripts/bench_summary.py gpurun_out/e_*.log
for W in resnet101 vgg16; do
  GVC_BENCH_NOPROF=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 45 --csv --log-file gpurun_out/e_launch_$W.csv python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline --no-north-star > /dev/null 2>&1
done
GVC_BENCH_NOPROF=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_collect|k_pass1" -s 6 -c 2 \
  -o gpurun_out/e_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-north-star > gpurun_out/e_full.log 2>&1
echo full rc=$?
