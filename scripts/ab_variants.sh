#!/bin/bash
# A/B of library builds on one box: bench summary per workload per scripts/probes/lib_<v>.so
L=paper_2305_12201_b200/libgravac_b200.so
cp $L /tmp/lib_keep.so
for v in ${VARIANTS}; do
  cp scripts/probes/lib_$v.so $L
  logs=""
  for w in ${WORKLOADS:-resnet101 vgg16}; do
    timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-north-star > gpurun_out/ab_${w}_$v.log 2>&1
    logs="$logs gpurun_out/ab_${w}_$v.log"
  done
  echo "== $v"; python scripts/bench_summary.py $logs
done
cp /tmp/lib_keep.so $L
