#!/bin/bash
# A/B of two builds of the library on one box: ncu launch list of the default bench with each.
L=paper_2305_12201_b200/libgravac_b200.so
for v in r1 new; do
  cp scripts/probes/lib_$v.so $L
  GVC_BENCH_NOPROF=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 40 --csv --log-file gpurun_out/ab_$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
