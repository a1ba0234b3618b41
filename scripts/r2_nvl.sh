#!/bin/bash
# NVLink evidence (one process, W GPUs) + the compress-API workloads.
W=${W:-2}
mkdir -p gpurun_out
timeout 300 python scripts/nvlink_probe.py $W > gpurun_out/nvl_probe_$W.log 2>&1; cat gpurun_out/nvl_probe_$W.log | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"k_tile" -c 24 --csv --log-file gpurun_out/nvl_ncu_$W.csv python scripts/nvlink_probe.py $W > gpurun_out/nvl_ncu_$W.log 2>&1
echo ncu rc=$?
if [ "$W" = "2" ]; then
  timeout 300 python bench.py --workload resnet101-layerwise --steps 10 --warmup 3 > gpurun_out/lw.log 2>&1; tail -1 gpurun_out/lw.log | cut -c1-400
  timeout 600 python bench.py --workload sweep --steps 5 --warmup 2 > gpurun_out/sweep.log 2>&1; tail -1 gpurun_out/sweep.log | cut -c1-300
fi
