#!/bin/bash
# N-GPU evidence: bench at N (ResNet101 + VGG16), one rank under ncu for the
# exchange kernel's time and NVLink bytes, and the multi-rank parity tests.
N=${N:-2}
mkdir -p gpurun_out
P=$((29500 + RANDOM % 1000))
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P \
    bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/m${N}_bench.log 2>&1; tail -1 gpurun_out/m${N}_bench.log | cut -c1-200
P=$((P + 1))
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P \
    bench.py --gpus $N --steps 20 --warmup 5 --workload vgg16 > gpurun_out/m${N}_vgg.log 2>&1
python scripts/bench_summary.py gpurun_out/m${N}_bench.log gpurun_out/m${N}_vgg.log
# rank N-1 under ncu (single-pass metrics: no kernel replay against live peers), the others plain
P=$((P + 1))
for r in $(seq 0 $((N - 1))); do
  if [ $r -eq $((N - 1)) ]; then
    MASTER_ADDR=127.0.0.1 MASTER_PORT=$P RANK=$r LOCAL_RANK=$r WORLD_SIZE=$N GVC_BENCH_NOPROF=1 GVC_BENCH_NOCLOCKS=1 \
      timeout 600 ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum --clock-control none \
      -k regex:"k_tile|k_emit|k_collect|k_dense" -c 30 --csv --log-file gpurun_out/m${N}_ncu_rank.csv \
      python bench.py --gpus $N --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/m${N}_ncu_rank.log 2>&1 &
  else
    MASTER_ADDR=127.0.0.1 MASTER_PORT=$P RANK=$r LOCAL_RANK=$r WORLD_SIZE=$N GVC_BENCH_NOPROF=1 GVC_BENCH_NOCLOCKS=1 \
      timeout 600 python bench.py --gpus $N --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/m${N}_plain_r$r.log 2>&1 &
  fi
done
wait
echo ncu-done
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -x -k "staged or epochs or dense" > gpurun_out/m${N}_tests.log 2>&1; tail -2 gpurun_out/m${N}_tests.log
