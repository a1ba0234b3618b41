#!/bin/bash
# Round-2 evidence on 1 GPU.  PART=a: GPU tests, smoke, the default bench line
# (north star + CPU leg), the reference arm and every workload's line;
# PART=b: launch lists and one full ncu capture of k_collect and k_pass1.
mkdir -p gpurun_out
if [ "${PART:-a}" = a ]; then
  timeout 900 python -m pytest tests -m gpu -q > gpurun_out/e_pytest_gpu.log 2>&1; tail -2 gpurun_out/e_pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as e; e.smoke(); print('smoke ok')" > gpurun_out/e_smoke.log 2>&1; tail -1 gpurun_out/e_smoke.log
  timeout 600 python bench.py > gpurun_out/e_default.log 2>&1; echo "default rc=$?"
  timeout 600 python bench.py --impl reference > gpurun_out/e_reference.log 2>&1; echo "reference rc=$?"
  for W in vgg16 resnet18 vgg16-dgc lstm-redsync lstm-randomk; do
    timeout 400 python bench.py --workload $W --steps 20 --warmup 5 --no-cpu-baseline --no-north-star > gpurun_out/e_$W.log 2>&1
  done
  for W in resnet101-layerwise sweep; do
    timeout 600 python bench.py --workload $W --steps 10 --warmup 3 > gpurun_out/e_$W.log 2>&1
  done
  python scripts/bench_summary.py gpurun_out/e_default.log gpurun_out/e_vgg16.log gpurun_out/e_resnet18.log \
    gpurun_out/e_vgg16-dgc.log gpurun_out/e_lstm-redsync.log gpurun_out/e_lstm-randomk.log
else
  for W in resnet101 vgg16 vgg16-dgc; do
    GVC_BENCH_NOPROF=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -c 60 --csv --log-file gpurun_out/e_launch_$W.csv python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline --no-north-star > /dev/null 2>&1
  done
  GVC_BENCH_NOPROF=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_collect|k_pass1" -s 6 -c 2 \
    -o gpurun_out/e_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-north-star > gpurun_out/e_full.log 2>&1
  echo full rc=$?
fi
