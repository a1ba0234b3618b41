# N = 1, 2, 4 bench lines (development aid): bash scripts/scale_run.sh [workload]
W=${1:-resnet101}
python bench.py --workload $W --no-cpu-baseline 2>&1 | grep '^{' > gpurun_out/scale_${W}_1.json
for N in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N --workload $W --no-cpu-baseline 2>&1 | grep '^{' > gpurun_out/scale_${W}_$N.json
done
for N in 1 2 4; do python -c "import json; d=json.load(open('gpurun_out/scale_${W}_$N.json')); print('$W N=$N', round(d['value'],1), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value'],1), 'collect frac', round(d['roofline']['frac'],3), d['clocks'].get('sm_mhz'))"; done
