T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 4 --steps 100 --warmup 5 --no-cpu-baseline"
for x in push pull nccl; do GVC_EXCHANGE=$x $T 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$x', round(d['value'],1), round(d['ms_per_step'],4), d['step_ms'], d['breakdown_ms'])"; done
