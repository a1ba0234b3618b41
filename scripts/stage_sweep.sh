# staged-pull parameter sweep (development aid): bash scripts/stage_sweep.sh N "chunk:copiers" ...
N=${1:-2}; shift
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $N --steps 60 --warmup 5 --no-cpu-baseline"
for cfg in "$@"; do
  ch=${cfg%%:*}; cp=${cfg##*:}
  GVC_EXCHANGE=staged GVC_STAGE_CHUNK=$ch GVC_STAGE_COPIERS=$cp $T 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$N chunk $ch copiers $cp', round(d['value'],1), round(d['ms_per_step'],4), round(d['step_ms']['median'],4))"
done
