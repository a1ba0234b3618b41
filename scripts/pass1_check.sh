#!/bin/bash
# parity suite + VGG16 / ResNet101 bench + launch list of one VGG16 step (dev loop for select-kernel changes)
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for w in vgg16 resnet101; do python bench.py --workload $w --no-cpu-baseline > gpurun_out/b_$w.log 2>&1; done
python scripts/bench_summary.py gpurun_out/b_vgg16.log gpurun_out/b_resnet101.log
GVC_BENCH_NOPROF=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -c 30 --csv \
    --log-file gpurun_out/vgg_l2.csv python bench.py --workload vgg16 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python - <<'PY'
import csv
r = list(csv.reader(open("gpurun_out/vgg_l2.csv")))
h = [i for i, x in enumerate(r) if "Kernel Name" in x][0]
H = r[h]
for x in r[h + 1:][-10:-1]:
    print(x[H.index("Kernel Name")][:30], x[H.index("Metric Value")])
PY
