#!/bin/bash
# A/B of library variants on the NVLink exchange probe (scripts/nvlink_probe.py, needs 2+ GPUs)
L=paper_2305_12201_b200/libgravac_b200.so
cp $L /tmp/lib_keep.so
for v in ${VARIANTS}; do
  cp scripts/probes/lib_$v.so $L
  echo "== $v"; timeout 120 python scripts/nvlink_probe.py ${W:-2} ${N:-44500000} 2>&1 | tail -2
done
cp /tmp/lib_keep.so $L
