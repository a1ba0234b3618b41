#!/bin/bash
# Per-kernel select timeline (scripts/phase_probe.py) with the stamped library variant
L=paper_2305_12201_b200/libgravac_b200.so
cp $L /tmp/lib_keep.so
cp scripts/probes/lib_${VARIANT:-stamps}.so $L
for n in ${SIZES:-44500000 138000000}; do
  echo "== n=$n"; timeout 300 python scripts/phase_probe.py $n
done
cp /tmp/lib_keep.so $L
