#!/bin/bash
# N-GPU A/B of library variants (staged exchange, ResNet101 44.5M)
L=paper_2305_12201_b200/libgravac_b200.so
cp $L /tmp/lib_keep.so
for v in ${VARIANTS}; do
  cp scripts/probes/lib_$v.so $L
  echo "== $v"; MODES=staged bash scripts/r2_n4_ab.sh
done
cp /tmp/lib_keep.so $L
