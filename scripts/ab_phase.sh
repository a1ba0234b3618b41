#!/bin/bash
# Per-kernel select timelines (scripts/phase_probe.py) for several stamped library variants
for v in ${VARIANTS}; do
  echo "#### $v"; VARIANT=$v SIZES="${SIZES:-44500000}" bash scripts/phase_run.sh 2>&1 | tail -4
done
