#!/bin/bash
# Per-stage timing of the narrow-row configs under env variants (under gpurun):
#   bash tools/head_timing.sh TAG "SNGB_HEAD=0" "SNGB_HEAD=1" ...
# Summarise with: python tools/ro_table.py gpurun_out/TAG/ro.log
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
for c in 5 3 4; do for v in "$@"; do
  echo "cfg$c $v" >> $OUT/ro.log
  env $v timeout 600 python tools/run_once.py --config $c --reps 2 >> $OUT/ro.log 2>&1
done; done
