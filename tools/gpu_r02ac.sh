#!/bin/bash
# source-level ncu of the two cfg5 kernels on the current tree (k_floyd_lean, k_gather_head)
OUT=gpurun_out/r02ac
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_floyd_lean|k_gather_head' -c 2 \
  -o $OUT/cfg5_two python tools/run_once.py --config 5 --reps 0 > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
ls -la $OUT
