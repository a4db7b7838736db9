#!/bin/bash
# source-level ncu of k_floyd_pipe on cfg5
OUT=gpurun_out/r02ah
mkdir -p $OUT
SNGB_FLOYD_PIPE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_floyd_pipe' -c 1 \
  -o $OUT/pipe_cfg5 python tools/run_once.py --config 5 --reps 0 > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
ls -la $OUT
