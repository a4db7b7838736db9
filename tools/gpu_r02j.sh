#!/bin/bash
OUT=gpurun_out/r02j
mkdir -p $OUT
SNGB_FUSED=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sample_head -c 1 \
   -o $OUT/fused2_cfg5 python tools/run_once.py --config 5 --reps 0 > $OUT/ncu_fused.log 2>&1; echo "rc=$?" >> $OUT/ncu_fused.log
tail -2 $OUT/ncu_fused.log
timeout 300 tools/tma_gather_ceiling w > $OUT/tma_wide.jsonl 2> $OUT/tma_wide.err; echo "rc=$?" >> $OUT/tma_wide.err
cat $OUT/tma_wide.jsonl; tail -2 $OUT/tma_wide.err
