#!/bin/bash
# r02g: fused v3 A/B on cfg3-5; cfg5 launch list; ncu full of the Floyd kernels (two-kernel and fused) on cfg5
OUT=gpurun_out/r02g
mkdir -p $OUT
timeout 900 python tools/ab_fused.py 3 4 5 > $OUT/ab.jsonl 2> $OUT/ab.err; echo "rc=$?" >> $OUT/ab.err
cat $OUT/ab.jsonl; tail -3 $OUT/ab.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches_cfg5.csv python tools/run_once.py --config 5 --reps 0 > $OUT/launches.log 2>&1; echo "rc=$?" >> $OUT/launches.log
tail -2 $OUT/launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_floyd_bloom -c 1 \
   -o $OUT/floyd_cfg5 python tools/run_once.py --config 5 --reps 0 > $OUT/ncu_floyd.log 2>&1; echo "rc=$?" >> $OUT/ncu_floyd.log
tail -2 $OUT/ncu_floyd.log
SNGB_FUSED=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_floyd_head -c 1 \
   -o $OUT/fused_cfg5 python tools/run_once.py --config 5 --reps 0 > $OUT/ncu_fused.log 2>&1; echo "rc=$?" >> $OUT/ncu_fused.log
tail -2 $OUT/ncu_fused.log
