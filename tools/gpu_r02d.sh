#!/bin/bash
# r02d: fused kernel with draws in smem -- parity, A/B, ncu of k_floyd_head on cfg5
OUT=gpurun_out/r02d
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "head or fused" > $OUT/parity.log 2>&1; echo "rc=$?" >> $OUT/parity.log
tail -3 $OUT/parity.log
timeout 900 python tools/ab_fused.py 3 4 5 > $OUT/ab.jsonl 2> $OUT/ab.err
cat $OUT/ab.jsonl; tail -3 $OUT/ab.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_floyd_head -c 1 \
   -o $OUT/fused_cfg5 python tools/run_once.py --config 5 --reps 0 > $OUT/ncu_fused.log 2>&1
tail -3 $OUT/ncu_fused.log
