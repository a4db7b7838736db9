#!/bin/bash
# r02n: fused v6 parity + A/B + ncu
OUT=gpurun_out/r02n
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or head or hook" > $OUT/parity.log 2>&1; echo "rc=$?" >> $OUT/parity.log
tail -4 $OUT/parity.log
timeout 900 python tools/ab_fused.py 3 4 5 > $OUT/ab.jsonl 2> $OUT/ab.err; echo "rc=$?" >> $OUT/ab.err
cat $OUT/ab.jsonl | cut -c1-200; tail -3 $OUT/ab.err
SNGB_FUSED=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sample_head -c 1 \
   -o $OUT/fused7_cfg5 python tools/run_once.py --config 5 --reps 0 > $OUT/ncu_fused.log 2>&1; echo "rc=$?" >> $OUT/ncu_fused.log
tail -2 $OUT/ncu_fused.log
