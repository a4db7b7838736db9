#!/bin/bash
# r02c: fused Floyd + head gather -- parity, then A/B timing (MINB 3 vs 4)
OUT=gpurun_out/r02c
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "head or fused" > $OUT/parity.log 2>&1; echo "rc=$?" >> $OUT/parity.log
tail -3 $OUT/parity.log
timeout 900 python tools/ab_fused.py 3 4 5 > $OUT/ab.jsonl 2> $OUT/ab.err
SNGB_LIBRARY=$PWD/tools/ab/libsngb_minb4.so timeout 600 python tools/ab_fused.py 4 5 >> $OUT/ab.jsonl 2>> $OUT/ab.err
cat $OUT/ab.jsonl; tail -3 $OUT/ab.err
