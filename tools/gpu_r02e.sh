#!/bin/bash
OUT=gpurun_out/r02e
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "head or fused" > $OUT/parity.log 2>&1; echo "rc=$?" >> $OUT/parity.log
tail -3 $OUT/parity.log
timeout 600 python tools/ab_fused.py 3 4 5 > $OUT/ab.jsonl 2> $OUT/ab.err
SNGB_LIBRARY=$PWD/tools/ab/libsngb_minb2.so timeout 600 python tools/ab_fused.py 5 >> $OUT/ab.jsonl 2>> $OUT/ab.err
cat $OUT/ab.jsonl; tail -3 $OUT/ab.err
