#!/bin/bash
OUT=gpurun_out/r02w
mkdir -p $OUT
for C in 5 4 3; do
SWEEP=rpb SWEEP_G=4 SWEEP_RPB=1,2,4,8,16 timeout 1200 python tools/overlap_sweep.py --config $C > $OUT/sweep$C.jsonl 2> $OUT/sweep$C.err; echo "rc=$?" >> $OUT/sweep$C.err
cat $OUT/sweep$C.jsonl | grep -v gather_rpb
done
