#!/bin/bash
OUT=gpurun_out/r02v
mkdir -p $OUT
SWEEP=rpb timeout 1200 python tools/overlap_sweep.py --config 5 > $OUT/sweep5.jsonl 2> $OUT/sweep5.err; echo "rc=$?" >> $OUT/sweep5.err
cat $OUT/sweep5.jsonl; tail -3 $OUT/sweep5.err
SWEEP=rpb timeout 600 python tools/overlap_sweep.py --config 4 > $OUT/sweep4.jsonl 2> $OUT/sweep4.err; echo "rc=$?" >> $OUT/sweep4.err
cat $OUT/sweep4.jsonl
