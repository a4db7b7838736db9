#!/bin/bash
OUT=gpurun_out/r02t
mkdir -p $OUT
for L in libsngb_fwr4 libsngb_fwr16; do
  SNGB_LIBRARY=$PWD/tools/ab/$L.so timeout 600 python tools/floyd_ab.py 3 4 5 >> $OUT/ab.jsonl 2>> $OUT/ab.err
done
timeout 600 python tools/floyd_ab.py 3 4 5 >> $OUT/ab.jsonl 2>> $OUT/ab.err
cat $OUT/ab.jsonl; tail -3 $OUT/ab.err
