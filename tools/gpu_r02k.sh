#!/bin/bash
OUT=gpurun_out/r02k
mkdir -p $OUT
timeout 600 compute-sanitizer --tool memcheck --show-backtrace device python tools/repro_fused.py > $OUT/memcheck.log 2>&1; echo "rc=$?" >> $OUT/memcheck.log
head -60 $OUT/memcheck.log
