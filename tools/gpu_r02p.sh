#!/bin/bash
OUT=gpurun_out/r02p
mkdir -p $OUT
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/repro_fw.py > $OUT/repro.log 2>&1; echo "rc=$?" >> $OUT/repro.log
tail -6 $OUT/repro.log
SNGB_FLOYD_BLOOM=1 timeout 300 python tools/repro_fw.py > $OUT/repro_bloom.log 2>&1; echo "rc=$?" >> $OUT/repro_bloom.log
tail -6 $OUT/repro_bloom.log
