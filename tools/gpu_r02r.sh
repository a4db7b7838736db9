#!/bin/bash
# r02r: fused v8 (k_floyd_warp's P1 + head gather, one pass) + k_floyd_warp parity; A/B; ncu
OUT=gpurun_out/r02r
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or head or hook or floyd_warp or irregular" > $OUT/parity.log 2>&1; echo "rc=$?" >> $OUT/parity.log
tail -4 $OUT/parity.log
AB_VARIANTS=fused,two_kernels timeout 900 python tools/ab_fused.py 3 4 5 > $OUT/ab.jsonl 2> $OUT/ab.err; echo "rc=$?" >> $OUT/ab.err
cat $OUT/ab.jsonl | cut -c1-200; tail -3 $OUT/ab.err
SNGB_FUSED=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sample_head -c 1 \
   -o $OUT/fused8_cfg5 python tools/run_once.py --config 5 --reps 0 > $OUT/ncu.log 2>&1; echo "rc=$?" >> $OUT/ncu.log
tail -2 $OUT/ncu.log
