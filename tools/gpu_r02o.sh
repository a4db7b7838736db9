#!/bin/bash
# r02q: k_floyd_warp (warp-per-vertex Floyd) parity + A/B vs k_floyd_bloom; ncu of it on cfg5
OUT=gpurun_out/r02q
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x > $OUT/parity.log 2>&1; echo "rc=$?" >> $OUT/parity.log
tail -4 $OUT/parity.log
AB_VARIANTS=two_kernels,two_kernels_bloom timeout 900 python tools/ab_fused.py 3 4 5 > $OUT/ab.jsonl 2> $OUT/ab.err; echo "rc=$?" >> $OUT/ab.err
cat $OUT/ab.jsonl | cut -c1-230; tail -3 $OUT/ab.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_floyd_warp -c 1 \
   -o $OUT/floydw_cfg5 python tools/run_once.py --config 5 --reps 0 > $OUT/ncu.log 2>&1; echo "rc=$?" >> $OUT/ncu.log
tail -2 $OUT/ncu.log
