#!/bin/bash
# r02i: warp-per-vertex fused kernel (k_sample_head): parity, then A/B against the two kernels
OUT=gpurun_out/r02i
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or head or hook" > $OUT/parity.log 2>&1; echo "rc=$?" >> $OUT/parity.log
tail -15 $OUT/parity.log
timeout 900 python tools/ab_fused.py 3 4 5 > $OUT/ab.jsonl 2> $OUT/ab.err; echo "rc=$?" >> $OUT/ab.err
cat $OUT/ab.jsonl; tail -3 $OUT/ab.err
{ time timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "rc=$?" >> $OUT/bench_ref.err; } 2> $OUT/bench_ref.time
tail -c 400 $OUT/bench_ref.json; tail -2 $OUT/bench_ref.err; cat $OUT/bench_ref.time
