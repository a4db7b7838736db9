#!/bin/bash
# r02f: re-establish this round's GPU evidence on the current tree
OUT=gpurun_out/r02f
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -x > $OUT/all.log 2>&1; echo "rc=$?" >> $OUT/all.log
tail -5 $OUT/all.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
tail -4 $OUT/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/bench_cfg5.json 2> $OUT/bench_cfg5.err
tail -c 3000 $OUT/bench_cfg5.json; tail -5 $OUT/bench_cfg5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
tail -c 1500 $OUT/bench_ref.json; tail -3 $OUT/bench_ref.err
