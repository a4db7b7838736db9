#!/bin/bash
# r02a: full-size parity cfg1-4, cfg5 + cfg4 bench lines with the new bench.py
OUT=gpurun_out/r02a
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "not 5" > $OUT/fullsize.log 2>&1; echo "rc=$?" >> $OUT/fullsize.log
timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/bench_cfg5.json 2> $OUT/bench_cfg5.err
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 > $OUT/bench_cfg4.json 2> $OUT/bench_cfg4.err
tail -3 $OUT/fullsize.log
tail -c 600 $OUT/bench_cfg5.json; tail -5 $OUT/bench_cfg5.err
