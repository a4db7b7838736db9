#!/bin/bash
# All five BASELINE shapes, one bench line each (under gpurun): bash tools/bench_all.sh TAG
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for c in 1 2 3; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err; done
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 > $OUT/bench_cfg4.json 2> $OUT/bench_cfg4.err
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 > $OUT/bench_cfg5.json 2> $OUT/bench_cfg5.err
for c in 1 2 3 4 5; do echo "cfg$c $(tail -c 300 $OUT/bench_cfg$c.json | head -c 300)"; done
