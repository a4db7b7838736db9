OUT=gpurun_out/r01k; mkdir -p $OUT
./tools/gather_ceiling q5 > $OUT/ceil.jsonl 2>&1
grep head $OUT/ceil.jsonl > $OUT/head_ceil.jsonl
cat $OUT/head_ceil.jsonl >> profiles/r01_gather_ceilings.jsonl
for c in 3 4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err; done
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 > $OUT/bench_cfg5.json 2> $OUT/bench_cfg5.err
