#!/bin/bash
# r02h: TMA gather microbenchmark; reference arm diagnosis (rc, memory)
OUT=gpurun_out/r02h
mkdir -p $OUT
(nproc; free -g) > $OUT/host.txt 2>&1
timeout 300 tools/tma_gather_ceiling > $OUT/tma_gather.jsonl 2> $OUT/tma_gather.err; echo "rc=$?" >> $OUT/tma_gather.err
cat $OUT/tma_gather.jsonl; tail -3 $OUT/tma_gather.err
(while true; do free -m | awk 'NR==2{print $3, $7}'; sleep 5; done) > $OUT/mem.txt 2>&1 &
MP=$!
{ time timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "rc=$?" >> $OUT/bench_ref.err; } 2> $OUT/bench_ref.time
kill $MP
tail -c 600 $OUT/bench_ref.json; tail -3 $OUT/bench_ref.err; cat $OUT/bench_ref.time; sort -n $OUT/mem.txt | tail -1; cat $OUT/host.txt
