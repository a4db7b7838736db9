#!/bin/bash
OUT=gpurun_out/r02x
mkdir -p $OUT
for C in 5 4; do
  timeout 900 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench$C.json 2> $OUT/bench$C.err
  python -c "import json;d=json.load(open('$OUT/bench$C.json'));print('cfg$C', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'], 'pageable', (d.get('e2e_pageable') or {}).get('ms_per_step'), d['stages_ms'])"
done
