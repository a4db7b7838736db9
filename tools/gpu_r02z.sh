#!/bin/bash
# k_floyd_lean: parity suite, A/B against k_floyd_bloom on cfg4/cfg5, bench, ncu of the kernel.
OUT=gpurun_out/r02z
mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
timeout 900 python tools/lean_ab.py 4 5 > $OUT/lean_ab.jsonl 2> $OUT/lean_ab.err; cat $OUT/lean_ab.jsonl
for C in 5 4; do
  timeout 900 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-pageable > $OUT/bench$C.json 2> $OUT/bench$C.err
  python -c "import json;d=json.load(open('$OUT/bench$C.json'));print('cfg$C', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'], d.get('stages_ms'))"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_floyd_lean -c 1 \
  -o $OUT/lean_cfg5 python tools/run_once.py --config 5 --reps 0 > $OUT/ncu_lean.log 2>&1; echo "ncu rc=$?"
