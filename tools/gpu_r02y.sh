#!/bin/bash
# Re-entry check of the restored tree: GPU suite, smoke, default bench (cfg5), cfg2/cfg4 lines.
OUT=gpurun_out/r02y
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
for C in 5 2 4; do
  timeout 900 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench$C.json 2> $OUT/bench$C.err
  python -c "import json;d=json.load(open('$OUT/bench$C.json'));print('cfg$C', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'], d.get('stages_ms'))"
done
