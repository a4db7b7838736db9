#!/bin/bash
# r02u: whole GPU suite on the current tree; cfg3 step A/B (warp vs bloom Floyd, default scheduling)
OUT=gpurun_out/r02u
mkdir -p $OUT
timeout 2400 python -m pytest tests -q -m gpu -x > $OUT/all.log 2>&1; echo "rc=$?" >> $OUT/all.log
tail -4 $OUT/all.log
for FW in 2 0; do
  SNGB_FLOYD_WARP=$FW timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench3_fw$FW.json 2> $OUT/bench3_fw$FW.err
  python -c "import json;d=json.load(open('$OUT/bench3_fw$FW.json'));print('FW=$FW cfg3', d['ms_per_step'], d['stages_ms'])"
done
