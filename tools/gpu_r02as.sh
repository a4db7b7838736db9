#!/bin/bash
OUT=gpurun_out/r02as
mkdir -p $OUT
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --no-pageable > $OUT/bench_cfg4_nvml.json 2> $OUT/err1.log
SNGB_BENCH_CLOCKS=smi timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --no-pageable > $OUT/bench_cfg4_smi.json 2> $OUT/err2.log
python - <<'P'
import json
for t in ('nvml','smi'):
    d=json.load(open(f'gpurun_out/r02as/bench_cfg4_{t}.json'))
    print(t, 'step', d['ms_per_step'], 'ms_total', d['stages_ms']['ms_total'], d['clocks'], 'e2e', d['e2e']['ms_per_step'])
P
tail -2 $OUT/err1.log
python tools/gap_probe.py 5 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "kat or golden or forced_irregular or floyd_pipe" 2>&1 | tail -2
