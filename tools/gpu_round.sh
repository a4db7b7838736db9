#!/bin/bash
# One GPU session: tests, bench (default + reference arm), launch list, ncu capture.
# Usage (from the repo root, under gpurun): bash tools/gpu_round.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
      python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_launch.log 2>&1
python tools/run_once.py --config 2 > $OUT/ro2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_gather -c 1 \
      -o $OUT/gather_cfg2 python tools/run_once.py --config 2 --reps 0 > $OUT/ncu_full.log 2>&1
tail -2 $OUT/pytest_gpu.log
# DRAM traffic of every gather launch of one cfg2 step (all L2 phases)
python tools/run_once.py --config 2 > $OUT/ro2b.log 2>&1 && \
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:k_gather -c 4 --csv --log-file $OUT/gather_traffic.csv \
      python tools/run_once.py --config 2 --reps 0 > $OUT/ncu_traffic.log 2>&1
