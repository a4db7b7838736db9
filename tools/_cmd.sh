OUT=gpurun_out/r01l; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --config 1 > $OUT/bench_cfg1.json 2> $OUT/bench_cfg1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
      python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_launch.log 2>&1
python tools/timeline.py --config 2 --reps 3 > $OUT/timeline_cfg2.txt 2>/dev/null
python tools/timeline.py --config 2 --reps 2 --host > $OUT/timeline_cfg2_host.txt 2>/dev/null
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
