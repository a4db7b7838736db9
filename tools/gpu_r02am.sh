#!/bin/bash
# r02 round check on the k_floyd_pipe tree: GPU suite, smoke, default bench (cfg5) + reference arm,
# launch list of the bench command, ncu --set full of the two cfg5 kernels.
OUT=gpurun_out/r02az
mkdir -p $OUT
(time timeout 1500 python -m pytest tests -q -m gpu -x) > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -4 $OUT/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_head -c 1 \
  -o $OUT/gather_cfg5 python tools/run_once.py --config 5 --reps 0 > $OUT/ncu_gather.log 2>&1; echo "ncu gather rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_floyd_pipe -c 1 \
  -o $OUT/pipe_cfg5 python tools/run_once.py --config 5 --reps 0 > $OUT/ncu_pipe.log 2>&1; echo "ncu pipe rc=$?"
ls -la $OUT
