mkdir -p gpurun_out/h1
./tools/gather_ceiling q5 > gpurun_out/h1/ceil.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k head > gpurun_out/h1/pytest.log 2>&1
for c in 5 3; do for m in 0 2; do echo "cfg$c HEAD=$m" >> gpurun_out/h1/ro.log; SNGB_HEAD=$m timeout 600 python tools/run_once.py --config $c --reps 2 >> gpurun_out/h1/ro.log 2>&1; done; done
