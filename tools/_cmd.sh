mkdir -p gpurun_out/ff
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_floyd or q8 or device_api" > gpurun_out/ff/pytest.log 2>&1
python tools/timeline.py --config 2 --reps 3 > gpurun_out/ff/cfg2.txt 2> gpurun_out/ff/cfg2.err
for v in "X=0" "SNGB_FUSE_FLOYD=0"; do
  echo "$v $(env $v timeout 300 python bench.py --config 2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["roofline"]["kernel_ms"],3), d["stages_ms"])')" >> gpurun_out/ff/b.log
done
