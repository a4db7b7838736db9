OUT=gpurun_out/h4; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "head" > $OUT/pytest.log 2>&1
for c in 5 3 4; do for ov in 0 2; do
  echo "cfg$c OVERLAP=$ov" >> $OUT/ro.log
  SNGB_OVERLAP=$ov timeout 600 python tools/run_once.py --config $c --reps 2 >> $OUT/ro.log 2>&1
done; done
