# head formats: parity + per-config timing of each format, with and without the sampler overlap
OUT=gpurun_out/h3; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_abi.py -q -x -k "head or abi" > $OUT/pytest.log 2>&1
for c in 5 3 4; do for k in 0 1 2; do for ov in 0 2; do
  echo "cfg$c KIND=$k OVERLAP=$ov" >> $OUT/ro.log
  SNGB_HEAD=2 SNGB_HEAD_KIND=$k SNGB_OVERLAP=$ov timeout 600 python tools/run_once.py --config $c --reps 2 >> $OUT/ro.log 2>&1
done; done; done
