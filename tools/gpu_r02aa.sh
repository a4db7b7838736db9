#!/bin/bash
# k_floyd_head: fused/lean parity tests, A/B vs two kernels on cfg4/cfg5, ncu of the kernel.
OUT=gpurun_out/r02aa
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fused or lean or floyd" > $OUT/pytest_sel.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_sel.log
tail -3 $OUT/pytest_sel.log
timeout 900 python tools/fh_ab.py 4 5 > $OUT/fh_ab.jsonl 2> $OUT/fh_ab.err; cat $OUT/fh_ab.jsonl; tail -3 $OUT/fh_ab.err
SNGB_FUSED=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_floyd_head -c 1 \
  -o $OUT/fh_cfg5 python tools/run_once.py --config 5 --reps 0 > $OUT/ncu_fh.log 2>&1; echo "ncu rc=$?"
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
