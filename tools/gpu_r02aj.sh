#!/bin/bash
# k_duo: parity tests, A/B against the two kernels on cfg4/cfg5
OUT=gpurun_out/r02aj
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "duo or floyd_pipe or fused" > $OUT/pytest_sel.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_sel.log
tail -15 $OUT/pytest_sel.log
timeout 1200 python tools/duo_ab.py 4 5 > $OUT/duo_ab.jsonl 2> $OUT/duo_ab.err; cat $OUT/duo_ab.jsonl; tail -3 $OUT/duo_ab.err
