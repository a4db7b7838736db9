#!/bin/bash
OUT=gpurun_out/r02ai
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "floyd_pipe" > $OUT/pytest_sel.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_sel.log
tail -3 $OUT/pytest_sel.log
timeout 900 python tools/pipe_ab.py 4 5 > $OUT/pipe_ab.jsonl 2> $OUT/pipe_ab.err; cat $OUT/pipe_ab.jsonl; tail -3 $OUT/pipe_ab.err
