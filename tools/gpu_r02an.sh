#!/bin/bash
# shared draws: parity tests, A/B on cfg4/cfg5
OUT=gpurun_out/r02an
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "shared_draws or floyd_pipe or duo or headpipe or lean" > $OUT/pytest_sel.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_sel.log
tail -15 $OUT/pytest_sel.log
timeout 1500 python tools/share_ab.py 4 5 > $OUT/share_ab.jsonl 2> $OUT/share_ab.err; cat $OUT/share_ab.jsonl; tail -3 $OUT/share_ab.err
