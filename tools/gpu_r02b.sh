#!/bin/bash
# r02b: new GPU tests (exact, multi-GPU C ABI, CLI, C++ mirror) + the whole -m gpu suite
OUT=gpurun_out/r02b
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_multi.py tests/test_cli.py tests/test_cpp_mirror.py -q -m gpu -x > $OUT/new.log 2>&1; echo "rc=$?" >> $OUT/new.log
timeout 1500 python -m pytest tests -q -m gpu --deselect tests/test_gpu_fullsize.py > $OUT/all.log 2>&1; echo "rc=$?" >> $OUT/all.log
tail -15 $OUT/new.log; tail -5 $OUT/all.log
