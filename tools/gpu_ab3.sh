#!/bin/bash
for i in 1 2; do
for lib in default tools/ab/libsngb_flagbar.so; do
  if [ "$lib" = default ]; then unset SNGB_LIBRARY; else export SNGB_LIBRARY=$PWD/$lib; fi
  echo "== $lib"; python tools/gap_probe.py 5 2>&1 | tail -5 | head -1; python tools/gap_probe.py 4 2>&1 | tail -5 | head -1
done
done
SNGB_LIBRARY=$PWD/tools/ab/libsngb_flagbar.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "floyd_pipe" 2>&1 | tail -1
