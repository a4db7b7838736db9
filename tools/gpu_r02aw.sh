#!/bin/bash
# head gather R / UF build variants on cfg5 and cfg4 (tools/ab/libsngb_*.so)
OUT=gpurun_out/r02aw
mkdir -p $OUT
for lib in default tools/ab/libsngb_r8.so tools/ab/libsngb_r2.so tools/ab/libsngb_uf4.so tools/ab/libsngb_uf1.so tools/ab/libsngb_r8uf4.so; do
  for c in 5 4; do
    if [ "$lib" = default ]; then unset SNGB_LIBRARY; else export SNGB_LIBRARY=$PWD/$lib; fi
    echo "== $lib cfg$c" >> $OUT/variants.log
    timeout 600 python tools/run_once.py --config $c --reps 3 2>&1 | tail -1 >> $OUT/variants.log
  done
done
cat $OUT/variants.log
