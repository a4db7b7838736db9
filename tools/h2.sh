# head filter: ncu captures on cfg5 / cfg3, cfg4 timing with the head forced
OUT=gpurun_out/h2; mkdir -p $OUT
for m in 0 2; do echo "cfg4 HEAD=$m" >> $OUT/ro.log; SNGB_HEAD=$m timeout 600 python tools/run_once.py --config 4 --reps 2 >> $OUT/ro.log 2>&1; done
for c in 5 3; do echo "cfg$c SEQ" >> $OUT/ro.log; SNGB_OVERLAP=0 timeout 600 python tools/run_once.py --config $c --reps 2 >> $OUT/ro.log 2>&1; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_head -c 1 -o $OUT/head_cfg5 python tools/run_once.py --config 5 --reps 0 > $OUT/ncu5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gather_head -c 1 -o $OUT/head_cfg3 python tools/run_once.py --config 3 --reps 0 > $OUT/ncu3.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_gather_head -c 1 --csv --log-file $OUT/traffic5.csv python tools/run_once.py --config 5 --reps 0 > $OUT/ncut.log 2>&1
