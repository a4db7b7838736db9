mkdir -p gpurun_out/fbn
python tools/run_once.py --config 2 > gpurun_out/fbn/ro.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_floyd_bitmap -c 1 -o gpurun_out/fbn/bitmap_cfg2 python tools/run_once.py --config 2 --reps 0 > gpurun_out/fbn/ncu.log 2>&1
