#!/bin/bash
OUT=gpurun_out/r02ao
mkdir -p $OUT
export SNGB_SHARE_SERIAL=1 SNGB_TBUF_MB=16384 SNGB_SAMPLER_RPB=64
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:'k_gather_head|k_floyd_pipe' --log-file $OUT/share_launches.csv \
      python tools/run_once.py --config 5 --reps 0 > $OUT/ncu.log 2>&1
echo rc=$?
python - <<'P'
import csv,collections
rows=[r for r in csv.reader(open('gpurun_out/r02ao/share_launches.csv')) if len(r)>10]
hdr=rows[0]; ki=hdr.index('Kernel Name'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); ii=hdr.index('ID')
d=collections.defaultdict(dict)
for r in rows[1:]:
    d[(r[ii],r[ki][:40])][r[mi]]=r[vi]
for k,v in list(d.items())[:12]: print(k, v)
P
