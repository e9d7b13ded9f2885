#!/bin/bash
# round 2, call 36: ncu evidence for the production step launches (tcgen05 kernel): c2, c3, c4, c5
# (one launch each, --set full, exported to csv) and the launch list of the default bench line
O=gpurun_out/r02c36; mkdir -p $O; T=/tmp/ncu36; mkdir -p $T
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --check 0"
$B --workload c2 > $O/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv $B --workload c2 > $O/ncu_launch_c2.log 2>&1
for wl in c2 c3 c4 c5; do
  $B --workload $wl > $O/plain_$wl.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_gqa_tc --launch-skip 3 --launch-count 1 \
    -o $T/step_$wl $B --workload $wl > $O/ncu_$wl.log 2>&1
  ncu -i $T/step_$wl.ncu-rep --page raw --csv > $O/step_${wl}_raw.csv 2>/dev/null
  ncu -i $T/step_$wl.ncu-rep --page details --csv > $O/step_${wl}_details.csv 2>/dev/null
  ncu -i $T/step_$wl.ncu-rep --page source --csv --print-source sass > $O/step_${wl}_source.csv 2>/dev/null
  ls -la $T >> $O/files.txt
done
du -sh $O >> $O/files.txt
