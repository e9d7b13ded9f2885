#!/bin/bash
# round 2 (session 3), call 97 (1 GPU): ncu of the final tcgen05 kernel on the C4@N=8-shaped
# launch (planner's split) and on C3 split 4 ways; details pages only
O=gpurun_out/r02c97; mkdir -p $O
timeout 300 ncu --set full --clock-control none -k regex:decode_gqa_tc -s 5 -c 1 -o /tmp/c4n8 python experiments/r02/tc_ab.py gqa_tc 16 8 1 128 32768 64 > $O/ncu_c4n8.log 2>&1
AB_SPLIT=1024 timeout 300 ncu --set full --clock-control none -k regex:decode_gqa_tc -s 5 -c 1 -o /tmp/c3s4 python experiments/r02/tc_ab.py gqa_tc 128 64 8 128 4096 64 > $O/ncu_c3s4.log 2>&1
for r in c4n8 c3s4; do
  ncu -i /tmp/$r.ncu-rep --page details --csv > $O/${r}_details.csv 2>&1
  ncu -i /tmp/$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>&1
done
echo done
