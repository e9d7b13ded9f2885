#!/bin/bash
# round 2 (session 3), call 88 (1 GPU): merges of 9..32 splits with batched partial loads (C,
# the build) vs sequential (A, experiments/r02/ab_A): C4@N=8 shape (S=16), C3 S=4 / S=1; ncu
# source captures of the S=16 launch for both
O=gpurun_out/r02c88; mkdir -p $O
LIB=paper_2405_01814_b200/lib/liblamina_attn.so
cp $LIB /tmp/C.so
for rep in 1 2; do
  for v in C A; do
    if [ $v = C ]; then cp /tmp/C.so $LIB; else cp experiments/r02/ab_A/liblamina_attn.so $LIB; fi
    AB_SPLIT=2048 timeout 120 python experiments/r02/tc_ab.py gqa_tc 16 8 1 128 32768 64 >> $O/c4n8_$v.log 2>&1
    AB_SPLIT=1024 timeout 120 python experiments/r02/tc_ab.py gqa_tc 128 64 8 128 4096 64 >> $O/c3s4_$v.log 2>&1
    timeout 120 python experiments/r02/tc_ab.py gqa_tc 128 64 8 128 4096 64 >> $O/c3_$v.log 2>&1
  done
done
cp /tmp/C.so $LIB
for v in C; do
  AB_SPLIT=2048 timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_gqa_tc -s 5 -c 1 -o /tmp/c4n8_$v python experiments/r02/tc_ab.py gqa_tc 16 8 1 128 32768 64 > $O/ncu_$v.log 2>&1
done
cp /tmp/C.so $LIB
ncu -i /tmp/c4n8_C.ncu-rep --page source --csv > $O/c4n8_C_source.csv 2>&1
ncu -i /tmp/c4n8_C.ncu-rep --page details --csv > $O/c4n8_C_details.csv 2>&1
echo done
