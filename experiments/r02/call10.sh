#!/bin/bash
# round 2, call 10: tcgen05 kernel with separate K / V rings: parity + A/B of 2K+4V vs 3K+3V
O=gpurun_out/r02c10; mkdir -p $O
timeout 300 python experiments/r02/tc_probe.py > $O/tc_probe.log 2>&1; echo "rc=$?" >> $O/tc_probe.log
for cfg in "gqa_mma 0 24" "gqa_tc 0 24" "gqa_tc 0 33" "gqa_tc 16 24" "gqa_mma 0 24" "gqa_tc 0 24" "gqa_tc 0 33"; do
  set -- $cfg
  LAM_DECODE_FLAGS=$2 LAM_TC_RING=$3 timeout 120 python experiments/r02/tc_ab.py $1 >> $O/ab.log 2>&1
done
