#!/bin/bash
# round 2, call 4: tcgen05 kernel diagnosis — pipeline-only (flags 16) and 2 vs 3 stages
O=gpurun_out/r02c05; mkdir -p $O
for cfg in "gqa_mma 0 3" "gqa_tc 0 3" "gqa_tc 16 3" "gqa_mma 16 3" "gqa_tc 0 2" "gqa_tc 16 2"; do
  set -- $cfg
  LAM_DECODE_FLAGS=$2 LAM_TC_STAGES=$3 timeout 120 python experiments/r02/tc_ab.py $1 >> $O/ab.log 2>&1
done
