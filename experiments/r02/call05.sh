#!/bin/bash
# round 2, call 5: tcgen05 kernel with split K / V stage barriers: parity probe + A/B
O=gpurun_out/r02c05; mkdir -p $O
timeout 300 python experiments/r02/tc_probe.py > $O/tc_probe.log 2>&1; echo "rc=$?" >> $O/tc_probe.log
for cfg in "gqa_mma 0 3" "gqa_tc 0 3" "gqa_tc 16 3" "gqa_mma 0 3" "gqa_tc 0 3"; do
  set -- $cfg
  LAM_DECODE_FLAGS=$2 LAM_TC_STAGES=$3 timeout 120 python experiments/r02/tc_ab.py $1 >> $O/ab.log 2>&1
done
