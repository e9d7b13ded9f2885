#!/bin/bash
# round 2, call 11: tcgen05 ring split A/B (3K3V vs 4K2V) on C3 and C2 (MHA) layer shapes
O=gpurun_out/r02c11; mkdir -p $O
for shape in "128 64 8 128 4096 64" "64 32 32 128 4096 64"; do
for cfg in "gqa_mma 33" "gqa_tc 33" "gqa_tc 42" "gqa_mma 33" "gqa_tc 33" "gqa_tc 42"; do
  set -- $cfg
  LAM_TC_RING=$2 timeout 120 python experiments/r02/tc_ab.py $1 $shape >> $O/ab.log 2>&1
done; done
