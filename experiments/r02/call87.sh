#!/bin/bash
# round 2 (session 3), call 87 (1 GPU): where the split path's per-item cost sits — the tcgen05
# kernel on C3 S=4 and the C4@N=8 shape (S=16) with the epilogue warp's work skipped
# (LAM_DECODE_FLAGS=32), the consumers' math skipped (16) and both (48)
O=gpurun_out/r02c87; mkdir -p $O
for fl in 0 32 16 48; do
  LAM_DECODE_FLAGS=$fl AB_SPLIT=1024 timeout 120 python experiments/r02/tc_ab.py gqa_tc 128 64 8 128 4096 64 >> $O/c3s4_f$fl.log 2>&1
  LAM_DECODE_FLAGS=$fl timeout 120 python experiments/r02/tc_ab.py gqa_tc 128 64 8 128 4096 64 >> $O/c3_f$fl.log 2>&1
  LAM_DECODE_FLAGS=$fl AB_SPLIT=2048 timeout 120 python experiments/r02/tc_ab.py gqa_tc 16 8 1 128 32768 64 >> $O/c4n8_f$fl.log 2>&1
done
echo done
