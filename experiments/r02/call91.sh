#!/bin/bash
# round 2 (session 3), call 91 (1 GPU): what the tcgen05 kernel's per-item cost is made of —
# C3 S=4 and S=1, and the same 2 GiB as 8192 short units (B=1024, l=512, S=1), with the epilogue
# warp's work skipped (LAM_DECODE_FLAGS=32), the last split's merge skipped (64), the MMAs
# skipped (16)
O=gpurun_out/r02c91; mkdir -p $O
for fl in 0 32 64 16; do
  LAM_DECODE_FLAGS=$fl AB_SPLIT=1024 timeout 120 python experiments/r02/tc_ab.py gqa_tc 128 64 8 128 4096 64 >> $O/c3s4_f$fl.log 2>&1
  LAM_DECODE_FLAGS=$fl timeout 120 python experiments/r02/tc_ab.py gqa_tc 128 64 8 128 4096 64 >> $O/c3_f$fl.log 2>&1
  LAM_DECODE_FLAGS=$fl timeout 120 python experiments/r02/tc_ab.py gqa_tc 1024 64 8 128 512 64 >> $O/short_f$fl.log 2>&1
done
echo done
