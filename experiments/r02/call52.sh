#!/bin/bash
# round 2, call 52 (1 GPU): where does the tcgen05 kernel's per-item cost come from? split sweep
# with and without the MMAs (LAM_DECODE_FLAGS=16: pipeline only), with claim records
O=gpurun_out/r02c52; mkdir -p $O
for fl in 0 16; do
for st in 4096 1024; do
  LAM_DECODE_FLAGS=$fl LAM_BENCH_SPLIT_TOKENS=$st timeout 300 python bench.py --workload c3 --steps 5 --warmup 3 --launch layer --no-cpu-baseline --no-e2e --check 0 > $O/f${fl}_s$st.json 2> $O/f${fl}_s$st.err
done
done
