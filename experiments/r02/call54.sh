#!/bin/bash
# round 2, call 54 (1 GPU): ncu source-level capture of the tcgen05 kernel, items of 1024 vs 4096
# tokens (c3 per-layer launches; the same command exited 0 without ncu in call 52)
O=gpurun_out/r02c54; mkdir -p $O
for st in 1024 4096; do
  LAM_BENCH_SPLIT_TOKENS=$st timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_gqa_tc --launch-skip 40 --launch-count 1 -f -o $O/tc_s$st python bench.py --workload c3 --steps 1 --warmup 3 --launch layer --no-cpu-baseline --no-e2e --check 0 > $O/ncu_s$st.log 2>&1
done
ls -la $O
