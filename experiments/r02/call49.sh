#!/bin/bash
# round 2, call 49 (1 GPU): per-item cost of the tcgen05 kernel: c3 per-layer launches with
# forced split sizes (4096 = one item per (request, kv head))
O=gpurun_out/r02c49; mkdir -p $O
for st in 4096 2048 1024 512; do
  LAM_BENCH_SPLIT_TOKENS=$st timeout 300 python bench.py --workload c3 --steps 5 --warmup 3 --launch layer --no-cpu-baseline --no-e2e --check 0 > $O/s$st.json 2> $O/s$st.err
done
for r in 33 24 42; do
  LAM_TC_RING=$r LAM_BENCH_SPLIT_TOKENS=1024 timeout 300 python bench.py --workload c3 --steps 5 --warmup 3 --launch layer --no-cpu-baseline --no-e2e --check 0 > $O/s1024_r$r.json 2> $O/s1024_r$r.err
done
