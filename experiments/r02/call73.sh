#!/bin/bash
# round 2, call 73 (1 GPU): K/V ring split of the tcgen05 kernel for short-item C5 vs C3
O=gpurun_out/r02c73; mkdir -p $O
for rep in 1 2; do
for r in 33 42 24; do
  for w in c5 c3; do
    LAM_TC_RING=$r timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --check 0 > $O/${w}_r${r}_$rep.json 2> $O/${w}_r${r}_$rep.err
  done
done
done
