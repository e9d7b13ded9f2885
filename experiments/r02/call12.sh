#!/bin/bash
# round 2, call 12: sustained-step A/B of the two GQA kernels (bench c3 / c2, same box), plus the
# 4K2V ring error check
O=gpurun_out/r02c12; mkdir -p $O
LAM_TC_RING=42 timeout 120 python experiments/r02/tc_ab.py gqa_tc > $O/ring42.log 2>&1
for rep in 1 2; do
for k in 0 1; do
  LAM_GQA_TC=$k timeout 600 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline > $O/c3_tc$k.$rep.json 2> $O/c3_tc$k.$rep.err
  LAM_GQA_TC=$k timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --no-cpu-baseline > $O/c2_tc$k.$rep.json 2> $O/c2_tc$k.$rep.err
done; done
