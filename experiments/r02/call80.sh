#!/bin/bash
# round 2 (session 3), call 80 (1 GPU): claim-ahead (LAM_CLAIM_AHEAD) A/B on C1, split-tail
# C1 grids, a C4@N=8-shaped tcgen05 launch and the unsplit C3 launch; decode tests with
# claim-ahead forced on
O=gpurun_out/r02c80; mkdir -p $O
c1() {  # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --workload c1 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --check 0 > $O/c1_$tag.json 2> $O/c1_$tag.err
}
for rep in 1 2; do
  c1 base_$rep
  c1 ca2_$rep LAM_CLAIM_AHEAD=2
  c1 ca6_$rep LAM_CLAIM_AHEAD=6
  c1 tail4_$rep LAM_TAIL_UNITS=108 LAM_TAIL_SPLITS=4 LAM_DECODE_CTAS=148
  c1 tail4ca_$rep LAM_TAIL_UNITS=108 LAM_TAIL_SPLITS=4 LAM_DECODE_CTAS=148 LAM_CLAIM_AHEAD=4
  c1 s4ca_$rep LAM_PLAN_CITEM_NS=100 LAM_CLAIM_AHEAD=4
done
for ca in 0 1 2 4; do
  LAM_CLAIM_AHEAD=$ca AB_SPLIT=2048 timeout 120 python experiments/r02/tc_ab.py gqa_tc 16 8 1 128 32768 64 >> $O/c4n8_ca$ca.log 2>&1
  LAM_CLAIM_AHEAD=$ca timeout 120 python experiments/r02/tc_ab.py gqa_tc 128 64 8 128 4096 64 >> $O/c3_ca$ca.log 2>&1
  LAM_CLAIM_AHEAD=$ca AB_SPLIT=1024 timeout 120 python experiments/r02/tc_ab.py gqa_tc 128 64 8 128 4096 64 >> $O/c3s4_ca$ca.log 2>&1
done
LAM_CLAIM_AHEAD=3 timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_step_gpu.py -x -q > $O/tests_ca3.txt 2>&1
echo done
