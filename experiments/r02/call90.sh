#!/bin/bash
# round 2 (session 3), call 90 (1 GPU): re-verify the MHA kernel choice on C2 after the SIMT
# re-tune (tcgen05 default vs SIMT variant 0 vs SIMT variant 7, LAM_MHA_MMA=0), same box,
# sustained steps; C1 split tails with the fp32 variant 7
O=gpurun_out/r02c90; mkdir -p $O
c2() {
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --check 0 > $O/c2_$tag.json 2> $O/c2_$tag.err
}
for rep in 1 2; do
  c2 tc_$rep
  c2 simt0_$rep LAM_MHA_MMA=0
  c2 simt7_$rep LAM_MHA_MMA=0 LAM_SIMT_VARIANT=7
done
c1() {
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --workload c1 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --check 0 > $O/c1_$tag.json 2> $O/c1_$tag.err
}
for rep in 1 2; do
  c1 base_$rep
  c1 tail2_$rep LAM_TAIL_UNITS=108 LAM_TAIL_SPLITS=2
  c1 tail4_$rep LAM_TAIL_UNITS=108 LAM_TAIL_SPLITS=4
done
echo done
