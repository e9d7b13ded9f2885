#!/bin/bash
# round 2 (session 3), call 84 (1 GPU): SIMT variants with NV 16-byte vectors per lane and row
# (7: 16 warps NV=2, 8: 8 warps NV=2, 9: 16 warps NV=4; 64-token fp32 tiles) vs 0 and 5 on C1;
# parity of each; C1 e2e with the best
O=gpurun_out/r02c84; mkdir -p $O
c1() {
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --workload c1 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --check 0 > $O/c1_$tag.json 2> $O/c1_$tag.err
}
for rep in 1 2; do
  for v in 0 5 7 8 9; do c1 v${v}_$rep LAM_SIMT_VARIANT=$v; done
  c1 v9c148_$rep LAM_SIMT_VARIANT=9 LAM_DECODE_CTAS=148
  c1 v7c148_$rep LAM_SIMT_VARIANT=7 LAM_DECODE_CTAS=148
done
for v in 7 9; do
  LAM_SIMT_VARIANT=$v timeout 600 python -m pytest tests/test_decode_gpu.py -x -q > $O/tests_v$v.txt 2>&1
  LAM_SIMT_VARIANT=$v LAM_MHA_MMA=0 timeout 600 python -m pytest tests/test_decode_gpu.py -x -q -k "not full_shape" > $O/tests_v${v}_mha16.txt 2>&1
done
echo done
