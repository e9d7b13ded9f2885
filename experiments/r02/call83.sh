#!/bin/bash
# round 2 (session 3), call 83 (1 GPU): fp32 SIMT variants with 64-token tiles (5: 16 warps,
# 6: 8 warps; 3 stages) against the default (32-token tiles, 6 stages) on C1; parity of each
O=gpurun_out/r02c83; mkdir -p $O
c1() {
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --workload c1 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --check 0 > $O/c1_$tag.json 2> $O/c1_$tag.err
}
for rep in 1 2; do
  c1 v0_$rep
  c1 v5_$rep LAM_SIMT_VARIANT=5
  c1 v6_$rep LAM_SIMT_VARIANT=6
  c1 v5c148_$rep LAM_SIMT_VARIANT=5 LAM_DECODE_CTAS=148
  c1 v6c148_$rep LAM_SIMT_VARIANT=6 LAM_DECODE_CTAS=148
  c1 v4_$rep LAM_SIMT_VARIANT=4
done
LAM_SIMT_VARIANT=5 timeout 600 python -m pytest tests/test_decode_gpu.py -x -q > $O/tests_v5.txt 2>&1
LAM_SIMT_VARIANT=6 timeout 600 python -m pytest tests/test_decode_gpu.py -x -q > $O/tests_v6.txt 2>&1
timeout 600 python -m pytest tests/test_decode_gpu.py -x -q -k "layers_host" > $O/tests_host.txt 2>&1
echo done
