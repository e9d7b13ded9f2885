#!/bin/bash
# overlap_prev (PDL: stream the first KV tiles while the previous layer drains): correctness, then
# bench A/B with --overlap-layers 0 / 1 on the same box
mkdir -p gpurun_out
exec > gpurun_out/call60.log 2>&1
timeout 600 python -m pytest tests/test_decode_gpu.py -x -q -k "overlap_prev" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_decode_gpu.py -x -q 2>&1 | tail -1
for R in 1 2; do
  for W in c2 c3 c1 c5; do
    for O in 0 1; do
      timeout 600 python bench.py --workload $W --no-cpu-baseline --no-e2e --overlap-layers $O 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ovl$O $W', round(d['value']), 'kern', round(d['roofline']['achieved']), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
    done
  done
done
