#!/bin/bash
# L2 bulk prefetch of tiles ahead of the ring (LAM_L2_AHEAD = 0 / 2 / 4 / 8), same box
mkdir -p gpurun_out
exec > gpurun_out/call65.log 2>&1
LAM_L2_AHEAD=4 timeout 600 python -m pytest tests/test_decode_gpu.py -x -q 2>&1 | tail -1
for R in 1 2; do
  for A in 0 2 4 8; do
    for C in c3n8 c1 c3 c2 c4n8; do
      LAM_L2_AHEAD=$A PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg $C --splits 0 --iters 30 2>&1 | grep -v Warn | sed "s/^/A$A /"
    done
  done
done
for A in 0 4; do
  for W in c2 c3 c1; do
    LAM_L2_AHEAD=$A timeout 600 python bench.py --workload $W --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench A$A $W', round(d['value']), 'kern', round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"
  done
done
