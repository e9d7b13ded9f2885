#!/bin/bash
# host-buffer path synchronised by sequence numbers (no events between launches): tests, then
# e2e A/B with LAM_HOST_FLAGS=0 / 1 on the same box
mkdir -p gpurun_out
exec > gpurun_out/call63.log 2>&1
timeout 600 python -m pytest tests/test_decode_gpu.py -x -q -k "layers_host" 2>&1 | tail -3
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for R in 1 2; do
  for W in c2 c3 c1; do
    for F in 0 1; do
      LAM_HOST_FLAGS=$F timeout 600 python bench.py --workload $W --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('flags$F $W value', round(d['value']), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])"
    done
  done
done
