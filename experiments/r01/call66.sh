#!/bin/bash
# tensor-map L2 promotion (0 none / 2 128B / 3 256B, default) in the sustained (power-capped) step
mkdir -p gpurun_out
exec > gpurun_out/call66.log 2>&1
for R in 1 2; do
  for P in 3 0 2; do
    for W in c2 c3; do
      LAM_TMAP_PROMOTION=$P timeout 600 python bench.py --workload $W --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('promo$P $W', round(d['value']), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
    done
  done
done
