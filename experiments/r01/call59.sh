#!/bin/bash
# rescale skip (warp-uniform alpha == 1) vs base: kernel alone and sustained bench (power cap)
mkdir -p gpurun_out
exec > gpurun_out/call59.log 2>&1
timeout 600 python -m pytest tests/test_decode_gpu.py -x -q 2>&1 | tail -1
for h in base skip; do
  (cd ab/$h && for C in c2 c3 c5; do PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg $C --splits 0 --iters 30 2>&1 | grep -v Warn | sed "s/^/$h /"; done)
done
for R in 1 2; do
for h in base skip; do
  for W in c2 c3; do
    (cd ab/$h && timeout 600 python bench.py --workload $W --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$h $W', round(d['value']), 'kern', round(d['roofline']['achieved']), d['clocks']['sm_mhz'], d['clocks']['reasons'])")
  done
done
done
