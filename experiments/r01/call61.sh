#!/bin/bash
# 2 GPUs: peer launches stream their first KV tiles before the inputs' sequence numbers arrive
# (LAM_PEER_PREFETCH=1, default) vs after (0); tests first
mkdir -p gpurun_out
exec > gpurun_out/call61.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "decode or dist or peer or request" 2>&1 | tail -2
for R in 1 2; do
  for W in c2 c3; do
    for F in 0 1; do
      LAM_PEER_PREFETCH=$F timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --workload $W --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('prefetch$F $W', round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
    done
  done
done
