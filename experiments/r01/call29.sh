#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/mg_sched.log 2>&1
for F in 0 4; do
  for WL in c3 c2; do
    LAM_DECODE_FLAGS=$F timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 --workload $WL --no-cpu-baseline --no-e2e 2>/dev/null | grep "^{" | python -c "
import sys,json
d=json.loads(sys.stdin.read()); r=d['roofline']; print('f$F', '$WL', 'value',round(d['value']),'ms',round(d['ms_per_step'],3),'kern',round(r['achieved']),'alone_ms',round(r['alone_launch_ms'],4),'launch_ms',round(r['avg_launch_ms'],4),'S',d['config']['splits'])"
  done
done
for F in 0 4; do LAM_DECODE_FLAGS=$F timeout 300 python scripts/exp_decode.py --cfg c2 --splits 0 | sed "s/^/f$F /"; done
