#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/mg_ab.log 2>&1
run() {  # $1 tag, $2 dir, $3 workload, $4 flags
  (cd $2 && LAM_DECODE_FLAGS=$4 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 --workload $3 --no-cpu-baseline --no-e2e 2>/dev/null) | grep "^{" | python -c "
import sys,json
d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', '$3', 'value',round(d['value']),'ms',round(d['ms_per_step'],3),'kern',round(r['achieved']),'launch_ms',round(r['avg_launch_ms'],4),'S',d['config']['splits'])"
}
for R in 1 2; do
run OLD $PWD/ab_old c3 0
run NEW $PWD c3 0
run NEWdyn $PWD c3 4
run OLD $PWD/ab_old c2 0
run NEW $PWD c2 0
run NEWdyn $PWD c2 4
done
