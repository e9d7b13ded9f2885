#!/bin/bash
mkdir -p gpurun_out
N=${NGPU:-2}
exec > gpurun_out/nccl_sweep.log 2>&1
for CH in default 1 2 4 8; do
  if [ $CH = default ]; then unset NCCL_MAX_NCHANNELS; else export NCCL_MAX_NCHANNELS=$CH; fi
  for WL in c3; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 10 --warmup 3 --workload $WL --no-cpu-baseline --no-e2e 2>/dev/null | grep "^{" | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('ch=$CH', '$WL', 'n$N', 'value',round(d['value']),'ms',round(d['ms_per_step'],3),'kern',round(d['roofline']['achieved']))"
  done
done
