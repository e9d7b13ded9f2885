#!/bin/bash
# in-kernel sequence numbers for the peer transport; planner defaults (RATE_SM 50, C_ITEM 2us)
mkdir -p gpurun_out
exec > gpurun_out/call34.log 2>&1
echo "== dist tests"
timeout 900 python -m pytest tests/test_dist_gpu.py -x -q 2>&1 | tail -4
run() {  # $1 transport, $2 workload, $3 sync
  LAM_PEER_SYNC=$3 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 2 --steps 10 --warmup 3 --workload $2 --no-cpu-baseline --transport $1 2>gpurun_out/err_$1_$2.log | grep "^{" | python -c "
import sys,json
d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', '$3', '$2', 'value',round(d['value']),'e2e',round(d['e2e']['value']),'ms',round(d['ms_per_step'],3),'kern',round(r['achieved']),'S',d['config'].get('splits'))"
  tail -2 gpurun_out/err_$1_$2.log
}
echo "== bench A/B"
for R in 1 2; do
  for C in c3 c2; do
    run nccl $C -
    run peer $C kernel
    run peer $C stream
  done
done
echo "== single GPU, new planner defaults"
for C in c1 c2 c3 c3n8 c4 c5; do
  PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg $C --splits 0 2>&1 | grep -v Warn
done
for C in c1 c2 c3 c4 c5; do
  timeout 600 python bench.py --workload $C --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "
import sys,json
d=json.loads(sys.stdin.read()); r=d['roofline']; print('bench', '$C', 'value',round(d['value']),'e2e',round(d['e2e']['value']),'ms',round(d['ms_per_step'],3),'kern',round(r['achieved']),'S',d['config'].get('splits'))"
done
