#!/bin/bash
# peer transport bring-up (2 GPUs) + planner constant sweep
mkdir -p gpurun_out
exec > gpurun_out/call33.log 2>&1
echo "== peer transport test"
for T in "peer 1 0" "peer 1 1"; do
  set -- $T
  LAM_TEST_TRANSPORT=$1 LAM_TEST_FUSED=$2 LAM_TEST_HOST=$3 PYTHONPATH=$PWD timeout 180 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 tests/dist_gpu_worker.py 2>&1 | grep -v Warn | tail -8
done
run() {  # $1 transport, $2 workload
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 2 --steps 10 --warmup 3 --workload $2 --no-cpu-baseline --transport $1 2>gpurun_out/err_$1_$2.log | grep "^{" | python -c "
import sys,json
d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', '$2', 'value',round(d['value']),'e2e',round(d['e2e']['value']),'ms',round(d['ms_per_step'],3),'kern',round(r['achieved']),'S',d['config'].get('splits'))"
  tail -3 gpurun_out/err_$1_$2.log
}
echo "== bench A/B"
for R in 1 2; do
  for C in c3 c2; do
    run nccl $C
    run peer $C
  done
done
echo "== planner sweep"
for K in "56 4000" "50 4000" "50 2000" "50 1000" "53 2000"; do
  set -- $K
  for C in c3 c3n8 c4 c5; do
    LAM_PLAN_RATE_SM=$1 LAM_PLAN_CITEM_NS=$2 PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg $C --splits 0 2>&1 | grep -v Warn | sed "s/^/$1 $2 /"
  done
done
for C in c4 c3n8; do
  PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg $C --splits 0,2048,4096,8192,16384 2>&1 | grep -v Warn | sed "s/^/forced /"
done
