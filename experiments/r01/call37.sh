#!/bin/bash
# bench C2 gap diagnosis; PDL-aware timing; N=1 engine vs plain; peer tests
mkdir -p gpurun_out
exec > gpurun_out/call37.log 2>&1
timeout 600 python -m pytest tests/test_peer_gpu.py -x -q 2>&1 | tail -3
PYTHONPATH=$PWD timeout 600 python scripts/exp_bench_c2.py --workload c2 2>&1 | grep -v Warn
PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg c2 --splits 0 2>&1 | grep -v Warn
b1() {  # $1 tag, rest: bench args
  tag=$1; shift
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" 2>gpurun_out/err_b1.log | grep "^{" | python -c "
import sys,json
d=json.loads(sys.stdin.read()); r=d['roofline']; print('N1', '$tag', 'value',round(d['value']),'e2e',round(d['e2e']['value']),'ms',round(d['ms_per_step'],3),'kern',round(r['achieved']),'alone',r.get('alone_launch_ms'),'S',d['config'].get('splits'))"
  tail -2 gpurun_out/err_b1.log
}
for C in c2 c3; do
  b1 plain --workload $C
  b1 engine --workload $C --engine peer --transport peer
done
run() {  # $1 transport, $2 workload
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 2 --steps 10 --warmup 3 --workload $2 --no-cpu-baseline --transport $1 2>gpurun_out/err_$1_$2.log | grep "^{" | python -c "
import sys,json
d=json.loads(sys.stdin.read()); r=d['roofline']; print('N2', '$1', '$2', 'value',round(d['value']),'e2e',round(d['e2e']['value']),'ms',round(d['ms_per_step'],3),'kern',round(r['achieved']),'alone',r.get('alone_launch_ms'),'S',d['config'].get('splits'))"
  tail -2 gpurun_out/err_$1_$2.log
}
for C in c3 c2; do
  run nccl $C
  run peer $C
done
