#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/call38.log 2>&1
timeout 600 python -m pytest tests/test_peer_gpu.py -x -q 2>&1 | tail -30
PYTHONPATH=$PWD timeout 900 python scripts/exp_bench_c2.py --workload c2 2>&1 | grep -v Warn
nvidia-smi -q -d PERFORMANCE,CLOCK | head -60
run() {  # $1 tag, $2 workload, $3 split tokens
  LAM_BENCH_SPLIT_TOKENS=$3 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 2 --steps 10 --warmup 3 --workload $2 --no-cpu-baseline --transport peer 2>gpurun_out/err_$2.log | grep "^{" | python -c "
import sys,json
d=json.loads(sys.stdin.read()); r=d['roofline']; print('N2', '$1', '$2', 'value',round(d['value']),'e2e',round(d['e2e']['value']),'ms',round(d['ms_per_step'],3),'kern',round(r['achieved']),'alone',r.get('alone_launch_ms'),'S',d['config'].get('splits'), 'clocks', d['clocks'])"
  tail -2 gpurun_out/err_$2.log
}
b1() {  # $1 tag, $2 workload, $3 split tokens, rest
  tag=$1; C=$2; st=$3; shift 3
  LAM_BENCH_SPLIT_TOKENS=$st timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --workload $C "$@" 2>gpurun_out/err_b1.log | grep "^{" | python -c "
import sys,json
d=json.loads(sys.stdin.read()); r=d['roofline']; print('N1', '$tag', '$C', 'value',round(d['value']),'e2e',round(d['e2e']['value']),'ms',round(d['ms_per_step'],3),'kern',round(r['achieved']),'alone',r.get('alone_launch_ms'),'S',d['config'].get('splits'), 'clocks', d['clocks'])"
  tail -2 gpurun_out/err_b1.log
}
for R in 1 2; do
  run s_auto c3 0
  run s_1 c3 4096
  b1 engine_s1 c3 4096 --engine peer --transport peer
  b1 plain c3 0
  b1 plain c2 0
done
