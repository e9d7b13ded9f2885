#!/bin/bash
# MHA on the tensor-core kernel (power-capped sustained runs); split tail; parity
mkdir -p gpurun_out
exec > gpurun_out/call40.log 2>&1
timeout 900 python -m pytest tests/test_decode_gpu.py -x -q -k "vs_oracle" 2>&1 | tail -3
for K in simt gqa_mma; do
  PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg c2 --splits 0 --kernels $K --iters 400 --warm 100 2>&1 | grep -v Warn | sed "s/^/sustained /"
  PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg c2 --splits 0 --kernels $K 2>&1 | grep -v Warn | sed "s/^/burst /"
done
LAM_MHA_MMA=0 timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "
import sys,json
d=json.loads(sys.stdin.read()); r=d['roofline']; print('bench simt', 'value',round(d['value']),'e2e',round(d['e2e']['value']),'kern',round(r['achieved']), d['clocks'])"
LAM_MHA_MMA=1 timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "
import sys,json
d=json.loads(sys.stdin.read()); r=d['roofline']; print('bench mma', 'value',round(d['value']),'e2e',round(d['e2e']['value']),'kern',round(r['achieved']), d['config']['kernel'], d['clocks'])"
echo "== split tail (sustained: 400 launches after 100 warm)"
for C in c2 c3 c3n8; do
  for T in "0 4" "74 4" "148 2" "148 4" "148 8" "296 4"; do
    set -- $T
    LAM_TAIL_UNITS=$1 LAM_TAIL_SPLITS=$2 PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg $C --splits 0 --iters 200 --warm 50 2>&1 | grep -v Warn | sed "s/^/tail $1 x$2 /"
  done
done
