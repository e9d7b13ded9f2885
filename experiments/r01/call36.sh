#!/bin/bash
# programmatic dependent launch for the peer engine; C2 footprint question
mkdir -p gpurun_out
exec > gpurun_out/call36.log 2>&1
echo "== dist tests"
timeout 900 python -m pytest tests/test_dist_gpu.py -x -q 2>&1 | tail -4
echo "== single-GPU tests"
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_dist_gpu.py 2>&1 | tail -3
run() {  # $1 transport, $2 workload, $3 PDL
  LAM_PDL=$3 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 2 --steps 10 --warmup 3 --workload $2 --no-cpu-baseline --transport $1 2>gpurun_out/err_$1_$2.log | grep "^{" | python -c "
import sys,json
d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', 'pdl$3', '$2', 'value',round(d['value']),'e2e',round(d['e2e']['value']),'ms',round(d['ms_per_step'],3),'kern',round(r['achieved']),'S',d['config'].get('splits'))"
  tail -2 gpurun_out/err_$1_$2.log
}
echo "== bench A/B"
for R in 1 2; do
  for C in c3 c2; do
    run nccl $C 0
    run peer $C 1
    run peer $C 0
  done
done
echo "== footprint"
for NB in 2 8 32; do
  PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg c2 --splits 0 --nbuf $NB 2>&1 | grep -v Warn | sed "s/^/nbuf$NB /"
done
