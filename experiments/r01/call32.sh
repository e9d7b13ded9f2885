#!/bin/bash
# restored 6dc8b57 scheduling: GPU tests + same-box A/B against b762168 (1 and 2 GPUs)
mkdir -p gpurun_out
exec > gpurun_out/call32.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for R in 1 2; do
  for C in c2 c3 c3n8 c4 c5; do
    PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg $C --splits 0 2>&1 | grep -v Warn | sed "s/^/CUR /"
    (cd ab/b762168 && PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg $C --splits 0 2>&1 | grep -v Warn | sed "s/^/OLD /")
  done
done
run() {  # $1 tag, $2 dir, $3 workload
  (cd $2 && timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 --workload $3 --no-cpu-baseline 2>/dev/null) | grep "^{" | python -c "
import sys,json
d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', '$3', 'value',round(d['value']),'e2e',round(d['e2e']['value']),'ms',round(d['ms_per_step'],3),'kern',round(r['achieved']),'S',d['config'].get('splits'))"
}
for R in 1 2; do
  for C in c2 c3; do
    run CUR $PWD $C
    run OLD $PWD/ab/b762168 $C
  done
done
