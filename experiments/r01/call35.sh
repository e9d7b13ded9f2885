#!/bin/bash
# why is the bench's C2 kernel slower than exp_decode's?  same-box A/B
mkdir -p gpurun_out
exec > gpurun_out/call35.log 2>&1
b() {  # $1 tag, rest: bench args
  tag=$1; shift
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | grep "^{" | python -c "
import sys,json
d=json.loads(sys.stdin.read()); r=d['roofline']; print('bench', '$tag', 'value',round(d['value']),'ms',round(d['ms_per_step'],3),'kern',round(r['achieved']),'S',d['config'].get('splits'), 'res', d['config']['kv_layers_resident'])"
}
for R in 1 2; do
  PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg c2 --splits 0 2>&1 | grep -v Warn
  PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg c2 --splits 0 --fused 2>&1 | grep -v Warn | sed "s/^/fused /"
  b c2fused --workload c2
  b c2sep --workload c2 --separate-append
  PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg c3 --splits 0 2>&1 | grep -v Warn
  PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg c3 --splits 0 --fused 2>&1 | grep -v Warn | sed "s/^/fused /"
  b c3fused --workload c3
  b c3sep --workload c3 --separate-append
done
