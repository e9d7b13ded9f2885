#!/bin/bash
# planner: even-round grid (ceil(items / k) CTAs) vs the previous build; split tail with the
# vectorised epilogue; one-GPU attention-worker engine vs plain launches
mkdir -p gpurun_out
exec > gpurun_out/call57.log 2>&1
timeout 600 python -m pytest tests/test_decode_gpu.py -x -q 2>&1 | tail -1
for R in 1 2; do
for h in ep plan; do
  (cd ab/$h && for C in c1 c2 c3 c4 c5 c3n8 c4n8; do PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg $C --splits 0 --iters 30 2>&1 | grep -v Warn | sed "s/^/$h /"; done)
done
done
cd ab/plan
for C in c3 c5; do
  for T in "148 2" "296 2"; do
    set -- $T
    LAM_TAIL_UNITS=$1 LAM_TAIL_SPLITS=$2 PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg $C --splits 0 --iters 30 2>&1 | grep -v Warn | sed "s/^/tail $1x$2 /"
  done
done
cd ../..
for W in c2 c3; do
  timeout 600 python bench.py --workload $W --no-cpu-baseline --no-e2e 2>/dev/null | cut -c1-200 | sed "s/^/plain $W /"
  timeout 600 python bench.py --workload $W --no-cpu-baseline --no-e2e --engine peer --transport peer 2>/dev/null | cut -c1-200 | sed "s/^/engine $W /"
done
