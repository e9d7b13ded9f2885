#!/bin/bash
# re-entry verification: all GPU tests, smoke, default bench, C3/C4/C5/C1 bench lines
mkdir -p gpurun_out
exec > gpurun_out/call42.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for W in c2 c3 c4 c5 c1; do
  timeout 600 python bench.py --workload $W 2>&1 | grep '^{' | sed "s/^/$W /"
done
