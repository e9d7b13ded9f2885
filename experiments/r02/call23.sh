#!/bin/bash
# round 2, call 23: step launches everywhere (tcgen05 default): GPU suite + N=1 bench lines with e2e
O=gpurun_out/r02c23; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for wl in c2 c3 c5 c4 c1; do
  timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --cpu-seconds 5 > $O/$wl.json 2> $O/$wl.err
done
