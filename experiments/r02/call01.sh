#!/bin/bash
# round 2, call 1: full GPU test suite (incl. new full-shape parity), bench lines with the output check
mkdir -p gpurun_out/r02c01
O=gpurun_out/r02c01
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for wl in c2 c1 c3; do
  timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 > $O/bench_$wl.json 2> $O/bench_$wl.err
  echo "$wl rc=$?" >> $O/rc.txt
done
