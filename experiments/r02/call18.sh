#!/bin/bash
O=gpurun_out/r02c18; mkdir -p $O
for wl in c3 c2; do for ln in step layer; do
  timeout 600 python bench.py --workload $wl --launch $ln --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/${wl}_${ln}.json 2> $O/${wl}_${ln}.err
done; done
