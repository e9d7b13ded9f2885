#!/bin/bash
# round 2, call 17: step launch vs per-layer launches, N=1, same box (c2, c3, c5; local and engine)
O=gpurun_out/r02c17; mkdir -p $O
for rep in 1 2; do
for wl in c2 c3 c5; do for ln in step layer; do
  timeout 600 python bench.py --workload $wl --launch $ln --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/${wl}_${ln}.$rep.json 2> $O/${wl}_${ln}.$rep.err
done; done; done
timeout 600 python bench.py --workload c3 --engine peer --launch step --steps 10 --warmup 3 --no-cpu-baseline > $O/c3_engine_step.json 2> $O/c3_engine_step.err
