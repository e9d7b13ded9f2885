#!/bin/bash
# round 2, call 20: is the step launch's loss tied to the span of pool layers? (resident 80 / 8 / 2)
O=gpurun_out/r02c20; mkdir -p $O
for res in 80 8 2; do for ln in step layer; do
  LAM_BENCH_RESIDENT=$res timeout 600 python bench.py --workload c3 --launch $ln --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --check 0 > $O/c3_${ln}_r$res.json 2> $O/c3_${ln}_r$res.err
done; done
