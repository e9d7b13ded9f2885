#!/bin/bash
# round 2, call 55 (1 GPU): double-buffered epilogue hand-off in the tcgen05 kernel
O=gpurun_out/r02c55; mkdir -p $O
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_step_gpu.py -x -q > $O/tests.txt 2>&1
for st in 4096 1024; do
  LAM_BENCH_SPLIT_TOKENS=$st timeout 300 python bench.py --workload c3 --steps 5 --warmup 3 --launch layer --no-cpu-baseline --no-e2e --check 0 > $O/s$st.json 2> $O/s$st.err
done
for w in c2 c3 c4 c5; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/$w.json 2> $O/$w.err
done
