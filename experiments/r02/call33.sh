#!/bin/bash
# round 2, call 33 (1 GPU): C1 — ncu full capture of the decode launch now; split / grid variants
O=gpurun_out/r02c33; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_simt --launch-skip 10 --launch-count 1 -o $O/c1_full \
  python bench.py --workload c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --check 0 > $O/ncu.log 2>&1
for cfg in "0 0" "512 0" "256 0" "0 148" "256 148" "128 148"; do
  set -- $cfg
  LAM_BENCH_SPLIT_TOKENS=$1 LAM_DECODE_CTAS=$2 timeout 300 python bench.py --workload c1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/c1_s$1_c$2.json 2> $O/c1_s$1_c$2.err
done
