#!/bin/bash
# round 2 (session 3), call 86 (1 GPU): static item bounds read while the slot is acquired;
# C1 on the full grid.  C1 lines, decode / step tests, C2 line, ncu of one C1 launch + launch list
O=gpurun_out/r02c86; mkdir -p $O
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_step_gpu.py tests/test_peer_gpu.py tests/test_bench_gpu.py -x -q > $O/tests.txt 2>&1
for rep in 1 2 3; do
  timeout 300 python bench.py --workload c1 --steps 200 --warmup 10 > $O/c1_$rep.json 2> $O/c1_$rep.err
done
timeout 600 python bench.py > $O/c2.json 2> $O/c2.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c1_launches.csv python bench.py --workload c1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --check 0 > $O/ncu_launches.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_simt -s 3 -c 1 -o $O/c1_simt python bench.py --workload c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --check 0 > $O/ncu_c1.log 2>&1
echo done
