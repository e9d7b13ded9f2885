#!/bin/bash
# round 2 (session 3), call 81 (1 GPU): batched last-split merge (S = 16 C4@N=8 shape, C3 S = 4),
# zero-copy host I/O for one-layer steps (C1 e2e), GPU tests of the changed paths, C1 and C2
# bench lines, an ncu capture of one C1 launch
O=gpurun_out/r02c81; mkdir -p $O
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_step_gpu.py tests/test_peer_gpu.py -x -q > $O/tests.txt 2>&1
for rep in 1 2; do
  AB_SPLIT=2048 timeout 120 python experiments/r02/tc_ab.py gqa_tc 16 8 1 128 32768 64 >> $O/c4n8.log 2>&1
  AB_SPLIT=1024 timeout 120 python experiments/r02/tc_ab.py gqa_tc 128 64 8 128 4096 64 >> $O/c3s4.log 2>&1
  AB_SPLIT=4096 timeout 120 python experiments/r02/tc_ab.py gqa_tc 16 8 1 128 32768 64 >> $O/c4n8_s8.log 2>&1
done
timeout 300 python bench.py --workload c1 --steps 200 --warmup 10 --no-cpu-baseline > $O/c1_zc.json 2> $O/c1_zc.err
LAM_HOST_ZERO_COPY=0 timeout 300 python bench.py --workload c1 --steps 200 --warmup 10 --no-cpu-baseline --check 0 > $O/c1_staged.json 2> $O/c1_staged.err
LAM_DECODE_CTAS=148 timeout 300 python bench.py --workload c1 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --check 0 > $O/c1_148.json 2> $O/c1_148.err
timeout 600 python bench.py > $O/c2.json 2> $O/c2.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_simt -s 12 -c 1 -o $O/c1_simt python bench.py --workload c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --check 0 > $O/ncu_c1.log 2>&1
echo done
