#!/bin/bash
# round 2 (session 3), call 92 (1 GPU): two epilogue warps in the tcgen05 kernel (one per
# hand-off buffer).  Same launches as call 91 (C3 S=4 / S=1, 8192 short units, C4@N=8 shape),
# tests of the tcgen05 paths, C2 / C3 / C5 step lines
O=gpurun_out/r02c92; mkdir -p $O
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_step_gpu.py tests/test_peer_gpu.py -x -q > $O/tests.txt 2>&1
for rep in 1 2; do
  AB_SPLIT=1024 timeout 120 python experiments/r02/tc_ab.py gqa_tc 128 64 8 128 4096 64 >> $O/c3s4.log 2>&1
  timeout 120 python experiments/r02/tc_ab.py gqa_tc 128 64 8 128 4096 64 >> $O/c3.log 2>&1
  timeout 120 python experiments/r02/tc_ab.py gqa_tc 1024 64 8 128 512 64 >> $O/short.log 2>&1
  timeout 120 python experiments/r02/tc_ab.py gqa_tc 16 8 1 128 32768 64 >> $O/c4n8.log 2>&1
  AB_SPLIT=2048 timeout 120 python experiments/r02/tc_ab.py gqa_tc 16 8 1 128 32768 64 >> $O/c4n8_s16.log 2>&1
done
timeout 600 python bench.py --no-cpu-baseline > $O/c2.json 2> $O/c2.err
for w in c3 c5; do timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > $O/$w.json 2> $O/$w.err; done
echo done
