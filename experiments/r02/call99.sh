#!/bin/bash
# round 2 (session 3), call 99 (1 GPU): tcgen05 warp roles — second epilogue warp on scheduler 1
# and the producer on warp 8 (new) vs epilogue warps 6 / 8 (head, experiments/r02/ab_head);
# tests of the new build
O=gpurun_out/r02c99; mkdir -p $O
LIB=paper_2405_01814_b200/lib/liblamina_attn.so
cp $LIB /tmp/new.so
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_step_gpu.py tests/test_peer_gpu.py tests/test_bench_gpu.py -x -q > $O/tests.txt 2>&1
for rep in 1 2; do
  for v in new head; do
    if [ $v = new ]; then cp /tmp/new.so $LIB; else cp experiments/r02/ab_head/liblamina_attn.so $LIB; fi
    AB_SPLIT=1024 timeout 120 python experiments/r02/tc_ab.py gqa_tc 128 64 8 128 4096 64 >> $O/c3s4_$v.log 2>&1
    timeout 120 python experiments/r02/tc_ab.py gqa_tc 128 64 8 128 4096 64 >> $O/c3_$v.log 2>&1
    timeout 120 python experiments/r02/tc_ab.py gqa_tc 1024 64 8 128 512 64 >> $O/short_$v.log 2>&1
    for w in c2 c5; do timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --check 0 > $O/${w}_${v}_$rep.json 2> $O/${w}_${v}_$rep.err; done
  done
done
cp /tmp/new.so $LIB
echo done
