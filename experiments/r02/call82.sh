#!/bin/bash
# round 2 (session 3), call 82 (1 GPU): same-box A/B of the batched last-split merge (new)
# against the per-head merge (experiments/r02/ab_merge_old), split launches and the unsplit C3
O=gpurun_out/r02c82; mkdir -p $O
LIB=paper_2405_01814_b200/lib/liblamina_attn.so
cp $LIB /tmp/new.so
for rep in 1 2; do
  for v in new old; do
    if [ $v = new ]; then cp /tmp/new.so $LIB; else cp experiments/r02/ab_merge_old/liblamina_attn.so $LIB; fi
    AB_SPLIT=2048 timeout 120 python experiments/r02/tc_ab.py gqa_tc 16 8 1 128 32768 64 >> $O/c4n8_$v.log 2>&1
    AB_SPLIT=1024 timeout 120 python experiments/r02/tc_ab.py gqa_tc 128 64 8 128 4096 64 >> $O/c3s4_$v.log 2>&1
    timeout 120 python experiments/r02/tc_ab.py gqa_tc 128 64 8 128 4096 64 >> $O/c3_$v.log 2>&1
  done
done
cp /tmp/new.so $LIB
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_simt -s 2 -c 1 -o $O/c1_simt python bench.py --workload c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --check 0 > $O/ncu_c1.log 2>&1
echo done
