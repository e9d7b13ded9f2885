#!/bin/bash
# round 2, call 56 (1 GPU): same-box A/B of the double-buffered epilogue hand-off (new) against
# the single-buffered build (experiments/r02/ab_old), step benches and a C4@N=8-shaped launch
O=gpurun_out/r02c56; mkdir -p $O
LIB=paper_2405_01814_b200/lib/liblamina_attn.so
cp $LIB /tmp/new.so
for rep in 1 2; do
  for v in new old; do
    if [ $v = new ]; then cp /tmp/new.so $LIB; else cp experiments/r02/ab_old/liblamina_attn.so $LIB; fi
    for w in c3 c4 c5; do
      timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --check 0 > $O/${w}_${v}_$rep.json 2> $O/${w}_${v}_$rep.err
    done
    # C4 at N=8 (strong): one KV head, 16 rows per micro-batch launch, 32 K tokens, S=16 (2 K-token items)
    AB_SPLIT=2048 timeout 120 python experiments/r02/tc_ab.py gqa_tc 16 8 1 128 32768 64 >> $O/c4n8_${v}.log 2>&1
    timeout 120 python experiments/r02/tc_ab.py gqa_tc 128 64 8 128 4096 64 >> $O/c3_unsplit_${v}.log 2>&1
  done
done
cp /tmp/new.so $LIB
