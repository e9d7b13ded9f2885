#!/bin/bash
# round 2, call 68 (1 GPU): release-only split / unit counting (acquire only by the last) vs the
# acq_rel build (experiments/r02/ab_old), same box
O=gpurun_out/r02c68; mkdir -p $O
LIB=paper_2405_01814_b200/lib/liblamina_attn.so
cp $LIB /tmp/new.so
for rep in 1 2; do
  for v in new old; do
    if [ $v = new ]; then cp /tmp/new.so $LIB; else cp experiments/r02/ab_old/liblamina_attn.so $LIB; fi
    for w in c4 c5; do
      timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --check 0 > $O/${w}_${v}_$rep.json 2> $O/${w}_${v}_$rep.err
    done
    LAM_BENCH_SPLIT_TOKENS=1024 timeout 300 python bench.py --workload c3 --launch layer --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --check 0 > $O/c3s1k_${v}_$rep.json 2> $O/c3s1k_${v}_$rep.err
    AB_SPLIT=2048 timeout 120 python experiments/r02/tc_ab.py gqa_tc 16 8 1 128 32768 64 >> $O/c4n8_${v}.log 2>&1
  done
done
cp /tmp/new.so $LIB
