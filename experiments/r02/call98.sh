#!/bin/bash
# round 2 (session 3), call 98 (1 GPU): planner item cost for the tcgen05 kernel after the merge
# fix — LAM_PLAN_CITEM_MMA_NS 5000 (default) / 2000 / 1000 on C4, the C4@N=8 shape, C3, and the
# 512-unit sharded C3 launch (c3n8)
O=gpurun_out/r02c98; mkdir -p $O
for rep in 1 2; do
  for c in 5000 2000 1000; do
    export LAM_PLAN_CITEM_MMA_NS=$c
    timeout 120 python experiments/r02/tc_ab.py gqa_tc 32 64 8 128 32768 64 >> $O/c4_c$c.log 2>&1
    timeout 120 python experiments/r02/tc_ab.py gqa_tc 16 8 1 128 32768 64 >> $O/c4n8_c$c.log 2>&1
    timeout 120 python experiments/r02/tc_ab.py gqa_tc 128 64 8 128 4096 64 >> $O/c3_c$c.log 2>&1
    timeout 120 python experiments/r02/tc_ab.py gqa_tc 512 8 1 128 4096 64 >> $O/c3n8_c$c.log 2>&1
  done
done
unset LAM_PLAN_CITEM_MMA_NS
for c in 5000 2000 1000; do
  LAM_PLAN_CITEM_MMA_NS=$c python - >> $O/plans.txt 2>&1 <<'PY'
import os, sys, torch
sys.path.insert(0, ".")
from paper_2405_01814_b200 import decode as dec
c = os.environ["LAM_PLAN_CITEM_MMA_NS"]
for name, B, Hq, Hkv, L in (("c4", 32, 64, 8, 32768), ("c4n8", 16, 8, 1, 32768), ("c3", 128, 64, 8, 4096), ("c3n8", 512, 8, 1, 4096)):
    npg = B * L // 64
    kp = torch.empty((npg, Hkv, 64, 128), dtype=torch.bfloat16, device="cuda")
    q = torch.empty((B, Hq, 128), dtype=torch.bfloat16, device="cuda")
    pt = torch.arange(npg, dtype=torch.int32, device="cuda").view(B, L // 64)
    lens = torch.full((B,), L, dtype=torch.int32, device="cuda")
    print(c, name, dec.plan(q, kp, kp, lens, page_table=pt, max_len=L), dec.plan_grid(q, kp, kp, lens, page_table=pt, max_len=L))
PY
done
echo done
