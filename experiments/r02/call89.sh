#!/bin/bash
# round 2 (session 3), call 89 (4 GPUs): validation of the committed state — GPU suite (dist
# tests at 2 and 4 ranks), default line + reference arm, C1, C3 / C4 / C5 strong at N=4, and the
# C4@N=8-shaped launch with the planner's split choice
O=gpurun_out/r02c89; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
timeout 600 python bench.py > $O/c2.json 2> $O/c2.err
timeout 600 python bench.py --impl reference > $O/c2_reference.json 2> $O/c2_reference.err
timeout 300 python bench.py --workload c1 --steps 200 --warmup 10 > $O/c1.json 2> $O/c1.err
for w in c3 c4 c5; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2954${w:1:1} bench.py --gpus 4 --workload $w --steps 10 --warmup 3 --no-cpu-baseline > $O/${w}n4.json 2> $O/${w}n4.err
done
for sp in 0 2048 4096; do
  AB_SPLIT=$sp timeout 120 python experiments/r02/tc_ab.py gqa_tc 16 8 1 128 32768 64 >> $O/c4n8_split$sp.log 2>&1
done
timeout 120 python experiments/r02/tc_ab.py gqa_tc 128 64 8 128 4096 64 >> $O/c3_unsplit.log 2>&1
echo done
