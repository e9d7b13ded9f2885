#!/bin/bash
# round 2 (session 3), call 96 (2 GPUs): validation of the final committed state — GPU suite
# (dist tests at 2 ranks), smoke, default line + reference arm, C1, C3 / C4 / C5 one GPU and C4 at N=2
O=gpurun_out/r02c96; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 600 python bench.py > $O/c2.json 2> $O/c2.err
timeout 600 python bench.py --impl reference > $O/c2_reference.json 2> $O/c2_reference.err
timeout 300 python bench.py --workload c1 --steps 200 --warmup 10 > $O/c1.json 2> $O/c1.err
for w in c3 c4 c5; do timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > $O/$w.json 2> $O/$w.err; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --workload c4 --steps 10 --warmup 3 --no-cpu-baseline > $O/c4n2.json 2> $O/c4n2.err
echo done
