#!/bin/bash
# round 2 (session 3), call 85 (2 GPUs): static first item per CTA (no claim before a launch's
# first loads) + fp32 MHA variant 7 default: full GPU suite, C1 / C2 / C3 / C5 lines, C3 at N=2
O=gpurun_out/r02c85; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1
timeout 300 python bench.py --workload c1 --steps 200 --warmup 10 > $O/c1.json 2> $O/c1.err
timeout 600 python bench.py > $O/c2.json 2> $O/c2.err
for w in c3 c4 c5; do timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > $O/$w.json 2> $O/$w.err; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --workload c3 --steps 10 --warmup 3 --no-cpu-baseline > $O/c3n2.json 2> $O/c3n2.err
echo done
