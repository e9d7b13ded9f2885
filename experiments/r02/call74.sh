#!/bin/bash
# round 2, call 74 (2 GPUs): primed timed region: C1 (20 and 200 steps), C2 default, a 2-rank
# C3 line, the bench self-check tests
O=gpurun_out/r02c74; mkdir -p $O
timeout 600 python bench.py --workload c1 > $O/c1.json 2> $O/c1.err
timeout 600 python bench.py --workload c1 --steps 200 --warmup 10 > $O/c1_200.json 2> $O/c1_200.err
timeout 600 python bench.py > $O/c2.json 2> $O/c2.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus 2 --workload c3 --steps 5 --warmup 3 --no-cpu-baseline > $O/c3n2.json 2> $O/c3n2.err
timeout 900 python -m pytest tests/test_bench_gpu.py -x -q > $O/tests.txt 2>&1
