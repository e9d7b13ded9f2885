#!/bin/bash
# round 2, call 2: the whole GPU suite (no -x) after the checker fix; c5 bench line with check
O=gpurun_out/r02c02; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err; echo "c5 rc=$?" >> $O/rc.txt
