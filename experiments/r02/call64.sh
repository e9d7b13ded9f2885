#!/bin/bash
# round 2, call 64 (1 GPU): final validation of the committed state: the GPU test suite, smoke,
# the default bench line, the reference arm, C1-C5 lines
O=gpurun_out/r02c64; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
for w in c3 c4 c5; do timeout 600 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 600 python bench.py --workload c1 --steps 200 --warmup 10 > $O/bench_c1.json 2> $O/bench_c1.err
