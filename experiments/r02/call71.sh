#!/bin/bash
# round 2, call 71 (1 GPU): final validation of the committed state
O=gpurun_out/r02c71; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q -rs > $O/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
