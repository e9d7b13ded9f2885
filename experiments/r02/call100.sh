#!/bin/bash
# round 2 (session 3), call 100 (1 GPU): the rebuilt in-tree library of the final commit — smoke,
# the decode / step GPU tests, the default bench line
O=gpurun_out/r02c100; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_step_gpu.py -x -q > $O/tests.txt 2>&1
timeout 600 python bench.py > $O/c2.json 2> $O/c2.err
echo done
