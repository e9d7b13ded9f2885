#!/bin/bash
# Final round-1 validation of the committed state: full -m gpu suite, smoke, default bench, reference arm.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/c67_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c67_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/c67_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/c67_smoke.log
timeout 600 python bench.py > gpurun_out/c67_bench.log 2>&1; echo "rc=$?" >> gpurun_out/c67_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/c67_ref.log 2>&1; echo "rc=$?" >> gpurun_out/c67_ref.log
tail -2 gpurun_out/c67_pytest.log; tail -1 gpurun_out/c67_smoke.log; tail -2 gpurun_out/c67_bench.log | cut -c1-400
