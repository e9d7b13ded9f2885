#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/call39.log 2>&1
timeout 600 python -m pytest tests/test_peer_gpu.py -x -q 2>&1 | tail -30
PYTHONPATH=$PWD timeout 900 python scripts/exp_bench_c2.py --workload c2 2>&1 | grep -v Warn
PYTHONPATH=$PWD timeout 900 python scripts/exp_bench_c2.py --workload c3 2>&1 | grep -v Warn
