#!/bin/bash
# round 2, call 70 (1 GPU): one host synchronisation per host-buffer instance call: the
# reference-API tests, the benchmark harness through the drop-in
O=gpurun_out/r02c70; mkdir -p $O
timeout 900 python -m pytest tests/test_reference_api_gpu.py tests/test_benchmarks_gpu.py tests/test_capi.py -x -q > $O/tests.txt 2>&1
timeout 600 benchmarks/bench_attention_b200 > $O/dropin_bench.txt 2>&1
