#!/bin/bash
# round 2, call 39: reference-API drop-in numbers next to the reference CPU code (same box), and
# the drop-in parity tests after the coalesced instance kernel
O=gpurun_out/r02c39; mkdir -p $O
timeout 600 python -m pytest tests/test_reference_api_gpu.py tests/test_benchmarks_gpu.py -q -p no:cacheprovider -rf > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 ./benchmarks/bench_attention_b200 > $O/bench_dropin.txt 2>&1
timeout 300 ./oracle/_ref/bench_attention_ref > $O/bench_reference_cpu.txt 2>&1
nproc > $O/nproc.txt; grep -m1 "model name" /proc/cpuinfo >> $O/nproc.txt
