#!/bin/bash
# round 2, call 37: compute-sanitizer memcheck over the small cases of every decode path
O=gpurun_out/r02c37; mkdir -p $O
timeout 600 python experiments/r02/sanitize_cases.py > $O/plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 50 python experiments/r02/sanitize_cases.py > $O/memcheck.log 2>&1; echo "rc=$?" >> $O/memcheck.log
