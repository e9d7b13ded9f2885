#!/bin/bash
mkdir -p gpurun_out
CMD="python scripts/exp_decode.py --cfg c3 --splits 1024 --iters 3"
timeout 300 $CMD > gpurun_out/p11_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_gqa -s 4 -c 1 -o gpurun_out/prof_c3s4 $CMD > gpurun_out/p11_ncu.log 2>&1
echo "rc=$?"
