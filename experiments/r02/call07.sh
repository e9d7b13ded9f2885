#!/bin/bash
O=gpurun_out/r02c07; mkdir -p $O
timeout 120 python experiments/r02/tc_debug.py > $O/debug.log 2>&1
