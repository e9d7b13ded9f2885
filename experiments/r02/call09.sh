#!/bin/bash
O=gpurun_out/r02c09; mkdir -p $O
timeout 120 python experiments/r02/tc_debug2.py > $O/debug2.log 2>&1
