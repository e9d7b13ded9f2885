#!/bin/bash
O=gpurun_out/r02c16; mkdir -p $O; rm -f $O/debug.log
for m in after cold; do timeout 120 python experiments/r02/step_debug.py auto $m >> $O/debug.log 2>&1; done
