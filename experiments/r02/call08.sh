#!/bin/bash
O=gpurun_out/r02c08; mkdir -p $O
timeout 120 python experiments/r02/tc_debug.py > $O/debug.log 2>&1
timeout 120 python experiments/r02/tc_probe.py parity > $O/probe.log 2>&1
