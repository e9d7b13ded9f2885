#!/bin/bash
O=gpurun_out/r02c35; mkdir -p $O
timeout 120 python experiments/r02/eager_debug.py > $O/debug.log 2>&1
