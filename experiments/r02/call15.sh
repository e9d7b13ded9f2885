#!/bin/bash
O=gpurun_out/r02c15; mkdir -p $O
timeout 600 python -m pytest tests/test_step_gpu.py -q -p no:cacheprovider -rf -x > $O/pytest_step.log 2>&1; echo "rc=$?" >> $O/pytest_step.log
