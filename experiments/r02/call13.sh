#!/bin/bash
# round 2, call 13: whole GPU suite with the tcgen05 kernel in the matrix and as the MHA default
O=gpurun_out/r02c13; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
