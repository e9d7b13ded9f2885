#!/bin/bash
# round 2, call 3: first run of the tcgen05 kernel (parity probe + C3-layer A/B vs mma.sync)
O=gpurun_out/r02c03; mkdir -p $O
timeout 300 python experiments/r02/tc_probe.py > $O/tc_probe.log 2>&1; echo "rc=$?" >> $O/tc_probe.log
nvidia-smi > $O/smi_after.txt 2>&1
