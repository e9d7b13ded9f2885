#!/bin/bash
# round 2, call 6: bisect the tcgen05 parity failure (K release after S vs after O)
O=gpurun_out/r02c06; mkdir -p $O
for f in 0 64; do echo "flags=$f" >> $O/probe.log; LAM_DECODE_FLAGS=$f timeout 120 python experiments/r02/tc_probe.py parity >> $O/probe.log 2>&1; done
