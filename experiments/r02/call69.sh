#!/bin/bash
# round 2, call 69 (2 GPUs): NVLink bytes of a peer launch (single process, rows on the other GPU)
O=gpurun_out/r02c69; mkdir -p $O
timeout 300 python experiments/r02/peer_nvlink.py > $O/plain.json 2> $O/plain.err && \
timeout 600 ncu --clock-control none -k regex:decode_gqa -c 1 --csv \
  --metrics nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  python experiments/r02/peer_nvlink.py > $O/ncu.csv 2> $O/ncu.err
