#!/bin/bash
# round 2, call 21: batched page-table lookups in the producer: per-layer and step launches, and a
# quick parity run of the decode tests
O=gpurun_out/r02c21; mkdir -p $O
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_step_gpu.py -q -x -p no:cacheprovider -m "gpu and not slow" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for wl in c3 c2; do for ln in step layer; do
  timeout 600 python bench.py --workload $wl --launch $ln --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/${wl}_${ln}.json 2> $O/${wl}_${ln}.err
done; done
