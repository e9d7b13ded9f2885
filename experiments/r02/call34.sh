#!/bin/bash
# round 2, call 34: eager q — tests and the per-layer latency experiment
O=gpurun_out/r02c34; mkdir -p $O
timeout 600 python -m pytest tests/test_peer_gpu.py tests/test_step_gpu.py -q -p no:cacheprovider -rf > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python experiments/r02/eager_latency.py > $O/eager.log 2>&1
