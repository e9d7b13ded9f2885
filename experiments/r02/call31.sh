#!/bin/bash
# round 2, call 31 (4 GPUs): step vs per-layer launches at N=4 for every workload (release-atomic
# unit counting); step tests
O=gpurun_out/r02c31; mkdir -p $O
timeout 600 python -m pytest tests/test_step_gpu.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
run() { local n=$1 np=$2; shift 2
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29520 bench.py --gpus $np "$@" --no-cpu-baseline --no-e2e --check 0 > $O/$n.json 2> $O/$n.err; }
for wl in c3 c2 c5 c4; do
  st=10; [ $wl = c4 -o $wl = c5 ] && st=5
  run ${wl}_step 4 --workload $wl --steps $st --warmup 2
  run ${wl}_layer 4 --workload $wl --steps $st --warmup 2 --launch layer
done
