#!/bin/bash
# vectorised epilogue (acq_rel publish, padded partial rows) vs the previous build, same box
mkdir -p gpurun_out
exec > gpurun_out/call54.log 2>&1
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_reference_api_gpu.py tests/test_peer_gpu.py -x -q 2>&1 | tail -2
for R in 1 2; do
for h in cur ep; do
  (cd ab/$h && for C in c2 c3 c5 c3n8 c1; do PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg $C --splits 0 --iters 30 2>&1 | grep -v Warn | sed "s/^/$h /"; done)
  (cd ab/$h && PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg c3 --splits 2048,1024 --iters 30 2>&1 | grep -v Warn | sed "s/^/$h /")
  (cd ab/$h && PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg c3n8 --splits 2048 --iters 30 2>&1 | grep -v Warn | sed "s/^/$h /")
  (cd ab/$h && PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg c4 --splits 32768,8192 --iters 30 2>&1 | grep -v Warn | sed "s/^/$h /")
done
done
cd ab/ep; LAM_DECODE_FLAGS=32 PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg c3 --splits 4096,1024 --iters 30 2>&1 | grep -v Warn | sed "s/^/ep-noepi /"
