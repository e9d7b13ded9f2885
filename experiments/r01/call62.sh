#!/bin/bash
# final single-GPU set: all GPU tests, smoke, every bench line (driver defaults), reference arm,
# ncu launch list + full capture of the default command
mkdir -p gpurun_out
exec > gpurun_out/call62.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for W in c2 c3 c4 c5 c1; do
  timeout 600 python bench.py --workload $W > gpurun_out/b62_$W.json 2>/dev/null; echo "bench $W rc=$?"
done
timeout 900 python bench.py --impl reference > gpurun_out/b62_ref.json 2>/dev/null; echo "ref rc=$?"
PROF_TAG=r01b_c2final PROF_KERNEL=decode_gqa BENCH_ARGS="--workload c2 --steps 2 --warmup 3" bash scripts/gpu_prof.sh
PROF_TAG=r01b_c1final PROF_KERNEL=decode_simt BENCH_ARGS="--workload c1 --steps 4 --warmup 3" bash scripts/gpu_prof.sh
timeout 600 python bench.py > gpurun_out/b62_c2_again.json 2>/dev/null; echo "bench c2 again rc=$?"
