#!/bin/bash
# ncu evidence for one bench command: plain run, launch list, then a full capture of the
# top kernel.  Usage: PROF_TAG=c2 PROF_KERNEL=decode_simt BENCH_ARGS="..." scripts/gpu_prof.sh
mkdir -p gpurun_out
TAG=${PROF_TAG:-c2}
CMD="python bench.py $BENCH_ARGS --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/prof_${TAG}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"${PROF_LIST_KERNELS:-decode|kv_append}" -c ${PROF_COUNT:-200} --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/prof_${TAG}_launches.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${PROF_KERNEL:-decode} -s ${PROF_SKIP:-8} -c 1 -o gpurun_out/prof_${TAG} $CMD > gpurun_out/prof_${TAG}_full.log 2>&1
echo "prof rc=$?"
