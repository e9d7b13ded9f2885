#!/bin/bash
# round 2, call 19: ncu of the c3 step launch vs one per-layer launch (why is the step slower?)
O=gpurun_out/r02c19; mkdir -p $O
M=gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum,gpc__cycles_elapsed.max,sm__cycles_active.avg
timeout 900 ncu --metrics $M --clock-control none -k regex:decode_gqa --launch-skip 3 --launch-count 1 --csv --log-file $O/ncu_step.csv \
  python bench.py --workload c3 --launch step --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --check 0 > $O/step.log 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:decode_gqa --launch-skip 400 --launch-count 3 --csv --log-file $O/ncu_layer.csv \
  python bench.py --workload c3 --launch layer --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --check 0 > $O/layer.log 2>&1
