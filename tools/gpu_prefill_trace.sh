#!/bin/bash
# Where a prefill item's time goes (under gpurun): role timelines of SM 0 from the
# -DDS_TRACE build (ab/trace), and SM-activity balance + tensor-pipe counters of one
# config-5 launch under ncu.
set -x
O=gpurun_out
mkdir -p $O
DS_PKG_ROOT=ab/trace timeout 300 python tools/trace_prefill.py 4x4096 > $O/trace_4x4096.txt 2>&1
DS_PKG_ROOT=ab/trace timeout 300 python tools/trace_prefill.py 8x1856 24 > $O/trace_8x1856_24.txt 2>&1
timeout 600 ncu --metrics sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_active.min,sm__cycles_elapsed.max,gpc__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.max,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:prefill_kernel -s 2 -c 1 --csv python tools/prefill_one.py c5 > $O/ncu_c5_balance.csv 2>&1
timeout 600 ncu --metrics sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_active.min,sm__cycles_elapsed.max,gpc__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.max,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:prefill_kernel -s 2 -c 1 --csv python tools/prefill_one.py 4x4096 > $O/ncu_4x4096_balance.csv 2>&1
