#!/bin/bash
# Round evidence on one B200 (run under gpurun): GPU tests, the default bench line,
# the reference (oracle) arm, the ncu launch list of one bench step and one
# ncu --set full capture per hot kernel at the bench configuration. Outputs in
# gpurun_out/; tools/summarize_round.sh turns them into profiles/<round>/.
set -x
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; tail -3 $O/gpu_tests.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; cat $O/bench.json
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; cat $O/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv \
  python bench.py --profile > $O/launches.log 2>&1
for k in decode_kernel prefill_kernel kv_local_kernel; do
  skip=3; [ $k = kv_local_kernel ] && skip=0
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
    -o $O/prof_$k python bench.py --profile > $O/ncu_$k.log 2>&1
done
ls -la $O
