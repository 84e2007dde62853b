#!/bin/bash
# Round-2 evidence on one B200 (under gpurun): every GPU test, the default bench line,
# the reference (oracle) arm, config 3/4/5 bench lines, the ncu launch list of one
# bench step, one ncu --set full capture per hot kernel at the bench configuration,
# and the kernel sweeps. Outputs in gpurun_out/ (summaries go to profiles/r02/).
set -x
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; tail -3 $O/gpu_tests.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; cat $O/bench.json
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
for c in 3 4 5; do
  timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > $O/bench_c$c.json 2> $O/bench_c$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv \
  python bench.py --profile > $O/launches.log 2>&1
for k in decode_kernel prefill_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o $O/prof_$k python bench.py --profile > $O/ncu_$k.log 2>&1
done
timeout 600 python tools/kernel_bench.py > $O/kb_all.jsonl 2>&1
timeout 300 python tools/pf_mix_probe.py > $O/mix.txt 2>&1
ls -la $O
