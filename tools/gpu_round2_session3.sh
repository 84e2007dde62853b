#!/bin/bash
# Round-2 (third session) evidence on one B200 with the final kernels: every GPU test,
# smoke, the default bench line, config 3/4/5 lines, the ncu launch list of one bench
# step and one ncu --set full capture of the decode kernel (DRAM bytes per launch).
set -x
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/s3_gpu_tests.log 2>&1; tail -2 $O/s3_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/s3_smoke.log 2>&1; tail -1 $O/s3_smoke.log
timeout 600 python bench.py > $O/s3_bench.json 2> $O/s3_bench.err; head -c 300 $O/s3_bench.json
for c in 3 4 5; do
  timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > $O/s3_bench_c$c.json 2> $O/s3_bench_c$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/s3_launches.csv \
  python bench.py --profile > $O/s3_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 \
  -o $O/s3_prof_decode_kernel python bench.py --profile > $O/s3_ncu_decode.log 2>&1
ls -la $O | grep s3_
