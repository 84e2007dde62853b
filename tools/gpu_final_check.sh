#!/bin/bash
# End-of-round check on one B200 (under gpurun): every GPU test, smoke(), the default
# bench line and the reference arm, with the final code.
set -x
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/final_gpu_tests.log 2>&1; tail -3 $O/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/final_smoke.log 2>&1; tail -2 $O/final_smoke.log
timeout 600 python bench.py > $O/final_bench.json 2> $O/final_bench.err; cat $O/final_bench.json
timeout 600 python bench.py --impl reference > $O/final_bench_ref.json 2> $O/final_bench_ref.err; cat $O/final_bench_ref.json
