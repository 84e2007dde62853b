#!/bin/bash
# A/B of the pair-streaming decode kernel (DS_DEC_PAIRS=k: used when B*n >= k*SMs)
# against decode_kernel on one B200: decode sweeps, then the decode GPU tests with it on.
O=gpurun_out
mkdir -p $O
for r in 1 2; do
  timeout 300 python tools/kernel_bench.py --what decode > $O/kbp_base_$r.jsonl 2>&1
  DS_DEC_PAIRS=${PAIRS:-1} timeout 300 python tools/kernel_bench.py --what decode > $O/kbp_pairs_$r.jsonl 2>&1
done
DS_DEC_PAIRS=${PAIRS:-1} timeout 900 python -m pytest tests -m gpu -q -x -k "decode or bench_step or end_to_end or config1" > $O/tests_pairs.log 2>&1
tail -3 $O/tests_pairs.log
