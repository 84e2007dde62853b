#!/bin/bash
# A/B of decode kernel variants on one B200 (under gpurun): decode sweeps (B = 1..256
# at 544 tokens, 8-layer CUDA graphs with early KV) of the product build and of each
# ab/<name> build given as arguments, repeated REPS times interleaved; then the decode
# GPU parity tests against each variant in TEST_VARIANTS (library swapped in place).
set -x
O=gpurun_out
mkdir -p $O
for r in $(seq 1 ${REPS:-2}); do
  timeout 300 python tools/kernel_bench.py --what decode > $O/kbd_base_$r.jsonl 2>&1
  for v in "$@"; do
    DS_PKG_ROOT=ab/$v timeout 300 python tools/kernel_bench.py --what decode > $O/kbd_${v}_$r.jsonl 2>&1
  done
done
cp paper_2401_09670_b200/libds.so /tmp/libds_base.so
for v in ${TEST_VARIANTS:-}; do
  cp ab/$v/paper_2401_09670_b200/libds.so paper_2401_09670_b200/libds.so
  timeout 900 python -m pytest tests -m gpu -q -x -k "decode or bench_step or end_to_end or config1" > $O/tests_$v.log 2>&1
  tail -2 $O/tests_$v.log
done
cp /tmp/libds_base.so paper_2401_09670_b200/libds.so
