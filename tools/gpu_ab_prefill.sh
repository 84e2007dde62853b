#!/bin/bash
# A/B of prefill kernel variants on one B200 (under gpurun): kernel sweeps of the
# product build and of each ab/<name> build given as arguments, then the prefill
# GPU parity tests against each variant's library (swapped in place; TEST_VARIANTS
# limits which).
set -x
O=gpurun_out
mkdir -p $O
[ -x tools/mma_smem_bench ] && timeout 120 tools/mma_smem_bench > $O/mma_smem.txt 2>&1
timeout 300 python tools/kernel_bench.py --what prefill > $O/kb_base.jsonl 2>&1
timeout 200 python tools/pf_mix_probe.py > $O/mix_base.txt 2>&1
for v in "$@"; do
  DS_PKG_ROOT=ab/$v timeout 300 python tools/kernel_bench.py --what prefill > $O/kb_$v.jsonl 2>&1
  DS_PKG_ROOT=ab/$v timeout 200 python tools/pf_mix_probe.py > $O/mix_$v.txt 2>&1
done
cp paper_2401_09670_b200/libds.so /tmp/libds_base.so
for v in ${TEST_VARIANTS:-$@}; do
  cp ab/$v/paper_2401_09670_b200/libds.so paper_2401_09670_b200/libds.so
  timeout 900 python -m pytest tests -m gpu -q -x -k "prefill or config1 or bench_step or end_to_end" > $O/tests_$v.log 2>&1
  tail -2 $O/tests_$v.log
done
cp /tmp/libds_base.so paper_2401_09670_b200/libds.so
