#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over a GPU parity subset (under
# gpurun). K selects the tests (pytest -k expression).
O=gpurun_out
mkdir -p $O
K=${K:-"config1 or work_stealing or tail_band or many_heads or push or chunked_prefill_parity or dynamic or item_space or early_kv"}
for tool in memcheck racecheck synccheck; do
  echo "== compute-sanitizer --tool $tool (tests/test_gpu_parity.py -k \"$K\")" >> $O/sanitizers.txt
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "$K" \
    > $O/san_$tool.log 2>&1
  grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY" $O/san_$tool.log | tail -3 >> $O/sanitizers.txt
done
cat $O/sanitizers.txt
