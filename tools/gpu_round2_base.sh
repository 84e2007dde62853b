set -x
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi0.txt
timeout 1200 python -m pytest tests -m gpu -q -x > $O/gpu_tests.log 2>&1; tail -3 $O/gpu_tests.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; cat $O/bench.json
timeout 600 python tools/kernel_bench.py --what prefill > $O/kb_prefill.jsonl 2>&1
timeout 300 python tools/pf_mix_probe.py > $O/pf_mix.txt 2>&1
