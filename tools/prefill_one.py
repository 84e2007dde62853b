"""One prefill configuration, a few launches (for ncu): python tools/prefill_one.py 4x4096"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import kernel_bench as kb  # noqa: E402

B, l = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "4x4096").split("x"))
print(kb.prefill_point([l] * B, 40, 128, reps=2, rot=2))
