"""One prefill configuration, a few launches (for ncu):
    python tools/prefill_one.py 4x4096        (B x l, 40 heads)
    python tools/prefill_one.py c5            (config 5: summarization mix, 24 heads)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import kernel_bench as kb  # noqa: E402
import synthetic as syn  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "4x4096"
if arg == "c5":
    print(kb.prefill_point([int(x) for x in syn.lengths_summarization(0, 8)[0]], 24, 128, reps=2, rot=2))
else:
    B, l = (int(x) for x in arg.split("x"))
    print(kb.prefill_point([l] * B, 40, 128, reps=2, rot=2))
