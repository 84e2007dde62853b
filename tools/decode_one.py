"""A few decode launches at one configuration (for ncu): python tools/decode_one.py 64 544"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import kernel_bench as kb  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 544
print(kb.decode_point(B, ctx, 40, 128, layers=4, reps=1))
