"""Decode launch floor: device time of ds_decode_attn for tiny problems (graph
replay of 8 layers), to expose fixed per-launch costs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import kernel_bench as kb  # noqa: E402

for B, ctx, n in ((1, 0, 1), (1, 15, 1), (1, 544, 1), (1, 544, 40), (4, 544, 40), (16, 544, 40), (64, 544, 40), (256, 544, 40)):
    print(json.dumps(kb.decode_point(B, ctx, n, 128, layers=8, reps=20)), flush=True)
