"""Cost of empty work items: the same 64 x 128-token prefill launched with
max_seqlen = 128 (1 q tile per sequence) and with a larger max_seqlen (the grid
then holds 15 empty q tiles per (sequence, head) that CTAs must skip)."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("DS_PKG_ROOT"):
    sys.path.insert(0, os.path.abspath(os.environ["DS_PKG_ROOT"]))
import paper_2401_09670_b200 as ds  # noqa: E402

B, l, n, d = 64, 128, 40, 128
T = B * l
q, k, v = (torch.randn((T, n, d), device="cuda", dtype=torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
pool = ds.Pool(B * 128 + 8)
cache = ds.KVCache.empty(1, B * 128 + 8, n, d)
tab = np.full((B, 128), -1, np.int32)
ds.ds_block_table(pool, ds.DS_BT_APPEND, [0] * B, [l] * B, tab)
tab_d = torch.from_numpy(tab).cuda()
cu = torch.arange(0, T + 1, l, dtype=torch.int32, device="cuda")
for maxl in (128, 512, 2048):
    f = lambda: ds.ds_prefill_attn(q, k, v, out, cu, maxl, cache, 0, tab_d, 1 / math.sqrt(d))  # noqa: E731
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"max_seqlen {maxl:5d}: {e0.elapsed_time(e1) / 20 * 1e3:8.1f} us  (grid {((maxl + 127) // 128) * n * B} items)")
