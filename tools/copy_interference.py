"""Does a concurrent host->device copy slow the decode kernel? Times 40 layers
of ds_decode_attn (B=64, ctx 544, OPT-13B heads; graph replay) alone and while a
side stream copies pinned host memory into (a) one 1 GB device buffer over and
over, (b) 24 distinct 1 GB device buffers in turn."""
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_09670_b200 as ds  # noqa: E402

B, ctx, n, d, L = 64, 544, 40, 128, 40
pages_per = -(-(ctx + 2) // 16)
nb = B * pages_per + 8
cache = ds.KVCache.empty(L, nb, n, d)
cache.tensor.normal_()
pool = ds.Pool(nb)
tab = np.full((B, pages_per), -1, np.int32)
ds.ds_block_table(pool, ds.DS_BT_APPEND, [0] * B, [ctx + 1] * B, tab)
tab_d = torch.from_numpy(tab).cuda()
cl = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
q = torch.randn((L, B, n, d), device="cuda", dtype=torch.bfloat16)
out = torch.empty((B, n, d), device="cuda", dtype=torch.bfloat16)
ws = torch.zeros(ds.ds_decode_workspace_bytes(B, n, d, ctx), dtype=torch.uint8, device="cuda")


def run():
    for l in range(L):
        ds.ds_decode_attn(q[l], q[l], q[l], out, cache, l, tab_d, cl, ctx, 1 / math.sqrt(d), ws)


run()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    run()
torch.cuda.synchronize()
GB = 1 << 30
host = torch.empty(GB // 2, dtype=torch.bfloat16).pin_memory()
bufs = [torch.empty(GB // 2, dtype=torch.bfloat16, device="cuda") for _ in range(24)]
cs = torch.cuda.Stream()


def timed(mode, reps=20):
    torch.cuda.synchronize()
    if mode != "alone":
        with torch.cuda.stream(cs):
            for i in range(40):  # ~0.8 s of copies, longer than the decode loop
                dst = bufs[0] if mode == "same_buffer" else bufs[i % len(bufs)]
                dst.copy_(host, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / L * 1e3


for mode in ("alone", "same_buffer", "24_buffers", "alone"):
    print(json.dumps({"mode": mode, "decode_us_per_layer": timed(mode)}), flush=True)
