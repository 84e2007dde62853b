"""Decode launch timing under input-layout variants (A/B aid): python tools/decode_variants.py
Prints one JSON line per variant: kernel_bench's decode_point setup (8-layer graph, early KV) with
  base      : q = k_new = v_new one tensor, sequences' pages contiguous (APPEND whole sequences)
  qkv       : distinct q / k_new / v_new tensors
  interleave: pages allocated 16 tokens at a time for all sequences (ids interleaved across sequences)
  both      : qkv + interleave
  bigpool   : qkv, 40 layers and a pool twice the batch's pages (bench.py's footprint: ~120 GB)"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("DS_PKG_ROOT"):
    sys.path.insert(0, os.path.abspath(os.environ["DS_PKG_ROOT"]))
import numpy as np
import torch

import paper_2401_09670_b200 as ds


def run(B, ctx, n, d, qkv, interleave, layers=8, reps=5, nb_scale=1):
    pages_per = -(-(ctx + 2) // 16)
    nb = (B * pages_per + 8) * nb_scale
    cache = ds.KVCache.empty(layers, nb, n, d)
    cache.tensor.normal_()
    pool = ds.Pool(nb)
    tab = np.full((B, pages_per), -1, np.int32)
    if interleave:
        cur = [0] * B
        while cur[0] < ctx + 1:
            add = [min(16, ctx + 1 - c) for c in cur]
            ds.ds_block_table(pool, ds.DS_BT_APPEND, cur, add, tab)
            cur = [c + a for c, a in zip(cur, add)]
    else:
        ds.ds_block_table(pool, ds.DS_BT_APPEND, [0] * B, [ctx + 1] * B, tab)
    tab_d = torch.from_numpy(tab).cuda()
    cl = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
    q = torch.randn((layers, B, n, d), device="cuda", dtype=torch.bfloat16)
    kn = torch.randn_like(q) if qkv else q
    vn = torch.randn_like(q) if qkv else q
    out = torch.empty((B, n, d), device="cuda", dtype=torch.bfloat16)
    ws = torch.zeros(ds.ds_decode_workspace_bytes(B, n, d, ctx), dtype=torch.uint8, device="cuda")
    scale = 1 / math.sqrt(d)

    def chain():
        for l in range(layers):
            ds.ds_decode_attn(q[l], kn[l], vn[l], out, cache, l, tab_d, cl, ctx, scale, ws, early_kv=l > 0)

    chain()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        chain()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    if os.environ.get("DS_DECODE_TRACE_OUT"):  # -DDS_TRACE builds: the last launch's warp timeline
        import ctypes
        f = ctypes.CDLL(ds.LIB_PATH).ds_debug_decode_trace
        f.argtypes = [ctypes.c_void_p, ctypes.c_int]
        buf = np.zeros(f(None, 0), np.uint64)
        f(buf.ctypes.data, 0)
        np.save(os.environ["DS_DECODE_TRACE_OUT"] + f".{'qkv' if qkv else 'same'}{'_il' if interleave else ''}.npy", buf)
    return e0.elapsed_time(e1) / reps / layers * 1e3


if __name__ == "__main__":
    B, ctx = int(os.environ.get("B", 128)), int(os.environ.get("CTX", 544))
    variants = (("base", False, False, 8, 1), ("qkv", True, False, 8, 1), ("interleave", False, True, 8, 1),
                ("both", True, True, 8, 1), ("bigpool", True, False, 40, 2))
    sel = os.environ.get("VARIANTS")
    for name, qkv, il, layers, nbs in variants:
        if sel and name not in sel.split(","):
            continue
        us = run(B, ctx, 40, 128, qkv, il, layers=layers, nb_scale=nbs)
        print(json.dumps({"variant": name, "kernel": ds.ds_decode_kernel(B, 40), "B": B, "ctx": ctx, "us": us}),
              flush=True)
