"""Per-warp timeline of ONE decode launch (A/B trace build only):
    tools/ab.sh trace "-DDS_TRACE"; DS_PKG_ROOT=ab/trace python tools/trace_decode.py 64 544
globaltimer (ns) stamps per warp: entry (after griddepcontrol.wait), prefix built,
first page ready, loop done."""
import ctypes
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import kernel_bench as kb  # noqa: E402,F401  (sys.path / DS_PKG_ROOT)
import paper_2401_09670_b200 as ds  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 544
    n, d = 40, 128
    lib = ctypes.CDLL(ds.LIB_PATH)
    f = lib.ds_debug_decode_trace
    f.argtypes = [ctypes.c_void_p, ctypes.c_int]
    pages_per = -(-(ctx + 2) // 16)
    nb = B * pages_per + 8
    cache = ds.KVCache.empty(2, nb, n, d)
    cache.tensor.normal_()
    pool = ds.Pool(nb)
    tab = np.full((B, pages_per), -1, np.int32)
    ds.ds_block_table(pool, ds.DS_BT_APPEND, [0] * B, [ctx + 1] * B, tab)
    tab_d = torch.from_numpy(tab).cuda()
    cl = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
    q = torch.randn((B, n, d), device="cuda", dtype=torch.bfloat16)
    out = torch.empty_like(q)
    ws = torch.zeros(ds.ds_decode_workspace_bytes(B, n, d, ctx), dtype=torch.uint8, device="cuda")
    for lyr in (0, 1, 0):
        ds.ds_decode_attn(q, q, q, out, cache, lyr, tab_d, cl, ctx, 1 / math.sqrt(d), ws)
    torch.cuda.synchronize()
    f(None, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ds.ds_decode_attn(q, q, q, out, cache, 1, tab_d, cl, ctx, 1 / math.sqrt(d), ws)
    e1.record()
    torch.cuda.synchronize()
    cnt = f(None, 0)
    buf = np.zeros(cnt, np.uint64)
    f(buf.ctypes.data, 0)
    t = buf.reshape(-1, 6)[:, :5].astype(np.int64)
    sm_of = np.arange(len(t)) // 16
    keep = t[:, 0] > 0
    t, sm_of = t[keep], sm_of[keep]
    t0 = t[:, 0].min()
    ent, pre, first, end = (t[:, k] - t0 for k in range(4))
    pages = t[:, 4]
    byts = B * n * (4 * ctx * d + 12 * d)
    print(f"event time {e0.elapsed_time(e1) * 1e3:.1f} us; warps {len(t)}; pages/warp {pages.mean():.1f}; "
          f"bytes {byts / 1e6:.1f} MB")
    for name, v in (("entry", ent), ("prefix built", pre), ("first page ready", first), ("loop done", end)):
        print(f"{name:18s} min {v.min() / 1e3:7.2f} us  median {np.median(v) / 1e3:7.2f}  max {v.max() / 1e3:7.2f}")
    span = (end.max() - ent.min()) / 1e3
    print(f"span entry->last done {span:.1f} us -> {byts / span / 1e3:.0f} GB/s over the span")
    sm_end = np.array([end[sm_of == k].max() for k in np.unique(sm_of)]) / 1e3
    sm_spread = np.array([end[sm_of == k].max() - end[sm_of == k].min() for k in np.unique(sm_of)]) / 1e3
    print(f"per-CTA (SM) last warp done: min {sm_end.min():.1f} median {np.median(sm_end):.1f} max {sm_end.max():.1f} us;"
          f" within-CTA spread median {np.median(sm_spread):.1f} max {sm_spread.max():.1f} us")
    order = np.argsort(sm_end)
    print("slowest CTAs (blockIdx: done us):", [(int(k), round(float(sm_end[k]), 1)) for k in order[-8:]])
    print("fastest CTAs:", [(int(k), round(float(sm_end[k]), 1)) for k in order[:8]])
    busy = (end - first)
    print(f"per-warp streaming time (first page -> done): median {np.median(busy) / 1e3:.1f} us; "
          f"rate per SM {byts / 148 / (np.median(busy) / 1e9) / 1e9:.1f} GB/s")


if __name__ == "__main__":
    main()
