"""Per-kernel timing sweeps (not the bench contract): ds_prefill_attn over prompt
lengths and ds_decode_attn over batch sizes, OPT-13B head geometry by default.
Device time with CUDA events over many launches that rotate through distinct
buffers (> L2), after warm-up. Prints one JSON line per point."""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("DS_PKG_ROOT"):  # an A/B variant build (tools/ab.sh)
    sys.path.insert(0, os.path.abspath(os.environ["DS_PKG_ROOT"]))

import numpy as np
import torch

import paper_2401_09670_b200 as ds

try:  # driver-measured on this pool; else the fallback B200_PROFILING.md states
    PEAKS = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
except OSError:
    PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def prefill_point(lens, n, d, reps=20, rot=4, warm=3, before_timed=None):
    T = sum(lens)
    bufs = [[torch.randn((T, n, d), device="cuda", dtype=torch.bfloat16) for _ in range(3)] for _ in range(rot)]
    out = torch.empty((T, n, d), device="cuda", dtype=torch.bfloat16)
    pages = sum(-(-l // 16) for l in lens)
    cache = ds.KVCache.empty(1, pages + 8, n, d)
    pool = ds.Pool(pages + 8)
    maxb = -(-max(lens) // 16)
    tab = np.full((len(lens), maxb), -1, np.int32)
    ds.ds_block_table(pool, ds.DS_BT_APPEND, [0] * len(lens), lens, tab)
    tab_d = torch.from_numpy(tab).cuda()
    cu = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)).cuda()
    scale = 1 / math.sqrt(d)
    for r in range(warm):
        q, k, v = bufs[r % rot]
        ds.ds_prefill_attn(q, k, v, out, cu, max(lens), cache, 0, tab_d, scale)
    torch.cuda.synchronize()
    if before_timed:
        before_timed()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for r in range(reps):
        q, k, v = bufs[r % rot]
        ds.ds_prefill_attn(q, k, v, out, cu, max(lens), cache, 0, tab_d, scale)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    flops = sum(n * 2 * d * l * (l + 1) for l in lens)
    byts = 12 * n * d * T
    roof = max(flops / (PEAKS["bf16_tflops"] * 1e12), byts / (PEAKS["hbm_gbs"] * 1e9))
    return {"kind": "prefill", "lens": f"{len(lens)}x{lens[0]}" if len(set(lens)) == 1 else f"{len(lens)} mixed",
            "n": n, "d": d, "us": t * 1e6, "tflops": flops / t / 1e12,
            "frac_tensor_peak": flops / t / 1e12 / PEAKS["bf16_tflops"], "frac_attainable": roof / t,
            "hbm_GBps_algorithmic": byts / t / 1e9}


def chunked_point(prefix, chunk, B, n, d, reps=20, rot=4):
    """NEXT-3: one chunk of `chunk` tokens per sequence on top of `prefix` cached tokens."""
    T = B * chunk
    bufs = [[torch.randn((T, n, d), device="cuda", dtype=torch.bfloat16) for _ in range(3)] for _ in range(rot)]
    out = torch.empty((T, n, d), device="cuda", dtype=torch.bfloat16)
    pages = B * -(-(prefix + chunk) // 16)
    cache = ds.KVCache.empty(1, pages + 8, n, d)
    cache.tensor.normal_()
    pool = ds.Pool(pages + 8)
    tab = np.full((B, -(-(prefix + chunk) // 16)), -1, np.int32)
    ds.ds_block_table(pool, ds.DS_BT_APPEND, [0] * B, [prefix + chunk] * B, tab)
    tab_d = torch.from_numpy(tab).cuda()
    cu = torch.from_numpy(np.arange(0, T + 1, chunk).astype(np.int32)).cuda()
    pl = torch.full((B,), prefix, dtype=torch.int32, device="cuda")
    scale = 1 / math.sqrt(d)
    run = lambda r: ds.ds_prefill_attn_chunked(bufs[r % rot][0], bufs[r % rot][1], bufs[r % rot][2], out, cu, pl,
                                               chunk, prefix + chunk, cache, 0, tab_d, scale)  # noqa: E731
    for r in range(3):
        run(r)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for r in range(reps):
        run(r)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    flops = B * n * 2 * d * chunk * (2 * prefix + chunk + 1)
    byts = B * n * d * (12 * chunk + 4 * prefix)
    roof = max(flops / (PEAKS["bf16_tflops"] * 1e12), byts / (PEAKS["hbm_gbs"] * 1e9))
    return {"kind": "chunked_prefill", "B": B, "prefix": prefix, "chunk": chunk, "n": n, "d": d, "us": t * 1e6,
            "tflops": flops / t / 1e12, "frac_tensor_peak": flops / t / 1e12 / PEAKS["bf16_tflops"],
            "frac_attainable": roof / t}


EARLY = os.environ.get("DS_EARLY_KV", "1") != "0"  # DS_DECODE_EARLY_KV on layers > 0, as bench.py


def decode_point(B, ctx, n, d, layers=8, reps=5):
    pages_per = -(-(ctx + 2) // 16)
    nb = B * pages_per + 8
    cache = ds.KVCache.empty(layers, nb, n, d)
    cache.tensor.normal_()
    pool = ds.Pool(nb)
    tab = np.full((B, pages_per), -1, np.int32)
    ds.ds_block_table(pool, ds.DS_BT_APPEND, [0] * B, [ctx + 1] * B, tab)
    tab_d = torch.from_numpy(tab).cuda()
    cl = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
    q = torch.randn((layers, B, n, d), device="cuda", dtype=torch.bfloat16)
    out = torch.empty((B, n, d), device="cuda", dtype=torch.bfloat16)
    ws = torch.zeros(ds.ds_decode_workspace_bytes(B, n, d, ctx), dtype=torch.uint8, device="cuda")
    scale = 1 / math.sqrt(d)

    def run():
        for l in range(layers):
            ds.ds_decode_attn(q[l], q[l], q[l], out, cache, l, tab_d, cl, ctx, scale, ws, early_kv=l > 0 and EARLY)

    run()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps / layers / 1e3
    byts = B * n * (4 * ctx * d + 12 * d) + 4 * B * -(-(ctx + 1) // 16)
    return {"kind": "decode", "B": B, "ctx": ctx, "n": n, "d": d, "us": t * 1e6, "GBps": byts / t / 1e9,
            "frac_hbm": byts / t / 1e9 / PEAKS["hbm_gbs"]}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--what", default="both", help="both | prefill | chunked | decode")
    p.add_argument("--n", type=int, default=40)
    p.add_argument("--d", type=int, default=128)
    a = p.parse_args()
    if a.what in ("both", "prefill"):
        for lens in ([512] * 16, [512] * 64, [128] * 64, [1024] * 8, [2048] * 4, [2048] * 16, [4096] * 4):
            print(json.dumps(prefill_point(lens, a.n, a.d)), flush=True)
        # config 5 (OPT-175B, TP4: 24 heads per GPU), LongBench-like prompts
        rng = np.random.default_rng(0)
        mix = [int(x) for x in rng.integers(1792, 1921, size=8)]
        print(json.dumps(prefill_point(mix, 24, a.d)), flush=True)
    if a.what in ("both", "chunked"):
        for prefix in (0, 512, 1024, 1536):
            print(json.dumps(chunked_point(prefix, 512, 16, a.n, a.d)), flush=True)
    if a.what in ("both", "decode"):
        for B in (1, 8, 16, 32, 64, 128, 256):
            print(json.dumps(decode_point(B, 544, a.n, a.d)), flush=True)


if __name__ == "__main__":
    main()
