"""Our a2 prefill and a7+a8 decode kernels beside the attention kernels the image
ships as LIBRARY code, on the same seeded shapes, same GPU, same timing (CUDA events
over launches that rotate through > L2 of distinct inputs, after warm-up).

Context, not the product: nothing here is on the product path. It answers "how do
the hand-written kernels compare with what a user could call instead on B200":

  prefill (causal, varlen, bf16, head_dim 128):
    ours       ds_prefill_attn          (also writes the paged K/V cache, a3)
    fa2        flash_attn 2.8.3 flash_attn_varlen_func (mma.sync, sm_100 build)
    fa4        vllm.vllm_flash_attn.cute flash_attn_varlen_func (CuTe-DSL tcgen05)
    trtllm     flashinfer trtllm_batch_context_with_kv_cache (NVIDIA trtllm-gen
               cubins; reads K/V from a 16-token paged cache — ours is written first)
  decode (one new token, paged cache of 16-token pages):
    ours       ds_decode_attn           (also appends the new token's K/V, a7 i)
    vllm_pa2   vLLM paged_attention_v2  (the PagedAttention kernel the paper's
               system used, in vLLM's current build)
    trtllm     flashinfer trtllm_batch_decode_with_kv_cache (reads OUR cache
               tensors directly: [pages][n][16][D] is its HND layout)
    fa4        vllm.vllm_flash_attn.cute with a page table (16-token pages,
               non-TMA paged path)

Each library output is compared with ours (max relative error) so a mis-called
library cannot report a fake time. Prints one JSON line per (shape, impl).
The flashinfer trtllm-gen launcher is JIT-built: tools/build_flashinfer_fmha.sh builds it
on the CPU host into .fi_ws/; export FLASHINFER_WORKSPACE_BASE=$PWD/.fi_ws and
FLASHINFER_CUDA_ARCH_LIST=10.0a on the box. DS_SUSTAINED_S=s also times each decode
shape after s seconds of back-to-back launches (the power-capped steady state of
bench.py's step; short runs measure boost clocks)."""
import argparse
import json
import math
import os
import sys
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2401_09670_b200 as ds

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUSTAINED = float(os.environ.get("DS_SUSTAINED_S", "0"))  # decode: also time after this many seconds of load
try:
    PEAKS = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
except OSError:
    PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def timed(run, reps, rot, graph=True):
    """device time per call of run(r) (r = rotation index), CUDA events"""
    for r in range(3):
        run(r % rot)
    torch.cuda.synchronize()
    g = None
    if graph:
        try:
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    for r in range(rot):
                        run(r)
            torch.cuda.current_stream().wait_stream(s)
            g.replay()
            torch.cuda.synchronize()
        except Exception:  # noqa: BLE001 — not capturable: time eagerly
            g = None
            torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if g is not None:
        n = max(1, reps // rot)
        e0.record()
        for _ in range(n):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / (n * rot) / 1e3, True
    e0.record()
    for r in range(reps):
        run(r % rot)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3, False


def timed_sustained(run, rot, seconds):
    """device time per call when the GPU has been busy for `seconds` (power-capped
    steady state, as inside bench.py's step): replay a graph of `rot` calls back to back,
    time the second half"""
    for r in range(rot):
        run(r)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for r in range(rot):
                run(r)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    n = max(2, int(seconds / (e0.elapsed_time(e1) / 1e3)))
    for _ in range(n // 2):
        g.replay()
    e0.record()
    for _ in range(n - n // 2):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / ((n - n // 2) * rot) / 1e3


def relerr(a, b):
    a, b = a.float(), b.float()
    return float(((a - b).abs().max() / b.abs().max().clamp_min(1e-6)).item())


def prefill_shape(lens, n, d, impls, reps=20, rot=4):
    T = sum(lens)
    g = torch.Generator(device="cuda").manual_seed(1234)
    bufs = [[torch.randn((T, n, d), device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(3)]
            for _ in range(rot)]
    cu = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)).cuda()
    maxl = max(lens)
    scale = 1 / math.sqrt(d)
    flops = sum(n * 2 * d * l * (l + 1) for l in lens)
    byts = 12 * n * d * T
    roof = max(flops / (PEAKS["bf16_tflops"] * 1e12), byts / (PEAKS["hbm_gbs"] * 1e9))
    # our kernel and its paged cache (one layer per rotation slot, so trtllm can read it)
    pages = sum(-(-l // 16) for l in lens)
    maxb = -(-maxl // 16)
    cache = ds.KVCache.empty(rot, pages + 8, n, d)
    pool = ds.Pool(pages + 8)
    tab = np.full((len(lens), maxb), -1, np.int32)
    ds.ds_block_table(pool, ds.DS_BT_APPEND, [0] * len(lens), lens, tab)
    tab_d = torch.from_numpy(tab).cuda()
    outs = {}

    def ours(r, out):
        q, k, v = bufs[r]
        ds.ds_prefill_attn(q, k, v, out, cu, maxl, cache, r, tab_d, scale)

    name = f"{len(lens)}x{lens[0]}" if len(set(lens)) == 1 else f"{len(lens)} mixed ({min(lens)}-{maxl})"
    res = []
    for impl in ["ours"] + [i for i in impls if i != "ours"]:
        out = torch.empty((T, n, d), device="cuda", dtype=torch.bfloat16)
        rec = {"kind": "prefill", "shape": name, "n": n, "d": d, "impl": impl}
        try:
            if impl == "ours":
                run = lambda r: ours(r, out)  # noqa: E731
            elif impl == "fa2":
                from flash_attn import flash_attn_varlen_func as fa2

                def run(r):  # FA2's varlen call allocates its output
                    q, k, v = bufs[r]
                    return fa2(q, k, v, cu, cu, maxl, maxl, softmax_scale=scale, causal=True)
            elif impl == "fa4":
                from vllm.vllm_flash_attn.cute.interface import _flash_attn_fwd as fa4

                def run(r):
                    q, k, v = bufs[r]
                    fa4(q, k, v, cu_seqlens_q=cu, cu_seqlens_k=cu, max_seqlen_q=maxl, max_seqlen_k=maxl,
                        softmax_scale=scale, causal=True, out=out)
            elif impl == "trtllm":
                from flashinfer.prefill import trtllm_batch_context_with_kv_cache as trt
                ws = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
                sl = torch.tensor(lens, dtype=torch.int32, device="cuda")

                def run(r):
                    q = bufs[r][0]
                    kv = (cache.tensor[r, 0], cache.tensor[r, 1])
                    trt(q, kv, ws, tab_d, sl, maxl, maxl, scale, 1.0, len(lens), cu, cu, out=out)
            else:
                raise ValueError(impl)
            # correctness vs ours on slot 0
            if impl == "ours":
                ours(0, out)
                outs["ours"] = out.clone()
            else:
                r0 = run(0)
                o = r0 if isinstance(r0, torch.Tensor) else out
                rec["max_rel_err_vs_ours"] = relerr(o, outs["ours"])
            t, graphed = timed(run, reps, rot)
            rec.update({"us": t * 1e6, "tflops": flops / t / 1e12,
                        "frac_tensor_peak": flops / t / 1e12 / PEAKS["bf16_tflops"], "frac_attainable": roof / t,
                        "graph": graphed})
            if SUSTAINED > 0 and graphed:
                ts = timed_sustained(run, rot, SUSTAINED)
                rec.update({"us_sustained": ts * 1e6, "tflops_sustained": flops / ts / 1e12,
                            "sustained_s": SUSTAINED})
        except Exception as e:  # noqa: BLE001
            rec["error"] = f"{type(e).__name__}: {str(e)[:300]}"
            traceback.print_exc(file=sys.stderr)
        print(json.dumps(rec), flush=True)
        res.append(rec)
    return res


def decode_shape(B, ctx, n, d, impls, layers=8):
    """B sequences with ctx cached tokens each, one new token: reads ctx + 1 keys"""
    pages_per = -(-(ctx + 2) // 16)
    nb = B * pages_per + 8
    scale = 1 / math.sqrt(d)
    g = torch.Generator(device="cuda").manual_seed(99)
    cache = ds.KVCache.empty(layers, nb, n, d)
    cache.tensor.normal_(generator=g)
    pool = ds.Pool(nb)
    tab = np.full((B, pages_per), -1, np.int32)
    ds.ds_block_table(pool, ds.DS_BT_APPEND, [0] * B, [ctx + 1] * B, tab)
    tab_d = torch.from_numpy(tab).cuda()
    cl = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
    q = torch.randn((layers, B, n, d), device="cuda", dtype=torch.bfloat16, generator=g)
    kn = torch.randn((layers, B, n, d), device="cuda", dtype=torch.bfloat16, generator=g)
    vn = torch.randn((layers, B, n, d), device="cuda", dtype=torch.bfloat16, generator=g)
    ws = torch.zeros(ds.ds_decode_workspace_bytes(B, n, d, ctx), dtype=torch.uint8, device="cuda")
    byts = B * n * (4 * ctx * d + 12 * d) + 4 * B * -(-(ctx + 1) // 16)
    res = []
    ref = None
    for impl in ["ours"] + [i for i in impls if i != "ours"]:
        out = torch.empty((B, n, d), device="cuda", dtype=torch.bfloat16)
        rec = {"kind": "decode", "B": B, "ctx": ctx, "n": n, "d": d, "impl": impl}
        extra = []
        try:
            if impl == "ours":
                def run(l):
                    ds.ds_decode_attn(q[l], kn[l], vn[l], out, cache, l, tab_d, cl, ctx, scale, ws,
                                      early_kv=l > 0)
                run(0)  # appends token ctx of layer 0; later calls rewrite the same bytes
                ref = out.clone()
            elif impl == "trtllm":
                from flashinfer.decode import trtllm_batch_decode_with_kv_cache as trt
                fws = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
                sl = torch.full((B,), ctx + 1, dtype=torch.int32, device="cuda")

                def run(l):
                    trt(q[l], (cache.tensor[l, 0], cache.tensor[l, 1]), fws, tab_d, sl, ctx + 1,
                        bmm1_scale=scale, bmm2_scale=1.0, out=out)
            elif impl == "vllm_pa2":
                import vllm._custom_ops as ops
                x = 8
                kc = torch.empty((layers, nb, n, d // x, 16, x), device="cuda", dtype=torch.bfloat16)
                vc = torch.empty((layers, nb, n, d, 16), device="cuda", dtype=torch.bfloat16)
                extra += [kc, vc]
                # the same values, in vLLM's layouts (K: [blk][n][d/x][16][x], V: [blk][n][d][16])
                for l in range(layers):
                    kc[l].copy_(cache.tensor[l, 0].view(nb, n, 16, d // x, x).permute(0, 1, 3, 2, 4))
                    vc[l].copy_(cache.tensor[l, 1].permute(0, 1, 3, 2))
                sl = torch.full((B,), ctx + 1, dtype=torch.int32, device="cuda")
                part = 512
                nparts = -(-(ctx + 1) // part)
                es = torch.empty((B, n, nparts), device="cuda", dtype=torch.float32)
                ml = torch.empty_like(es)
                tmp = torch.empty((B, n, nparts, d), device="cuda", dtype=torch.bfloat16)
                one = torch.ones((), device="cuda", dtype=torch.float32)

                def run(l):
                    ops.paged_attention_v2(out, es, ml, tmp, q[l], kc[l], vc[l], n, scale, tab_d, sl, 16, ctx + 1,
                                           None, "auto", one, one)
            elif impl == "fa4":
                from vllm.vllm_flash_attn.cute.interface import _flash_attn_fwd as fa4
                kc = torch.empty((layers, nb, 16, n, d), device="cuda", dtype=torch.bfloat16)
                vc = torch.empty_like(kc)
                extra += [kc, vc]
                for l in range(layers):
                    kc[l].copy_(cache.tensor[l, 0].permute(0, 2, 1, 3))
                    vc[l].copy_(cache.tensor[l, 1].permute(0, 2, 1, 3))
                sl = torch.full((B,), ctx + 1, dtype=torch.int32, device="cuda")
                o4 = out.view(B, 1, n, d)

                def run(l):
                    fa4(q[l].view(B, 1, n, d), kc[l], vc[l], seqused_k=sl, page_table=tab_d, softmax_scale=scale,
                        causal=False, out=o4)
            else:
                raise ValueError(impl)
            if impl != "ours":
                run(0)
                rec["max_rel_err_vs_ours"] = relerr(out, ref)
            t, graphed = timed(run, 5 * layers, layers)
            rec.update({"us": t * 1e6, "GBps": byts / t / 1e9, "frac_hbm": byts / t / 1e9 / PEAKS["hbm_gbs"],
                        "graph": graphed})
            if SUSTAINED > 0 and graphed:
                ts = timed_sustained(run, layers, SUSTAINED)
                rec.update({"us_sustained": ts * 1e6, "GBps_sustained": byts / ts / 1e9,
                            "sustained_s": SUSTAINED})
        except Exception as e:  # noqa: BLE001
            rec["error"] = f"{type(e).__name__}: {str(e)[:300]}"
            traceback.print_exc(file=sys.stderr)
        del extra
        print(json.dumps(rec), flush=True)
        res.append(rec)
    return res


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--what", default="both", help="both | prefill | decode")
    p.add_argument("--impls", default="ours,fa2,fa4,trtllm,vllm_pa2")
    p.add_argument("--batches", default="16,64,128,256", help="decode batch sizes")
    p.add_argument("--shapes", default="128x512,16x512,16x2048,4x4096,mix5", help="prefill shapes")
    a = p.parse_args()
    impls = a.impls.split(",")
    torch.cuda.set_device(0)
    if a.what in ("both", "prefill"):
        pi = [i for i in impls if i in ("ours", "fa2", "fa4", "trtllm")]
        rng = np.random.default_rng(0)
        mix5 = [int(x) for x in rng.integers(1792, 1921, size=8)]
        shapes = {"128x512": ([512] * 128, 40), "16x512": ([512] * 16, 40), "16x2048": ([2048] * 16, 40),
                  "4x4096": ([4096] * 4, 40), "mix5": (mix5, 24)}
        for key in a.shapes.split(","):
            lens, n = shapes[key]
            prefill_shape(lens, n, 128, pi)
            torch.cuda.empty_cache()
    if a.what in ("both", "decode"):
        di = [i for i in impls if i in ("ours", "trtllm", "vllm_pa2", "fa4")]
        for B in [int(x) for x in a.batches.split(",")]:
            decode_shape(B, 544, 40, 128, di)
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
