"""NEXT-1 measurement: the TP/PP-mismatched resharding of the placements the paper
chose — every decode rank gathers the (layer, head) rectangle it owns from
every prefill rank (pairing.reshard_plan), through the page-gather kernel (LOCAL: all
'ranks' are pools on one GPU, so this times the kernel against HBM; across GPUs the
same kernel reads the peer pool over NVLink, PULL). One batch of 8 x 512-token prompts.

    python tools/reshard_bench.py        -> one JSON line per placement

Bytes: every migrated page (K and V, whole 16-token pages) is read once and written
once, so the HBM roofline of a launch sequence is 2 x page bytes / copy peak."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("DS_PKG_ROOT"):
    sys.path.insert(0, os.path.abspath(os.environ["DS_PKG_ROOT"]))

import numpy as np
import torch

import paper_2401_09670_b200 as ds
from paper_2401_09670_b200 import pairing

try:
    PEAKS = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
except OSError:
    PEAKS = {"hbm_gbs": 6650.0}

# (model, layers, heads, prefill (tp, pp), decode (tp, pp)) — P:735-739
PLACEMENTS = [
    ("OPT-13B", 40, 40, (2, 1), (1, 1)),
    ("OPT-66B", 64, 72, (4, 1), (2, 2)),
    ("OPT-175B", 96, 96, (3, 3), (4, 3)),
]


def run(model, L, n, prefill, decode, B=8, l=512, d=128, reps=5):
    (tp_p, pp_p), (tp_d, pp_d) = prefill, decode
    plan = pairing.reshard_plan(L, n, prefill, decode)
    pairing.check_reshard(plan, L, n, prefill, decode)
    lp, hp, ld, hd = L // pp_p, n // tp_p, L // pp_d, n // tp_d
    pages = B * (l // 16)
    ids = torch.arange(pages, dtype=torch.int32, device="cuda")
    src = [ds.KVCache.empty(lp, pages, hp, d) for _ in range(tp_p * pp_p)]
    dst = [ds.KVCache.empty(ld, pages, hd, d) for _ in range(tp_d * pp_d)]
    n_src = tp_p * pp_p

    def go():
        for p in plan:
            ds.ds_kv_migrate(None, ds.DS_MIGRATE_LOCAL, 0, src[p.src], p.src_layer_begin, p.layer_count, ids,
                             p.src_head_begin, p.head_count, None, dst_cache=dst[p.dst - n_src], dst_block_ids=ids,
                             dst_head_begin=p.dst_head_begin, dst_layer_begin=p.dst_layer_begin)

    go()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        go()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    page_bytes = L * n * 2 * pages * 16 * d * 2  # the whole model's K+V pages of the batch, each moved once
    return {"model": model, "prefill_tp_pp": prefill, "decode_tp_pp": decode, "slices": len(plan),
            "batch": f"{B}x{l}", "page_bytes": page_bytes, "ms": t * 1e3, "GBps": page_bytes / t / 1e9,
            "frac_of_hbm": 2 * page_bytes / t / 1e9 / PEAKS["hbm_gbs"]}


def main():
    for m in PLACEMENTS:
        print(json.dumps(run(*m)), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
