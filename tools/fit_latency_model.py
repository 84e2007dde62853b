"""NEXT-4: fit the Appendix A attention coefficients (C2, C5) to this
build's kernels on B200 and write profiles/<round>/latency_model_b200.json.

  python tools/fit_latency_model.py [--out profiles/r01/latency_model_b200.json]

Prefill points: uniform batches B x l and the three length mixes of the paper's
workloads (synthetic.lengths_*), OPT-13B per-GPU heads (n = 40, s = 128); one
ds_prefill_attn launch = one layer. Decode points: B x context grid; one
ds_decode_attn launch = one layer. Device time per launch from
tools/kernel_bench.py (CUDA events, inputs rotated beyond L2).
"""
import argparse
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import kernel_bench as kb  # noqa: E402

import synthetic as syn  # noqa: E402
from paper_2401_09670_b200 import latency_model as lm  # noqa: E402

N, S = 40, 128


def prefill_sets():
    out = [[l] * B for l, B in ((128, 16), (128, 64), (256, 32), (512, 8), (512, 32), (512, 64), (1024, 8),
                                (1024, 16), (2048, 4), (2048, 8), (4096, 2), (4096, 4))]
    for name, fn in (("chatbot", syn.lengths_chatbot), ("code", syn.lengths_code),
                     ("summarization", syn.lengths_summarization)):
        for seed, B in ((1, 16), (2, 48)):
            out.append([int(x) for x in fn(seed, B)[0]])
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--out", default=os.path.join(os.path.dirname(HERE), "profiles", "r01",
                                                 "latency_model_b200.json"))
    a = p.parse_args()
    pre = []
    for lens in prefill_sets():
        r = kb.prefill_point(lens, N, S)
        pre.append({"lens_B": len(lens), "t": sum(lens), "t2": sum(l * l for l in lens), "max_len": max(lens),
                    "x": lm.prefill_feature(lens, N, S), "x_lin": lm.prefill_linear_feature(lens, N, S),
                    "us": r["us"]})
        print(json.dumps(pre[-1]), flush=True)
    dec = []
    for B in (1, 4, 16, 64, 128, 256):
        for ctx in (128, 544, 1024, 2048):
            if B * ctx > 256 * 1024:  # bounded pool (8 layers x B x ctx pages)
                continue
            r = kb.decode_point(B, ctx, N, S, layers=8, reps=10)
            dec.append({"B": B, "ctx": ctx, "x": lm.decode_feature([ctx + 1] * B, N, S), "us": r["us"]})
            print(json.dumps(dec[-1]), flush=True)
    fits = {}
    for name, pts in (("prefill_C2", pre), ("decode_C5", dec)):
        x = [q["x"] for q in pts]
        y = [q["us"] * 1e-6 for q in pts]
        fits[name] = {"with_intercept": lm.fit(x, y).as_dict(), "paper_form_no_intercept": lm.fit(x, y, False).as_dict()}
        if name == "prefill_C2":  # the exact count before the approximation of P:671: + 2 h t
            fits[name]["full_quadratic_plus_linear"] = lm.fit([[q["x"], q["x_lin"]] for q in pts], y).as_dict()
    res = {"model": "PAPER.md Appendix A: T2 = C2 * 3 h t2 / b (P:673), T4 = C5 * 3 h t (P:699); per layer, "
                    "h = n*s per GPU; b = %d; decode l_i = c_i + 1" % lm.B_PREFILL,
           "geometry": {"n": N, "s": S}, "fits": fits, "prefill_points": pre, "decode_points": dec}
    dc = fits["decode_C5"]["with_intercept"]["coef"][0]
    # 3 h t element reads at 2 bytes: the bandwidth C5 implies (K and V dominate)
    res["decode_C5_implied_GBps_per_element_byte"] = 2.0 / dc / 1e9 if dc > 0 else None
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({"fits": fits}), flush=True)


if __name__ == "__main__":
    main()
