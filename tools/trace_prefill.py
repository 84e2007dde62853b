"""Timeline of the prefill kernel's roles on SM 0 (A/B trace build only):
    tools/ab.sh trace "-DDS_TRACE"; DS_PKG_ROOT=ab/trace python tools/trace_prefill.py 4x4096
Prints per-tile medians (clock cycles) of: S MMA issue -> softmax sees S, softmax
compute (S seen -> last warp's P published), MMA wait for P, and a short
interleaved timeline of the CTAs resident on SM 0."""
import collections
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import kernel_bench as kb  # noqa: E402  (honours DS_PKG_ROOT)
import paper_2401_09670_b200 as ds  # noqa: E402

NAMES = {1: "sm_wait_S", 2: "sm_got_S", 3: "sm_P", 4: "mma_S", 5: "mma_wait_P", 6: "mma_PV", 7: "sm_epi_done",
         8: "ld_K", 9: "ld_V", 10: "sm_epi_pv"}


def main():
    B, l = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "4x4096").split("x"))
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    lib = ctypes.CDLL(ds.LIB_PATH)
    f = lib.ds_debug_prefill_trace
    f.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
    # warm-up launches, then exactly one traced launch
    print(kb.prefill_point([l] * B, n, 128, reps=1, rot=1, warm=2, before_timed=lambda: f(None, 0, 1)))
    cap = f(None, 0, 0)
    buf = np.zeros(2 * cap, np.uint64)
    f(buf.ctypes.data, cap, 1)
    rec = buf.reshape(-1, 2)
    rec = rec[rec[:, 0] != 0]
    cnt = len(rec)
    clk, tag = rec[:, 0].astype(np.int64), rec[:, 1]
    ev = (tag >> np.uint64(56)).astype(int)
    cta = ((tag >> np.uint64(32)) & np.uint64(0xFFFFFF)).astype(int)
    g = (tag & np.uint64(0xFFFFFFFF)).astype(int)
    t0 = clk.min()
    clk = clk - t0
    print(f"{cnt} records, span {clk.max()} cycles, CTAs {len(set(cta))}")
    by = collections.defaultdict(dict)  # (cta, g) -> {event: clock}
    for c, e, gg, t in zip(cta, ev, g, clk):
        d = by[(c, gg)]
        if 32 <= e < 48:
            d[f"epi{e - 32}"] = t
            continue
        if e >= 16:
            d["P_last"] = max(d.get("P_last", 0), t)
            d.setdefault("P_first", t)
            d["P_first"] = min(d["P_first"], t)
        else:
            d[NAMES.get(e, e)] = t
    stats = collections.defaultdict(list)
    for (c, gg), d in by.items():
        if "mma_S" in d and "sm_got_S" in d:
            stats["S issue -> softmax sees S"].append(d["sm_got_S"] - d["mma_S"])
        if "sm_wait_S" in d and "sm_got_S" in d:
            stats["softmax idle waiting for S"].append(d["sm_got_S"] - d["sm_wait_S"])
        if "sm_got_S" in d and "P_last" in d:
            stats["softmax: S seen -> last warp P"].append(d["P_last"] - d["sm_got_S"])
            stats["warp skew (last - first P)"].append(d["P_last"] - d["P_first"])
        if "mma_wait_P" in d and "mma_PV" in d:
            stats["MMA blocked on P (wait -> PV issued)"].append(d["mma_PV"] - d["mma_wait_P"])
        if "P_last" in d and "mma_PV" in d:
            stats["P published -> PV issued"].append(d["mma_PV"] - d["P_last"])
        if "ld_K" in d and "mma_S" in d:
            stats["K load issued -> S issued"].append(d["mma_S"] - d["ld_K"])
    for k, v in stats.items():
        v = np.array(v)
        print(f"{k:40s} n={len(v):6d} median={np.median(v):8.0f} p10={np.percentile(v, 10):8.0f} "
              f"p90={np.percentile(v, 90):8.0f}")
    # epilogue: the item's last tile g (sm_epi_done recorded with g = last tile)
    epi = []
    for (c, gg), d in by.items():
        if "sm_epi_done" in d and "P_last" in d:
            epi.append(d["sm_epi_done"] - d["P_last"])
    epv = [d["sm_epi_pv"] - d["P_last"] for d in by.values() if "sm_epi_pv" in d and "P_last" in d]
    if epv:
        print(f"{'epilogue wait for last P.V':40s} n={len(epv):6d} median={np.median(epv):8.0f}")
    for k in range(8):
        a_ = [d[f"epi{k}"] - d["sm_epi_pv"] for d in by.values() if f"epi{k}" in d and "sm_epi_pv" in d]
        if a_:
            print(f"  epilogue chunk {k // 2} {'loaded' if k % 2 == 0 else 'stored'} at +{np.median(a_):.0f} after the P.V wait")
    if epi:
        print(f"{'epilogue (last P -> O stored)':40s} n={len(epi):6d} median={np.median(epi):8.0f} "
              f"p90={np.percentile(epi, 90):8.0f}")
    # per-CTA tile rate
    per = collections.defaultdict(list)
    for (c, gg), d in by.items():
        if "sm_got_S" in d:
            per[c].append(d["sm_got_S"])
    rates = [np.median(np.diff(sorted(v))) for v in per.values() if len(v) > 4]
    print("median cycles between consecutive tiles of one CTA:", np.median(rates) if rates else None)
    # short timeline window
    order = np.argsort(clk)
    mid = clk.max() // 2
    sel = [i for i in order if mid <= clk[i] < mid + 6000]
    for i in sel[:120]:
        e = ev[i]
        name = f"sm_P_w{e - 16}" if e >= 16 else NAMES.get(e, e)
        print(f"{clk[i]:10d} cta{cta[i]:6d} g{g[i]:5d} {name}")


if __name__ == "__main__":
    main()
