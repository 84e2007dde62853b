"""bench.py — DistServe KV-cache data path on B200 (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ds|reference]

One STEP = one pass of the whole hot path over one batch of B synthetic
requests with OPT-13B attention geometry (40 layers x 40 heads x 128), prompt
512 / output 64 (BASELINE config 2):
  a1  block tables for the batch (prefill pool ALLOC; decode pool ALLOC/APPEND/FREE)
  a2+a3  40 x ds_prefill_attn (one per layer, fused paged K/V write)
  a4-a6  ds_kv_migrate of all 40 layers' pages prefill pool -> decode pool
  a7+a8  64 decode steps x 40 layers of ds_decode_attn (append + split-K attention)
At N=1 one GPU plays both instances (migration is the LOCAL page copy); at
N>1 ranks [0, N/2) are prefill instances and [N/2, N) decode instances, paired
r <-> r + N/2 (independent pairs, one p2p exchange per pair per step; the
prefill of batch k+1 overlaps the decode of batch k).

value = (prompt + generated) tokens of all pairs / max-over-ranks step time.
Inputs are resident in HBM and larger than L2 (each layer's Q/K/V is 252 MB,
each layer's decode KV ~180 MB, layers rotate), so no L2 flush is needed.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "prefill tok/s, decode tok/s/GPU, KV migrate GB/s at 1/2/4/8 B200 vs roofline"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
NVLINK_GBS = 900.0  # nominal per direction per GPU (B200_PROFILING.md; measured peer copy 770)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--batch", type=int, default=16)
    p.add_argument("--prompt", type=int, default=512)
    p.add_argument("--output", type=int, default=64)
    p.add_argument("--impl", default="ds", choices=["ds", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=2)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--profile", action="store_true", help="one short pass for ncu (no JSON)")
    p.add_argument("--no-graphs", action="store_true", help="eager decode launches (no CUDA graphs)")
    return p.parse_args()


def load_peaks():
    try:
        d = json.load(open(PEAKS_PATH))
        return d, "measured"
    except Exception:
        return FALLBACK_PEAKS, "fallback"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------- workload
class Workload:
    """Synthetic OPT-13B-geometry batch; identical on every rank of a pair."""

    def __init__(self, batch, prompt, output, layers=40, heads=40, head_dim=128):
        self.B, self.l0, self.out_len = batch, prompt, output
        self.L, self.n, self.d = layers, heads, head_dim
        self.lens = [prompt] * batch
        self.T = prompt * batch
        self.scale = 1.0 / math.sqrt(head_dim)
        self.pages_per_seq = -(-prompt // 16)
        self.maxb = -(-(prompt + output) // 16)

    # algorithmic work
    def prefill_flops_per_layer(self):
        return sum(self.n * 2 * self.d * l * (l + 1) for l in self.lens)

    def prefill_bytes_per_layer(self):
        return 12 * self.n * self.d * self.T

    def decode_bytes(self, ctx):  # one layer, cache lengths ctx (tokens already cached)
        pages = sum(-(-(c + 1) // 16) for c in ctx)
        return sum(self.n * (4 * c * self.d + 12 * self.d) for c in ctx) + 4 * pages

    def kv_payload_bytes(self):  # valid tokens, all layers, K+V
        return 2 * self.L * self.T * self.n * self.d * 2

    def kv_page_bytes(self):  # whole pages actually moved
        return 2 * self.L * self.B * self.pages_per_seq * 16 * self.n * self.d * 2


def _i32(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()


class Engine:
    """Device state of one rank: pools, resident inputs, staging, launch helpers."""

    def __init__(self, w: Workload, role: str, comm, peer, seed, torch, ds):
        self.w, self.role, self.comm, self.peer, self.torch, self.ds = w, role, comm, peer, torch, ds
        dev = "cuda"
        bf = torch.bfloat16
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        self.pf = role in ("both", "prefill")
        self.dc = role in ("both", "decode")
        # pools sized for 2 batches in flight (pipelined N>1) + headroom
        nb = 2 * w.B * w.maxb + 64
        if self.pf:
            self.P = ds.KVCache.empty(w.L, nb, w.n, w.d)
            self.pool_p = ds.Pool(nb)
            shape = (w.T, w.n, w.d)
            # per-layer resident prefill inputs (N(0,1) bf16; each layer 3 x 84 MB)
            self.q = [torch.randn(shape, generator=g, device=dev, dtype=torch.float32).to(bf) for _ in range(w.L)]
            self.k = [torch.randn(shape, generator=g, device=dev, dtype=torch.float32).to(bf) for _ in range(w.L)]
            self.v = [torch.randn(shape, generator=g, device=dev, dtype=torch.float32).to(bf) for _ in range(w.L)]
            self.out = torch.empty(shape, dtype=bf, device=dev)
            self.cu = _i32(torch, np.concatenate([[0], np.cumsum(w.lens)]))
        if self.dc:
            self.D = ds.KVCache.empty(w.L, nb, w.n, w.d)
            self.pool_d = ds.Pool(nb)
            dshape = (w.out_len, w.L, w.B, w.n, w.d)
            self.dq = torch.randn(dshape, generator=g, device=dev, dtype=torch.float32).to(bf)
            self.dk = torch.randn(dshape, generator=g, device=dev, dtype=torch.float32).to(bf)
            self.dv = torch.randn(dshape, generator=g, device=dev, dtype=torch.float32).to(bf)
            self.dout = torch.empty((w.out_len, w.B, w.n, w.d), dtype=bf, device=dev)
            self.max_c = w.l0 + w.out_len - 1  # largest cache length of the batch (validation only)
            self.ws = torch.zeros(max(16, ds.ds_decode_workspace_bytes(w.B, w.n, w.d, self.max_c)),
                                  dtype=torch.uint8, device=dev)
            # fixed device block table / lengths read by the captured decode graphs
            self.dtab = torch.full((w.B, w.maxb), -1, dtype=torch.int32, device=dev)
            self.dlen = torch.zeros((w.B,), dtype=torch.int32, device=dev)
            self.h_tab2 = [torch.empty((w.B, w.maxb), dtype=torch.int32).pin_memory() for _ in range(2)]
            self.h_len2 = [torch.empty((w.B,), dtype=torch.int32).pin_memory() for _ in range(2)]
            self.h_ev2 = [None, None]
            self.hslot = 0
            self.graphs = None
        nblk = w.B * w.pages_per_seq
        mrole = {"both": ds.DS_MIGRATE_LOCAL, "prefill": ds.DS_MIGRATE_SEND, "decode": ds.DS_MIGRATE_RECV}[role]
        self.mrole = mrole
        cache_for_size = self.P if self.pf else self.D
        sbytes = ds.ds_kv_migrate_staging_bytes(cache_for_size, mrole, w.L, nblk, w.n)
        self.staging = torch.empty(sbytes, dtype=torch.uint8, device=dev) if sbytes else None
        # pinned host ring for the per-step block-table / cache-length uploads (async H2D)
        self.ring = w.out_len + 2
        self.h_tab = torch.empty((self.ring, w.B, w.maxb), dtype=torch.int32).pin_memory()
        self.h_len = torch.empty((self.ring, w.B), dtype=torch.int32).pin_memory()
        self.d_tab = torch.empty((self.ring, w.B, w.maxb), dtype=torch.int32, device=dev)
        self.d_len = torch.empty((self.ring, w.B), dtype=torch.int32, device=dev)
        self.h_ev = [None] * self.ring
        self.slot = 0
        self.stream = torch.cuda.current_stream()
        self.launches = 0
        self.decode_events = []

    def upload_fixed(self, table: np.ndarray, lens):
        """async H2D of the decode block table + lengths into the graphs' fixed buffers"""
        i = self.hslot
        self.hslot ^= 1
        if self.h_ev2[i] is not None:
            self.h_ev2[i].synchronize()
        self.h_tab2[i].numpy()[:] = table
        self.h_len2[i].numpy()[:] = lens
        self.dtab.copy_(self.h_tab2[i], non_blocking=True)
        self.dlen.copy_(self.h_len2[i], non_blocking=True)
        ev = self.torch.cuda.Event()
        ev.record()
        self.h_ev2[i] = ev

    def decode_layers(self, s):
        """ds_decode_attn for every layer of decode step s (reads dtab / dlen)"""
        w, ds = self.w, self.ds
        for layer in range(w.L):
            ds.ds_decode_attn(self.dq[s, layer], self.dk[s, layer], self.dv[s, layer], self.dout[s], self.D, layer,
                              self.dtab, self.dlen, self.max_c, w.scale, self.ws)

    def capture_decode_graphs(self):
        """one CUDA graph per decode step: the 40-layer loop becomes a single launch"""
        torch = self.torch
        self.graphs = []
        for s in range(self.w.out_len):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.decode_layers(s)
            self.graphs.append(g)
        torch.cuda.synchronize()

    def upload(self, table: np.ndarray, lens):
        """async H2D of a block table (+ lengths) through the pinned ring"""
        s = self.slot
        self.slot = (s + 1) % self.ring
        if self.h_ev[s] is not None:
            self.h_ev[s].synchronize()  # the previous copy out of this slot has completed
        self.h_tab[s].numpy()[:, :table.shape[1]] = table
        self.h_len[s].numpy()[:] = lens
        self.d_tab[s].copy_(self.h_tab[s], non_blocking=True)
        self.d_len[s].copy_(self.h_len[s], non_blocking=True)
        ev = self.torch.cuda.Event()
        ev.record()
        self.h_ev[s] = ev
        return self.d_tab[s], self.d_len[s]

    # -- one step ------------------------------------------------------------------
    def step(self, events=None, time_decode=False):
        torch, ds, w = self.torch, self.ds, self.w
        ev = events or {}
        nblk = w.B * w.pages_per_seq
        if "start" in ev:
            ev["start"].record()
        if self.pf:
            tp = np.full((w.B, w.maxb), -1, np.int32)
            ds.ds_block_table(self.pool_p, ds.DS_BT_APPEND, [0] * w.B, w.lens, tp)
            tp_d, _ = self.upload(tp, w.lens)
            for layer in range(w.L):
                ds.ds_prefill_attn(self.q[layer], self.k[layer], self.v[layer], self.out, self.cu, w.l0, self.P, layer,
                                   tp_d, w.scale)
            self.launches += w.L
            src_ids = tp_d[:, :w.pages_per_seq].reshape(-1).contiguous()
        if "prefill_end" in ev:
            ev["prefill_end"].record()
        if self.dc:
            td = np.full((w.B, w.maxb), -1, np.int32)
            ds.ds_block_table(self.pool_d, ds.DS_BT_APPEND, [0] * w.B, w.lens, td)
            td_d, _ = self.upload(td, w.lens)
            dst_ids = td_d[:, :w.pages_per_seq].reshape(-1).contiguous()
        # migration (pull: the decode side has admitted the batch above)
        if self.mrole == ds.DS_MIGRATE_LOCAL:
            ds.ds_kv_migrate(None, self.mrole, 0, self.P, 0, w.L, src_ids, 0, w.n, None,
                             dst_cache=self.D, dst_block_ids=dst_ids)
            self.launches += 1
        else:
            chunk_rows = max(1, (64 << 20) // (w.n * 16 * w.d * 2))
            self.launches += -(-(2 * w.L * nblk) // chunk_rows)  # pack or unpack kernels (+ NCCL's own)
            if self.pf:
                ds.ds_kv_migrate(self.comm, self.mrole, self.peer, self.P, 0, w.L, src_ids, 0, w.n, self.staging)
            else:
                ds.ds_kv_migrate(self.comm, self.mrole, self.peer, self.D, 0, w.L, dst_ids, 0, w.n, self.staging)
        if self.pf:
            ds.ds_block_table(self.pool_p, ds.DS_BT_FREE, w.lens, None, tp)
        if "migrate_end" in ev:
            ev["migrate_end"].record()
        if self.dc:
            cur = list(w.lens)
            for s in range(w.out_len):
                ds.ds_block_table(self.pool_d, ds.DS_BT_APPEND, cur, [1] * w.B, td)
                self.upload_fixed(td, cur)
                if self.graphs is not None:
                    self.graphs[s].replay()
                else:
                    self.decode_layers(s)
                self.launches += 2 * w.L  # decode_kernel + decode_combine_kernel per layer
                cur = [c + 1 for c in cur]
            ds.ds_block_table(self.pool_d, ds.DS_BT_FREE, cur, None, td)
        if "end" in ev:
            ev["end"].record()


def dist_setup(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1 and world % 2:
        raise SystemExit("N>1 needs an even number of GPUs (prefill/decode pairs)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def pair_of(rank, world):
    """(role, peer): ranks [0, N/2) prefill, [N/2, N) decode; pair r <-> r + N/2."""
    if world == 1:
        return "both", 0
    half = world // 2
    return ("prefill", rank + half) if rank < half else ("decode", rank - half)


def make_comm(world, rank, ds):
    import torch.distributed as dist
    if world == 1:
        return None  # both instances on one GPU: LOCAL page copy, no communicator
    obj = [ds.ds_comm_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return ds.ds_comm_init(obj[0], world, rank)


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ----------------------------------------------------------------------------- CPU oracle
def oracle_sample_tok_s(w: Workload, target_s: float = 15.0):
    """Time the fp64 C oracle (as it stands) on a bounded sample of the same
    workload and scale linearly to tok/s: prefill of one 512-token request over
    all 40 heads of one layer, plus decode steps (c = 512..) of one request over
    one layer. Work is linear in layers, heads and requests."""
    import oracle
    import synthetic as syn
    threads = os.cpu_count() or 1
    b = syn.prefill_batch(0, [w.l0], w.n, w.d)
    t0 = time.perf_counter()
    oracle.prefill(b.q, b.k, b.v, b.cu_seqlens, w.scale, nthreads=threads)
    t_pf = time.perf_counter() - t0  # one request, one layer
    pool = oracle.Pool(1, w.pages_per_seq + w.out_len // 16 + 2, w.n, w.d)
    table = np.full((1, w.maxb + 1), -1, np.int32)
    pool.append([0], [w.l0], table)
    pool.write_prefill(0, b.k, b.v, b.cu_seqlens, table)
    n_dec, t_dec, c = 0, 0.0, w.l0
    while n_dec < w.out_len and t_dec < target_s:
        pool.append([c], [1], table)
        db = syn.decode_batch(n_dec, 1, w.n, w.d)
        t0 = time.perf_counter()
        pool.decode(0, db.q, db.k_new, db.v_new, table, [c], w.scale, nthreads=threads)
        t_dec += time.perf_counter() - t0
        c += 1
        n_dec += 1
    per_req = w.L * (t_pf + t_dec / n_dec * w.out_len)  # all layers, one request
    tok_s = (w.l0 + w.out_len) / per_req
    sample = (f"1 request x 1 layer x {w.n} heads: prefill {w.l0} tokens ({t_pf:.2f} s) + {n_dec} decode steps "
              f"({t_dec:.2f} s); scaled linearly to {w.L} layers and {w.out_len} steps")
    return tok_s, threads, sample, t_pf + t_dec


# ----------------------------------------------------------------------------- main arms
def run_reference(args):
    """--impl reference: the oracle as it stands on the host cores, same config/metric."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = Workload(args.batch, args.prompt, args.output)
    vals = []
    for _ in range(max(args.steps, 1)):
        tok_s, threads, sample, spent = oracle_sample_tok_s(w, target_s=5.0)
        vals.append(tok_s * w.B / w.B)  # per-request rate == whole-batch rate (linear)
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tok/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": w.B * (w.l0 + w.out_len) / v * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"OPT-13B attention geometry, {w.B} req x {w.l0} in / {w.out_len} out",
                       "batch": w.B, "prompt": w.l0, "output": w.out_len},
            "cpu_baseline": {"value": v, "unit": "tok/s", "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ds(args):
    import torch
    world, rank, local = dist_setup(args)
    import paper_2401_09670_b200 as ds
    role, peer = pair_of(rank, world)
    w = Workload(args.batch, args.prompt, args.output)
    comm = make_comm(world, rank, ds)
    eng = Engine(w, role, comm, peer, seed=1234 + (rank % max(1, world // 2)), torch=torch, ds=ds)
    torch.cuda.synchronize()
    if args.profile:
        eng.step()
        torch.cuda.synchronize()
        return
    for _ in range(args.warmup):
        eng.step()
    torch.cuda.synchronize()
    if eng.dc and not args.no_graphs:
        eng.capture_decode_graphs()
        eng.step()  # one graph-replay warm-up step
        torch.cuda.synchronize()
    barrier(world)
    sampler = ClockSampler(local)
    sampler.start()
    phase = []
    eng.launches = 0
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    t_start.record()
    for s in range(args.steps):
        evs = {k: torch.cuda.Event(enable_timing=True) for k in ("start", "prefill_end", "migrate_end", "end")}
        eng.step(evs)
        phase.append(evs)
    t_end.record()
    torch.cuda.synchronize()
    barrier(world)
    clocks = sampler.stop()
    total_ms = t_start.elapsed_time(t_end)
    total_ms = max_over_ranks(total_ms, world)
    launches = eng.launches
    ms_step = total_ms / args.steps
    pairs = max(1, world // 2)
    tokens_step = pairs * w.B * (w.l0 + w.out_len)
    value = tokens_step / (ms_step / 1e3)

    peaks, peak_kind = load_peaks()
    comp = {}
    # phase breakdown on this rank (device time between events)
    if eng.pf:
        pf_ms = statistics.median(e["start"].elapsed_time(e["prefill_end"]) for e in phase)
        comp["prefill_ms_per_step"] = pf_ms
        comp["prefill_tok_s_per_gpu"] = w.T / (pf_ms / 1e3)
        comp["prefill_tflops"] = w.L * w.prefill_flops_per_layer() / (pf_ms / 1e3) / 1e12
        comp["prefill_frac_of_tensor_peak"] = comp["prefill_tflops"] / peaks["bf16_tflops"]
        t_roof = max(w.prefill_flops_per_layer() / (peaks["bf16_tflops"] * 1e12),
                     w.prefill_bytes_per_layer() / (peaks["hbm_gbs"] * 1e9)) * w.L
        comp["prefill_frac_of_attainable_roofline"] = t_roof / (pf_ms / 1e3)
        mig_ms = statistics.median(e["prefill_end"].elapsed_time(e["migrate_end"]) for e in phase)
        comp["migrate_ms_per_step"] = mig_ms
        comp["kv_migrate_GBps"] = w.kv_payload_bytes() / (mig_ms / 1e3) / 1e9
        comp["kv_migrate_page_GBps"] = w.kv_page_bytes() / (mig_ms / 1e3) / 1e9
    dec_kernel = None
    if eng.dc:
        dec_ms = statistics.median(e["migrate_end"].elapsed_time(e["end"]) for e in phase)
        comp["decode_ms_per_step"] = dec_ms
        comp["decode_tok_s_per_gpu"] = w.B * w.out_len / (dec_ms / 1e3)
        ctx_steps = [[c + s for c in w.lens] for s in range(w.out_len)]
        avg_bytes = sum(w.decode_bytes(c) for c in ctx_steps) / w.out_len
        avg_ms = dec_ms / (w.out_len * w.L)  # device time per ds_decode_attn call (both kernels + gaps)
        dec_kernel = (avg_bytes, avg_ms)
        comp["decode_attn_GBps"] = avg_bytes / (avg_ms / 1e3) / 1e9
        comp["decode_attn_frac_of_hbm"] = comp["decode_attn_GBps"] / peaks["hbm_gbs"]
        comp["decode_attn_us_per_launch"] = avg_ms * 1e3
        comp["decode_graphs"] = eng.graphs is not None
    roofline = None
    if dec_kernel:
        achieved = dec_kernel[0] / (dec_kernel[1] / 1e3) / 1e9
        roofline = {"kernel": "ds_decode_attn (decode_kernel + decode_combine_kernel)", "bound": "hbm", "achieved": achieved,
                    "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                    "traffic": None, "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
                    "algorithmic_bytes_per_launch": dec_kernel[0]}
    line = {"metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"OPT-13B attention geometry (40 layers x 40 heads x 128), "
                                   f"{w.B} requests x {w.l0} prompt / {w.out_len} output per pair; "
                                   f"prefill->migrate->decode per step",
                       "batch": w.B, "prompt": w.l0, "output": w.out_len, "pairs": pairs,
                       "parallelism": "single GPU (P+D)" if world == 1 else f"{pairs}P:{pairs}D pairs",
                       "l2": "inputs larger than L2 (252 MB/layer prefill, ~180 MB/layer decode KV)"},
            "components": comp, "roofline": roofline, "clocks": clocks, "gpu_launches": launches}
    # e2e through the public API with host buffers
    if not args.no_e2e:
        line["e2e"] = run_e2e(args, eng, w, world, torch, ds)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        tok_s, threads, sample, _ = oracle_sample_tok_s(w)
        line["cpu_baseline"] = {"value": tok_s, "unit": "tok/s", "cores": threads, "kind": "oracle",
                                "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_e2e(args, eng, w, world, torch, ds):
    """Same step, but every layer's prefill inputs are copied host(pinned)->device
    and the decode inputs too; the last layer's decode outputs are read back."""
    bf = torch.bfloat16
    h2d = d2h = 0
    host = {}
    if eng.pf:
        shape = (w.T, w.n, w.d)
        host["qkv"] = torch.randn((3,) + shape, dtype=torch.float32).to(bf).pin_memory()
    if eng.dc:
        host["dec"] = torch.randn((3, w.out_len, w.L, w.B, w.n, w.d), dtype=torch.float32).to(bf).pin_memory()
        host["out"] = torch.empty((w.out_len, w.B, w.n, w.d), dtype=bf).pin_memory()

    def step():
        nonlocal h2d, d2h
        if eng.pf:
            for layer in range(w.L):
                eng.q[layer].copy_(host["qkv"][0], non_blocking=True)
                eng.k[layer].copy_(host["qkv"][1], non_blocking=True)
                eng.v[layer].copy_(host["qkv"][2], non_blocking=True)
                h2d += 3 * host["qkv"][0].numel() * 2
        if eng.dc:
            eng.dq.copy_(host["dec"][0], non_blocking=True)
            eng.dk.copy_(host["dec"][1], non_blocking=True)
            eng.dv.copy_(host["dec"][2], non_blocking=True)
            h2d += 3 * eng.dq.numel() * 2
        eng.step()
        if eng.dc:
            host["out"].copy_(eng.dout, non_blocking=True)
            d2h += eng.dout.numel() * 2

    step()
    torch.cuda.synchronize()
    h2d = d2h = 0
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.e2e_steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1), world) / args.e2e_steps
    pairs = max(1, world // 2)
    return {"value": pairs * w.B * (w.l0 + w.out_len) / (ms / 1e3), "unit": "tok/s",
            "h2d_bytes_per_step": h2d // args.e2e_steps, "d2h_bytes_per_step": d2h // args.e2e_steps,
            "ms_per_step": ms, "steps": args.e2e_steps}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ds(args)


if __name__ == "__main__":
    main()
