"""bench.py — the DistServe KV-cache data path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2|1|3|4|5] [--batch B]
                    [--impl ds|reference]

One STEP = one pass of the whole hot path over one batch
of B synthetic requests:
  a1     block tables (prefill pool ALLOC/FREE; decode pool ALLOC/APPEND/FREE)
  a2+a3  ds_prefill_attn for every local layer (fused paged K/V write)
  a4-a6  the pages of all local layers, prefill -> decode: at N=1 fused into the
         prefill kernel (ds_prefill_attn_push into the decode pool); at N>1
         ds_kv_migrate_contig (NCCL pool to pool), or pull / push over CUDA IPC
  a7+a8  `output` decode steps x local layers of ds_decode_attn
Default workload = BASELINE configs[1] (config 2): OPT-13B attention geometry
(40 layers x 40 heads x 128), 128 requests x 512 prompt / 64 output (the decode
batch a dedicated decode instance accumulates — decoding is batched as far as
memory allows; at N=1 both instances' pools, 2 x 56 GB, share the GPU;
SURVEY §8d sweeps B = 1..256, profiles/r01/sweep_bench_c2_b*.json).
At N=1 one GPU plays both instances (migration fused into the prefill); at N>1
ranks [0, N/2) are prefill and [N/2, N) decode instances, paired by
paper_2401_09670_b200.pairing (same layers/heads), migration = NCCL
p2p over NVLink (pool to pool); each replica pair serves its own batch (weak scaling) and the
prefill of batch k+1 overlaps the decode of batch k.

value = (prompt + generated) tokens of all replicas / max-over-ranks step time.
Inputs are resident and larger than L2: prefill inputs rotate over >= 1 GB of
distinct buffers, each layer's decode KV is >= ~180 MB at B = 16 and the 40
layers rotate, so no L2 flush is needed.
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

import synthetic as syn  # noqa: E402

METRIC = "prefill tok/s, decode tok/s/GPU, KV migrate GB/s at 1/2/4/8 B200 vs roofline"
# the decode kernel reads ~99.9 % of its bytes; the roofline peak is the driver's copy
# (read + write) figure, so frac can exceed 1 — a pure streaming read of this part
# reaches 7.1-7.3 TB/s (tools/hbm_read_bench.cu, profiles/r01/hbm_read_bench.txt)
DECODE_PEAK_NOTE = ("peak = driver-measured copy bandwidth (read+write); decode is ~99.9% reads, whose streaming "
                    "ceiling measured 7.1-7.3 TB/s on this part, 7.0-7.1 TB/s for its page-ring pattern sustained "
                    "for 5 s (profiles/r01/hbm_read_bench.txt, profiles/r02/hbm_read_bench_sustained.txt)")
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
NVLINK_GBS = 900.0  # nominal per direction per GPU (770 measured peer copy, B200_PROFILING.md)

# BASELINE.json configs. mix: prompt-length source; output = decode steps run.
CONFIGS = {
    "1": dict(geom=syn.TINY, mix="fixed", prompt=32, output=8, batch=1, tp=1, pp=1,
              desc="config 1: 1 layer x 4 heads x 64, prompt 32 + 8 decode steps"),
    "2": dict(geom=syn.OPT_13B, mix="fixed", prompt=512, output=64, batch=128, tp=1, pp=1,
              desc="config 2: OPT-13B attention geometry, 512 in / 64 out"),
    "3": dict(geom=syn.OPT_13B, mix="chatbot", prompt=0, output=64, batch=64, tp=1, pp=1,
              desc="config 3: OPT-13B, ShareGPT-like chatbot length mix"),
    "4": dict(geom=syn.OPT_66B, mix="code", prompt=0, output=64, batch=32, tp=2, pp=2,
              desc="config 4: OPT-66B, HumanEval-like code lengths, TP2 x PP2 per phase"),
    "5": dict(geom=syn.OPT_175B, mix="summarization", prompt=0, output=32, batch=8, tp=4, pp=1,
              desc="config 5: OPT-175B, LongBench-like summarization lengths, TP4 -> TP4"),
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="2", choices=sorted(CONFIGS))
    p.add_argument("--batch", type=int, default=0, help="requests per batch (0 = config default)")
    p.add_argument("--prompt", type=int, default=0, help="fixed prompt length override")
    p.add_argument("--output", type=int, default=0, help="decode steps override")
    p.add_argument("--impl", default="ds", choices=["ds", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=6)
    p.add_argument("--stream-layers", action="store_true",
                   help="migrate each layer's pages right after its prefill (NEXT-2; LOCAL/NCCL transports)")
    p.add_argument("--e2e-trace", action="store_true", help="print a per-step copy/compute timeline to stderr")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-graphs", action="store_true", help="eager decode launches (no CUDA graphs)")
    p.add_argument("--packed-migration", action="store_true",
                   help="N>1 NCCL: pack -> send/recv -> unpack through staging (default: zero-copy pool-to-pool "
                        "ds_kv_migrate_contig, the batch's pages being one run of ids at both ends)")
    p.add_argument("--no-fused-migration", action="store_true",
                   help="N=1: prefill into the prefill pool, then a LOCAL page-copy migration (default: the "
                        "prefill kernel stores the pages straight into the decode pool, ds_prefill_attn_push)")
    p.add_argument("--transport", default="nccl", choices=["nccl", "pull", "push"],
                   help="N>1 KV migration: NCCL send/recv (default), one-sided CUDA-IPC pull by the decoder, or "
                        "push: the prefill kernel stores the pages into the decoder's IPC-mapped pool (fused)")
    p.add_argument("--pg-backend", default="nccl", choices=["nccl", "gloo"],
                   help="torch.distributed backend for plumbing (gloo lets 2 ranks share one GPU for rehearsal)")
    p.add_argument("--prefill-instances", type=int, default=0,
                   help="N>1: prefill instances (0 = balance the phases with the roofline cost model)")
    p.add_argument("--profile", action="store_true", help="one short pass for ncu (no JSON)")
    return p.parse_args()


def ncu_traffic(args, w, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture
    of this configuration (profiles/<round>/ncu_traffic.json), else None."""
    import glob
    key = f"config{args.config}_B{w.B}"
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_traffic.json")), reverse=True):
        try:
            d = json.load(open(path))[key][kernel]
            return d["dram_read"] + d["dram_write"]
        except Exception:
            continue
    return None


def load_peaks():
    try:
        return json.load(open(PEAKS_PATH)), "measured"
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
    """One batch of one replica on one rank: prompt lengths, decode steps and the
    rank's local shard (layers of its PP stage, heads of its TP rank)."""

    def __init__(self, cfg: dict, args, role):
        g = cfg["geom"]
        B = args.batch or cfg["batch"]
        mix = "fixed" if args.prompt else cfg["mix"]
        if mix == "fixed":
            lens = [args.prompt or cfg["prompt"]] * B
        elif mix == "chatbot":
            lens = list(syn.lengths_chatbot(0, B)[0])
        elif mix == "code":
            inp = syn.lengths_code(0)[0]
            lens = [int(inp[i % len(inp)]) for i in range(B)]
        else:
            lens = list(syn.lengths_summarization(0, B)[0])
        self.cfg, self.mix, self.geom = cfg, mix, g
        self.B, self.lens = B, [int(x) for x in lens]
        self.out_len = args.output or cfg["output"]
        self.L, self.n, self.d = role.layer_count, role.head_count, g.head_dim
        self.L_full, self.n_full = g.layers, g.heads
        self.T = sum(self.lens)
        self.scale = 1.0 / math.sqrt(self.d)
        self.pages = [-(-l // 16) for l in self.lens]
        self.maxb = -(-(max(self.lens) + self.out_len) // 16)
        self.max_len = max(self.lens)

    def describe(self):
        return (f"{self.cfg['desc']}; {self.B} requests (prompt tokens {self.T}, max {self.max_len}), "
                f"{self.out_len} decode steps; per GPU {self.L} layers x {self.n} heads x {self.d}")

    # algorithmic work
    def prefill_flops_per_layer(self):
        return sum(self.n * 2 * self.d * l * (l + 1) for l in self.lens)

    def prefill_bytes_per_layer(self):
        return 12 * self.n * self.d * self.T

    def decode_bytes(self, ctx):  # one layer, cache lengths ctx (tokens already cached)
        pages = sum(-(-(c + 1) // 16) for c in ctx)
        return sum(self.n * (4 * c * self.d + 12 * self.d) for c in ctx) + 4 * pages

    def kv_payload_bytes(self):  # valid tokens, local layers and heads, K+V
        return 2 * self.L * self.T * self.n * self.d * 2

    def kv_page_bytes(self):  # whole pages actually moved
        return 2 * self.L * sum(self.pages) * 16 * self.n * self.d * 2


def _i32(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()


class Engine:
    """Device state of one rank: pools, resident inputs, staging, CUDA graphs."""

    def __init__(self, w: Workload, role, comm, seed, torch, ds, transport="nccl", stream_layers=False,
                 fused=False, no_contig=False):
        self.w, self.role, self.comm, self.torch, self.ds = w, role, comm, torch, ds
        dev = "cuda"
        bf = torch.bfloat16
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        self.pf = role.phase in ("both", "prefill")
        self.dc = role.phase in ("both", "decode")
        # one batch per pool: the prefill side's pages are reused for batch k+1 only after
        # the (stream-ordered) migration of batch k; the decode side admits k+1 after k ends
        nb_p = sum(w.pages) * (2 * len(role.peers) if (transport == "pull" and role.phase == "prefill") else 1) + 16
        nb_d = sum(-(-(l + w.out_len) // 16) for l in w.lens) + 16
        if transport == "push" and role.phase == "decode":
            nb_d = 2 * nb_d  # the batch being decoded + the next one, admitted ahead and pushed into
        if self.pf:
            self.P = ds.KVCache.empty(w.L, nb_p, w.n, w.d)
            self.pool_p = ds.Pool(nb_p)
            shape = (w.T, w.n, w.d)
            # resident prefill inputs, N(0,1) bf16: distinct buffers rotate over the layers,
            # enough of them (>= 2, >= 1 GB) that no layer's inputs are still in the 126 MB L2
            per_layer = 3 * w.T * w.n * w.d * 2
            n_in = min(w.L, max(2, -(-(1 << 30) // per_layer)))
            self.q = [torch.randn(shape, generator=g, device=dev, dtype=torch.float32).to(bf) for _ in range(n_in)]
            self.k = [torch.randn(shape, generator=g, device=dev, dtype=torch.float32).to(bf) for _ in range(n_in)]
            self.v = [torch.randn(shape, generator=g, device=dev, dtype=torch.float32).to(bf) for _ in range(n_in)]
            self.out = torch.empty(shape, dtype=bf, device=dev)
            self.cu = _i32(torch, syn.cu_seqlens(w.lens))
        if self.dc:
            self.D = ds.KVCache.empty(w.L, nb_d, w.n, w.d)
            self.pool_d = ds.Pool(nb_d)
            dshape = (w.out_len, w.L, w.B, w.n, w.d)
            self.dq = torch.randn(dshape, generator=g, device=dev, dtype=torch.float32).to(bf)
            self.dk = torch.randn(dshape, generator=g, device=dev, dtype=torch.float32).to(bf)
            self.dv = torch.randn(dshape, generator=g, device=dev, dtype=torch.float32).to(bf)
            self.dout = torch.empty((w.out_len, w.B, w.n, w.d), dtype=bf, device=dev)
            self.max_c = w.max_len + w.out_len - 1  # largest cache length of the batch (validation only)
            self.ws = torch.zeros(max(16, ds.ds_decode_workspace_bytes(w.B, w.n, w.d, self.max_c)),
                                  dtype=torch.uint8, device=dev)
            # per-step device block tables / lengths read by the captured decode graphs:
            # the scheduler runs a batch's APPENDs for all its steps up front (fixed output
            # lengths) and uploads them in one copy, so no small per-step H2D copy queues
            # behind bulk transfers on the copy engine
            self.dtab = torch.full((w.out_len, w.B, w.maxb), -1, dtype=torch.int32, device=dev)
            self.dlen = torch.zeros((w.out_len, w.B), dtype=torch.int32, device=dev)
            self.h_tab2 = [torch.empty((w.out_len, w.B, w.maxb), dtype=torch.int32).pin_memory() for _ in range(2)]
            self.h_len2 = [torch.empty((w.out_len, w.B), dtype=torch.int32).pin_memory() for _ in range(2)]
            self.h_ev2 = [None] * 2
            self.hslot = 0
            self.graphs = None
        nblk = sum(w.pages)
        self.transport = "local" if role.phase == "both" else transport
        # a2-a6 fused (ds_prefill_attn_push): with both instances on one GPU the prefill
        # kernel writes the pages straight into the decode pool admitted for the batch
        self.fused = fused and self.transport == "local" and not stream_layers
        self.no_contig = no_contig
        self.contig = None
        # NEXT-2: migrate layer l as soon as its prefill is done, so the
        # transfer overlaps the prefill of the next layers (LOCAL: on a side stream;
        # NCCL: the library's own side stream). PULL stays whole-batch.
        self.stream_layers = stream_layers and self.transport in ("local", "nccl")
        self.mig_stream = torch.cuda.Stream() if (self.stream_layers and self.pf) else None
        self.mrole = {"local": ds.DS_MIGRATE_LOCAL, "pull": ds.DS_MIGRATE_PULL}.get(
            self.transport, ds.DS_MIGRATE_SEND if role.phase == "prefill" else ds.DS_MIGRATE_RECV)
        cache_for_size = self.P if self.pf else self.D
        sbytes = ds.ds_kv_migrate_staging_bytes(cache_for_size, self.mrole, w.L, nblk, w.n)
        self.staging = torch.empty(sbytes, dtype=torch.uint8, device=dev) if sbytes else None
        # pinned host ring for prefill / admission table uploads (async H2D)
        self.ring = 4
        self.h_tab = torch.empty((self.ring, w.B, w.maxb), dtype=torch.int32).pin_memory()
        self.d_tab = torch.empty((self.ring, w.B, w.maxb), dtype=torch.int32, device=dev)
        self.h_ev = [None] * self.ring
        self.d_free = [None] * self.ring  # events: device slot no longer read
        self.slot = 0
        self.copy_stream = None  # e2e: table uploads share the bulk-copy stream
        self.dec_free = None  # event: the decode graphs of the last batch are done with dtab/dlen
        self.launches = 0
        self.layer_hook = None  # e2e: per-layer input copies overlapped with the prefill
        self.step_trace = None  # --e2e-trace: an event after every decode step
        idx = np.concatenate([np.arange(b * w.maxb, b * w.maxb + p) for b, p in enumerate(w.pages)])
        self._idx = _i32(torch, idx).long()

    # -- host -> device block tables ------------------------------------------------
    def _h2d(self, copies, free_ev):
        """Async H2D of small tables; returns the event that marks their arrival.
        With copy_stream set (e2e), they ride the same FIFO stream as the bulk input
        copies: a copy engine serves H2D copies in the order they become ready, so a
        table upload on another stream would wait behind every bulk copy that became
        ready first. free_ev: the device buffer may be overwritten once it completes."""
        torch = self.torch
        if self.copy_stream is None:
            for dst, src in copies:
                dst.copy_(src, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            return ev
        main, cs = torch.cuda.current_stream(), self.copy_stream
        with torch.cuda.stream(cs):
            if free_ev is not None:
                cs.wait_event(free_ev)
            for dst, src in copies:
                dst.copy_(src, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        main.wait_event(ev)
        return ev

    def upload(self, table: np.ndarray):
        s = self.slot
        self.slot = (s + 1) % self.ring
        # every consumer of the previous upload is enqueued by now: its slot is free
        # once the caller's stream gets here
        mark = self.torch.cuda.Event()
        mark.record()
        self.d_free[(s - 1) % self.ring] = mark
        if self.h_ev[s] is not None:
            self.h_ev[s].synchronize()  # the previous copy out of this slot has completed
        self.h_tab[s].numpy()[:] = table
        self.h_ev[s] = self._h2d([(self.d_tab[s], self.h_tab[s])], self.d_free[s])
        return self.d_tab[s]

    def upload_decode(self, tables: np.ndarray, lens: np.ndarray):
        """one async H2D of a batch's per-step decode tables + lengths into the graphs' buffers"""
        i = self.hslot
        self.hslot ^= 1
        if self.h_ev2[i] is not None:
            self.h_ev2[i].synchronize()  # the upload of two batches ago has left this slot
        self.h_tab2[i].numpy()[:] = tables
        self.h_len2[i].numpy()[:] = lens
        self.h_ev2[i] = self._h2d([(self.dtab, self.h_tab2[i]), (self.dlen, self.h_len2[i])], self.dec_free)

    def page_ids(self, table_dev):
        """the batch's page ids in logical order (device gather of the table rows)"""
        return table_dev.reshape(-1).index_select(0, self._idx).contiguous()

    # -- decode ---------------------------------------------------------------------
    def decode_layers(self, s):
        """ds_decode_attn for every local layer of decode step s (reads dtab / dlen)"""
        w, ds = self.w, self.ds
        for layer in range(w.L):
            # layers > 0: the kernel just ahead is layer-1's decode, which writes none of
            # layer's pages, the table or the lengths -> DS_DECODE_EARLY_KV is safe
            ds.ds_decode_attn(self.dq[s, layer], self.dk[s, layer], self.dv[s, layer], self.dout[s], self.D, layer,
                              self.dtab[s], self.dlen[s], self.max_c, w.scale, self.ws, early_kv=layer > 0)

    def capture_decode_graphs(self):
        """one CUDA graph per decode step: the layer loop becomes a single launch"""
        torch = self.torch
        self.graphs = []
        for s in range(self.w.out_len):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.decode_layers(s)
            self.graphs.append(g)
        torch.cuda.synchronize()

    # -- one step -------------------------------------------------------------------
    def _mark(self, marks, label):
        if marks is not None:
            e = self.torch.cuda.Event(enable_timing=True)
            e.record()
            marks.append((label, e))

    def prefill_and_send(self, peer, marks):
        """a1 + a2/a3 for one batch, then a4-a6 towards decode rank `peer`."""
        ds, w = self.ds, self.w
        if self.transport == "push":
            return self.push_batch(peer, marks)
        if self.transport == "pull":
            self.pull_reclaim(peer, keep=1)  # a pool slot for this batch
        tp = np.full((w.B, w.maxb), -1, np.int32)
        ds.ds_block_table(self.pool_p, ds.DS_BT_APPEND, [0] * w.B, w.lens, tp)
        tp_d = self.upload(tp)
        self.contig = self.contig_run(tp)
        src_ids = self.page_ids(tp_d)
        for layer in range(w.L):
            i = layer % len(self.q)
            if self.layer_hook:
                self.layer_hook("before", layer)
            if self.fused:
                ds.ds_prefill_attn_push(self.q[i], self.k[i], self.v[i], self.out, self.cu, w.max_len, self.P, layer,
                                        tp_d, self.D, layer, self.td_dev, w.scale, write_local=False)
            else:
                ds.ds_prefill_attn(self.q[i], self.k[i], self.v[i], self.out, self.cu, w.max_len, self.P, layer,
                                   tp_d, w.scale)
            if self.layer_hook:
                self.layer_hook("after", layer)
            if self.stream_layers:
                self.migrate_layers(peer, src_ids, layer, 1)
        self.launches += w.L
        self._mark(marks, "prefill")
        if self.transport == "pull":  # publish the batch; the decoder fetches it when it has memory
            self.pull_publish(peer, tp)
            self._mark(marks, "migrate")
            return
        if not self.stream_layers and not self.fused:
            self.migrate_layers(peer, src_ids, 0, w.L)
        if self.mig_stream is not None:
            self.torch.cuda.current_stream().wait_stream(self.mig_stream)
        # the pages are free again once the (stream-ordered) migration has read them
        ds.ds_block_table(self.pool_p, ds.DS_BT_FREE, w.lens, None, tp)
        self._mark(marks, "migrate")

    def migrate_layers(self, peer, src_ids, layer_begin, layer_count):
        """a4-a6 for layers [layer_begin, +layer_count) of this batch towards `peer`"""
        ds, w, torch = self.ds, self.w, self.torch
        if self.transport == "local":
            st = self.mig_stream
            if st is not None:
                st.wait_stream(torch.cuda.current_stream())  # the prefill of these layers is done
            with torch.cuda.stream(st if st is not None else torch.cuda.current_stream()):
                ds.ds_kv_migrate(None, self.mrole, 0, self.P, layer_begin, layer_count, src_ids, 0, w.n, None,
                                 dst_cache=self.D, dst_block_ids=self.dst_ids)
            self.launches += 1
        else:
            # streamed per layer: the sends run on a side stream, after this layer's
            # prefill, while the main stream goes on with the next layers
            st = self.mig_stream
            if st is not None:
                st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st if st is not None else torch.cuda.current_stream()):
                if self.contig is not None:  # zero-copy: the batch's pages are one run in both pools
                    ds.ds_kv_migrate_contig(self.comm, self.mrole, peer, self.P, layer_begin, layer_count,
                                            self.contig, sum(w.pages))
                else:
                    ds.ds_kv_migrate(self.comm, self.mrole, peer, self.P, layer_begin, layer_count, src_ids, 0,
                                     w.n, self.staging)
                    self.launches += self.migrate_chunks(layer_count)

    # -- one-sided pull (CUDA IPC) ----------------------------------------------------
    def pull_setup(self, roles, ctl):
        """Exchange pool / event handles: prefill ranks export their pool and one
        'ready' event per (decoder, slot); decoders export one 'done' event per slot."""
        import torch.distributed as dist
        ds, w, role = self.ds, self.w, self.role
        self.ctl = ctl
        info = {"rank": role.rank}
        if role.phase == "prefill":
            self.ready = {p: [ds.IpcEvent() for _ in range(2)] for p in role.peers}
            h, off = ds.ds_ipc_export_mem(self.P.tensor)
            info.update(pool=(h, off, self.P.num_blocks), ready={p: [e.handle for e in evs] for p, evs in self.ready.items()})
        else:
            self.done = [ds.IpcEvent() for _ in range(2)]
            info.update(done=[e.handle for e in self.done])
        self.pending = []  # outstanding non-blocking control messages (work, tensor)
        allinfo = [None] * role.world
        dist.all_gather_object(allinfo, info, group=ctl)
        if role.phase == "prefill":
            self.peer_done = {p: [ds.IpcEvent(hd) for hd in allinfo[p]["done"]] for p in role.peers}
            self.inflight = {p: [] for p in role.peers}
            self.sent = {p: 0 for p in role.peers}
        else:
            src = allinfo[role.peer]
            h, off, nb = src["pool"]
            self.remote = ds.RemoteKVCache(h, off, w.L, nb, w.n, w.d)
            self.peer_ready = [ds.IpcEvent(hd) for hd in src["ready"][role.rank]]
            self.recvd = 0

    def pull_publish(self, peer, tp):
        torch, w = self.torch, self.w
        k = self.sent[peer]
        self.ready[peer][k % 2].record()
        ids = torch.from_numpy(np.concatenate([[k], tp[:, :max(w.pages)].reshape(-1)]).astype(np.int32))
        # non-blocking: a blocking send here could wait on a decoder that is itself
        # blocked handing back its 'done' for an earlier batch
        self.pending.append((torch.distributed.isend(ids, peer, group=self.ctl), ids))
        self.inflight[peer].append((k, tp))
        self.sent[peer] = k + 1

    def pull_reclaim(self, peer, keep):
        """free this decoder's batches once it has pulled them (at most `keep` left in flight... 2 slots)"""
        torch, ds, w = self.torch, self.ds, self.w
        while len(self.inflight[peer]) > keep:
            k, tp = self.inflight[peer].pop(0)
            msg = torch.zeros(1, dtype=torch.int32)
            torch.distributed.recv(msg, peer, group=self.ctl)
            assert int(msg[0]) == k, (int(msg[0]), k)
            self.peer_done[peer][k % 2].wait()  # the decoder's pull kernel has read the pages
            ds.ds_block_table(self.pool_p, ds.DS_BT_FREE, w.lens, None, tp)

    def pull_drain(self):
        if self.transport != "pull":
            return
        if self.role.phase == "prefill":
            for peer in self.role.peers:
                self.pull_reclaim(peer, keep=0)
        for work, _ in self.pending:
            work.wait()
        self.pending = []

    # -- fused push (CUDA IPC): the prefill kernel stores into the decoder's pool ----------
    def push_setup(self, roles, ctl):
        """Decoders export their pool and one 'free' event per slot; prefill ranks map
        every peer's pool and export one 'ready' event per (decoder, slot)."""
        import torch.distributed as dist
        ds, w, role = self.ds, self.w, self.role
        self.ctl = ctl
        info = {"rank": role.rank}
        if role.phase == "prefill":
            self.ready = {p: [ds.IpcEvent() for _ in range(2)] for p in role.peers}
            info.update(ready={p: [e.handle for e in evs] for p, evs in self.ready.items()})
        else:
            self.free = [ds.IpcEvent() for _ in range(2)]
            h, off = ds.ds_ipc_export_mem(self.D.tensor)
            info.update(pool=(h, off, self.D.num_blocks), free=[e.handle for e in self.free])
        self.pending = []
        allinfo = [None] * role.world
        dist.all_gather_object(allinfo, info, group=ctl)
        if role.phase == "prefill":
            self.remotes = {p: ds.RemoteKVCache(*allinfo[p]["pool"][:2], w.L, allinfo[p]["pool"][2], w.n, w.d)
                            for p in role.peers}
            self.peer_free = {p: [ds.IpcEvent(hd) for hd in allinfo[p]["free"]] for p in role.peers}
        else:
            self.peer_ready = [ds.IpcEvent(hd) for hd in allinfo[role.peer]["ready"][role.rank]]
            self.announced = []  # host tables of admitted batches, in order
            self.recvd = 0

    def push_announce(self):
        """decoder: admit the next batch (pages for its prompts) and send the table to
        the prefill rank, which pushes the pages straight into them"""
        torch, ds, w = self.torch, self.ds, self.w
        td = np.full((w.B, w.maxb), -1, np.int32)
        ds.ds_block_table(self.pool_d, ds.DS_BT_APPEND, [0] * w.B, w.lens, td)
        k = self.recvd + len(self.announced)
        msg = torch.from_numpy(np.concatenate([[k], td.reshape(-1)]).astype(np.int32))
        self.pending.append((torch.distributed.isend(msg, self.role.peer, group=self.ctl), msg))
        self.announced.append(td)

    def push_batch(self, peer, marks):
        """prefill rank: receive the decoder's table of batch k, then prefill with the
        page stores going into its pool (ds_prefill_attn_push, write_local = 0)"""
        ds, w, torch = self.ds, self.w, self.torch
        msg = torch.zeros(1 + w.B * w.maxb, dtype=torch.int32)
        torch.distributed.recv(msg, peer, group=self.ctl)
        k = int(msg[0])
        td = msg[1:].numpy().reshape(w.B, w.maxb)
        tp = np.full((w.B, w.maxb), -1, np.int32)
        ds.ds_block_table(self.pool_p, ds.DS_BT_APPEND, [0] * w.B, w.lens, tp)
        tp_d, td_d = self.upload(tp), self.upload(td)
        if k >= 2:
            self.peer_free[peer][k % 2].wait()  # batch k-2 (same pages' slot parity) has been decoded
        for layer in range(w.L):
            i = layer % len(self.q)
            if self.layer_hook:
                self.layer_hook("before", layer)
            ds.ds_prefill_attn_push(self.q[i], self.k[i], self.v[i], self.out, self.cu, w.max_len, self.P, layer,
                                    tp_d, self.remotes[peer], layer, td_d, w.scale, write_local=False)
            if self.layer_hook:
                self.layer_hook("after", layer)
        self.launches += w.L
        self._mark(marks, "prefill")
        self.ready[peer][k % 2].record()
        note = torch.tensor([k], dtype=torch.int32)
        self.pending.append((torch.distributed.isend(note, peer, group=self.ctl), note))
        ds.ds_block_table(self.pool_p, ds.DS_BT_FREE, w.lens, None, tp)
        self._mark(marks, "migrate")

    def push_drain(self):
        """after the timed loop: every decoder announced one batch ahead; the prefill
        ranks take those tables without pushing, decoders return the pages"""
        if self.transport != "push":
            return
        torch, w = self.torch, self.w
        if self.role.phase == "prefill":
            for peer in self.role.peers:
                msg = torch.zeros(1 + w.B * w.maxb, dtype=torch.int32)
                torch.distributed.recv(msg, peer, group=self.ctl)
        else:
            for td in self.announced:
                self.ds.ds_block_table(self.pool_d, self.ds.DS_BT_FREE, w.lens, None, td)
            self.announced = []
        for work, _ in self.pending:
            work.wait()
        self.pending = []

    def receive(self, marks):
        """decode rank: admit the batch, then migrate it in (NCCL recv, or PULL)"""
        ds, w, role, torch = self.ds, self.w, self.role, self.torch
        if self.transport == "push":
            if not self.announced:
                self.push_announce()
            self.push_announce()  # the next batch's pages, pushed while this one decodes
            note = torch.zeros(1, dtype=torch.int32)
            torch.distributed.recv(note, role.peer, group=self.ctl)
            k = int(note[0])
            assert k == self.recvd, (k, self.recvd)
            self.peer_ready[k % 2].wait()  # the prefill kernels of batch k have stored its pages
            self.td = self.announced.pop(0)
            self.recvd = k + 1
            self._mark(marks, "migrate")
            return
        if self.transport == "pull":
            ids = torch.zeros(1 + w.B * max(w.pages), dtype=torch.int32)
            torch.distributed.recv(ids, role.peer, group=self.ctl)
            k = int(ids[0])
            assert k == self.recvd, (k, self.recvd)
            tab = ids[1:].numpy().reshape(w.B, max(w.pages))
            src = np.concatenate([tab[b, :p] for b, p in enumerate(w.pages)])
            self.admit()
            self.peer_ready[k % 2].wait()  # the prefill of this batch has finished
            ds.ds_kv_migrate(None, ds.DS_MIGRATE_PULL, 0, self.remote, 0, w.L, _i32(torch, src), 0, w.n, None,
                             dst_cache=self.D, dst_block_ids=self.dst_ids)
            self.done[k % 2].record()
            msg = torch.tensor([k], dtype=torch.int32)
            self.pending.append((torch.distributed.isend(msg, role.peer, group=self.ctl), msg))
            self.recvd = k + 1
            self.launches += 1
        else:
            self.admit()
            # the receiver posts the same per-layer (or whole-batch) calls as its sender
            per = [(l, 1) for l in range(w.L)] if self.stream_layers else [(0, w.L)]
            for l0, nl in per:
                if self.contig is not None:
                    ds.ds_kv_migrate_contig(self.comm, self.mrole, role.peer, self.D, l0, nl, self.contig,
                                            sum(w.pages))
                else:
                    ds.ds_kv_migrate(self.comm, self.mrole, role.peer, self.D, l0, nl, self.dst_ids, 0, w.n,
                                     self.staging)
                    self.launches += self.migrate_chunks(nl)
        self._mark(marks, "migrate")

    def migrate_chunks(self, layers):
        w = self.w
        chunk_rows = max(1, (64 << 20) // (w.n * 16 * w.d * 2))
        return -(-(2 * layers * sum(w.pages)) // chunk_rows)  # pack or unpack kernels (+ NCCL's own)

    def contig_run(self, table):
        """NCCL transport: first id if the batch's pages (logical order) are one run of
        consecutive ids — always, since each pool holds one batch at a time and hands
        out the lowest free ids — so the zero-copy ds_kv_migrate_contig applies; both
        ends decide the same way (their pools are built alike), else None"""
        if self.transport != "nccl" or self.no_contig:
            return None
        ids = np.concatenate([table[b, :p] for b, p in enumerate(self.w.pages)])
        run = self.ds.contiguous_run(ids)
        if run is None:
            raise RuntimeError("batch pages are not one run: the zero-copy migration would mismatch its peer")
        return run

    def admit(self):
        """decode-side admission of one batch (pull): pages for the prompts"""
        ds, w = self.ds, self.w
        self.td = np.full((w.B, w.maxb), -1, np.int32)
        ds.ds_block_table(self.pool_d, ds.DS_BT_APPEND, [0] * w.B, w.lens, self.td)
        self.td_dev = self.upload(self.td)
        self.dst_ids = self.page_ids(self.td_dev)
        self.contig = self.contig_run(self.td)

    def decode_batch(self, marks):
        """a1 (APPEND per step) + a7/a8 for `output` steps, then FREE"""
        ds, w = self.ds, self.w
        cur = list(w.lens)
        tabs = np.empty((w.out_len, w.B, w.maxb), np.int32)
        lens = np.empty((w.out_len, w.B), np.int32)
        for s in range(w.out_len):  # a1: one APPEND per step (a page whenever a sequence crosses 16k)
            ds.ds_block_table(self.pool_d, ds.DS_BT_APPEND, cur, [1] * w.B, self.td)
            tabs[s], lens[s] = self.td, cur
            cur = [c + 1 for c in cur]
        self.upload_decode(tabs, lens)
        for s in range(w.out_len):
            if self.graphs is not None:
                self.graphs[s].replay()
            else:
                self.decode_layers(s)
            if self.step_trace is not None:
                ev = self.torch.cuda.Event(enable_timing=True)
                ev.record()
                self.step_trace.append(ev)
            self.launches += w.L  # one decode_kernel per layer (split merge fused)
        self.dec_free = self.torch.cuda.Event()
        self.dec_free.record()
        ds.ds_block_table(self.pool_d, ds.DS_BT_FREE, cur, None, self.td)
        self._mark(marks, "decode")

    def step(self, marks=None):
        """N=1: one batch through prefill -> LOCAL migrate -> decode.
        prefill rank: one batch per decoding rank it feeds (round-robin dispatch).
        decode rank: receive one batch, decode it."""
        ds, w, role = self.ds, self.w, self.role
        self._mark(marks, "start")
        if role.phase == "both":
            self.admit()
            self.prefill_and_send(0, marks)
            self.decode_batch(marks)
        elif role.phase == "prefill":
            for peer in role.peers:
                self.prefill_and_send(peer, marks)
        else:
            self.receive(marks)
            self.decode_batch(marks)
            if self.transport == "push":
                self.free[(self.recvd - 1) % 2].record()  # batch recvd-1's pages are read


# ----------------------------------------------------------------------------- distributed
def dist_setup(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        if args.pg_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return world, rank, local


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ----------------------------------------------------------------------------- CPU oracle
def oracle_sample_tok_s(w: Workload, target_s: float = 15.0):
    """Time the fp64 C oracle (as it stands) on a bounded sample of the same
    workload and scale linearly to tok/s: prefill of the batch's longest request
    over all local heads of one layer, plus decode steps of it over one layer.
    Work is linear in layers and heads; requests are scaled by their cost share
    (l(l+1) for prefill, context length for decode)."""
    import oracle
    threads = os.cpu_count() or 1
    l0 = w.max_len
    b = syn.prefill_batch(0, [l0], w.n, w.d)
    t0 = time.perf_counter()
    oracle.prefill(b.q, b.k, b.v, b.cu_seqlens, w.scale, nthreads=threads)
    t_pf = time.perf_counter() - t0
    cols = -(-(l0 + w.out_len + 1) // 16)
    pool = oracle.Pool(1, cols + 1, w.n, w.d)
    table = np.full((1, cols), -1, np.int32)
    pool.append([0], [l0], table)
    pool.write_prefill(0, b.k, b.v, b.cu_seqlens, table)
    n_dec, t_dec, c = 0, 0.0, l0
    while n_dec < w.out_len and t_dec < target_s:
        pool.append([c], [1], table)
        db = syn.decode_batch(n_dec, 1, w.n, w.d)
        t0 = time.perf_counter()
        pool.decode(0, db.q, db.k_new, db.v_new, table, [c], w.scale, nthreads=threads)
        t_dec += time.perf_counter() - t0
        c += 1
        n_dec += 1
    pf_all = t_pf * sum(l * (l + 1) for l in w.lens) / (l0 * (l0 + 1))
    dec_all = (t_dec / n_dec) * w.out_len * sum(w.lens) / l0
    per_batch = w.L_full * (w.n_full / w.n) * (pf_all + dec_all)  # all layers and heads of the model
    tok_s = (w.T + w.B * w.out_len) / per_batch
    sample = (f"1 request ({l0} tokens) x 1 layer x {w.n} heads: prefill ({t_pf:.2f} s) + {n_dec} decode steps "
              f"({t_dec:.2f} s) with {threads} threads; scaled linearly to the batch and all "
              f"{w.L_full} layers x {w.n_full} heads")
    return tok_s, threads, sample


# ----------------------------------------------------------------------------- arms
def _config_line(w, world, replicas, roles=None):
    tp, pp = (1, 1) if world == 1 else (w.cfg["tp"], w.cfg["pp"])
    n_p = 0 if world == 1 else sum(1 for r in roles if r.phase == "prefill") // (tp * pp)
    return {"workload": w.describe(), "batch": w.B, "prompt_tokens": w.T, "max_prompt": w.max_len,
            "decode_steps": w.out_len, "mix": w.mix, "decode_instances": replicas, "prefill_instances": n_p,
            "tp": tp, "pp": pp,
            "parallelism": "single GPU (P+D)" if world == 1 else
            f"{n_p} prefill : {replicas} decode instances, TP{tp} PP{pp} each (round-robin dispatch)",
            "l2": "inputs larger than L2; no flush"}


def stage_costs(cfg, args):
    """Roofline estimate (s) of one batch on a prefill rank (prefill + send) and on
    a decoding rank (receive + decode) — the latency model that picks the split."""
    from paper_2401_09670_b200.pairing import assign
    g = cfg["geom"]
    tp, pp = cfg["tp"], cfg["pp"]
    role = assign(0, 2 * tp * pp, g.layers, g.heads, tp, pp)
    w = Workload(cfg, args, role)
    peaks, _ = load_peaks()
    hbm, tc, nvl = 0.7 * peaks["hbm_gbs"] * 1e9, 0.5 * peaks["bf16_tflops"] * 1e12, 0.7 * NVLINK_GBS * 1e9
    mig = w.kv_page_bytes() / nvl
    t_p = w.L * max(w.prefill_flops_per_layer() / tc, w.prefill_bytes_per_layer() / hbm) + mig
    t_d = sum(w.decode_bytes([c + s for c in w.lens]) for s in range(w.out_len)) * w.L / (0.85 * peaks["hbm_gbs"] * 1e9) + mig
    return t_p, t_d


def roles_for(cfg, world, args):
    from paper_2401_09670_b200 import pairing
    g = cfg["geom"]
    if world == 1:
        return [pairing.assign(0, 1, g.layers, g.heads)]
    tp, pp = cfg["tp"], cfg["pp"]
    n_p = args.prefill_instances
    if n_p <= 0:
        t_p, t_d = stage_costs(cfg, args)
        n_p = pairing.balanced_prefill_instances(world, tp, pp, t_p, t_d)
    return pairing.all_roles(world, g.layers, g.heads, tp, pp, n_p)


def _role_for(cfg, rank, world, args=None):
    if args is None:
        from paper_2401_09670_b200.pairing import assign
        g = cfg["geom"]
        return assign(0, 1, g.layers, g.heads) if world == 1 else \
            assign(rank, world, g.layers, g.heads, cfg["tp"], cfg["pp"])
    return roles_for(cfg, world, args)[rank]


def run_reference(args):
    """--impl reference: the oracle as it stands on the host cores, same config and metric."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    w = Workload(cfg, args, _role_for(cfg, 0, world))
    vals, sample, threads = [], "", 1
    for _ in range(max(args.steps, 1)):
        tok_s, threads, sample = oracle_sample_tok_s(w, target_s=4.0)
        vals.append(tok_s)
    v = statistics.median(vals)
    replicas = 1 if world == 1 else world // 2 // (cfg["tp"] * cfg["pp"])
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tok/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": (w.T + w.B * w.out_len) / v * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config_line(w, world, replicas),
            "cpu_baseline": {"value": v, "unit": "tok/s", "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ds(args):
    import torch
    world, rank, local = dist_setup(args)
    import paper_2401_09670_b200 as ds
    from paper_2401_09670_b200 import pairing
    cfg = CONFIGS[args.config]
    roles = roles_for(cfg, world, args)
    role = roles[rank]
    w = Workload(cfg, args, role)
    if world == 1 or args.transport in ("pull", "push"):
        comm = None  # one GPU (fused / LOCAL) or CUDA-IPC pull / push: no NCCL communicator
    else:
        import torch.distributed as dist
        comm = ds.ds_comm_init(pairing.bootstrap_unique_id(ds.ds_comm_get_unique_id, rank, world, dist), world, rank)
    replicas = 1 if world == 1 else sum(1 for r in roles if r.phase == "decode") // (cfg["tp"] * cfg["pp"])
    eng = Engine(w, role, comm, seed=1234 + role.replica * 7919 + role.stage * 131 + role.tp_rank, torch=torch,
                 ds=ds, transport=args.transport, stream_layers=args.stream_layers,
                 fused=not args.no_fused_migration, no_contig=args.packed_migration)
    if world > 1 and args.transport in ("pull", "push"):
        import torch.distributed as dist
        ctl = dist.group.WORLD if args.pg_backend == "gloo" else dist.new_group(backend="gloo")
        (eng.pull_setup if args.transport == "pull" else eng.push_setup)(roles, ctl)
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
    eng.step()  # one more warm-up step on every rank (graph replay on decoders; keeps the pairs in step)
    torch.cuda.synchronize()
    barrier(world)
    sampler = ClockSampler(local)
    sampler.start()
    phase = []
    eng.launches = 0
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    t_start.record()
    for _ in range(args.steps):
        marks = []
        eng.step(marks)
        phase.append(marks)
    t_end.record()
    torch.cuda.synchronize()
    barrier(world)
    clocks = sampler.stop()
    total_ms = max_over_ranks(t_start.elapsed_time(t_end), world)
    ms_step = total_ms / args.steps
    n_dec = 1 if world == 1 else sum(1 for r in roles if r.phase == "decode") // (cfg["tp"] * cfg["pp"])
    value = n_dec * (w.T + w.B * w.out_len) / (ms_step / 1e3)

    peaks, peak_kind = load_peaks()
    comp = {"phase": role.phase}

    def phase_ms(label):  # median over steps of the summed device time of `label` segments
        per_step = []
        for marks in phase:
            t = sum(marks[k - 1][1].elapsed_time(marks[k][1]) for k in range(1, len(marks)) if marks[k][0] == label)
            per_step.append(t)
        return statistics.median(per_step)
    nb = len(role.peers) if role.phase == "prefill" else 1  # batches this rank handles per step
    if eng.pf:
        pf_ms = phase_ms("prefill") / nb
        comp["prefill_ms_per_batch"] = pf_ms
        comp["prefill_tok_s_per_gpu"] = w.T / (pf_ms / 1e3)
        comp["prefill_tflops"] = w.L * w.prefill_flops_per_layer() / (pf_ms / 1e3) / 1e12
        comp["prefill_frac_of_tensor_peak"] = comp["prefill_tflops"] / peaks["bf16_tflops"]
        # the prefill runs inside a long step (every layer's prefill, then the decode
        # graphs), so the sustained bf16 figure is its denominator; the burst one
        # (a kernel timed alone) is kept beside it
        sustained = peaks.get("bf16_tflops_sustained", FALLBACK_PEAKS["bf16_tflops_sustained"])
        comp["prefill_frac_of_tensor_peak_sustained"] = comp["prefill_tflops"] / sustained
        comp["prefill_tensor_peaks_tflops"] = {"burst": peaks["bf16_tflops"], "sustained": sustained}
        t_roof = w.L * max(w.prefill_flops_per_layer() / (peaks["bf16_tflops"] * 1e12),
                           w.prefill_bytes_per_layer() / (peaks["hbm_gbs"] * 1e9))
        comp["prefill_frac_of_attainable_roofline"] = t_roof / (pf_ms / 1e3)
    if eng.pf and eng.stream_layers:
        # per-layer migration is issued inside the prefill loop: the prefill segment holds
        # both, the migrate segment only the tail the last layers' transfer adds
        comp["migration"] = "streamed per layer (overlaps prefill)"
        comp["prefill_with_migration_ms_per_batch"] = pf_ms + phase_ms("migrate") / nb
        comp["migrate_tail_ms_per_batch"] = phase_ms("migrate") / nb
    elif world > 1 and args.transport == "push":
        comp["kv_migrate_path"] = ("fused into the prefill kernel: its page stores go into the decoder's "
                                   "IPC-mapped pool over NVLink (ds_prefill_attn_push)")
    elif (role.phase != "decode" or world > 1) and not (args.transport == "pull" and role.phase == "prefill"):
        mig_ms = phase_ms("migrate") / nb  # (a pull prefill rank only publishes; its decoders move the bytes)
        comp["migrate_ms_per_batch"] = mig_ms
        if eng.fused:  # no separate pass: the page bytes are part of the prefill kernel's writes
            comp["kv_migrate_GBps"] = comp["kv_migrate_page_GBps"] = None
        else:
            comp["kv_migrate_GBps"] = w.kv_payload_bytes() / (mig_ms / 1e3) / 1e9
            comp["kv_migrate_page_GBps"] = w.kv_page_bytes() / (mig_ms / 1e3) / 1e9
        comp["kv_migrate_path"] = ("fused into the prefill kernel: pages stored straight into the decode pool "
                                   "(ds_prefill_attn_push)" if eng.fused else
                                   "LOCAL page copy (one GPU)" if world == 1 else
                                   ("NCCL p2p over NVLink, pool to pool (zero-copy)" if eng.contig is not None
                                    else "NCCL p2p over NVLink (pack / unpack via staging)")
                                   if args.transport == "nccl" else
                                   "one-sided pull: decoder's kernel reads the IPC-mapped prefill pool")
        if world > 1:
            comp["kv_migrate_frac_of_nvlink"] = comp["kv_migrate_page_GBps"] / NVLINK_GBS
    dec_kernel = None
    if eng.dc:
        dec_ms = phase_ms("decode")
        comp["decode_ms_per_batch"] = dec_ms
        comp["decode_tok_s_per_gpu"] = w.B * w.out_len / (dec_ms / 1e3)
        ctx_steps = [[c + s for c in w.lens] for s in range(w.out_len)]
        avg_bytes = sum(w.decode_bytes(c) for c in ctx_steps) / w.out_len
        avg_ms = dec_ms / (w.out_len * w.L)  # device time per ds_decode_attn call (incl. table upload, gaps)
        dec_kernel = (avg_bytes, avg_ms)
        comp["decode_attn_GBps"] = avg_bytes / (avg_ms / 1e3) / 1e9
        comp["decode_attn_frac_of_hbm"] = comp["decode_attn_GBps"] / peaks["hbm_gbs"]
        comp["decode_attn_us_per_launch"] = avg_ms * 1e3
        comp["decode_graphs"] = eng.graphs is not None
    roofline = None  # the dominant kernel of this rank's step
    dec_name = ds.ds_decode_kernel(w.B, w.n) if eng.dc else "decode_kernel"
    traffic = ncu_traffic(args, w, dec_name)
    if dec_kernel:
        achieved = dec_kernel[0] / (dec_kernel[1] / 1e3) / 1e9
        roofline = {"kernel": f"ds_decode_attn ({dec_name}, split merge fused)", "bound": "hbm",
                    "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                    "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
                    "peak_note": DECODE_PEAK_NOTE, "algorithmic_bytes_per_launch": dec_kernel[0]}
    elif eng.pf:
        t_layer = comp["prefill_ms_per_batch"] / w.L / 1e3
        fl, by = w.prefill_flops_per_layer(), w.prefill_bytes_per_layer()
        if fl / by >= peaks["bf16_tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9):
            roofline = {"kernel": "ds_prefill_attn (prefill_kernel)", "bound": "tensor",
                        "achieved": fl / t_layer / 1e12, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                        "frac": fl / t_layer / 1e12 / peaks["bf16_tflops"], "traffic": None}
        else:
            roofline = {"kernel": "ds_prefill_attn (prefill_kernel)", "bound": "hbm", "achieved": by / t_layer / 1e9,
                        "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": by / t_layer / 1e9 / peaks["hbm_gbs"],
                        "traffic": None}
    paper = {"note": "end-to-end serving figures of the paper on 32 x A100-80GB (context, not a target): "
                     "up to 7.4x more requests and 12.6x tighter SLO than vLLM (P:33); KV transfer < 0.1% of "
                     "latency, > 95% of OPT-175B requests < 30 ms (P:512); 1.13 GB KV per OPT-66B 512-token "
                     "request (P:265)", "goodput_x_vs_vllm": 7.4, "slo_x_vs_vllm": 12.6}
    line = {"metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": _config_line(w, world, replicas, roles), "components": comp, "roofline": roofline,
            "clocks": clocks, "gpu_launches": eng.launches, "paper_context": paper}
    eng.pull_drain()
    eng.push_drain()
    if world > 1 and args.transport != "push":  # push: the migration is inside the prefill kernel
        comp.update(measure_migration(eng, w, world, torch))
    elif world == 1 and eng.transport == "local":
        comp.update(measure_local_migration(eng, w, torch))
    if not args.no_e2e:
        line["e2e"] = run_e2e(args, eng, w, world, replicas, torch)
        eng.pull_drain()
        eng.push_drain()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        tok_s, threads, sample = oracle_sample_tok_s(w)
        line["cpu_baseline"] = {"value": tok_s, "unit": "tok/s", "cores": threads, "kind": "oracle",
                                "sample": sample}
    if world > 1:  # every rank's components (prefill ranks report migrate, decode ranks decode)
        import torch.distributed as dist
        objs = [None] * world
        dist.all_gather_object(objs, comp)
        line["components_by_rank"] = {str(r): c for r, c in enumerate(objs)}
        decs = [c for c in objs if "decode_attn_GBps" in c]
        if decs:  # the decode kernel dominates the job; report it from the first decode rank
            d0 = decs[0]
            line["roofline"] = {"kernel": f"ds_decode_attn ({ds.ds_decode_kernel(w.B, w.n)}, split merge fused)",
                                "bound": "hbm",
                                "achieved": d0["decode_attn_GBps"], "peak": peaks["hbm_gbs"], "unit": "GB/s",
                                "frac": d0["decode_attn_GBps"] / peaks["hbm_gbs"], "traffic": None, "peak_note": DECODE_PEAK_NOTE,
                                "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if os.environ.get("DS_DECODE_TRACE_OUT"):  # -DDS_TRACE builds only: the last decode launch's warp timeline
        import ctypes
        import numpy as np
        f = ctypes.CDLL(ds.LIB_PATH).ds_debug_decode_trace
        f.argtypes = [ctypes.c_void_p, ctypes.c_int]
        buf = np.zeros(f(None, 0), np.uint64)
        f(buf.ctypes.data, 0)
        np.save(os.environ["DS_DECODE_TRACE_OUT"], buf)
    if comm is not None:
        comm.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def measure_migration(eng, w, world, torch, reps=3):
    """N>1: the KV migration alone, all pairs in lockstep after a barrier (the
    pipelined step also contains waits for the peer, so its migrate segments
    understate the link). NCCL: per prefill rank, page bytes sent / device time.
    PULL: per decoding rank, page bytes pulled / device time."""
    ds, role = eng.ds, eng.role
    pull = eng.transport == "pull"
    if eng.pf:
        tp = np.full((w.B, w.maxb), -1, np.int32)
        ds.ds_block_table(eng.pool_p, ds.DS_BT_APPEND, [0] * w.B, w.lens, tp)
        src_ids = eng.page_ids(eng.upload(tp))
        if pull:
            for peer in role.peers:  # publish the same pages to every decoder it feeds
                ids = torch.from_numpy(np.concatenate([[-1], tp[:, :max(w.pages)].reshape(-1)]).astype(np.int32))
                eng.pending.append((torch.distributed.isend(ids, peer, group=eng.ctl), ids))
    else:
        eng.admit()
        if pull:
            ids = torch.zeros(1 + w.B * max(w.pages), dtype=torch.int32)
            torch.distributed.recv(ids, role.peer, group=eng.ctl)
            tab = ids[1:].numpy().reshape(w.B, max(w.pages))
            pull_src = _i32(torch, np.concatenate([tab[b, :p] for b, p in enumerate(w.pages)]))
    run = None if pull else eng.contig_run(tp if eng.pf else eng.td)
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        if pull:
            if not eng.pf:
                ds.ds_kv_migrate(None, ds.DS_MIGRATE_PULL, 0, eng.remote, 0, w.L, pull_src, 0, w.n, None,
                                 dst_cache=eng.D, dst_block_ids=eng.dst_ids)
        elif eng.pf:
            for peer in role.peers:
                if run is not None:  # the step's default: zero-copy pool to pool
                    ds.ds_kv_migrate_contig(eng.comm, eng.mrole, peer, eng.P, 0, w.L, run, sum(w.pages))
                else:
                    ds.ds_kv_migrate(eng.comm, eng.mrole, peer, eng.P, 0, w.L, src_ids, 0, w.n, eng.staging)
        elif run is not None:
            ds.ds_kv_migrate_contig(eng.comm, eng.mrole, role.peer, eng.D, 0, w.L, run, sum(w.pages))
        else:
            ds.ds_kv_migrate(eng.comm, eng.mrole, role.peer, eng.D, 0, w.L, eng.dst_ids, 0, w.n, eng.staging)
    e1.record()
    torch.cuda.synchronize()
    barrier(world)
    ms = e0.elapsed_time(e1)
    if eng.pf:
        ds.ds_block_table(eng.pool_p, ds.DS_BT_FREE, w.lens, None, tp)
    else:
        ds.ds_block_table(eng.pool_d, ds.DS_BT_FREE, w.lens, None, eng.td)
    eng.pull_drain()
    if pull and eng.pf:
        return {}
    nb = len(role.peers) if eng.pf else 1
    gbps = reps * nb * w.kv_page_bytes() / (ms / 1e3) / 1e9
    return {"kv_migrate_isolated_GBps": gbps, "kv_migrate_isolated_frac_of_nvlink": gbps / NVLINK_GBS,
            "kv_migrate_isolated_ms_per_batch": ms / (reps * nb)}


def measure_local_migration(eng, w, torch, reps=3):
    """N=1: the one-GPU step fuses the migration into the prefill kernel (no pass of its
    own); this times the separate LOCAL page copy (ds_kv_migrate LOCAL, prefill pool ->
    decode pool, one batch, all layers) alone, for the migrate metric at one GPU."""
    ds, peaks = eng.ds, load_peaks()[0]
    tp = np.full((w.B, w.maxb), -1, np.int32)
    ds.ds_block_table(eng.pool_p, ds.DS_BT_APPEND, [0] * w.B, w.lens, tp)
    src_ids = eng.page_ids(eng.upload(tp))
    eng.admit()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ds.ds_kv_migrate(None, ds.DS_MIGRATE_LOCAL, 0, eng.P, 0, w.L, src_ids, 0, w.n, None, dst_cache=eng.D,
                     dst_block_ids=eng.dst_ids)  # warm-up
    e0.record()
    for _ in range(reps):
        ds.ds_kv_migrate(None, ds.DS_MIGRATE_LOCAL, 0, eng.P, 0, w.L, src_ids, 0, w.n, None, dst_cache=eng.D,
                         dst_block_ids=eng.dst_ids)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ds.ds_block_table(eng.pool_p, ds.DS_BT_FREE, w.lens, None, tp)
    ds.ds_block_table(eng.pool_d, ds.DS_BT_FREE, w.lens, None, eng.td)
    gbps = w.kv_page_bytes() / (ms / 1e3) / 1e9
    return {"kv_migrate_local_GBps": gbps, "kv_migrate_local_ms_per_batch": ms,
            "kv_migrate_local_frac_of_hbm": 2 * gbps / peaks["hbm_gbs"],
            "kv_migrate_local_note": "one-GPU LOCAL page copy (prefill pool -> decode pool) timed alone; reads and "
                                     "writes each page once, so its HBM roofline is 2 x bytes / copy peak; the "
                                     "bench step itself fuses the migration into the prefill kernel"}


def run_e2e(args, eng, w, world, replicas, torch):
    """The same step through the same API, but every layer's prefill inputs and
    every decode step's inputs are copied host(pinned)->device inside the timed
    region, and the decode outputs are read back."""
    bf = torch.bfloat16
    h2d = d2h = 0
    host = {}
    if eng.pf:
        host["qkv"] = torch.randn((3, w.T, w.n, w.d), dtype=torch.float32).to(bf).pin_memory()
    if eng.dc:
        host["dec"] = torch.randn((3,) + tuple(eng.dq.shape), dtype=torch.float32).to(bf).pin_memory()
        host["out"] = torch.empty(tuple(eng.dout.shape), dtype=bf).pin_memory()

    # host->device copies ride a separate stream so PCIe overlaps the kernels:
    # layer l's inputs land in rotating buffer l % n_in, and a copy into buffer i
    # waits only until the prefill that last read buffer i is done — so the next
    # batch's prompt copies stream in while this batch decodes (PCIe stays busy).
    main, cs = torch.cuda.current_stream(), torch.cuda.Stream()
    if eng.pf:  # more landing buffers (free HBM permitting) so the copies can run a whole decode ahead
        per_buf = 3 * eng.q[0].numel() * 2
        spare = max(0, torch.cuda.mem_get_info()[0] - (12 << 30)) // per_buf
        for _ in range(min(w.L, 24) - len(eng.q)):
            if spare <= 0:
                break
            for lst in (eng.q, eng.k, eng.v):
                lst.append(torch.empty_like(lst[0]))
            spare -= 1
    n_in = len(eng.q) if eng.pf else 0
    copied = [torch.cuda.Event() for _ in range(w.L)]
    buf_free = [None] * n_in  # event: the last prefill reading buffer i has finished

    trace = []  # --e2e-trace: (label, event) on the stream that does the work
    step_traces = []  # --e2e-trace: per batch, decode-step completion times (ms from decode start)

    def tmark(label, stream):
        if args.e2e_trace:
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            trace.append((label, e))

    def copy_layer(layer):
        nonlocal h2d
        i = layer % n_in
        with torch.cuda.stream(cs):
            if buf_free[i] is not None:
                cs.wait_event(buf_free[i])
            if layer in (0, w.L - 1):
                tmark(f"copy{layer}", cs)
            eng.q[i].copy_(host["qkv"][0], non_blocking=True)
            eng.k[i].copy_(host["qkv"][1], non_blocking=True)
            eng.v[i].copy_(host["qkv"][2], non_blocking=True)
            copied[layer].record(cs)
        h2d += 3 * host["qkv"][0].numel() * 2

    def hook(when, layer):
        if when == "before":
            main.wait_event(copied[layer])
        else:
            ev = torch.cuda.Event()
            ev.record(main)
            buf_free[layer % n_in] = ev
            if layer + n_in < w.L:
                copy_layer(layer + n_in)

    def copy_prefill_inputs():
        for layer in range(min(n_in, w.L)):
            copy_layer(layer)

    dec_ready = torch.cuda.Event()

    def decode_io(after):
        nonlocal h2d, d2h
        if not after:
            with torch.cuda.stream(cs):
                cs.wait_stream(main)
                eng.dq.copy_(host["dec"][0], non_blocking=True)
                eng.dk.copy_(host["dec"][1], non_blocking=True)
                eng.dv.copy_(host["dec"][2], non_blocking=True)
                dec_ready.record(cs)
            h2d += 3 * eng.dq.numel() * 2
        else:
            host["out"].copy_(eng.dout, non_blocking=True)
            d2h += eng.dout.numel() * 2

    def decode_after_inputs():
        main.wait_event(dec_ready)
        tmark("decode", main)
        if args.e2e_trace:
            eng.step_trace = []
        eng.decode_batch(None)
        tmark("decode_end", main)
        if args.e2e_trace:
            step_traces.append((trace[-2][1], eng.step_trace))
            eng.step_trace = None

    def step():  # Engine.step with the host <-> device traffic of every batch
        role = eng.role
        eng.layer_hook = hook if eng.pf else None
        if role.phase == "both":
            eng.admit()
            copy_prefill_inputs()  # prompt copies before the decode inputs: they wait on prefill, not decode
            decode_io(False)
            tmark("prefill", main)
            eng.prefill_and_send(0, None)
            decode_after_inputs()
            decode_io(True)
        elif role.phase == "prefill":
            for peer in role.peers:
                copy_prefill_inputs()
                eng.prefill_and_send(peer, None)
        else:
            decode_io(False)
            eng.receive(None)
            decode_after_inputs()
            decode_io(True)
        eng.layer_hook = None

    eng.copy_stream = cs
    step()
    torch.cuda.synchronize()
    h2d = d2h = 0
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.e2e_steps):
        step()
    main.wait_stream(cs)
    e1.record()
    torch.cuda.synchronize()
    eng.copy_stream = None
    if trace:
        t0 = trace[0][1]
        sys.stderr.write("e2e trace (ms): " + " ".join(f"{l}@{t0.elapsed_time(e):.1f}" for l, e in trace) + "\n")
        for t0, evs in step_traces:
            sys.stderr.write(f"e2e decode steps (ms): {[round(t0.elapsed_time(e), 1) for e in evs]}\n")
    ms = max_over_ranks(e0.elapsed_time(e1), world) / args.e2e_steps
    if world > 1:  # whole-job host <-> device bytes
        import torch.distributed as dist
        t = torch.tensor([float(h2d), float(d2h)], dtype=torch.float64,
                         device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t)
        h2d, d2h = int(t[0].item()), int(t[1].item())
    return {"value": replicas * (w.T + w.B * w.out_len) / (ms / 1e3), "unit": "tok/s",
            "h2d_bytes_per_step": h2d // args.e2e_steps, "d2h_bytes_per_step": d2h // args.e2e_steps,
            "ms_per_step": ms, "steps": args.e2e_steps,
            # the end-to-end step is bound by the host -> device link: every step's inputs
            # (each layer's Q/K/V and every decode step's q/k_new/v_new) cross it once
            "h2d_GBps": (h2d // args.e2e_steps) / (ms / 1e3) / 1e9 / max(1, world),
            "bound": "host->device copies (pinned H2D; tools/h2d_probe.py measures the link)"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ds(args)


if __name__ == "__main__":
    main()
