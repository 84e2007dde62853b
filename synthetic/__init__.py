"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no attention, no softmax, no
paging): it only draws random numbers and rounds them to the bf16 bit patterns
that both `oracle/` and the CUDA path consume, plus the request-length mixes
that stand in for the paper's datasets.

Everything is deterministic under its seed (numpy PCG64).

Citations (PAPER.md line numbers, `P:n`):
  * OPT head geometries: P:454 (OPT-13B/66B/175B), hidden sizes per BASELINE.json.
  * Dataset stand-ins: ShareGPT chatbot P:456, HumanEval code completion P:457,
    LongBench summarisation P:458 (inputs capped so input+output <= 2048).
    The paper only plots the length distributions (fig:dataset; image
    missing) so the parameters below are OUR assumptions, fixed for comparability.
"""
from __future__ import annotations

import dataclasses
import numpy as np

BLOCK_SIZE = 16  # KV page size in tokens (BASELINE.json; the paper never states one)


@dataclasses.dataclass(frozen=True)
class Geometry:
    name: str
    layers: int
    heads: int
    head_dim: int

    @property
    def hidden(self) -> int:
        return self.heads * self.head_dim


# BASELINE.json configs; SURVEY.md §8 "Geometries".
TINY = Geometry("config1-tiny", 1, 4, 64)
OPT_13B = Geometry("OPT-13B", 40, 40, 128)
OPT_66B = Geometry("OPT-66B", 64, 72, 128)
OPT_175B = Geometry("OPT-175B", 96, 96, 128)
GEOMETRIES = {g.name: g for g in (TINY, OPT_13B, OPT_66B, OPT_175B)}


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round float32 values to bf16 (round-to-nearest-even); return uint16 bits.

    Input-representation helper only (how the synthetic numbers are stored);
    inputs are finite by construction."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return rounded.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bits to float32 (for building inputs/fixtures)."""
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def normal_bf16(seed: int, shape, sigma: float = 1.0) -> np.ndarray:
    """N(0, sigma^2) drawn in float32 then rounded to bf16 bits."""
    g = rng(seed)
    return f32_to_bf16_bits(g.standard_normal(size=shape, dtype=np.float32) * np.float32(sigma))


def cu_seqlens(lens) -> np.ndarray:
    lens = np.asarray(lens, dtype=np.int64)
    out = np.zeros(len(lens) + 1, dtype=np.int32)
    out[1:] = np.cumsum(lens)
    return out


@dataclasses.dataclass
class PrefillBatch:
    lens: np.ndarray        # int32 [B]
    cu_seqlens: np.ndarray  # int32 [B+1]
    q: np.ndarray           # uint16 bf16 bits [T][n][d]
    k: np.ndarray
    v: np.ndarray


def prefill_batch(seed: int, lens, heads: int, head_dim: int, q_sigma: float = 1.0,
                  kv_sigma: float = 1.0) -> PrefillBatch:
    lens = np.asarray(lens, dtype=np.int32)
    T = int(lens.sum())
    shape = (T, heads, head_dim)
    return PrefillBatch(lens=lens, cu_seqlens=cu_seqlens(lens),
                        q=normal_bf16(seed * 3 + 0, shape, q_sigma),
                        k=normal_bf16(seed * 3 + 1, shape, kv_sigma),
                        v=normal_bf16(seed * 3 + 2, shape, kv_sigma))


@dataclasses.dataclass
class DecodeBatch:
    q: np.ndarray      # uint16 [B][n][d]
    k_new: np.ndarray
    v_new: np.ndarray


def decode_batch(seed: int, batch: int, heads: int, head_dim: int, q_sigma: float = 1.0) -> DecodeBatch:
    shape = (batch, heads, head_dim)
    return DecodeBatch(q=normal_bf16(seed * 3 + 100001, shape, q_sigma),
                       k_new=normal_bf16(seed * 3 + 100002, shape),
                       v_new=normal_bf16(seed * 3 + 100003, shape))


# ---------------------------------------------------------------------------
# Length mixes (SURVEY.md §8(d) "Concrete synthetic inputs"). Our assumptions.
# ---------------------------------------------------------------------------
MAX_CONTEXT = 2048  # OPT learned positions; LongBench capped at 2048 (P:458 footnote)


def lengths_chatbot(seed: int, n: int):
    """ShareGPT stand-in: input ~ LogNormal(median 256, sigma 1.0) clipped
    [4, 2048-out]; output ~ LogNormal(median 128, sigma 1.0) clipped [1, 1024]."""
    g = rng(seed)
    out = np.clip(np.round(np.exp(np.log(128.0) + g.standard_normal(n))), 1, 1024).astype(np.int32)
    inp = np.round(np.exp(np.log(256.0) + g.standard_normal(n)))
    inp = np.clip(inp, 4, MAX_CONTEXT - out).astype(np.int32)
    return inp, out


def lengths_code(seed: int = 0, n: int = 164):
    """HumanEval stand-in (P:457, 164 problems): input ~ N(160, 60) clipped
    [32, 512]; output ~ N(120, 60) clipped [8, 384]."""
    g = rng(seed)
    inp = np.clip(np.round(g.normal(160.0, 60.0, n)), 32, 512).astype(np.int32)
    out = np.clip(np.round(g.normal(120.0, 60.0, n)), 8, 384).astype(np.int32)
    return inp, out


def lengths_summarization(seed: int, n: int):
    """LongBench stand-in: input 70% U[1792,1920], 30% U[512,1792];
    output ~ LogNormal(median 128, sigma 0.5) clipped [16, 256]; in+out <= 2048."""
    g = rng(seed)
    long_mask = g.random(n) < 0.7
    inp = np.where(long_mask, g.integers(1792, 1921, n), g.integers(512, 1793, n))
    out = np.clip(np.round(np.exp(np.log(128.0) + 0.5 * g.standard_normal(n))), 16, 256)
    inp = np.minimum(inp, MAX_CONTEXT - out)
    return inp.astype(np.int32), out.astype(np.int32)


def pack_prefill_batches(inp_lens, token_budget: int = 8192):
    """Greedy in-order grouping of prompts into prefill batches whose total stays
    <= token_budget (the L_m-style batching of P:377); a prompt longer than the
    budget forms its own batch. Returns a list of index lists."""
    batches, cur, tot = [], [], 0
    for i, l in enumerate(inp_lens):
        l = int(l)
        if cur and tot + l > token_budget:
            batches.append(cur)
            cur, tot = [], 0
        cur.append(i)
        tot += l
    if cur:
        batches.append(cur)
    return batches


def decode_snapshot_contexts(seed: int, inp, out):
    """Decode-batch snapshot: context = input + U[0, output-1]."""
    g = rng(seed)
    inp = np.asarray(inp, dtype=np.int64)
    out = np.asarray(out, dtype=np.int64)
    return (inp + g.integers(0, np.maximum(out, 1))).astype(np.int32)


def fragmented_free_order(seed: int, num_blocks: int, num_prefree: int):
    """Block ids to pre-allocate-then-free in a random order, so that the pool is
    fragmented before the test allocates (T1 'fragmented pools')."""
    g = rng(seed)
    return g.permutation(num_blocks)[:num_prefree].astype(np.int32)
