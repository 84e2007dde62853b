"""Rank roles and prefill->decode pairing for the disaggregated data path.

Host-side plumbing only (no kernels): which GPU is a prefill or a decode
instance, which layers and heads it owns, and which peer it migrates KV pages
with. Follows the paper's placement structure:
  * disaggregation: prefill and decoding instances run on disjoint GPUs
    (PAPER.md P:150-152); ranks [0, N/2) are prefill, [N/2, N) decode;
  * intra-op (tensor) parallelism divides the heads: rank t of a TP group owns
    heads [t*n/tp, (t+1)*n/tp) (reading R11);
  * inter-op (pipeline) parallelism groups layers into stages; stage k owns
    layers [k*L/pp, (k+1)*L/pp) (reading R12);
  * "KV cache transfer occurs exclusively between corresponding layers"
    (P:363): the prefill rank (replica, stage, tp) pairs with the decode rank
    (replica, stage, tp) — same layer range, same head range;
  * replication: independent (prefill, decode) instance pairs.
Both phases use the same (tp, pp) here (BASELINE configs 3-5; reading R18);
TP-mismatched resharding is SURVEY §8f NEXT-1.
"""
from __future__ import annotations

import dataclasses


@dataclasses.dataclass(frozen=True)
class RankRole:
    rank: int
    world: int
    phase: str          # "prefill", "decode", or "both" (N = 1: one GPU plays both)
    replica: int        # instance pair index
    stage: int          # PP stage within the instance
    tp_rank: int        # TP rank within the stage
    peer: int           # the rank this one migrates pages with
    layer_begin: int
    layer_count: int
    head_begin: int
    head_count: int


def assign(rank: int, world: int, layers: int, heads: int, tp: int = 1, pp: int = 1) -> RankRole:
    """Role of `rank` among `world` ranks for a model with `layers` x `heads`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if heads % tp or layers % pp:
        raise ValueError(f"tp={tp} must divide heads={heads} and pp={pp} must divide layers={layers}")
    per_inst = tp * pp
    if world == 1:
        if per_inst != 1:
            raise ValueError("one GPU hosts a single TP1/PP1 instance pair")
        return RankRole(0, 1, "both", 0, 0, 0, 0, 0, layers, 0, heads)
    if world % 2 or (world // 2) % per_inst:
        raise ValueError(f"world={world} must be 2 x (replicas x tp x pp = {per_inst})")
    half = world // 2
    phase = "prefill" if rank < half else "decode"
    local = rank % half
    replica, idx = divmod(local, per_inst)
    stage, tp_rank = divmod(idx, tp)
    peer = rank + half if phase == "prefill" else rank - half
    lc, hc = layers // pp, heads // tp
    return RankRole(rank, world, phase, replica, stage, tp_rank, peer, stage * lc, lc, tp_rank * hc, hc)


def all_roles(world: int, layers: int, heads: int, tp: int = 1, pp: int = 1):
    return [assign(r, world, layers, heads, tp, pp) for r in range(world)]


def check_pairing(roles) -> None:
    """Invariants of a placement: symmetric pairs, corresponding layer and head
    ranges, every (layer, head) of every replica covered exactly once per phase."""
    by_rank = {r.rank: r for r in roles}
    for r in roles:
        if r.phase == "both":
            continue
        p = by_rank[r.peer]
        assert p.peer == r.rank and p.phase != r.phase
        assert (p.replica, p.stage, p.tp_rank) == (r.replica, r.stage, r.tp_rank)
        assert (p.layer_begin, p.layer_count, p.head_begin, p.head_count) == \
               (r.layer_begin, r.layer_count, r.head_begin, r.head_count)
    cover = {}
    for r in roles:
        for l in range(r.layer_begin, r.layer_begin + r.layer_count):
            for h in range(r.head_begin, r.head_begin + r.head_count):
                key = (r.phase, r.replica, l, h)
                assert key not in cover, f"(layer {l}, head {h}) owned twice"
                cover[key] = r.rank


def bootstrap_unique_id(get_id, rank: int, world: int, dist=None) -> bytes:
    """Rank 0 creates the 128-byte NCCL unique id; it reaches every rank through
    torch.distributed (any backend). `get_id` is ds_comm_get_unique_id."""
    if world == 1:
        return get_id()
    obj = [get_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]
