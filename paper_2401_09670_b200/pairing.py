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
  * replication: independent (prefill, decode) instance pairs;
  * unequal phase sizes: "allocation of multiple prefill instances to a single
    decoding instance" — and, for attention-only work where decode
    dominates, one prefill instance feeding several decoding instances; each
    prefill instance dispatches its batches round-robin over the decoding
    instances it serves (FCFS to the least-loaded decoder, degenerates
    to round-robin for equal batches). The split is chosen from the workload's
    roofline cost (`balanced_prefill_instances`), as the paper's placement
    step chooses it from its latency model.
`assign` uses the same (tp, pp) in both phases (BASELINE configs 3-5; reading
R18). `reshard_plan` covers the placements the paper actually chose, where the
phases differ (Table tab:parallel_config: 13B P-TP2 -> D-TP1; 66B
P-TP4 -> D-TP2 PP2; 175B P-TP3 PP3 -> D-TP4 PP3): each decode
rank receives the intersection of its (layer, head) rectangle with every prefill
rank's rectangle.
"""
from __future__ import annotations

import dataclasses


@dataclasses.dataclass(frozen=True)
class RankRole:
    rank: int
    world: int
    phase: str          # "prefill", "decode", or "both" (N = 1: one GPU plays both)
    replica: int        # instance index within its phase
    stage: int          # PP stage within the instance
    tp_rank: int        # TP rank within the stage
    peer: int           # decode: the prefill rank it receives from; prefill: its first decode peer
    layer_begin: int
    layer_count: int
    head_begin: int
    head_count: int
    peers: tuple = ()   # prefill: every decode rank it feeds, in dispatch order


def assign(rank: int, world: int, layers: int, heads: int, tp: int = 1, pp: int = 1,
           n_prefill: int | None = None) -> RankRole:
    """Role of `rank` among `world` ranks for a model with `layers` x `heads`.

    n_prefill = number of prefill INSTANCES (each tp*pp ranks); default world/2
    ranks' worth (1:1). Instances [0, n_prefill) are prefill, the rest decode;
    decode instance j receives from prefill instance j % n_prefill."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if heads % tp or layers % pp:
        raise ValueError(f"tp={tp} must divide heads={heads} and pp={pp} must divide layers={layers}")
    per_inst = tp * pp
    if world == 1:
        if per_inst != 1:
            raise ValueError("one GPU hosts a single TP1/PP1 instance pair")
        return RankRole(0, 1, "both", 0, 0, 0, 0, 0, layers, 0, heads, (0,))
    if world % per_inst:
        raise ValueError(f"world={world} must be a multiple of tp x pp = {per_inst}")
    n_inst = world // per_inst
    if n_prefill is None:
        if n_inst % 2:
            raise ValueError(f"world={world} must be 2 x (instances x tp x pp = {per_inst}) for 1:1 pairs")
        n_prefill = n_inst // 2
    if not 1 <= n_prefill < n_inst:
        raise ValueError(f"need 1 <= prefill instances ({n_prefill}) < instances ({n_inst})")
    n_decode = n_inst - n_prefill
    inst, idx = divmod(rank, per_inst)
    stage, tp_rank = divmod(idx, tp)
    lc, hc = layers // pp, heads // tp
    if inst < n_prefill:
        served = tuple((n_prefill + j) * per_inst + idx for j in range(n_decode) if j % n_prefill == inst)
        if not served:
            raise ValueError(f"prefill instance {inst} feeds no decoding instance ({n_prefill}:{n_decode})")
        return RankRole(rank, world, "prefill", inst, stage, tp_rank, served[0], stage * lc, lc, tp_rank * hc, hc,
                        served)
    j = inst - n_prefill
    peer = (j % n_prefill) * per_inst + idx
    return RankRole(rank, world, "decode", j, stage, tp_rank, peer, stage * lc, lc, tp_rank * hc, hc, (peer,))


def balanced_prefill_instances(world: int, tp: int, pp: int, t_prefill: float, t_decode: float) -> int:
    """Prefill instances that balance the two phases for a workload whose one
    batch costs t_prefill on a prefill instance and t_decode on a decoding one
    (throughput = min(n_p / t_prefill, n_d / t_decode)); at least one of each."""
    n_inst = world // (tp * pp)
    if n_inst < 2:
        raise ValueError("need at least one prefill and one decoding instance")
    best, best_tp = 1, -1.0
    for n_p in range(1, n_inst):
        thr = min(n_p / t_prefill, (n_inst - n_p) / t_decode)
        if thr > best_tp + 1e-12:
            best, best_tp = n_p, thr
    return best


def all_roles(world: int, layers: int, heads: int, tp: int = 1, pp: int = 1, n_prefill: int | None = None):
    return [assign(r, world, layers, heads, tp, pp, n_prefill) for r in range(world)]


def check_pairing(roles) -> None:
    """Invariants of a placement: every decode rank receives from exactly one
    prefill rank that lists it; the two hold corresponding layer and head ranges
    (P:363); every (layer, head) of every instance is covered exactly once."""
    by_rank = {r.rank: r for r in roles}
    for r in roles:
        if r.phase == "decode":
            p = by_rank[r.peer]
            assert p.phase == "prefill" and r.rank in p.peers
            assert (p.stage, p.tp_rank) == (r.stage, r.tp_rank)
            assert (p.layer_begin, p.layer_count, p.head_begin, p.head_count) == \
                   (r.layer_begin, r.layer_count, r.head_begin, r.head_count)
        elif r.phase == "prefill":
            for d in r.peers:
                assert by_rank[d].phase == "decode" and by_rank[d].peer == r.rank
    fed = [d for r in roles if r.phase == "prefill" for d in r.peers]
    assert len(fed) == len(set(fed)) == sum(r.phase == "decode" for r in roles)
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


@dataclasses.dataclass(frozen=True)
class ReshardSlice:
    """Pages of `layer_count` layers x `head_count` heads moving from prefill rank
    `src` to decode rank `dst`; begins are LOCAL indices in each rank's pool."""
    src: int
    dst: int
    src_layer_begin: int
    dst_layer_begin: int
    layer_count: int
    src_head_begin: int
    dst_head_begin: int
    head_count: int
    global_layer_begin: int
    global_head_begin: int


def reshard_plan(layers: int, heads: int, prefill=(1, 1), decode=(1, 1)):
    """Migration plan from ONE prefill instance (tp_p x pp_p ranks 0..) to ONE
    decoding instance (tp_d x pp_d ranks following it), rank = stage * tp + tp_rank
    inside each instance; KV moves only between corresponding layers and
    TP ranks hold contiguous head ranges (R11). Returns the slices sorted by
    (dst, src)."""
    (tp_p, pp_p), (tp_d, pp_d) = prefill, decode
    for tp, pp in (prefill, decode):
        if heads % tp or layers % pp:
            raise ValueError(f"tp={tp}/pp={pp} must divide heads={heads}/layers={layers}")
    lp, hp, ld, hd = layers // pp_p, heads // tp_p, layers // pp_d, heads // tp_d
    n_src = tp_p * pp_p
    out = []
    for d in range(tp_d * pp_d):
        sd, td = divmod(d, tp_d)
        for s in range(n_src):
            sp, tpp = divmod(s, tp_p)
            l0, l1 = max(sd * ld, sp * lp), min((sd + 1) * ld, (sp + 1) * lp)
            h0, h1 = max(td * hd, tpp * hp), min((td + 1) * hd, (tpp + 1) * hp)
            if l0 < l1 and h0 < h1:
                out.append(ReshardSlice(s, n_src + d, l0 - sp * lp, l0 - sd * ld, l1 - l0, h0 - tpp * hp,
                                        h0 - td * hd, h1 - h0, l0, h0))
    return out


def check_reshard(plan, layers: int, heads: int, prefill=(1, 1), decode=(1, 1)) -> None:
    """Every (layer, head) of every decode rank arrives exactly once, from the
    prefill rank that computed it, at the same global (layer, head)."""
    (tp_p, pp_p), (tp_d, pp_d) = prefill, decode
    lp, hp, ld, hd = layers // pp_p, heads // tp_p, layers // pp_d, heads // tp_d
    n_src = tp_p * pp_p
    got = {}
    for sl in plan:
        sp, tpp = divmod(sl.src, tp_p)
        sd, td = divmod(sl.dst - n_src, tp_d)
        for dl in range(sl.layer_count):
            for dh in range(sl.head_count):
                g_src = (sp * lp + sl.src_layer_begin + dl, tpp * hp + sl.src_head_begin + dh)
                g_dst = (sd * ld + sl.dst_layer_begin + dl, td * hd + sl.dst_head_begin + dh)
                assert g_src == g_dst, (sl, g_src, g_dst)
                assert 0 <= sl.src_layer_begin + dl < lp and 0 <= sl.src_head_begin + dh < hp
                assert 0 <= sl.dst_layer_begin + dl < ld and 0 <= sl.dst_head_begin + dh < hd
                key = (sl.dst, g_dst)
                assert key not in got, f"{key} delivered twice"
                got[key] = sl.src
    assert len(got) == tp_d * pp_d * ld * hd  # == layers * heads: everything arrives
