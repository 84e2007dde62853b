"""Multi-process host logic on CPU (gloo, world_size 2 and 4): rank roles and
prefill<->decode pairing, the NCCL unique-id bootstrap
through torch.distributed, and the max-over-ranks timing reduction used by
bench.py. The NCCL data path itself needs GPUs (tests/test_gpu_parity.py covers
SELF/LOCAL on one GPU)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2401_09670_b200 import pairing


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        role = pairing.assign(rank, world, layers=40, heads=40)
        # unique id: rank 0's bytes reach everybody unchanged
        uid = pairing.bootstrap_unique_id(lambda: bytes(range(128)) if rank == 0 else None, rank, world, dist)
        # max over ranks (bench.py reduces the device time this way)
        t = torch.tensor([float(rank + 1) * 1.5], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        # each pair exchanges its (layer, head) ranges: they must agree (corresponding layers)
        mine = torch.tensor([role.layer_begin, role.layer_count, role.head_begin, role.head_count])
        theirs = torch.zeros_like(mine)
        if role.phase == "prefill":
            dist.send(mine, role.peer)
            dist.recv(theirs, role.peer)
        else:
            dist.recv(theirs, role.peer)
            dist.send(mine, role.peer)
        q.put((rank, role.phase, role.peer, uid, float(t.item()), bool(torch.equal(mine, theirs))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_pairing_bootstrap_and_max(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    half = world // 2
    for rank, phase, peer, uid, tmax, same in res:
        assert phase == ("prefill" if rank < half else "decode")
        assert peer == (rank + half if rank < half else rank - half)
        assert uid == bytes(range(128))
        assert tmax == world * 1.5
        assert same


@pytest.mark.parametrize("world,layers,heads,tp,pp", [
    (1, 40, 40, 1, 1), (2, 40, 40, 1, 1), (8, 40, 40, 1, 1),   # config 3: 1:1 .. 4:4 replicas
    (8, 64, 72, 2, 2),                                          # config 4: OPT-66B TP2 x PP2 per phase
    (8, 96, 96, 4, 1),                                          # config 5: OPT-175B TP4 -> TP4
])
def test_placements_pair_corresponding_layers_and_heads(world, layers, heads, tp, pp):
    roles = pairing.all_roles(world, layers, heads, tp, pp)
    pairing.check_pairing(roles)
    if world > 1:
        per_phase = sum(r.layer_count * r.head_count for r in roles if r.phase == "prefill")
        assert per_phase == (world // 2) // (tp * pp) * layers * heads
    if (tp, pp) == (2, 2):
        r = pairing.assign(5, 8, layers, heads, tp, pp)  # decode rank 5 = replica 0, stage 0, tp 1
        assert (r.stage, r.tp_rank, r.layer_begin, r.layer_count, r.head_begin, r.head_count) == (0, 1, 0, 32, 36, 36)
        assert r.peer == 1


@pytest.mark.parametrize("world,n_p", [(4, 1), (8, 1), (8, 2), (8, 3), (3, 1)])
def test_unequal_prefill_decode_split(world, n_p):
    roles = pairing.all_roles(world, 40, 40, n_prefill=n_p)
    pairing.check_pairing(roles)
    pre = [r for r in roles if r.phase == "prefill"]
    dec = [r for r in roles if r.phase == "decode"]
    assert len(pre) == n_p and len(dec) == world - n_p
    loads = sorted(len(r.peers) for r in pre)
    assert loads[-1] - loads[0] <= 1  # round-robin dispatch balances the decoders per prefill rank


def test_balanced_split_follows_stage_costs():
    # decode 6x costlier than prefill: 1 prefill rank for up to ~7 ranks
    assert pairing.balanced_prefill_instances(2, 1, 1, 1.0, 6.0) == 1
    assert pairing.balanced_prefill_instances(8, 1, 1, 1.0, 6.0) == 1
    assert pairing.balanced_prefill_instances(8, 1, 1, 1.0, 1.0) == 4
    assert pairing.balanced_prefill_instances(8, 1, 1, 3.0, 1.0) == 6
    assert pairing.balanced_prefill_instances(8, 2, 2, 1.0, 1.0) == 1


def test_bad_placements_rejected():
    for args in ((3, 40, 40, 1, 1), (4, 40, 40, 3, 1), (8, 40, 40, 1, 3), (6, 40, 40, 2, 1)):
        with pytest.raises(ValueError):
            pairing.all_roles(*args)
    with pytest.raises(ValueError):
        pairing.all_roles(4, 40, 40, n_prefill=4)  # no decoding instance


@pytest.mark.parametrize("layers,heads,prefill,decode", [
    (40, 40, (2, 1), (1, 1)),    # OPT-13B: P TP2 -> D TP1
    (64, 72, (4, 1), (2, 2)),    # OPT-66B: P TP4 -> D TP2 PP2
    (96, 96, (3, 3), (4, 3)),    # OPT-175B: P TP3 PP3 -> D TP4 PP3
    (8, 12, (3, 2), (2, 4)),     # odd mix: both TP and PP differ
    (4, 4, (1, 1), (1, 1)),
])
def test_reshard_plan_covers_everything_once(layers, heads, prefill, decode):
    plan = pairing.reshard_plan(layers, heads, prefill, decode)
    pairing.check_reshard(plan, layers, heads, prefill, decode)


def test_reshard_plan_175b_overlaps():
    # TP3 -> TP4 over 96 heads: decode rank (tp 1) gets heads 24..31 from P tp0 and 32..47 from P tp1
    plan = [p for p in pairing.reshard_plan(96, 96, (3, 3), (4, 3)) if p.dst == 9 + 1]
    assert [(p.src, p.global_head_begin, p.head_count) for p in plan] == [(0, 24, 8), (1, 32, 16)]
    assert all(p.layer_count == 32 and p.src_layer_begin == 0 and p.dst_layer_begin == 0 for p in plan)
