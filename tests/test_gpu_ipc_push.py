"""Fused prefill + migration across processes (CUDA IPC), on one GPU (-m gpu).

This "decoding instance" process admits a batch into its (fragmented) pool and
exports the pool; a spawned "prefill instance" maps it and runs
ds_prefill_attn_push: the prefill kernel's TMA page stores land directly in the
other process's allocation (across GPUs the same stores cross NVLink), then it
records an inter-process event. After waiting on it, the decoding side's pages
must be bit-exact with the oracle and one decode step within tolerance
(P:233 the decode instance receives the KV caches; P:407 transfers that avoid
blocking the computation)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

import paper_2401_09670_b200 as ds  # noqa: E402
import synthetic as syn  # noqa: E402
from gpu_util import i32, pages_match, to_bits, to_dev, to_f64  # noqa: E402

pytestmark = pytest.mark.gpu
LENS, N, D, L = [70, 33, 129, 1], 4, 128, 2


def _ceil(a, b):
    return -(-a // b)


def _prefill_instance(q_in, q_out):
    import paper_2401_09670_b200 as ds
    torch.cuda.set_device(0)
    handle, off, nb_d, td = q_in.get(timeout=300)
    remote = ds.RemoteKVCache(handle, off, L, nb_d, N, D)
    b = syn.prefill_batch(43, LENS, N, D)
    cache = ds.KVCache.empty(L, 40, N, D)  # the prefill pool (not written: write_local = False)
    cache.tensor.zero_()
    pool = ds.Pool(40)
    table = np.full((len(LENS), 9), -1, np.int32)
    ds.ds_block_table(pool, ds.DS_BT_APPEND, [0] * len(LENS), LENS, table)
    out = torch.empty((sum(LENS), N, D), dtype=torch.bfloat16, device="cuda")
    for layer in range(L):
        ds.ds_prefill_attn_push(to_dev(b.q), to_dev(b.k), to_dev(b.v), out, i32(b.cu_seqlens), max(LENS), cache,
                                layer, i32(table), remote, layer, i32(td), 1 / math.sqrt(D), write_local=False)
    ev = ds.IpcEvent()
    ev.record()
    torch.cuda.synchronize()
    untouched = bool((cache.tensor.view(torch.int16) == 0).all())
    q_out.put((ev.handle, untouched))
    assert q_in.get(timeout=300) == "done"
    remote.close()


def test_push_migration_across_processes(oracle_mod):
    ctx = mp.get_context("spawn")
    q_in, q_out = ctx.Queue(), ctx.Queue()
    child = ctx.Process(target=_prefill_instance, args=(q_in, q_out))
    child.start()
    try:
        dcache = ds.KVCache.empty(L, 48, N, D)
        dcache.tensor.view(torch.int16).fill_(0x7FC0)  # never-written slots: NaN
        dpool = ds.Pool(48)
        opool_d = oracle_mod.Pool(L, 48, N, D)
        junk = np.full((5, 1), -1, np.int32)
        ds.ds_block_table(dpool, ds.DS_BT_APPEND, [0] * 5, [16] * 5, junk)
        opool_d.append([0] * 5, [16] * 5, junk.copy())
        maxb = _ceil(max(LENS) + 1, 16)
        td = np.full((len(LENS), maxb), -1, np.int32)
        tdo = td.copy()
        ds.ds_block_table(dpool, ds.DS_BT_APPEND, [0] * len(LENS), LENS, td)  # admission before the prefill
        opool_d.append([0] * len(LENS), LENS, tdo)
        handle, off = ds.ds_ipc_export_mem(dcache.tensor)
        q_in.put((handle, off, 48, td))
        ev_handle, untouched = q_out.get(timeout=300)
        assert untouched, "write_local = False must leave the prefill pool untouched"
        ready = ds.IpcEvent(ev_handle)
        ready.wait()
        torch.cuda.synchronize()
        b = syn.prefill_batch(43, LENS, N, D)
        for layer in range(L):
            opool_d.write_prefill(layer, b.k, b.v, b.cu_seqlens, tdo)
        bits = to_bits(dcache.tensor)
        for layer in range(L):
            assert pages_match(bits, opool_d, layer, LENS, td)
        ds.ds_block_table(dpool, ds.DS_BT_APPEND, LENS, [1] * len(LENS), td)
        opool_d.append(LENS, [1] * len(LENS), tdo)
        db = syn.decode_batch(78, len(LENS), N, D)
        o = torch.empty((len(LENS), N, D), dtype=torch.bfloat16, device="cuda")
        ws = torch.zeros(ds.ds_decode_workspace_bytes(len(LENS), N, D, max(LENS)), dtype=torch.uint8, device="cuda")
        ds.ds_decode_attn(to_dev(db.q), to_dev(db.k_new), to_dev(db.v_new), o, dcache, 1, i32(td), i32(LENS),
                          max(LENS), 1 / math.sqrt(D), ws)
        ref = opool_d.decode(1, db.q, db.k_new, db.v_new, tdo, LENS, 1 / math.sqrt(D))
        assert oracle_mod.max_rel_err(to_f64(o), ref) <= 5e-3
        q_in.put("done")
        ready.close()
    finally:
        child.join(timeout=120)
    assert child.exitcode == 0
