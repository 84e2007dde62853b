"""One-sided PULL migration across processes (CUDA IPC), on one GPU (-m gpu).

A spawned "prefill instance" process runs ds_prefill_attn into its pool, records
an inter-process event and exports the pool; this "decoding instance" process
maps the pool, waits on the event, pulls the pages into its own (fragmented)
pool with ds_kv_migrate(DS_MIGRATE_PULL) and decodes one step — pages must be
bit-exact with the oracle and the decode output within tolerance (P:382 pull,
P:407 asynchronous copies)."""
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
LENS, N, D, L = [70, 33, 129], 4, 128, 2


def _ceil(a, b):
    return -(-a // b)


def _prefill_instance(q_out, q_in):
    import paper_2401_09670_b200 as ds
    torch.cuda.set_device(0)
    b = syn.prefill_batch(41, LENS, N, D)
    cache = ds.KVCache.empty(L, 40, N, D)
    pool = ds.Pool(40)
    junk = np.full((1, 1), -1, np.int32)
    ds.ds_block_table(pool, ds.DS_BT_APPEND, [0], [16 * 3], np.full((1, 3), -1, np.int32))  # offset the ids
    table = np.full((len(LENS), 9), -1, np.int32)
    ds.ds_block_table(pool, ds.DS_BT_APPEND, [0] * len(LENS), LENS, table)
    out = torch.empty((sum(LENS), N, D), dtype=torch.bfloat16, device="cuda")
    for layer in range(L):
        ds.ds_prefill_attn(to_dev(b.q), to_dev(b.k), to_dev(b.v), out, i32(b.cu_seqlens), max(LENS), cache, layer,
                           i32(table), 1 / math.sqrt(D))
    ev = ds.IpcEvent()
    ev.record()
    handle, off = ds.ds_ipc_export_mem(cache.tensor)
    q_out.put((handle, off, ev.handle, table, cache.num_blocks))
    assert q_in.get(timeout=300) == "done"  # keep the pool alive until the pull finished
    del junk


def test_pull_migration_across_processes(oracle_mod):
    ctx = mp.get_context("spawn")
    q_out, q_in = ctx.Queue(), ctx.Queue()
    child = ctx.Process(target=_prefill_instance, args=(q_out, q_in))
    child.start()
    try:
        handle, off, ev_handle, table_p, nb_p = q_out.get(timeout=300)
        remote = ds.RemoteKVCache(handle, off, L, nb_p, N, D)
        ready = ds.IpcEvent(ev_handle)
        # decode-side admission (pull happens when the decoder has memory)
        dcache = ds.KVCache.empty(L, 48, N, D)
        dcache.tensor.zero_()
        dpool = ds.Pool(48)
        opool_d = oracle_mod.Pool(L, 48, N, D)
        junk = np.full((5, 1), -1, np.int32)
        ds.ds_block_table(dpool, ds.DS_BT_APPEND, [0] * 5, [16] * 5, junk)
        opool_d.append([0] * 5, [16] * 5, junk.copy())
        maxb = _ceil(max(LENS) + 1, 16)
        td = np.full((len(LENS), maxb), -1, np.int32)
        tdo = td.copy()
        ds.ds_block_table(dpool, ds.DS_BT_APPEND, [0] * len(LENS), LENS, td)
        opool_d.append([0] * len(LENS), LENS, tdo)
        src = np.concatenate([table_p[i, :_ceil(l, 16)] for i, l in enumerate(LENS)])
        dst = np.concatenate([td[i, :_ceil(l, 16)] for i, l in enumerate(LENS)])
        ready.wait()
        ds.ds_kv_migrate(None, ds.DS_MIGRATE_PULL, 0, remote, 0, L, i32(src), 0, N, None, dst_cache=dcache,
                         dst_block_ids=i32(dst))
        torch.cuda.synchronize()
        q_in.put("done")
        # oracle: the same prompt K/V written into the prefill-side pool, migrated
        b = syn.prefill_batch(41, LENS, N, D)
        opool_p = oracle_mod.Pool(L, 40, N, D)
        for layer in range(L):
            opool_p.write_prefill(layer, b.k, b.v, b.cu_seqlens, table_p)
        oracle_mod.migrate(opool_p, opool_d, 0, L, src, dst, 0, 0, N)
        bits = to_bits(dcache.tensor)
        for layer in range(L):
            assert pages_match(bits, opool_d, layer, LENS, td)
        # one decode step on the pulled cache
        ds.ds_block_table(dpool, ds.DS_BT_APPEND, LENS, [1] * len(LENS), td)
        opool_d.append(LENS, [1] * len(LENS), tdo)
        db = syn.decode_batch(77, len(LENS), N, D)
        o = torch.empty((len(LENS), N, D), dtype=torch.bfloat16, device="cuda")
        ws = torch.zeros(ds.ds_decode_workspace_bytes(len(LENS), N, D, max(LENS)), dtype=torch.uint8, device="cuda")
        ds.ds_decode_attn(to_dev(db.q), to_dev(db.k_new), to_dev(db.v_new), o, dcache, 1, i32(td), i32(LENS),
                          max(LENS), 1 / math.sqrt(D), ws)
        ref = opool_d.decode(1, db.q, db.k_new, db.v_new, tdo, LENS, 1 / math.sqrt(D))
        assert oracle_mod.max_rel_err(to_f64(o), ref) <= 5e-3
        remote.close()
        ready.close()
    finally:
        child.join(timeout=120)
    assert child.exitcode == 0
