"""C-ABI boundary tests that run without a GPU (-m "not gpu").

* libds.so loads and exports every entry point include/ds.h declares;
* a1 (ds_block_table, host code) is bit-exact against the oracle allocator on
  randomised APPEND/FREE traces, including exhaustion (all-or-nothing);
* argument validation rejects bad calls with DS_ERR_INVALID_ARG before touching
  the device, and a well-formed compute call on a GPU-less host fails loudly
  with DS_ERR_CUDA (no CPU fallback).
"""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2401_09670_b200 as ds
import synthetic as syn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    txt = open(os.path.join(ROOT, "include", "ds.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ds_[a-z_0-9]+)\s*\(", txt)))


def test_header_symbols_exported():
    declared = _declared_symbols()
    assert len(declared) >= 17
    lib = ctypes.CDLL(ds.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(ds.EXPORTED) == declared


def test_build_info_reports_nccl():
    info = ds.ds_build_info()
    assert info.startswith("libds sm_100a nccl 2.")


def _rand_trace(seed, nseq=6, steps=60):
    g = syn.rng(seed)
    ops = []
    lens = np.zeros(nseq, dtype=np.int32)
    live = np.zeros(nseq, dtype=bool)
    for _ in range(steps):
        s = int(g.integers(nseq))
        r = g.random()
        if live[s] and r < 0.2:
            ops.append(("free", s, int(lens[s])))
            lens[s] = 0
            live[s] = False
        else:
            add = int(g.integers(1, 40)) if r < 0.6 else 1
            ops.append(("append", s, int(lens[s]), add))
            lens[s] += add
            live[s] = True
    return ops


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_block_table_bit_exact_vs_oracle(oracle_mod, seed):
    nseq, nb, maxb = 6, 40, 16
    pool = ds.Pool(nb)
    opool = oracle_mod.Pool(1, nb, 1, 64)
    t_ds = np.full((nseq, maxb), -1, dtype=np.int32)
    t_or = t_ds.copy()
    for op in _rand_trace(seed, nseq):
        if op[0] == "append":
            _, s, cur, add = op
            row_ds, row_or = t_ds[s:s + 1].copy(), t_or[s:s + 1].copy()
            try:
                ds.ds_block_table(pool, ds.DS_BT_APPEND, [cur], [add], row_ds)
                rc_ds = 0
            except ds.DSError as e:
                rc_ds = e.status
            rc_or = opool.append([cur], [add], row_or)
            assert rc_ds == rc_or
            t_ds[s], t_or[s] = row_ds[0], row_or[0]
            if rc_ds != 0:
                # undo the host-side length bookkeeping of this trace step: sequence is reset
                row = t_ds[s:s + 1].copy()
                ds.ds_block_table(pool, ds.DS_BT_FREE, [cur], None, row)
                opool.free([cur], t_or[s:s + 1].copy()) if cur else None
                t_or[s:s + 1] = -1
                t_ds[s:s + 1] = -1
        else:
            _, s, cur = op
            row_ds, row_or = t_ds[s:s + 1].copy(), t_or[s:s + 1].copy()
            ds.ds_block_table(pool, ds.DS_BT_FREE, [cur], None, row_ds)
            assert opool.free([cur], row_or) == 0
            t_ds[s], t_or[s] = row_ds[0], row_or[0]
        assert np.array_equal(t_ds, t_or)
        assert pool.num_free == opool.num_free


def test_block_table_batch_and_exhaustion(oracle_mod):
    lens = [33, 1, 16, 17, 200]
    pool, opool = ds.Pool(21), oracle_mod.Pool(1, 21, 1, 64)
    t1, t2 = np.full((5, 16), -1, np.int32), np.full((5, 16), -1, np.int32)
    nf = ds.ds_block_table(pool, ds.DS_BT_APPEND, [0] * 5, lens, t1)
    assert opool.append([0] * 5, lens, t2) == 0
    assert np.array_equal(t1, t2) and nf == opool.num_free == 21 - 20
    t3 = np.full((1, 16), -1, np.int32)
    with pytest.raises(ds.DSError) as ei:
        ds.ds_block_table(pool, ds.DS_BT_APPEND, [0], [33], t3)
    assert ei.value.status == ds.DS_ERR_NO_BLOCKS
    assert np.all(t3 == -1) and pool.num_free == 1


def test_block_table_rejects_bad_args():
    pool = ds.Pool(8)
    t = np.full((1, 2), -1, np.int32)
    for args in ((ds.DS_BT_APPEND, [-1], [1]), (ds.DS_BT_APPEND, [0], [33]), (7, [0], [1])):
        with pytest.raises(ds.DSError) as ei:
            ds.ds_block_table(pool, args[0], args[1], args[2], t)
        assert ei.value.status == ds.DS_ERR_INVALID_ARG
    with pytest.raises(ds.DSError):  # FREE of never-allocated ids
        ds.ds_block_table(pool, ds.DS_BT_FREE, [16], None, np.array([[3, -1]], np.int32))
    assert pool.num_free == 8


def test_block_table_free_rejects_duplicate_ids():
    """the same page listed twice in one FREE must not be freed twice
    (num_free would overcount and a later APPEND would hand out page -1)."""
    pool = ds.Pool(8)
    t = np.full((2, 2), -1, np.int32)
    ds.ds_block_table(pool, ds.DS_BT_APPEND, [0, 0], [32, 16], t)  # pages 0,1 | 2
    assert pool.num_free == 5
    dup = np.array([[0, 1], [1, -1]], np.int32)  # page 1 in both rows
    with pytest.raises(ds.DSError) as ei:
        ds.ds_block_table(pool, ds.DS_BT_FREE, [32, 16], None, dup)
    assert ei.value.status == ds.DS_ERR_INVALID_ARG
    assert pool.num_free == 5 and np.array_equal(dup, [[0, 1], [1, -1]])  # nothing freed
    same_row = np.array([[2, 2]], np.int32)
    with pytest.raises(ds.DSError):
        ds.ds_block_table(pool, ds.DS_BT_FREE, [32], None, same_row)
    assert pool.num_free == 5
    # the pool is intact: the real tables free cleanly and everything is allocatable again
    ds.ds_block_table(pool, ds.DS_BT_FREE, [32, 16], None, t)
    assert pool.num_free == 8 and np.all(t == -1)
    full = np.full((1, 8), -1, np.int32)
    ds.ds_block_table(pool, ds.DS_BT_APPEND, [0], [128], full)
    assert sorted(full[0].tolist()) == list(range(8)) and pool.num_free == 0


def _cache(base=0x10000, L=2, NB=64, n=4, D=64):
    return ds.ds_kv_cache(base, L, NB, n, 16, D)


FAKE = 0x7F0000000000  # aligned non-null address; never dereferenced on a GPU-less host


def test_prefill_validation_then_no_device():
    lib = ds.lib()
    c = _cache()
    args = lambda **kw: dict(dict(q=FAKE, k=FAKE, v=FAKE, out=FAKE, cu=FAKE, B=2, T=40, maxl=33,
                                  layer=1, bt=FAKE, maxb=4, scale=0.125), **kw)
    def call(a, cache=c):
        return lib.ds_prefill_attn(a["q"], a["k"], a["v"], a["out"], a["cu"], a["B"], a["T"], a["maxl"],
                                   ctypes.byref(cache), a["layer"], a["bt"], a["maxb"], a["scale"], None)
    assert call(args(q=FAKE + 2)) == ds.DS_ERR_INVALID_ARG
    assert call(args(layer=2)) == ds.DS_ERR_INVALID_ARG
    assert call(args(maxb=2)) == ds.DS_ERR_INVALID_ARG
    assert call(args(scale=0.0)) == ds.DS_ERR_INVALID_ARG
    assert call(args(), cache=_cache(D=96)) == ds.DS_ERR_INVALID_ARG
    assert call(args(B=0)) == ds.DS_OK  # empty batch is a no-op
    rc = call(args())
    assert rc == ds.DS_ERR_CUDA, ds.ds_last_error()
    assert "ds_prefill_attn" in ds.ds_last_error()


def test_prefill_push_validation_then_no_device():
    lib = ds.lib()
    c = _cache(n=4)

    def call(dst, dst_layer=0, head0=0, wl=1, dbt=FAKE, dmaxb=4):
        return lib.ds_prefill_attn_push(FAKE, FAKE, FAKE, FAKE, FAKE, 2, 40, 33, ctypes.byref(c), 1, FAKE, 4,
                                        ctypes.byref(dst), dst_layer, dbt, dmaxb, head0, wl, 0.125, None)
    assert call(_cache(n=8, D=128)) == ds.DS_ERR_INVALID_ARG           # head_dim differs
    assert call(_cache(n=8), dst_layer=2) == ds.DS_ERR_INVALID_ARG     # dst layer out of range
    assert call(_cache(n=8), head0=5) == ds.DS_ERR_INVALID_ARG         # 5 + 4 heads > 8
    assert call(_cache(n=8), wl=2) == ds.DS_ERR_INVALID_ARG
    assert call(_cache(n=8), dbt=None) == ds.DS_ERR_INVALID_ARG
    assert call(_cache(n=8), dmaxb=2) == ds.DS_ERR_INVALID_ARG         # 33 tokens need 3 pages
    rc = call(_cache(n=8), head0=4)
    assert rc == ds.DS_ERR_CUDA, ds.ds_last_error()
    assert "ds_prefill_attn_push" in ds.ds_last_error()


def test_decode_validation_and_workspace():
    lib = ds.lib()
    c = _cache(n=4, D=128)
    assert ds.ds_decode_workspace_bytes(1, 4, 128, 543) >= 4 * (128 + 2) * 4
    ws = ds.ds_decode_workspace_bytes(1, 4, 128, 543)
    call = lambda maxc, ws_ptr, ws_bytes: lib.ds_decode_attn(FAKE, FAKE, FAKE, FAKE, ctypes.byref(c), 0, FAKE, 40,
                                                           FAKE, 1, maxc, 0.088, ws_ptr, ws_bytes, None)
    assert call(543, None, 0) == ds.DS_ERR_INVALID_ARG  # needs split workspace
    assert call(640, FAKE, ws) == ds.DS_ERR_INVALID_ARG  # 640/16 >= 40 pages
    assert call(543, FAKE, ws) == ds.DS_ERR_CUDA
    call_ex = lambda flags: lib.ds_decode_attn_ex(FAKE, FAKE, FAKE, FAKE, ctypes.byref(c), 0, FAKE, 40, FAKE, 1,
                                                  543, 0.088, FAKE, ws, flags, None)
    assert call_ex(2) == ds.DS_ERR_INVALID_ARG and "flags" in ds.ds_last_error()
    assert call_ex(ds.DS_DECODE_EARLY_KV) == ds.DS_ERR_CUDA  # a valid call, no device here


def test_decode_kernel_query():
    """ds_decode_kernel names the kernel a batch shape gets (no device work): the
    page-range kernel by default; decode_pairs_kernel only when DS_DEC_PAIRS opts in
    (read once per process: checked in a child with it set)."""
    import os
    import subprocess
    import sys
    names = {ds.ds_decode_kernel(b, n) for b in (1, 64, 128, 4096) for n in (1, 40)}
    expect = {"decode_kernel"} if not os.environ.get("DS_DEC_PAIRS") else {"decode_kernel", "decode_pairs_kernel"}
    assert names <= expect, names
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import paper_2401_09670_b200 as ds; "
            "print(ds.ds_decode_kernel(1, 4), ds.ds_decode_kernel(128, 40))")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=120,
                       env=dict(os.environ, DS_DEC_PAIRS="4"))
    assert r.returncode == 0, r.stderr[-2000:]
    # 4 pairs per SM: 1 x 4 pairs -> page ranges; 128 x 40 = 5120 pairs -> pair streaming
    assert r.stdout.split() == ["decode_kernel", "decode_pairs_kernel"], r.stdout


def test_decode_workspace_holds_the_dynamic_chunks():
    """The workspace grows with the batch's page count once the dynamic tail is on
    (>= 64 pages per warp of the largest grid: 160 SMs x 16 warps): 10 % of the
    pages in 8-page chunks, two (D + 4)-float partial rows per chunk."""
    f = ds.ds_decode_workspace_bytes
    # 64 x 40 x 35 pages stay static: the size does not depend on the lengths
    assert f(64, 40, 128, 1000) == f(64, 40, 128, 543)
    big_b = 1024
    pages = big_b * 40 * ((543 + 1 + 15) // 16)
    assert pages >= 64 * 160 * 16
    chunks = (pages * 10 // 100) // 8
    base = f(big_b, 40, 128, 0)  # one page per sequence: static
    assert f(big_b, 40, 128, 543) == base + chunks * 2 * (128 + 4) * 4
    assert f(big_b, 40, 128, 1000) > f(big_b, 40, 128, 543)  # more pages -> more chunk rows


def test_decode_workspace_tickets_fixed_region():
    """the merge tickets live in one fixed region at a fixed
    offset, so a workspace reused by calls with other batch shapes or head_dim never
    finds its tickets on top of another call's partial rows. The size therefore has
    a fixed 2 MiB ticket part (4096 x 128 pairs) plus parts that grow with the call."""
    f = ds.ds_decode_workspace_bytes
    fixed = 16 + (1 << 19) * 4
    rows = 160 * 16 * 2 * (128 + 4) * 4  # static partial rows of the largest grid
    assert f(1, 1, 128, 0) == fixed + rows
    assert f(1000, 100, 128, 0) == fixed + rows  # the ticket part does not grow (no dynamic chunks here)
    lib = ds.lib()
    c = _cache(n=256, D=128, NB=4096)
    ws = f(4096, 256, 128, 15)
    call = lambda B: lib.ds_decode_attn(FAKE, FAKE, FAKE, FAKE, ctypes.byref(c), 0, FAKE, 40, FAKE, B, 15, 0.088,
                                        FAKE, ws, None)
    assert call(2048) == ds.DS_ERR_CUDA          # 2048 x 256 = 2^19 pairs: accepted (no device here)
    assert call(2049) == ds.DS_ERR_INVALID_ARG   # one pair over the ticket region
    assert "n_loc" in ds.ds_last_error()


def test_wrapper_shape_checks():
    """the Python wrappers reject shape mismatches the C side cannot
    see (device array sizes) before any pointer crosses the boundary"""
    import torch

    class FakeCache:
        heads, head_dim = 4, 64
    q = torch.zeros(8, 4, 64)
    ds._check_activations(q, ((torch.zeros(8, 4, 64), "k"),), FakeCache)
    with pytest.raises(ValueError, match="k_new"):
        ds._check_activations(q, ((torch.zeros(7, 4, 64), "k_new"),), FakeCache)
    with pytest.raises(ValueError, match="matching the cache"):
        ds._check_activations(torch.zeros(8, 5, 64), (), FakeCache)
    with pytest.raises(ValueError, match="block_table"):
        ds._check_table(torch.zeros(3, 4), 4, "block_table")
    with pytest.raises(ValueError, match="block_table"):
        ds._check_table(torch.zeros(12), 4, "block_table")
    ds._check_table(torch.zeros(5, 4), 4, "block_table")
    with pytest.raises(ValueError, match="total_tokens"):
        ds._check_seqlens(torch.zeros(3), 9, 8)


def test_staging_sizes():
    c = _cache(L=40, NB=1000, n=40, D=128)
    assert ds.lib().ds_kv_staging_bytes(ctypes.byref(c), 40, 32, 40) == 40 * 2 * 32 * 40 * 4096
    # per request of OPT-13B at 512 tokens: 419,430,400 bytes
    assert ds.lib().ds_kv_staging_bytes(ctypes.byref(c), 40, 32, 40) == 419_430_400
    row = 40 * 4096
    mig = ds.lib().ds_kv_migrate_staging_bytes(ctypes.byref(c), ds.DS_MIGRATE_SEND, 40, 32, 40)
    assert mig == 2 * ((64 << 20) // row) * row
    mig_self = ds.lib().ds_kv_migrate_staging_bytes(ctypes.byref(c), ds.DS_MIGRATE_SELF, 40, 32, 40)
    assert mig_self == 2 * mig
    small = ds.lib().ds_kv_migrate_staging_bytes(ctypes.byref(c), ds.DS_MIGRATE_SEND, 1, 1, 40)
    assert small == 2 * 2 * row  # chunk clamps to the 2 rows that exist


def test_pack_validation():
    lib = ds.lib()
    c = _cache(L=2, NB=16, n=4, D=64)
    assert lib.ds_kv_pack(ctypes.byref(c), 1, 2, FAKE, 3, 0, 4, FAKE, 1 << 20, None) == ds.DS_ERR_INVALID_ARG
    assert lib.ds_kv_pack(ctypes.byref(c), 0, 2, FAKE, 3, 2, 3, FAKE, 1 << 20, None) == ds.DS_ERR_INVALID_ARG
    assert lib.ds_kv_pack(ctypes.byref(c), 0, 2, FAKE, 3, 0, 4, FAKE, 100, None) == ds.DS_ERR_INVALID_ARG
    assert lib.ds_kv_pack(ctypes.byref(c), 0, 2, FAKE, 3, 0, 4, FAKE, 1 << 20, None) == ds.DS_ERR_CUDA


def test_contiguous_run_helper():
    """the host check that picks the zero-copy migration (ds_kv_migrate_contig)"""
    assert ds.contiguous_run([3, 4, 5, 6]) == 3
    assert ds.contiguous_run(np.array([[0, 1], [2, 3]])) == 0
    assert ds.contiguous_run([3, 5]) is None
    assert ds.contiguous_run([4, 3]) is None
    assert ds.contiguous_run([]) is None
