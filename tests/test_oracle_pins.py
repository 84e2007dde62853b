"""Pins for the fp64 CPU oracle (-m "not gpu").

Each test pins the oracle to something other than itself: the paper's printed
numbers (tests/golden/), closed forms, a brute-force numpy path, invariants of
the mathematics, or small exhaustive cases. A plausible mistake in the oracle
(a dropped term, wrong sign/index, transposed operand, off-by-one mask,
missing 1/Z, wrong page index) fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest

import synthetic as syn
from oracle.dense_ref import bits_to_f64, dense_causal_attention

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
BS = syn.BLOCK_SIZE


def _bits(x):
    return syn.f32_to_bf16_bits(np.asarray(x, dtype=np.float32))


# ----------------------------------------------------------------------------
# a2 prefill attention
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("lens,n,d", [([1], 1, 64), ([5, 17, 1, 33], 3, 64), ([64], 4, 128),
                                      ([16, 15, 31], 2, 128)])
def test_prefill_matches_dense_bruteforce(oracle_mod, lens, n, d):
    b = syn.prefill_batch(7, lens, n, d)
    scale = 1.0 / math.sqrt(d)
    got = oracle_mod.prefill(b.q, b.k, b.v, b.cu_seqlens, scale, nthreads=3)
    ref = dense_causal_attention(b.q, b.k, b.v, b.cu_seqlens, scale)
    assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


def test_worked_example_golden(oracle_mod):
    g = json.load(open(os.path.join(GOLDEN, "worked_example_two_tokens.json")))
    q = _bits(np.array(g["q"])[:, None, :])
    k = _bits(np.array(g["k"])[:, None, :])
    v = _bits(np.array(g["v"])[:, None, :])
    out = oracle_mod.prefill(q, k, v, [0, 2], g["scale"])[:, 0, :]
    e = math.e
    expected = np.array([[1, 0, 0, 0], [1 / (1 + e), e / (1 + e), 0, 0]])
    assert np.abs(out - expected).max() < 1e-15


def test_q_zero_gives_prefix_mean(oracle_mod):
    b = syn.prefill_batch(3, [40, 7], 2, 64)
    q = np.zeros_like(b.q)
    out = oracle_mod.prefill(q, b.k, b.v, b.cu_seqlens, 0.125)
    v = bits_to_f64(b.v)
    for r in range(2):
        s0, s1 = b.cu_seqlens[r], b.cu_seqlens[r + 1]
        pref = np.cumsum(v[s0:s1], axis=0) / np.arange(1, s1 - s0 + 1)[:, None, None]
        assert np.abs(out[s0:s1] - pref).max() < 1e-13


def test_single_token_returns_v_exactly(oracle_mod):
    b = syn.prefill_batch(11, [1, 1, 1], 4, 128)
    out = oracle_mod.prefill(b.q, b.k, b.v, b.cu_seqlens, 1 / math.sqrt(128))
    assert np.array_equal(out, bits_to_f64(b.v))


def test_equal_keys_give_prefix_mean(oracle_mod):
    b = syn.prefill_batch(5, [24], 2, 64)
    k = np.broadcast_to(b.k[:1], b.k.shape).copy()
    out = oracle_mod.prefill(b.q, k, b.v, b.cu_seqlens, 0.125)
    v = bits_to_f64(b.v)
    pref = np.cumsum(v, axis=0) / np.arange(1, 25)[:, None, None]
    assert np.abs(out - pref).max() < 1e-13


def test_dominant_key_selects_its_value(oracle_mod):
    d, l = 64, 20
    b = syn.prefill_batch(9, [l], 1, d)
    q = np.zeros_like(b.q)
    k = np.zeros_like(b.k)
    q[:, 0, 0] = _bits([32.0])[0]
    j0 = 6
    k[j0, 0, 0] = _bits([32.0])[0]  # logit scale*32*32 = 128 >= 80 above all others (0)
    out = oracle_mod.prefill(q, k, b.v, b.cu_seqlens, 1 / 8)
    v = bits_to_f64(b.v)
    # rows i >= j0 see the dominant key: weight of the rest <= (i)e^-128
    assert np.abs(out[j0:, 0] - v[j0, 0]).max() < 1e-30
    # rows i < j0 do not see it (causality) -> prefix mean of v
    pref = np.cumsum(v[:j0, 0], axis=0) / np.arange(1, j0 + 1)[:, None]
    assert np.abs(out[:j0, 0] - pref).max() < 1e-13


def test_softmax_rows_sum_to_one(oracle_mod):
    b = syn.prefill_batch(13, [50, 3], 3, 64, q_sigma=4.0)
    ones = np.full_like(b.v, _bits(1.0))
    out = oracle_mod.prefill(b.q, b.k, ones, b.cu_seqlens, 0.125)
    assert np.abs(out - 1.0).max() < 1e-12


def test_causality_future_tokens_do_not_matter(oracle_mod):
    b = syn.prefill_batch(17, [30], 2, 64)
    out1 = oracle_mod.prefill(b.q, b.k, b.v, b.cu_seqlens, 0.125)
    i = 12
    q2, k2, v2 = b.q.copy(), b.k.copy(), b.v.copy()
    g = syn.normal_bf16(99, q2[i + 1:].shape)
    q2[i + 1:], k2[i + 1:], v2[i + 1:] = g, g[::-1], g
    out2 = oracle_mod.prefill(q2, k2, v2, b.cu_seqlens, 0.125)
    assert np.array_equal(out1[: i + 1], out2[: i + 1])
    assert not np.array_equal(out1[i + 1:], out2[i + 1:])


def test_sequences_do_not_attend_across(oracle_mod):
    b = syn.prefill_batch(19, [10, 12], 2, 64)
    both = oracle_mod.prefill(b.q, b.k, b.v, b.cu_seqlens, 0.125)
    second = oracle_mod.prefill(b.q[10:], b.k[10:], b.v[10:], [0, 12], 0.125)
    assert np.array_equal(both[10:], second)


def test_head_independence(oracle_mod):
    b = syn.prefill_batch(23, [9, 21], 4, 64)
    perm = np.array([2, 0, 3, 1])
    out = oracle_mod.prefill(b.q, b.k, b.v, b.cu_seqlens, 0.125)
    outp = oracle_mod.prefill(b.q[:, perm], b.k[:, perm], b.v[:, perm], b.cu_seqlens, 0.125)
    assert np.array_equal(out[:, perm], outp)


def test_linearity_in_v(oracle_mod):
    b = syn.prefill_batch(29, [33], 2, 64)
    g = syn.rng(5)
    v1 = g.integers(-8, 9, b.v.shape).astype(np.float32)
    v2 = g.integers(-8, 9, b.v.shape).astype(np.float32)
    o1 = oracle_mod.prefill(b.q, b.k, _bits(v1), b.cu_seqlens, 0.125)
    o2 = oracle_mod.prefill(b.q, b.k, _bits(v2), b.cu_seqlens, 0.125)
    o12 = oracle_mod.prefill(b.q, b.k, _bits(v1 + v2), b.cu_seqlens, 0.125)
    o_2 = oracle_mod.prefill(b.q, b.k, _bits(2 * v1), b.cu_seqlens, 0.125)
    assert np.abs(o12 - (o1 + o2)).max() < 1e-12
    assert np.abs(o_2 - 2 * o1).max() < 1e-12


def test_row_i_equals_shorter_prefill(oracle_mod):
    b = syn.prefill_batch(31, [26], 2, 64)
    full = oracle_mod.prefill(b.q, b.k, b.v, b.cu_seqlens, 0.125)
    for i in (0, 7, 15, 25):
        part = oracle_mod.prefill(b.q[: i + 1], b.k[: i + 1], b.v[: i + 1], [0, i + 1], 0.125)
        assert np.array_equal(full[i], part[i])
        row = oracle_mod.prefill_row(b.q, b.k, b.v, b.cu_seqlens, 0, i, 1, 0.125)
        assert np.array_equal(row, full[i, 1])


def test_scale_enters_as_multiplier(oracle_mod):
    # doubling q (exact in bf16) equals doubling the scale; a missing or squared
    # scale would break this.
    b = syn.prefill_batch(37, [19], 2, 64)
    q2 = _bits(2 * bits_to_f64(b.q).astype(np.float32))
    a = oracle_mod.prefill(q2, b.k, b.v, b.cu_seqlens, 0.125)
    c = oracle_mod.prefill(b.q, b.k, b.v, b.cu_seqlens, 0.25)
    assert np.abs(a - c).max() < 1e-13


# ----------------------------------------------------------------------------
# a1 block table / allocator
# ----------------------------------------------------------------------------
def _ceil(a, b):
    return -(-a // b)


def test_block_table_bijection_and_lowest_first(oracle_mod):
    pool = oracle_mod.Pool(1, 64, 1, 64)
    lens = [1, 16, 17, 33, 0, 100]
    table = np.full((len(lens), 8), -1, dtype=np.int32)
    assert pool.append([0] * len(lens), lens, table) == 0
    ids = [int(x) for x in table.ravel() if x >= 0]
    assert ids == list(range(sum(_ceil(l, BS) for l in lens)))  # lowest first, arg + logical order
    assert len(set(ids)) == len(ids)
    assert pool.num_free == 64 - len(ids)
    # every (seq, token) maps to a distinct (block, slot)
    slots = {(int(table[s, t // BS]), t % BS) for s, l in enumerate(lens) for t in range(l)}
    assert len(slots) == sum(lens)


def test_append_allocates_iff_page_boundary(oracle_mod):
    pool = oracle_mod.Pool(1, 16, 1, 64)
    table = np.full((1, 16), -1, dtype=np.int32)
    c = 0
    for step in range(70):
        before = pool.num_free
        assert pool.append([c], [1], table) == 0
        assert before - pool.num_free == (1 if c % BS == 0 else 0)
        c += 1
    assert [int(x) for x in table[0] if x >= 0] == list(range(_ceil(70, BS)))


def test_all_or_nothing_state_unchanged(oracle_mod):
    pool = oracle_mod.Pool(1, 10, 1, 64)
    t = np.full((2, 8), -1, dtype=np.int32)
    assert pool.append([0, 0], [64, 48], t) == 0  # 4 + 3 pages
    snap = t.copy()
    t2 = np.full((2, 8), -1, dtype=np.int32)
    assert pool.append([0, 0], [32, 33], t2) == oracle_mod.NO_BLOCKS  # 2 + 3 > 3 free
    assert np.array_equal(t2, np.full((2, 8), -1)) and pool.num_free == 3
    assert np.array_equal(t, snap)
    # free seq 0 (4 pages: ids 0..3) then re-alloc returns the same lowest ids
    t0 = t[:1].copy()
    assert pool.free([64], t0) == 0 and np.all(t0 == -1) and pool.num_free == 7
    t3 = np.full((1, 8), -1, dtype=np.int32)
    assert pool.append([0], [50], t3) == 0
    assert list(t3[0, :4]) == [0, 1, 2, 3]


def test_invalid_append_rejected(oracle_mod):
    pool = oracle_mod.Pool(1, 10, 1, 64)
    t = np.full((1, 2), -1, dtype=np.int32)
    assert pool.append([0], [33], t) == oracle_mod.INVALID  # 3 pages > max_blocks 2
    assert pool.num_free == 10


# ----------------------------------------------------------------------------
# a3 paged write + a7 decode
# ----------------------------------------------------------------------------
def test_paged_write_scatter_gather_identity(oracle_mod):
    lens, n, d = [5, 16, 37], 3, 64
    b = syn.prefill_batch(41, lens, n, d)
    pool = oracle_mod.Pool(2, 32, n, d)
    # fragment the pool first: 9 one-page rows, then free rows 1, 4, 5, 8
    junk = np.full((9, 1), -1, dtype=np.int32)
    assert pool.append([0] * 9, [16] * 9, junk) == 0
    sel = [1, 4, 5, 8]
    assert pool.free([16] * 4, np.ascontiguousarray(junk[sel])) == 0
    table = np.full((3, 8), -1, dtype=np.int32)
    assert pool.append([0, 0, 0], lens, table) == 0
    assert list(table[0, :1]) == [1] and list(table[1, :1]) == [4] and list(table[2, :3]) == [5, 8, 9]
    pool.write_prefill(1, b.k, b.v, b.cu_seqlens, table)
    for r, l in enumerate(lens):
        for t in range(l):
            for h in range(n):
                tok = b.cu_seqlens[r] + t
                assert np.array_equal(pool.page(1, 0, table[r, t // BS], h)[t % BS], b.k[tok, h])
                assert np.array_equal(pool.page(1, 1, table[r, t // BS], h)[t % BS], b.v[tok, h])


@pytest.mark.parametrize("ctx", [[0], [15, 16, 17, 31, 32, 1]])
def test_decode_equals_last_prefill_row(oracle_mod, ctx):
    n, d = 2, 64
    B = len(ctx)
    full = syn.prefill_batch(43, [c + 1 for c in ctx], n, d)
    pool = oracle_mod.Pool(1, 64, n, d)
    table = np.full((B, 8), -1, dtype=np.int32)
    assert pool.append([0] * B, ctx, table) == 0
    # cached part = first c tokens of each sequence
    hist_idx = np.concatenate([np.arange(full.cu_seqlens[i], full.cu_seqlens[i] + c) for i, c in enumerate(ctx)]).astype(np.int64)
    cu_hist = syn.cu_seqlens(ctx)
    pool.write_prefill(0, full.k[hist_idx], full.v[hist_idx], cu_hist, table)
    assert pool.append(ctx, [1] * B, table) == 0
    last = full.cu_seqlens[1:] - 1
    out = pool.decode(0, full.q[last], full.k[last], full.v[last], table, ctx, 0.125)
    ref = oracle_mod.prefill(full.q, full.k, full.v, full.cu_seqlens, 0.125)[last]
    assert np.abs(out - ref).max() <= 1e-12
    # the append wrote the new token at position c
    for i, c in enumerate(ctx):
        assert np.array_equal(pool.page(0, 0, table[i, c // BS], 1)[c % BS], full.k[last[i], 1])


# ----------------------------------------------------------------------------
# a4-a6 migration + KV sizing
# ----------------------------------------------------------------------------
def test_paper_kv_size_golden(oracle_mod):
    g = json.load(open(os.path.join(GOLDEN, "paper_kv_sizing.json")))
    nbytes = oracle_mod.kv_bytes(g["layers"], g["prompt_tokens"], g["heads"], g["head_dim"], g["elem_bytes"])
    assert nbytes == 1_207_959_552
    # the paper prints 3 significant figures: the exact value must lie within half a
    # unit of the last printed digit (inclusive: 1.125 prints as 1.13 rounding half up)
    gib = nbytes / 2**30
    assert abs(gib - g["printed_kv_gib_per_request"]) <= 0.005 + 1e-12
    per_s = gib * g["arrival_rate_rps"]
    assert abs(per_s - g["printed_gib_per_second"]) <= 0.05 + 1e-12
    assert abs(per_s * 8 - g["printed_gibit_per_second"]) <= 0.5 + 1e-12
    # and the decimal-GB reading would NOT match the printed 1.13 (R7)
    assert abs(nbytes / 1e9 - g["printed_kv_gib_per_request"]) > 0.005


def test_migrate_moves_pages_between_corresponding_layers(oracle_mod):
    L, n, d = 3, 4, 64
    lens = [20, 33]
    b = syn.prefill_batch(47, lens, n, d)
    P = oracle_mod.Pool(L, 16, n, d)
    D = oracle_mod.Pool(L, 24, 2, d)  # decode rank holds 2 heads (TP slice)
    tp = np.full((2, 4), -1, dtype=np.int32)
    assert P.append([0, 0], lens, tp) == 0
    for layer in range(L):
        P.write_prefill(layer, b.k, b.v, b.cu_seqlens, tp)
    junk = np.full((1, 4), -1, dtype=np.int32)
    D.append([0], [40], junk)  # D's ids differ from P's
    td = np.full((2, 4), -1, dtype=np.int32)
    assert D.append([0, 0], lens, td) == 0
    src = np.concatenate([tp[i, :_ceil(l, BS)] for i, l in enumerate(lens)])
    dst = np.concatenate([td[i, :_ceil(l, BS)] for i, l in enumerate(lens)])
    nbytes = oracle_mod.migrate(P, D, 1, 2, src, dst, 2, 0, 2)  # heads 2..3 -> 0..1, layers 1..2
    n_pages = len(src)
    assert nbytes == n_pages * 2 * 2 * 2 * BS * d * 2
    # payload bytes for the valid tokens equal kv_bytes scaled by layers/heads share
    assert oracle_mod.kv_bytes(2, sum(lens), 2, d) <= nbytes
    for r, l in enumerate(lens):
        for t in range(l):
            tok = b.cu_seqlens[r] + t
            for layer in (1, 2):
                for hd in range(2):
                    pg_k = D.page(layer, 0, td[r, t // BS], hd)[t % BS]
                    pg_v = D.page(layer, 1, td[r, t // BS], hd)[t % BS]
                    assert np.array_equal(pg_k, b.k[tok, 2 + hd]) and np.array_equal(pg_v, b.v[tok, 2 + hd])
            assert not D.page(0, 0, td[r, 0], 0).any()  # layer 0 not migrated


def test_max_rel_err_metric(oracle_mod):
    r = np.array([[1.0, -2.0, 0.5], [0.0, 0.0, 0.0]])
    g = r + np.array([[0.02, 0.0, 0.0], [1e-7, 0.0, 0.0]])
    assert oracle_mod.max_rel_err(g, r) == pytest.approx(0.1)  # 1e-7 / 1e-6 floor


# ----------------------------------------------------------------------------
# NEXT-3 chunked prefill over a paged prefix
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("chunks", [[(0, 30)], [(17, 20), (0, 5), (64, 1)], [(100, 37), (3, 3)]])
def test_chunked_prefill_equals_rows_of_full_prefill(oracle_mod, chunks):
    """chunk (c, l) of a sequence == rows c..c+l-1 of plain prefill over c+l tokens."""
    n, d = 2, 64
    full = syn.prefill_batch(53, [c + l for c, l in chunks], n, d)
    pool = oracle_mod.Pool(1, 64, n, d)
    B = len(chunks)
    table = np.full((B, 16), -1, np.int32)
    pref = [c for c, _ in chunks]
    assert pool.append([0] * B, pref, table) == 0
    hist = [np.arange(full.cu_seqlens[i], full.cu_seqlens[i] + c) for i, (c, _) in enumerate(chunks)]
    idx = np.concatenate(hist).astype(np.int64) if any(pref) else np.zeros(0, np.int64)
    pool.write_prefill(0, full.k[idx], full.v[idx], syn.cu_seqlens(pref), table)
    assert pool.append(pref, [l for _, l in chunks], table) == 0
    cidx = np.concatenate([np.arange(full.cu_seqlens[i] + c, full.cu_seqlens[i + 1])
                           for i, (c, _) in enumerate(chunks)]).astype(np.int64)
    out = oracle_mod.chunked_prefill(pool, 0, full.q[cidx], full.k[cidx], full.v[cidx],
                                     syn.cu_seqlens([l for _, l in chunks]), pref, table, 0.125)
    ref = oracle_mod.prefill(full.q, full.k, full.v, full.cu_seqlens, 0.125)[cidx]
    assert np.abs(out - ref).max() <= 1e-12
    # the chunk's K/V landed at positions c..c+l-1
    for i, (c, l) in enumerate(chunks):
        for t in range(c, c + l):
            assert np.array_equal(pool.page(0, 0, table[i, t // BS], 1)[t % BS], full.k[full.cu_seqlens[i] + t, 1])
