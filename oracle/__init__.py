"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/oracle.c header).

Python face of the plain fp64 C oracle. Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / `--impl reference` legs may import this package. The
product library (paper_2401_09670_b200, libds.so) never imports it, and this
package imports nothing from the product.

All array arguments are numpy arrays: bf16 inputs as uint16 bit patterns,
int32 tables/lengths, float64 outputs.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

OK, INVALID, NO_BLOCKS = 0, 1, 3


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain C, -O2, no fast-math: IEEE fp64)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math",
                               "-ffp-contract=off", "-o", tmp, _SRC, "-lm", "-lpthread"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i32, i64, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        _lib.oracle_prefill.argtypes = [P, P, P, P, i32, i32, i32, f64, P, i32]
        _lib.oracle_prefill_row.argtypes = [P, P, P, P, i32, i32, i32, i32, i32, f64, P]
        _lib.oracle_pool_create.argtypes = [i32, i32, i32, i32, i32]
        _lib.oracle_pool_create.restype = P
        _lib.oracle_pool_destroy.argtypes = [P]
        _lib.oracle_pool_num_free.argtypes = [P]
        _lib.oracle_pool_num_free.restype = i32
        _lib.oracle_pool_page.argtypes = [P, i32, i32, i32, i32]
        _lib.oracle_pool_page.restype = P
        _lib.oracle_bt_append.argtypes = [P, i32, P, P, P, i32, i32]
        _lib.oracle_bt_free.argtypes = [P, i32, P, P, i32, i32]
        _lib.oracle_pool_write_prefill.argtypes = [P, i32, P, P, P, i32, P, i32]
        _lib.oracle_decode.argtypes = [P, i32, P, P, P, P, i32, P, i32, f64, P, i32]
        _lib.oracle_migrate.argtypes = [P, P, i32, i32, P, P, i32, i32, i32, i32]
        _lib.oracle_migrate.restype = i64
        _lib.oracle_chunked_prefill.argtypes = [P, i32, P, P, P, P, P, i32, P, i32, f64, P, i32]
        _lib.oracle_kv_bytes.argtypes = [i32, i64, i32, i32, i32]
        _lib.oracle_kv_bytes.restype = i64
    return _lib


def _p(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.c_void_p)


def _u16(a):
    return np.ascontiguousarray(a, dtype=np.uint16)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def default_threads() -> int:
    return os.cpu_count() or 1


def prefill(q, k, v, cu_seqlens, scale: float, nthreads: int | None = None) -> np.ndarray:
    """a2: causal attention per (sequence, head), fp64 output [T][n][d]."""
    q, k, v, cu = _u16(q), _u16(k), _u16(v), _i32(cu_seqlens)
    T, n, d = q.shape
    out = np.zeros((T, n, d), dtype=np.float64)
    rc = lib().oracle_prefill(_p(q), _p(k), _p(v), _p(cu), len(cu) - 1, n, d, scale, _p(out),
                              nthreads or default_threads())
    if rc != OK:
        raise ValueError(f"oracle_prefill rc={rc}")
    return out


def prefill_row(q, k, v, cu_seqlens, r: int, i: int, h: int, scale: float) -> np.ndarray:
    """One output row (sequence r, row i, head h) — for sampled full-size checks."""
    q, k, v, cu = _u16(q), _u16(k), _u16(v), _i32(cu_seqlens)
    _, n, d = q.shape
    out = np.zeros(d, dtype=np.float64)
    rc = lib().oracle_prefill_row(_p(q), _p(k), _p(v), _p(cu), r, i, h, n, d, scale, _p(out))
    if rc != OK:
        raise ValueError(f"oracle_prefill_row rc={rc}")
    return out


def kv_bytes(layers: int, tokens: int, heads: int, head_dim: int, elem_bytes: int = 2) -> int:
    return int(lib().oracle_kv_bytes(layers, tokens, heads, head_dim, elem_bytes))


class Pool:
    """Paged KV pool model + lowest-free-first allocator (a1, a3, a6, a7)."""

    def __init__(self, layers: int, num_blocks: int, heads: int, head_dim: int, block_size: int = 16):
        self.layers, self.num_blocks, self.heads = layers, num_blocks, heads
        self.head_dim, self.block_size = head_dim, block_size
        self._h = lib().oracle_pool_create(layers, num_blocks, heads, block_size, head_dim)
        if not self._h:
            raise MemoryError("oracle_pool_create failed")

    def close(self):
        if self._h:
            lib().oracle_pool_destroy(self._h)
            self._h = None

    __del__ = close

    @property
    def num_free(self) -> int:
        return int(lib().oracle_pool_num_free(self._h))

    def page(self, layer: int, kv: int, block: int, head: int) -> np.ndarray:
        """Copy of page (layer, kv, block, head): uint16 [block_size][head_dim]."""
        ptr = lib().oracle_pool_page(self._h, layer, kv, block, head)
        n = self.block_size * self.head_dim
        buf = (ctypes.c_uint16 * n).from_address(ptr)
        return np.frombuffer(buf, dtype=np.uint16, count=n).reshape(self.block_size, self.head_dim).copy()

    def append(self, cur_lens, add_lens, table: np.ndarray) -> int:
        cur, add = _i32(cur_lens), _i32(add_lens)
        assert table.dtype == np.int32 and table.flags.c_contiguous
        return int(lib().oracle_bt_append(self._h, len(cur), _p(cur), _p(add), _p(table),
                                          table.shape[1], self.block_size))

    def free(self, cur_lens, table: np.ndarray) -> int:
        cur = _i32(cur_lens)
        assert table.dtype == np.int32 and table.flags.c_contiguous
        return int(lib().oracle_bt_free(self._h, len(cur), _p(cur), _p(table), table.shape[1],
                                        self.block_size))

    def write_prefill(self, layer: int, k, v, cu_seqlens, table: np.ndarray) -> None:
        k, v, cu = _u16(k), _u16(v), _i32(cu_seqlens)
        rc = lib().oracle_pool_write_prefill(self._h, layer, _p(k), _p(v), _p(cu), len(cu) - 1,
                                             _p(table), table.shape[1])
        if rc != OK:
            raise ValueError(f"oracle_pool_write_prefill rc={rc}")

    def decode(self, layer: int, q, k_new, v_new, table: np.ndarray, cache_lens, scale: float,
               nthreads: int | None = None) -> np.ndarray:
        q, kn, vn, cl = _u16(q), _u16(k_new), _u16(v_new), _i32(cache_lens)
        B, n, d = q.shape
        out = np.zeros((B, n, d), dtype=np.float64)
        rc = lib().oracle_decode(self._h, layer, _p(q), _p(kn), _p(vn), _p(table), table.shape[1],
                                 _p(cl), B, scale, _p(out), nthreads or default_threads())
        if rc != OK:
            raise ValueError(f"oracle_decode rc={rc}")
        return out


def chunked_prefill(pool: "Pool", layer: int, q, k, v, cu_seqlens, prefix_lens, table: np.ndarray, scale: float,
                    nthreads: int | None = None) -> np.ndarray:
    """NEXT-3: append a chunk per sequence after its cached prefix and attend
    (rows of the chunk, fp64 [T][n][d])."""
    q, k, v, cu, pl = _u16(q), _u16(k), _u16(v), _i32(cu_seqlens), _i32(prefix_lens)
    T, n, d = q.shape
    out = np.zeros((T, n, d), dtype=np.float64)
    rc = lib().oracle_chunked_prefill(pool._h, layer, _p(q), _p(k), _p(v), _p(cu), _p(pl), len(cu) - 1, _p(table),
                                      table.shape[1], scale, _p(out), nthreads or default_threads())
    if rc != OK:
        raise ValueError(f"oracle_chunked_prefill rc={rc}")
    return out


def migrate(src: Pool, dst: Pool, layer_begin: int, layer_count: int, src_blocks, dst_blocks,
            src_head0: int, dst_head0: int, head_count: int) -> int:
    sb, db = _i32(src_blocks), _i32(dst_blocks)
    assert len(sb) == len(db)
    nbytes = lib().oracle_migrate(src._h, dst._h, layer_begin, layer_count, _p(sb), _p(db), len(sb),
                                  src_head0, dst_head0, head_count)
    if nbytes < 0:
        raise ValueError("oracle_migrate rejected its arguments")
    return int(nbytes)


def max_rel_err(gpu: np.ndarray, ref: np.ndarray) -> float:
    """per (token, head) vector err = max_k|g-r| / max(max_k|r|, 1e-6);
    returns the maximum over vectors. Arrays [..., d]."""
    g = np.asarray(gpu, dtype=np.float64)
    r = np.asarray(ref, dtype=np.float64)
    num = np.abs(g - r).max(axis=-1)
    den = np.maximum(np.abs(r).max(axis=-1), 1e-6)
    return float((num / den).max()) if num.size else 0.0
