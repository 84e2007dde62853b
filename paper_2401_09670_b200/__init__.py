"""Python binding of libds.so — the B200-native DistServe KV-cache data path.

Thin ctypes marshalling over the C ABI in include/ds.h: every function keeps
the C name and only turns torch tensors into (pointer, size) arguments; all
compute runs in the library's sm_100a kernels. PyTorch is used for device
memory, streams and process groups only.

There is no fallback of any kind: if libds.so is missing or cannot load, the
import raises; on a device that is not sm_100, every compute call raises
DSError (DS_ERR_CUDA).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libds.so")

DS_OK, DS_ERR_INVALID_ARG, DS_ERR_UNSUPPORTED, DS_ERR_NO_BLOCKS, DS_ERR_CUDA, DS_ERR_NCCL, DS_ERR_STATE = range(7)
DS_BT_APPEND, DS_BT_FREE = 0, 1
DS_MIGRATE_SEND, DS_MIGRATE_RECV, DS_MIGRATE_SELF, DS_MIGRATE_LOCAL, DS_MIGRATE_PULL = 0, 1, 2, 3, 4
DS_DECODE_EARLY_KV = 1  # ds_decode_attn_ex flag
BLOCK_SIZE = 16

# every symbol include/ds.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "ds_last_error", "ds_build_info", "ds_pool_create", "ds_pool_destroy", "ds_pool_num_free",
    "ds_block_table", "ds_prefill_attn", "ds_decode_workspace_bytes", "ds_decode_attn", "ds_decode_attn_ex",
    "ds_decode_kernel",
    "ds_kv_staging_bytes", "ds_kv_pack", "ds_kv_unpack", "ds_comm_get_unique_id", "ds_comm_init",
    "ds_comm_destroy", "ds_kv_migrate_staging_bytes", "ds_kv_migrate", "ds_ipc_export_mem", "ds_ipc_open_mem",
    "ds_ipc_close_mem", "ds_event_create_ipc", "ds_event_open_ipc", "ds_event_record", "ds_event_wait",
    "ds_event_destroy", "ds_prefill_attn_chunked", "ds_prefill_attn_push", "ds_kv_migrate_contig",
)


class DSError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"ds status {status}: {msg}")
        self.status = status


class ds_kv_cache(ctypes.Structure):
    _fields_ = [("base", ctypes.c_void_p), ("num_layers", ctypes.c_int32),
                ("num_blocks", ctypes.c_int32), ("num_heads", ctypes.c_int32),
                ("block_size", ctypes.c_int32), ("head_dim", ctypes.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python paper_2401_09670_b200/build.py` "
                          "(there is no fallback implementation)")
    lib = ctypes.CDLL(LIB_PATH)
    P, i32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t
    f32, cache_p = ctypes.c_float, ctypes.POINTER(ds_kv_cache)
    sig = {
        "ds_last_error": ([], ctypes.c_char_p),
        "ds_build_info": ([], ctypes.c_char_p),
        "ds_pool_create": ([i32, ctypes.POINTER(P)], ctypes.c_int),
        "ds_pool_destroy": ([P], ctypes.c_int),
        "ds_pool_num_free": ([P, ctypes.POINTER(i32)], ctypes.c_int),
        "ds_block_table": ([P, i32, i32, P, P, P, i32, i32, ctypes.POINTER(i32)], ctypes.c_int),
        "ds_prefill_attn": ([P, P, P, P, P, i32, i32, i32, cache_p, i32, P, i32, f32, P], ctypes.c_int),
        "ds_prefill_attn_push": ([P, P, P, P, P, i32, i32, i32, cache_p, i32, P, i32, cache_p, i32, P, i32, i32, i32,
                                  f32, P], ctypes.c_int),
        "ds_prefill_attn_chunked": ([P, P, P, P, P, P, i32, i32, i32, i32, cache_p, i32, P, i32, f32, P],
                                    ctypes.c_int),
        "ds_decode_workspace_bytes": ([i32, i32, i32, i32], sz),
        "ds_decode_kernel": ([i32, i32], ctypes.c_char_p),
        "ds_decode_attn": ([P, P, P, P, cache_p, i32, P, i32, P, i32, i32, f32, P, sz, P], ctypes.c_int),
        "ds_decode_attn_ex": ([P, P, P, P, cache_p, i32, P, i32, P, i32, i32, f32, P, sz, ctypes.c_uint32, P],
                              ctypes.c_int),
        "ds_kv_staging_bytes": ([cache_p, i32, i32, i32], sz),
        "ds_kv_pack": ([cache_p, i32, i32, P, i32, i32, i32, P, sz, P], ctypes.c_int),
        "ds_kv_unpack": ([cache_p, i32, i32, P, i32, i32, i32, P, sz, P], ctypes.c_int),
        "ds_comm_get_unique_id": ([P], ctypes.c_int),
        "ds_comm_init": ([P, i32, i32, ctypes.POINTER(P)], ctypes.c_int),
        "ds_comm_destroy": ([P], ctypes.c_int),
        "ds_kv_migrate_staging_bytes": ([cache_p, i32, i32, i32, i32], sz),
        "ds_kv_migrate_contig": ([P, i32, i32, cache_p, i32, i32, i32, i32, cache_p, i32, P], ctypes.c_int),
        "ds_kv_migrate": ([P, i32, i32, cache_p, i32, i32, P, i32, i32, i32, cache_p, P, i32, i32, P, sz, P],
                          ctypes.c_int),
        "ds_ipc_export_mem": ([P, P, ctypes.POINTER(sz)], ctypes.c_int),
        "ds_ipc_open_mem": ([P, ctypes.POINTER(P)], ctypes.c_int),
        "ds_ipc_close_mem": ([P], ctypes.c_int),
        "ds_event_create_ipc": ([ctypes.POINTER(P), P], ctypes.c_int),
        "ds_event_open_ipc": ([P, ctypes.POINTER(P)], ctypes.c_int),
        "ds_event_record": ([P, P], ctypes.c_int),
        "ds_event_wait": ([P, P], ctypes.c_int),
        "ds_event_destroy": ([P], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes, fn.restype = args, res
    return lib


_lib = _load()


def lib():
    return _lib


def ds_last_error() -> str:
    return _lib.ds_last_error().decode()


def ds_build_info() -> str:
    return _lib.ds_build_info().decode()


def _check(status: int):
    if status != DS_OK:
        raise DSError(status, ds_last_error())


# --------------------------------------------------------------------- helpers
def _torch():
    import torch
    return torch


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream) -> int | None:
    torch = _torch()
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _dev(t, dtype, name):
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _check_activations(q, others, cache, what="T"):
    """q [rows][n_loc][head_dim] matching the cache; every tensor in `others` the
    same shape (the C side cannot see device array sizes: a mismatch here would be
    an out-of-bounds device access there)"""
    if q.dim() != 3 or q.shape[1] != cache.heads or q.shape[2] != cache.head_dim:
        raise ValueError(f"q must be [{what}][n_loc][head_dim] matching the cache")
    for t, nm in others:
        if t.shape != q.shape:
            raise ValueError(f"{nm} must have q's shape {tuple(q.shape)}, got {tuple(t.shape)}")


def _check_table(table, rows: int, name: str):
    if table.dim() != 2 or table.shape[0] < rows:
        raise ValueError(f"{name} must be 2-D with at least {rows} rows, got {tuple(table.shape)}")


def _check_seqlens(cu_seqlens, T: int, q_rows: int):
    if cu_seqlens.dim() != 1 or cu_seqlens.numel() < 1:
        raise ValueError("cu_seqlens must be 1-D [num_seqs + 1]")
    if T > q_rows:
        raise ValueError(f"total_tokens {T} exceeds the {q_rows} rows of q")


class KVCache:
    """Caller-owned paged KV pool of one rank: bf16 [L][2][num_blocks][n][16][D]."""

    def __init__(self, tensor):
        torch = _torch()
        _dev(tensor, torch.bfloat16, "cache")
        if tensor.dim() != 6 or tensor.shape[1] != 2 or tensor.shape[4] != BLOCK_SIZE:
            raise ValueError("cache must be [L][2][num_blocks][n][16][head_dim]")
        self.tensor = tensor
        L, _, NB, n, bs, D = tensor.shape
        self.desc = ds_kv_cache(tensor.data_ptr(), L, NB, n, bs, D)

    @classmethod
    def empty(cls, layers, num_blocks, heads, head_dim, device="cuda"):
        torch = _torch()
        return cls(torch.empty((layers, 2, num_blocks, heads, BLOCK_SIZE, head_dim),
                               dtype=torch.bfloat16, device=device))

    @property
    def layers(self):
        return self.desc.num_layers

    @property
    def num_blocks(self):
        return self.desc.num_blocks

    @property
    def heads(self):
        return self.desc.num_heads

    @property
    def head_dim(self):
        return self.desc.head_dim

    def ref(self):
        return ctypes.byref(self.desc)


# --------------------------------------------------------------------- a1
class Pool:
    """ds_pool: library-owned free set of page ids [0, num_blocks)."""

    def __init__(self, num_blocks: int):
        h = ctypes.c_void_p()
        _check(_lib.ds_pool_create(num_blocks, ctypes.byref(h)))
        self._h = h
        self._lib = _lib  # kept alive for __del__ at interpreter shutdown

    def close(self):
        if getattr(self, "_h", None):
            self._lib.ds_pool_destroy(self._h)
            self._h = None

    __del__ = close

    @property
    def num_free(self) -> int:
        n = ctypes.c_int32()
        _check(_lib.ds_pool_num_free(self._h, ctypes.byref(n)))
        return n.value


def ds_block_table(pool: Pool, op: int, cur_lens, add_lens, table: np.ndarray,
                   block_size: int = BLOCK_SIZE) -> int:
    """Host block-table op (APPEND / FREE). `table` is an int32 numpy array
    [num_seqs][max_blocks_per_seq] updated in place; returns the free count."""
    cur = np.ascontiguousarray(cur_lens, dtype=np.int32)
    add = None if add_lens is None else np.ascontiguousarray(add_lens, dtype=np.int32)
    if table.dtype != np.int32 or not table.flags.c_contiguous or table.ndim != 2:
        raise ValueError("table must be a C-contiguous int32 [num_seqs][max_blocks] array")
    if table.shape[0] != len(cur) or (add is not None and len(add) != len(cur)):
        raise ValueError("table rows, cur_lens and add_lens must agree")
    nf = ctypes.c_int32()
    _check(_lib.ds_block_table(pool._h, op, len(cur), cur.ctypes.data, None if add is None else add.ctypes.data,
                               table.ctypes.data, table.shape[1], block_size, ctypes.byref(nf)))
    return nf.value


# --------------------------------------------------------------------- a2 + a3
def ds_prefill_attn(q, k, v, out, cu_seqlens, max_seqlen: int, cache: KVCache, layer: int,
                    block_table, softmax_scale: float, stream=None, total_tokens: int | None = None):
    torch = _torch()
    for t, nm in ((q, "q"), (k, "k"), (v, "v"), (out, "out")):
        _dev(t, torch.bfloat16, nm)
    _dev(cu_seqlens, torch.int32, "cu_seqlens")
    _dev(block_table, torch.int32, "block_table")
    T = q.shape[0] if total_tokens is None else total_tokens
    _check_activations(q, ((k, "k"), (v, "v"), (out, "out")), cache)
    _check_seqlens(cu_seqlens, T, q.shape[0])
    _check_table(block_table, cu_seqlens.numel() - 1, "block_table")
    _check(_lib.ds_prefill_attn(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                cu_seqlens.data_ptr(), cu_seqlens.numel() - 1, T, max_seqlen,
                                cache.ref(), layer, block_table.data_ptr(), block_table.shape[1],
                                softmax_scale, _stream(stream)))


def ds_prefill_attn_push(q, k, v, out, cu_seqlens, max_seqlen: int, cache: KVCache, layer: int, block_table,
                         dst_cache: KVCache, dst_layer: int, dst_block_table, softmax_scale: float,
                         dst_head0: int = 0, write_local: bool = True, stream=None, total_tokens: int | None = None):
    """a2-a6 fused: prefill whose page stores also land in `dst_cache` (the
    decoding instance's pool; a peer GPU's pool mapped through IPC or a pool of
    this GPU) at `dst_layer` / `dst_block_table` / `dst_head0`."""
    torch = _torch()
    for t, nm in ((q, "q"), (k, "k"), (v, "v"), (out, "out")):
        _dev(t, torch.bfloat16, nm)
    _dev(cu_seqlens, torch.int32, "cu_seqlens")
    _dev(block_table, torch.int32, "block_table")
    _dev(dst_block_table, torch.int32, "dst_block_table")
    T = q.shape[0] if total_tokens is None else total_tokens
    _check_activations(q, ((k, "k"), (v, "v"), (out, "out")), cache)
    _check_seqlens(cu_seqlens, T, q.shape[0])
    _check_table(block_table, cu_seqlens.numel() - 1, "block_table")
    _check_table(dst_block_table, cu_seqlens.numel() - 1, "dst_block_table")
    _check(_lib.ds_prefill_attn_push(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                     cu_seqlens.data_ptr(), cu_seqlens.numel() - 1, T, max_seqlen, cache.ref(), layer,
                                     block_table.data_ptr(), block_table.shape[1], dst_cache.ref(), dst_layer,
                                     dst_block_table.data_ptr(), dst_block_table.shape[1], dst_head0,
                                     1 if write_local else 0, softmax_scale, _stream(stream)))


def ds_prefill_attn_chunked(q, k, v, out, cu_seqlens, prefix_lens, max_chunk_len: int, max_context_len: int,
                            cache: KVCache, layer: int, block_table, softmax_scale: float, stream=None):
    """NEXT-3: attend each sequence's next chunk over its cached prefix + itself,
    then append the chunk's K/V to the pages."""
    torch = _torch()
    for t, nm in ((q, "q"), (k, "k"), (v, "v"), (out, "out")):
        _dev(t, torch.bfloat16, nm)
    _dev(cu_seqlens, torch.int32, "cu_seqlens")
    _dev(prefix_lens, torch.int32, "prefix_lens")
    _dev(block_table, torch.int32, "block_table")
    _check_activations(q, ((k, "k"), (v, "v"), (out, "out")), cache)
    _check_seqlens(cu_seqlens, q.shape[0], q.shape[0])
    B = cu_seqlens.numel() - 1
    if prefix_lens.dim() != 1 or prefix_lens.numel() < B:
        raise ValueError(f"prefix_lens must be 1-D with at least {B} entries")
    _check_table(block_table, B, "block_table")
    _check(_lib.ds_prefill_attn_chunked(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                        cu_seqlens.data_ptr(), prefix_lens.data_ptr(), cu_seqlens.numel() - 1,
                                        q.shape[0], max_chunk_len, max_context_len, cache.ref(), layer,
                                        block_table.data_ptr(), block_table.shape[1], softmax_scale,
                                        _stream(stream)))


# --------------------------------------------------------------------- a7 + a8
def ds_decode_kernel(num_seqs: int, n_loc: int) -> str:
    """name of the kernel ds_decode_attn launches for this batch shape"""
    return _lib.ds_decode_kernel(num_seqs, n_loc).decode()


def ds_decode_workspace_bytes(num_seqs: int, n_loc: int, head_dim: int, max_cache_len: int) -> int:
    return int(_lib.ds_decode_workspace_bytes(num_seqs, n_loc, head_dim, max_cache_len))


def ds_decode_attn(q, k_new, v_new, out, cache: KVCache, layer: int, block_table, cache_lens,
                   max_cache_len: int, softmax_scale: float, workspace, stream=None, early_kv: bool = False):
    """early_kv=True: DS_DECODE_EARLY_KV (include/ds.h) — the caller guarantees the
    kernel just ahead on the stream writes neither the lengths, the table nor this
    layer's pages"""
    torch = _torch()
    for t, nm in ((q, "q"), (k_new, "k_new"), (v_new, "v_new"), (out, "out")):
        _dev(t, torch.bfloat16, nm)
    _dev(block_table, torch.int32, "block_table")
    _dev(cache_lens, torch.int32, "cache_lens")
    B = q.shape[0]
    _check_activations(q, ((k_new, "k_new"), (v_new, "v_new"), (out, "out")), cache, "B")
    if cache_lens.dim() != 1 or cache_lens.numel() < B:
        raise ValueError(f"cache_lens must be 1-D with at least {B} entries")
    _check_table(block_table, B, "block_table")
    ws_ptr, ws_bytes = (None, 0) if workspace is None else (workspace.data_ptr(),
                                                            workspace.numel() * workspace.element_size())
    _check(_lib.ds_decode_attn_ex(q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(), out.data_ptr(),
                                  cache.ref(), layer, block_table.data_ptr(), block_table.shape[1],
                                  cache_lens.data_ptr(), B, max_cache_len, softmax_scale, ws_ptr,
                                  ws_bytes, DS_DECODE_EARLY_KV if early_kv else 0, _stream(stream)))


# --------------------------------------------------------------------- a4 / a6
def ds_kv_staging_bytes(cache: KVCache, layer_count: int, num_blocks: int, head_count: int) -> int:
    return int(_lib.ds_kv_staging_bytes(cache.ref(), layer_count, num_blocks, head_count))


def _nbytes(t):
    return t.numel() * t.element_size()


def ds_kv_pack(cache: KVCache, layer_begin: int, layer_count: int, block_ids, head_begin: int,
               head_count: int, staging, stream=None):
    torch = _torch()
    _dev(block_ids, torch.int32, "block_ids")
    _check(_lib.ds_kv_pack(cache.ref(), layer_begin, layer_count, block_ids.data_ptr(), block_ids.numel(),
                           head_begin, head_count, staging.data_ptr(), _nbytes(staging), _stream(stream)))


def ds_kv_unpack(cache: KVCache, layer_begin: int, layer_count: int, block_ids, head_begin: int,
                 head_count: int, staging, stream=None):
    torch = _torch()
    _dev(block_ids, torch.int32, "block_ids")
    _check(_lib.ds_kv_unpack(cache.ref(), layer_begin, layer_count, block_ids.data_ptr(), block_ids.numel(),
                             head_begin, head_count, staging.data_ptr(), _nbytes(staging), _stream(stream)))


# --------------------------------------------------------------------- a5
def ds_comm_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.ds_comm_get_unique_id(buf))
    return buf.raw


class Comm:
    """ds_comm: library-owned NCCL communicator (+ side stream) for KV migration."""

    def __init__(self, unique_id: bytes, nranks: int, rank: int):
        if len(unique_id) != 128:
            raise ValueError("unique_id must be 128 bytes")
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(unique_id, 128)
        _check(_lib.ds_comm_init(buf, nranks, rank, ctypes.byref(h)))
        self._h, self.rank, self.nranks = h, rank, nranks
        self._lib = _lib

    def close(self):
        if getattr(self, "_h", None):
            self._lib.ds_comm_destroy(self._h)
            self._h = None

    __del__ = close


def ds_comm_init(unique_id: bytes, nranks: int, rank: int) -> Comm:
    return Comm(unique_id, nranks, rank)


def ds_kv_migrate_staging_bytes(cache: KVCache, role: int, layer_count: int, num_blocks: int,
                                head_count: int) -> int:
    return int(_lib.ds_kv_migrate_staging_bytes(cache.ref(), role, layer_count, num_blocks, head_count))


def ds_kv_migrate(comm: Comm | None, role: int, peer: int, cache, layer_begin: int, layer_count: int,
                  block_ids, head_begin: int, head_count: int, staging, dst_cache: KVCache | None = None,
                  dst_block_ids=None, dst_head_begin: int = 0, dst_layer_begin: int | None = None, stream=None):
    """`cache` is a KVCache, or (PULL) a RemoteKVCache mapped from another process."""
    torch = _torch()
    _dev(block_ids, torch.int32, "block_ids")
    if dst_block_ids is not None:
        _dev(dst_block_ids, torch.int32, "dst_block_ids")
    _check(_lib.ds_kv_migrate(None if comm is None else comm._h, role, peer, cache.ref(), layer_begin, layer_count,
                              block_ids.data_ptr(), block_ids.numel(), head_begin, head_count,
                              None if dst_cache is None else dst_cache.ref(), _ptr(dst_block_ids),
                              dst_head_begin, layer_begin if dst_layer_begin is None else dst_layer_begin,
                              _ptr(staging), 0 if staging is None else _nbytes(staging), _stream(stream)))


def ds_kv_migrate_contig(comm: Comm, role: int, peer: int, cache, layer_begin: int, layer_count: int,
                         block_begin: int, num_blocks: int, dst_cache: KVCache | None = None,
                         dst_block_begin: int = 0, stream=None):
    """a5 zero-copy: pages [block_begin, +num_blocks) of every layer move pool to pool
    through NCCL (consecutive ids at both ends, all heads)."""
    _check(_lib.ds_kv_migrate_contig(comm._h, role, peer, cache.ref(), layer_begin, layer_count, block_begin,
                                     num_blocks, None if dst_cache is None else dst_cache.ref(), dst_block_begin,
                                     _stream(stream)))


def contiguous_run(ids) -> int | None:
    """first id if `ids` (host, logical order) are consecutive, else None"""
    a = np.asarray(ids).reshape(-1)
    if a.size == 0 or not np.array_equal(a, np.arange(a[0], a[0] + a.size)):
        return None
    return int(a[0])


# --------------------------------------------------------------------- a5, one-sided pull (CUDA IPC)
def ds_ipc_export_mem(tensor) -> tuple[bytes, int]:
    """(64-byte handle of the cudaMalloc allocation holding tensor.data_ptr(),
    byte offset of the tensor inside it)."""
    buf = ctypes.create_string_buffer(64)
    off = ctypes.c_size_t()
    _check(_lib.ds_ipc_export_mem(tensor.data_ptr(), buf, ctypes.byref(off)))
    return buf.raw, off.value


class RemoteKVCache:
    """A prefill rank's KV pool mapped into this process (ds_ipc_open_mem);
    usable as the source `cache` of ds_kv_migrate(DS_MIGRATE_PULL)."""

    def __init__(self, handle: bytes, offset: int, layers: int, num_blocks: int, heads: int, head_dim: int):
        base = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(handle, 64)
        _check(_lib.ds_ipc_open_mem(buf, ctypes.byref(base)))
        self.base = base.value
        self._lib = _lib
        self.desc = ds_kv_cache(self.base + offset, layers, num_blocks, heads, BLOCK_SIZE, head_dim)

    def ref(self):
        return ctypes.byref(self.desc)

    def close(self):
        if getattr(self, "base", None):
            self._lib.ds_ipc_close_mem(self.base)
            self.base = None

    __del__ = close


class IpcEvent:
    """Inter-process CUDA event: create() here and share .handle, or open(handle)."""

    def __init__(self, handle: bytes | None = None):
        h = ctypes.c_void_p()
        if handle is None:
            buf = ctypes.create_string_buffer(64)
            _check(_lib.ds_event_create_ipc(ctypes.byref(h), buf))
            self.handle = buf.raw
        else:
            _check(_lib.ds_event_open_ipc(ctypes.create_string_buffer(handle, 64), ctypes.byref(h)))
            self.handle = handle
        self._h = h
        self._lib = _lib

    def record(self, stream=None):
        _check(_lib.ds_event_record(self._h, _stream(stream)))

    def wait(self, stream=None):
        _check(_lib.ds_event_wait(self._h, _stream(stream)))

    def close(self):
        if getattr(self, "_h", None):
            self._lib.ds_event_destroy(self._h)
            self._h = None

    __del__ = close
