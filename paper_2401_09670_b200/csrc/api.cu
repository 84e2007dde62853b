// api.cu — the C ABI of libds.so (include/ds.h): validation, TMA descriptor
// encoding, launch planning. Every entry point returns ds_status, never throws.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <string>

#include "../../include/ds.h"
#include "internal.h"
#include "kernels.h"

namespace ds {

static thread_local std::string g_last_error;

ds_status fail(ds_status st, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

static ds_status cuda_fail(cudaError_t e, const char *where) {
  return fail(DS_ERR_CUDA, "%s: %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
}

// sm_100 (B200) only; no fallback.
static ds_status require_sm100(const char *where) {
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, where);
  static int cached[64];  // 0 unknown, 1 ok, 2 bad
  if (dev >= 0 && dev < 64 && cached[dev] == 1) return DS_OK;
  int major = 0, minor = 0;
  e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (e != cudaSuccess) return cuda_fail(e, where);
  if (major != 10 || minor != 0)
    return fail(DS_ERR_CUDA, "%s: device %d is sm_%d%d; libds is built for sm_100a only", where,
                dev, major, minor);
  if (dev >= 0 && dev < 64) cached[dev] = 1;
  return DS_OK;
}

static bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

static ds_status check_cache(const ds_kv_cache *c, const char *where) {
  if (!c) return fail(DS_ERR_INVALID_ARG, "%s: cache is NULL", where);
  if (!c->base || !aligned16(c->base)) return fail(DS_ERR_INVALID_ARG, "%s: cache base NULL or not 16-B aligned", where);
  if (c->block_size != 16) return fail(DS_ERR_INVALID_ARG, "%s: block_size must be 16", where);
  if (c->head_dim != 64 && c->head_dim != 128) return fail(DS_ERR_INVALID_ARG, "%s: head_dim must be 64 or 128", where);
  if (c->num_layers <= 0 || c->num_blocks <= 0 || c->num_heads <= 0)
    return fail(DS_ERR_INVALID_ARG, "%s: cache dimensions must be > 0", where);
  return DS_OK;
}

// ----------------------------------------------------------- TMA descriptors
typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                    const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                    const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

static ds_status encode(CUtensorMap *m, void *base, int rank, const cuuint64_t *dims,
                        const cuuint64_t *strides_bytes, const cuuint32_t *box, const char *where,
                        CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B) {
  PFN_encodeTiled fn = get_encode();
  if (!fn) return fail(DS_ERR_CUDA, "%s: cuTensorMapEncodeTiled unavailable", where);
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, base, dims, strides_bytes, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DS_ERR_CUDA, "%s: cuTensorMapEncodeTiled failed (%d)", where, (int)r);
  return DS_OK;
}

// [T][n][D] token-major activations, box = `rows` tokens x 64 dims of one head
static ds_status qkv_map(CUtensorMap *m, const void *p, int T, int n, int D, int rows, const char *where) {
  const cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)n, (cuuint64_t)T};
  const cuuint64_t str[2] = {(cuuint64_t)D * 2, (cuuint64_t)n * D * 2};
  const cuuint32_t box[3] = {64, 1, (cuuint32_t)rows};
  return encode(m, const_cast<void *>(p), 3, dims, str, box, where);
}

// prefill output [T][n][D]: box = 32 tokens x 32 dims of one head, 64-B swizzle (the
// epilogue of one softmax warp: its 32 q rows, one 32-column TMEM chunk at a time)
static ds_status out_map(CUtensorMap *m, void *p, int T, int n, int D, const char *where) {
  const cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)n, (cuuint64_t)T};
  const cuuint64_t str[2] = {(cuuint64_t)D * 2, (cuuint64_t)n * D * 2};
  const cuuint32_t box[3] = {32, 1, 32};
  return encode(m, p, 3, dims, str, box, where, CU_TENSOR_MAP_SWIZZLE_64B);
}

// pool [L*2*NB][n][16][D]; box = one 16-token page x 64 dims
static ds_status cache_map(CUtensorMap *m, const ds_kv_cache *c, const char *where) {
  const int D = c->head_dim;
  const cuuint64_t dims[4] = {(cuuint64_t)D, 16, (cuuint64_t)c->num_heads,
                              (cuuint64_t)c->num_layers * 2 * c->num_blocks};
  const cuuint64_t str[3] = {(cuuint64_t)D * 2, 16ull * D * 2, (cuuint64_t)c->num_heads * 16 * D * 2};
  const cuuint32_t box[4] = {64, 16, 1, 1};
  return encode(m, c->base, 4, dims, str, box, where);
}

// ----------------------------------------------------------- decode planning
static int device_sms() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess &&
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0)
    return sms < kDecodeMaxSMs ? sms : kDecodeMaxSMs;
  return 148;
}

}  // namespace ds

using namespace ds;

extern "C" const char *ds_last_error(void) { return g_last_error.c_str(); }

// Push target of the fused prefill + migration (nullptr: plain prefill).
struct PushTarget {
  const ds_kv_cache *cache;
  int32_t layer;
  const int32_t *block_table;
  int32_t max_blocks, head0, write_local;
};

static ds_status prefill_impl(const char *W, const void *q, const void *k, const void *v, void *out,
                              const int32_t *cu_seqlens, int32_t num_seqs, int32_t total_tokens,
                              int32_t max_seqlen, const ds_kv_cache *cache, int32_t layer,
                              const int32_t *block_table, int32_t max_blocks_per_seq, float softmax_scale,
                              const PushTarget *push, void *stream) {
  if (num_seqs < 0) return fail(DS_ERR_INVALID_ARG, "%s: num_seqs < 0", W);
  if (ds_status s = check_cache(cache, W)) return s;
  if (push) {
    if (ds_status s = check_cache(push->cache, W)) return s;
    if (push->cache->head_dim != cache->head_dim)
      return fail(DS_ERR_INVALID_ARG, "%s: destination pool head_dim differs", W);
    if (push->layer < 0 || push->layer >= push->cache->num_layers)
      return fail(DS_ERR_INVALID_ARG, "%s: dst_layer out of range", W);
    if (push->head0 < 0 || push->head0 + cache->num_heads > push->cache->num_heads)
      return fail(DS_ERR_INVALID_ARG, "%s: dst_head0 + n_loc exceeds the destination pool's heads", W);
    if (push->write_local != 0 && push->write_local != 1)
      return fail(DS_ERR_INVALID_ARG, "%s: write_local must be 0 or 1", W);
  }
  if (num_seqs == 0) return DS_OK;
  if (!q || !k || !v || !out || !cu_seqlens || !block_table || (push && !push->block_table))
    return fail(DS_ERR_INVALID_ARG, "%s: NULL pointer argument", W);
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(out))
    return fail(DS_ERR_INVALID_ARG, "%s: q/k/v/out must be 16-B aligned", W);
  if (total_tokens < num_seqs || max_seqlen < 1 || max_seqlen > total_tokens)
    return fail(DS_ERR_INVALID_ARG, "%s: need num_seqs <= total_tokens and 1 <= max_seqlen <= total_tokens", W);
  if (layer < 0 || layer >= cache->num_layers) return fail(DS_ERR_INVALID_ARG, "%s: layer out of range", W);
  if ((max_seqlen + 15) / 16 > max_blocks_per_seq || (push && (max_seqlen + 15) / 16 > push->max_blocks))
    return fail(DS_ERR_INVALID_ARG, "%s: max_seqlen needs more than max_blocks_per_seq pages", W);
  if (!(softmax_scale > 0.f) || !isfinite(softmax_scale))
    return fail(DS_ERR_INVALID_ARG, "%s: softmax_scale must be finite and > 0", W);
  if (ds_status s = require_sm100(W)) return s;
  const int D = cache->head_dim, n = cache->num_heads;
  // kernel choice: one 128-row q tile per CTA, two CTAs per SM (measured fastest
  // at every length, profiles/r01). DS_PREFILL_KERNEL=2q selects the experimental
  // ping-pong pair-of-q-tiles CTA (prefill2q.cu; parity-tested, slower today).
  static const char *force = getenv("DS_PREFILL_KERNEL");
  const bool two_q = force && strcmp(force, "2q") == 0 && !push;
  const int kv_rows = two_q ? 128 : kPrefillKVRows;
  CUtensorMap tq, tk, tv, tc, to, tdst;
  if (ds_status s = qkv_map(&tq, q, total_tokens, n, D, kPrefillQRows, W)) return s;
  if (ds_status s = out_map(&to, out, total_tokens, n, D, W)) return s;
  if (ds_status s = qkv_map(&tk, k, total_tokens, n, D, kv_rows, W)) return s;
  if (ds_status s = qkv_map(&tv, v, total_tokens, n, D, kv_rows, W)) return s;
  if (ds_status s = cache_map(&tc, cache, W)) return s;
  if (push)
    if (ds_status s = cache_map(&tdst, push->cache, W)) return s;
  PrefillArgs a{};
  a.out = out;
  a.cu_seqlens = cu_seqlens;
  a.prefix_lens = nullptr;
  a.block_table = block_table;
  a.num_seqs = num_seqs;
  a.n_loc = n;
  a.max_blocks = max_blocks_per_seq;
  a.num_q_tiles = two_q ? (max_seqlen + 255) / 256 : (max_seqlen + 127) / 128;
  a.persistent = prefill_persistent(max_seqlen);
  prefill_set_grid(a, total_tokens);
  a.layer = layer;
  a.num_blocks = cache->num_blocks;
  a.scale_log2 = softmax_scale * 1.4426950408889634f;
  a.write_local = 1;
  if (push) {
    a.dst_block_table = push->block_table;
    a.dst_max_blocks = push->max_blocks;
    a.dst_layer = push->layer;
    a.dst_num_blocks = push->cache->num_blocks;
    a.dst_head0 = push->head0;
    a.write_local = push->write_local;
  }
  cudaError_t e = two_q ? launch_prefill2q(a, tq, tk, tv, tc, to, D, static_cast<cudaStream_t>(stream))
                        : launch_prefill(a, tq, tk, tv, tc, to, push ? &tdst : nullptr, D,
                                         static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, W);
  return DS_OK;
}

extern "C" ds_status ds_prefill_attn(const void *q, const void *k, const void *v, void *out,
                                     const int32_t *cu_seqlens, int32_t num_seqs,
                                     int32_t total_tokens, int32_t max_seqlen,
                                     const ds_kv_cache *cache, int32_t layer,
                                     const int32_t *block_table, int32_t max_blocks_per_seq,
                                     float softmax_scale, void *stream) {
  return prefill_impl("ds_prefill_attn", q, k, v, out, cu_seqlens, num_seqs, total_tokens, max_seqlen, cache, layer,
                      block_table, max_blocks_per_seq, softmax_scale, nullptr, stream);
}

extern "C" ds_status ds_prefill_attn_push(const void *q, const void *k, const void *v, void *out,
                                          const int32_t *cu_seqlens, int32_t num_seqs, int32_t total_tokens,
                                          int32_t max_seqlen, const ds_kv_cache *cache, int32_t layer,
                                          const int32_t *block_table, int32_t max_blocks_per_seq,
                                          const ds_kv_cache *dst_cache, int32_t dst_layer,
                                          const int32_t *dst_block_table, int32_t dst_max_blocks_per_seq,
                                          int32_t dst_head0, int32_t write_local, float softmax_scale,
                                          void *stream) {
  const PushTarget push{dst_cache, dst_layer, dst_block_table, dst_max_blocks_per_seq, dst_head0, write_local};
  return prefill_impl("ds_prefill_attn_push", q, k, v, out, cu_seqlens, num_seqs, total_tokens, max_seqlen, cache,
                      layer, block_table, max_blocks_per_seq, softmax_scale, &push, stream);
}

extern "C" ds_status ds_prefill_attn_chunked(const void *q, const void *k, const void *v, void *out,
                                             const int32_t *cu_seqlens, const int32_t *prefix_lens,
                                             int32_t num_seqs, int32_t total_tokens, int32_t max_chunk_len,
                                             int32_t max_context_len, const ds_kv_cache *cache, int32_t layer,
                                             const int32_t *block_table, int32_t max_blocks_per_seq,
                                             float softmax_scale, void *stream) {
  const char *W = "ds_prefill_attn_chunked";
  if (num_seqs < 0) return fail(DS_ERR_INVALID_ARG, "%s: num_seqs < 0", W);
  if (ds_status s = check_cache(cache, W)) return s;
  if (num_seqs == 0) return DS_OK;
  if (!q || !k || !v || !out || !cu_seqlens || !prefix_lens || !block_table)
    return fail(DS_ERR_INVALID_ARG, "%s: NULL pointer argument", W);
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(out))
    return fail(DS_ERR_INVALID_ARG, "%s: q/k/v/out must be 16-B aligned", W);
  if (total_tokens < num_seqs || max_chunk_len < 1 || max_chunk_len > total_tokens || max_context_len < max_chunk_len)
    return fail(DS_ERR_INVALID_ARG, "%s: bad lengths", W);
  if (layer < 0 || layer >= cache->num_layers) return fail(DS_ERR_INVALID_ARG, "%s: layer out of range", W);
  if ((max_context_len + 15) / 16 > max_blocks_per_seq)
    return fail(DS_ERR_INVALID_ARG, "%s: prefix + chunk needs more than max_blocks_per_seq pages", W);
  if (!(softmax_scale > 0.f) || !isfinite(softmax_scale))
    return fail(DS_ERR_INVALID_ARG, "%s: softmax_scale must be finite and > 0", W);
  if (ds_status s = require_sm100(W)) return s;
  const int D = cache->head_dim, n = cache->num_heads;
  CUtensorMap tq, tk, tv, tc, to;
  if (ds_status s = qkv_map(&tq, q, total_tokens, n, D, kPrefillQRows, W)) return s;
  if (ds_status s = out_map(&to, out, total_tokens, n, D, W)) return s;
  if (ds_status s = qkv_map(&tk, k, total_tokens, n, D, kPrefillKVRows, W)) return s;
  if (ds_status s = qkv_map(&tv, v, total_tokens, n, D, kPrefillKVRows, W)) return s;
  if (ds_status s = cache_map(&tc, cache, W)) return s;
  PrefillArgs a{};
  a.out = out;
  a.cu_seqlens = cu_seqlens;
  a.prefix_lens = prefix_lens;
  a.block_table = block_table;
  a.num_seqs = num_seqs;
  a.n_loc = n;
  a.max_blocks = max_blocks_per_seq;
  a.num_q_tiles = (max_chunk_len + 127) / 128;
  a.persistent = prefill_persistent(max_context_len);  // an item attends the prefix + its chunk rows
  prefill_set_grid(a, total_tokens);
  a.layer = layer;
  a.num_blocks = cache->num_blocks;
  a.scale_log2 = softmax_scale * 1.4426950408889634f;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = launch_prefill(a, tq, tk, tv, tc, to, nullptr, D, st);  // reads the prefix pages + the chunk
  if (e != cudaSuccess) return cuda_fail(e, W);
  KvAppendArgs ap{};  // then the chunk's K/V join the pages (positions prefix + t)
  ap.k = static_cast<const uint16_t *>(k);
  ap.v = static_cast<const uint16_t *>(v);
  ap.cache = static_cast<uint16_t *>(cache->base);
  ap.cu_seqlens = cu_seqlens;
  ap.prefix_lens = prefix_lens;
  ap.block_table = block_table;
  ap.num_seqs = num_seqs;
  ap.n_loc = n;
  ap.head_dim = D;
  ap.max_blocks = max_blocks_per_seq;
  ap.layer = layer;
  ap.num_blocks = cache->num_blocks;
  ap.total_tokens = total_tokens;
  e = launch_kv_append(ap, st);
  if (e != cudaSuccess) return cuda_fail(e, W);
  return DS_OK;
}

extern "C" const char *ds_decode_kernel(int32_t num_seqs, int32_t n_loc) {
  return decode_uses_pairs(num_seqs, n_loc, device_sms()) ? "decode_pairs_kernel" : "decode_kernel";
}

extern "C" size_t ds_decode_workspace_bytes(int32_t num_seqs, int32_t n_loc, int32_t head_dim,
                                            int32_t max_cache_len) {
  if (num_seqs <= 0 || n_loc <= 0 || (head_dim != 64 && head_dim != 128) || max_cache_len < 0) return 0;
  return decode_layout(num_seqs, n_loc, head_dim, kDecodeMaxSMs, max_cache_len).total;
}

extern "C" ds_status ds_decode_attn_ex(const void *q, const void *k_new, const void *v_new, void *out,
                                       const ds_kv_cache *cache, int32_t layer,
                                       const int32_t *block_table, int32_t max_blocks_per_seq,
                                       const int32_t *cache_lens, int32_t num_seqs,
                                       int32_t max_cache_len, float softmax_scale, void *workspace,
                                       size_t workspace_bytes, uint32_t flags, void *stream) {
  const char *W = "ds_decode_attn";
  if (flags & ~(uint32_t)DS_DECODE_EARLY_KV) return fail(DS_ERR_INVALID_ARG, "%s: unknown flags", W);
  if (num_seqs < 0) return fail(DS_ERR_INVALID_ARG, "%s: num_seqs < 0", W);
  if (ds_status s = check_cache(cache, W)) return s;
  if (num_seqs == 0) return DS_OK;
  if (num_seqs > kDecodeMaxSeqs)
    return fail(DS_ERR_INVALID_ARG, "%s: at most %d sequences per call", W, kDecodeMaxSeqs);
  if ((int64_t)num_seqs * cache->num_heads > kDecodeMaxPairs)
    return fail(DS_ERR_INVALID_ARG, "%s: num_seqs * n_loc must be <= %d", W, kDecodeMaxPairs);
  if (!q || !k_new || !v_new || !out || !block_table || !cache_lens)
    return fail(DS_ERR_INVALID_ARG, "%s: NULL pointer argument", W);
  if (!aligned16(q) || !aligned16(k_new) || !aligned16(v_new) || !aligned16(out))
    return fail(DS_ERR_INVALID_ARG, "%s: q/k_new/v_new/out must be 16-B aligned", W);
  if (layer < 0 || layer >= cache->num_layers) return fail(DS_ERR_INVALID_ARG, "%s: layer out of range", W);
  if (max_cache_len < 0 || max_cache_len / 16 >= max_blocks_per_seq)
    return fail(DS_ERR_INVALID_ARG, "%s: max_cache_len out of range for max_blocks_per_seq", W);
  if (!(softmax_scale > 0.f) || !isfinite(softmax_scale))
    return fail(DS_ERR_INVALID_ARG, "%s: softmax_scale must be finite and > 0", W);
  const int D = cache->head_dim, n = cache->num_heads;
  const size_t need = ds_decode_workspace_bytes(num_seqs, n, D, max_cache_len);
  if (!workspace || workspace_bytes < need || !aligned16(workspace))
    return fail(DS_ERR_INVALID_ARG, "%s: workspace must be >= %zu bytes and 16-B aligned", W, need);
  if (ds_status s = require_sm100(W)) return s;
  DecodeArgs a{};
  a.q = static_cast<const uint16_t *>(q);
  a.k_new = static_cast<const uint16_t *>(k_new);
  a.v_new = static_cast<const uint16_t *>(v_new);
  a.out = out;
  a.cache = static_cast<const uint16_t *>(cache->base);
  a.block_table = block_table;
  a.cache_lens = cache_lens;
  const DecodeLayout L = decode_layout(num_seqs, n, D, kDecodeMaxSMs, max_cache_len);
  char *wsb = static_cast<char *>(workspace);
  a.dyn = reinterpret_cast<int32_t *>(wsb + L.dyn_off);
  a.workspace = reinterpret_cast<float *>(wsb + L.rows_off);
  a.tickets = reinterpret_cast<int32_t *>(wsb + L.tickets_off);
  a.chunk_rows = reinterpret_cast<float *>(wsb + L.chunk_off);
  a.max_chunks = L.max_chunks;
  a.max_cache_len = max_cache_len;
  a.early_kv = (flags & DS_DECODE_EARLY_KV) ? 1 : 0;
  a.layer = layer;
  a.num_blocks = cache->num_blocks;
  a.n_loc = n;
  a.max_blocks = max_blocks_per_seq;
  a.num_seqs = num_seqs;
  a.scale_log2 = softmax_scale * 1.4426950408889634f;
  cudaError_t e = launch_decode(a, D, device_sms(), static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, W);
  return DS_OK;
}

extern "C" ds_status ds_decode_attn(const void *q, const void *k_new, const void *v_new, void *out,
                                    const ds_kv_cache *cache, int32_t layer,
                                    const int32_t *block_table, int32_t max_blocks_per_seq,
                                    const int32_t *cache_lens, int32_t num_seqs,
                                    int32_t max_cache_len, float softmax_scale, void *workspace,
                                    size_t workspace_bytes, void *stream) {
  return ds_decode_attn_ex(q, k_new, v_new, out, cache, layer, block_table, max_blocks_per_seq, cache_lens,
                           num_seqs, max_cache_len, softmax_scale, workspace, workspace_bytes, 0u, stream);
}

// ----------------------------------------------------------- a4 / a6
extern "C" size_t ds_kv_staging_bytes(const ds_kv_cache *cache, int32_t layer_count,
                                      int32_t num_blocks, int32_t head_count) {
  if (!cache || layer_count < 0 || num_blocks < 0 || head_count < 0) return 0;
  return (size_t)layer_count * 2 * num_blocks * head_count * 16 * cache->head_dim * 2;
}

namespace ds {
ds_status kv_copy_checked(const ds_kv_cache *cache, int32_t layer_begin, int32_t layer_count,
                          const int32_t *block_ids, int32_t num_blocks, int32_t head_begin,
                          int32_t head_count, void *staging, size_t staging_bytes,
                          int64_t row_begin, int64_t row_end, bool pack, cudaStream_t stream,
                          const char *W, bool dry_run = false) {
  if (ds_status s = check_cache(cache, W)) return s;
  if (layer_count < 0 || num_blocks < 0 || head_count < 0)
    return fail(DS_ERR_INVALID_ARG, "%s: negative count", W);
  if (layer_begin < 0 || layer_begin + layer_count > cache->num_layers)
    return fail(DS_ERR_INVALID_ARG, "%s: layer range outside the pool", W);
  if (head_begin < 0 || head_begin + head_count > cache->num_heads)
    return fail(DS_ERR_INVALID_ARG, "%s: head slice outside n_loc", W);
  const int64_t rows = (int64_t)layer_count * 2 * num_blocks;
  if (row_end <= row_begin || rows == 0 || head_count == 0) return DS_OK;
  if (!block_ids || !staging) return fail(DS_ERR_INVALID_ARG, "%s: NULL pointer argument", W);
  if (!aligned16(staging)) return fail(DS_ERR_INVALID_ARG, "%s: staging must be 16-B aligned", W);
  const size_t row_bytes = (size_t)head_count * 16 * cache->head_dim * 2;
  if (staging_bytes < (size_t)(row_end - row_begin) * row_bytes)
    return fail(DS_ERR_INVALID_ARG, "%s: staging_bytes too small", W);
  if (ds_status s = require_sm100(W)) return s;
  if (dry_run) return DS_OK;  // every check passed; the caller launches later
  KvCopyArgs a{};
  a.cache = static_cast<uint16_t *>(cache->base);
  a.staging = static_cast<uint16_t *>(staging);
  a.block_ids = block_ids;
  a.layer_begin = layer_begin;
  a.num_blocks_sel = num_blocks;
  a.head_begin = head_begin;
  a.head_count = head_count;
  a.pool_blocks = cache->num_blocks;
  a.n_loc = cache->num_heads;
  a.head_dim = cache->head_dim;
  a.row_begin = row_begin;
  a.row_end = row_end;
  cudaError_t e = launch_kv_copy(a, pack, stream);
  if (e != cudaSuccess) return cuda_fail(e, W);
  return DS_OK;
}
}  // namespace ds

extern "C" ds_status ds_kv_pack(const ds_kv_cache *cache, int32_t layer_begin, int32_t layer_count,
                                const int32_t *block_ids, int32_t num_blocks, int32_t head_begin,
                                int32_t head_count, void *staging, size_t staging_bytes,
                                void *stream) {
  return kv_copy_checked(cache, layer_begin, layer_count, block_ids, num_blocks, head_begin,
                         head_count, staging, staging_bytes, 0,
                         (int64_t)layer_count * 2 * num_blocks, true,
                         static_cast<cudaStream_t>(stream), "ds_kv_pack");
}

extern "C" ds_status ds_kv_unpack(const ds_kv_cache *cache, int32_t layer_begin,
                                  int32_t layer_count, const int32_t *block_ids,
                                  int32_t num_blocks, int32_t head_begin, int32_t head_count,
                                  const void *staging, size_t staging_bytes, void *stream) {
  return kv_copy_checked(cache, layer_begin, layer_count, block_ids, num_blocks, head_begin,
                         head_count, const_cast<void *>(staging), staging_bytes, 0,
                         (int64_t)layer_count * 2 * num_blocks, false,
                         static_cast<cudaStream_t>(stream), "ds_kv_unpack");
}
