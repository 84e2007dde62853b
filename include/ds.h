/*
 * ds.h — C ABI of the B200-native DistServe KV-cache data path (libds.so).
 *
 * DistServe (arXiv 2401.09670) disaggregates LLM serving into a prefill
 * instance and a decoding instance. The prefill instance
 * computes the prompt's KV cache and keeps it in its GPU memory;
 * the decoding instance receives "the KV caches and the first output token"
 * by pulling them into paged memory (PagedAttention, P:251,
 * P:407) and then generates one token per step.
 * Tensor parallelism divides the heads; KV moves only between
 * corresponding layers.
 *
 * This header is the whole boundary of the hot path:
 *   a1  ds_block_table      page allocation / block tables (host)
 *   a2+a3 ds_prefill_attn   causal prefill attention + paged K/V write
 *   a2-a6 ds_prefill_attn_push  the same with the migration fused in (pages
 *                           stored straight into the decoding instance's pool)
 *   a4  ds_kv_pack          gather pages of a head slice into a staging buffer
 *   a5  ds_kv_migrate       pack -> NCCL send/recv over NVLink -> unpack
 *   a6  ds_kv_unpack        scatter a staging buffer into pages
 *   a7+a8 ds_decode_attn    decode append + split-K paged attention + combine
 *
 * Conventions (all entry points):
 *  - Every call returns ds_status and never throws or aborts. On a non-OK
 *    status, ds_last_error() returns thread-local text describing it.
 *  - Validation is synchronous and happens before any launch; a rejected call
 *    launches nothing and changes nothing.
 *  - GPU work is stream-ordered and asynchronous on the caller's `stream`
 *    (a cudaStream_t passed as void*; NULL = legacy default stream). Device
 *    faults surface at the caller's next synchronisation.
 *  - Pointers are DEVICE pointers unless the name ends in `_h` (host).
 *  - All K/V/Q/O tensors are bf16 (2 bytes); there is no dtype or arch dispatch:
 *    bf16 and sm_100a only. There is no CPU fallback: without a usable sm_100
 *    device every compute entry point returns DS_ERR_CUDA.
 *  - Ownership: all tensors, tables, workspaces and staging buffers are owned
 *    by the caller (allocated with torch in the Python layer). The library owns
 *    only the opaque handles (ds_pool, ds_comm) and cached TMA descriptors.
 *    Pointer arguments are not retained after the call's stream work completes.
 *
 * KV cache layout (one allocation per pool and rank; reading R3/R-layout):
 *   base[L_loc][2 (0=K,1=V)][num_blocks][n_loc][block_size=16][head_dim]
 * A page (layer, kv, block, head) is 16*head_dim*2 bytes contiguous (4 KiB at
 * head_dim 128); a head range inside one block is contiguous.
 */
#ifndef DS_H_
#define DS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DS_OK = 0,
  DS_ERR_INVALID_ARG = 1, /* argument validation failed; nothing launched */
  DS_ERR_UNSUPPORTED = 2, /* valid request this build does not implement */
  DS_ERR_NO_BLOCKS = 3,   /* pool too small; all-or-nothing, nothing changed */
  DS_ERR_CUDA = 4,        /* CUDA runtime/launch error or no sm_100 device */
  DS_ERR_NCCL = 5,        /* NCCL error (text from ncclGetErrorString) */
  DS_ERR_STATE = 6        /* handle misuse (destroyed, wrong role, ...) */
} ds_status;

/* Thread-local description of the last non-OK status on this thread. */
const char *ds_last_error(void);

/* Library/build identification: e.g. "libds sm_100a nccl 2.28.9". */
const char *ds_build_info(void);

/* Caller-owned paged KV pool of one rank (layout above). */
typedef struct {
  void *base;         /* device, 16-B aligned */
  int32_t num_layers; /* L_loc  (PP stage's layer count)  */
  int32_t num_blocks; /* pages per (layer, kv, head)              */
  int32_t num_heads;  /* n_loc  (TP rank's head count)     */
  int32_t block_size; /* must be 16 (BASELINE.json)               */
  int32_t head_dim;   /* 64 or 128                                */
} ds_kv_cache;

/* ======================================================================
 * a1 — page allocation and block tables (host, synchronous).
 * PagedAttention-style fixed-size pages with a per-request logical->physical
 * map. The paper gives no policy; ours (reading R13):
 * lowest free id first, sequences in argument order, blocks in logical order.
 * ==================================================================== */
typedef struct ds_pool_s *ds_pool; /* library-owned free set of [0, num_blocks) */

ds_status ds_pool_create(int32_t num_blocks, ds_pool *out_h);
ds_status ds_pool_destroy(ds_pool pool);
/* Number of free pages (host). */
ds_status ds_pool_num_free(ds_pool pool, int32_t *num_free_h);

enum { DS_BT_APPEND = 0, DS_BT_FREE = 1 };

/* op = DS_BT_APPEND: for each sequence s grow from cur_lens_h[s] to
 *   cur_lens_h[s] + add_lens_h[s] tokens; a page is taken for each logical block
 *   in [ceil(cur/bs), ceil((cur+add)/bs)) and written to table_h[s][block].
 *   ALLOC is APPEND from cur_len 0. Entries below ceil(cur/bs) are not touched.
 *   If the pool cannot satisfy the whole call: DS_ERR_NO_BLOCKS, nothing changes
 *   (SPEC CapacityError / up-front admission).
 * op = DS_BT_FREE: return the ceil(cur_lens_h[s]/bs) pages of each row to the
 *   pool and set those entries to -1 (add_lens_h ignored, may be NULL).
 * table_h: host int32 [num_seqs][max_blocks_per_seq], row-major, -1 = no page.
 * block_size must be 16. num_seqs == 0 is a no-op. num_free_h may be NULL.
 * Errors: DS_ERR_INVALID_ARG (negative lengths, ceil(len/bs) > max_blocks_per_seq,
 * FREE of an id that is not allocated or that appears twice in the call; a
 * rejected FREE frees nothing), DS_ERR_NO_BLOCKS, DS_ERR_STATE (free set
 * inconsistent; nothing allocated). */
ds_status ds_block_table(ds_pool pool, int32_t op, int32_t num_seqs,
                         const int32_t *cur_lens_h, const int32_t *add_lens_h,
                         int32_t *table_h, int32_t max_blocks_per_seq,
                         int32_t block_size, int32_t *num_free_h);

/* ======================================================================
 * a2 + a3 — prefill causal attention of one layer, fused paged K/V write.
 * For every sequence r, head h, row i < l_r (§2.1; App. A:
 * attention only among the tokens of the same request; readings R1, R2):
 *   out[i] = sum_{j<=i} softmax_j(scale * q[i].k[j]) v[j]
 * and (a3, "KV caches ... saved in GPU memory"):
 *   cache[layer][K][block_table[r][t/16]][h][t%16][:] = k[t][h][:]   (and V)
 *
 * q, k, v, out : bf16 [T][n_loc][head_dim], packed varlen (token-major), T =
 *                total_tokens = cu_seqlens[num_seqs] (host value; sizes the TMA
 *                descriptors); row stride n_loc*head_dim.
 * cu_seqlens   : device int32 [num_seqs+1], cu[0]=0, non-decreasing, every
 *                length >= 1; max_seqlen >= every length (host value).
 * block_table  : device int32 [num_seqs][max_blocks_per_seq]; row r must hold
 *                ceil(l_r/16) valid page ids (from ds_block_table APPEND).
 * cache        : host pointer to the pool descriptor; cache->num_heads must
 *                equal n_loc. layer in [0, num_layers).
 * Numerics: bf16 inputs, fp32 S and O accumulation (tcgen05, TMEM), online
 * base-2 softmax, P rounded to bf16 for the P.V MMA, bf16 output (RNE).
 * Page slots at positions >= l_r in a sequence's last page are unspecified.
 * Errors: DS_ERR_INVALID_ARG (head_dim not 64/128, block_size != 16, misaligned
 * pointers, num_seqs < 0, max_seqlen < 1, layer out of range), DS_ERR_CUDA. */
ds_status ds_prefill_attn(const void *q, const void *k, const void *v, void *out,
                          const int32_t *cu_seqlens, int32_t num_seqs, int32_t total_tokens,
                          int32_t max_seqlen,
                          const ds_kv_cache *cache, int32_t layer,
                          const int32_t *block_table, int32_t max_blocks_per_seq,
                          float softmax_scale, void *stream);

/* ======================================================================
 * a2 + a3 + a4-a6 fused — prefill with the page migration inside the kernel
 * ("push"): as ds_prefill_attn, and every K/V page the kernel writes is also
 * stored, from the same shared-memory tile, into a DESTINATION pool — the
 * decoding instance's ("the decode instance receives the KV caches"),
 * either a peer GPU's pool mapped with ds_ipc_open_mem (the stores cross NVLink
 * while the attention of later tiles runs) or another pool of this GPU:
 *   dst[dst_layer][K|V][dst_block_table[r][t/16]][dst_head0 + h][t%16] = k|v[t][h]
 * The decoding side must have admitted the batch (allocated its pages) before
 * the call — the paper's pull lets the prefill GPU buffer the pages
 * until the decoder has memory; this push is the variant for a decoder that
 * already has it, and costs no separate migration pass.
 * dst_cache      : host descriptor of the destination pool (base may be a
 *                  peer-mapped pointer); same head_dim and block size;
 *                  dst_head0 + n_loc <= dst_cache->num_heads.
 * dst_block_table: device int32 [num_seqs][dst_max_blocks_per_seq] (this
 *                  GPU's memory), ceil(l_r/16) valid destination page ids per row.
 * write_local    : 1 also writes the source pool as ds_prefill_attn does;
 *                  0 writes the pages only to the destination.
 * Errors as ds_prefill_attn, plus DS_ERR_INVALID_ARG for a bad destination.
 * ==================================================================== */
ds_status ds_prefill_attn_push(const void *q, const void *k, const void *v, void *out,
                               const int32_t *cu_seqlens, int32_t num_seqs, int32_t total_tokens,
                               int32_t max_seqlen, const ds_kv_cache *cache, int32_t layer,
                               const int32_t *block_table, int32_t max_blocks_per_seq,
                               const ds_kv_cache *dst_cache, int32_t dst_layer,
                               const int32_t *dst_block_table, int32_t dst_max_blocks_per_seq,
                               int32_t dst_head0, int32_t write_local, float softmax_scale, void *stream);

/* ======================================================================
 * NEXT-3 — chunked prefill over a paged prefix, the technique the
 * paper contrasts with disaggregation ("segmenting long prefill into
 * chunks": chunk k re-reads the KV of all earlier chunks). Sequence r
 * already holds c_r = prefix_lens[r] tokens in the pool; its next chunk of l_r
 * tokens (q, k, v packed by cu_seqlens) is attended and appended:
 *   out[i] = sum_{j <= c_r + i} softmax_j(scale * q[i].key[j]) value[j]
 * with keys/values j < c_r read from the pages (block_table) and j >= c_r the
 * chunk's own; then cache[...][pos = c_r + t] = k[t], v[t]. With every c_r = 0
 * this is ds_prefill_attn. The block table must already hold the pages of
 * positions [0, c_r + l_r). prefix_lens: device int32 [num_seqs];
 * max_chunk_len >= every l_r and max_context_len >= every c_r + l_r: host bounds. Two launches (attention, then
 * the page append of the chunk). Errors as ds_prefill_attn.
 * ==================================================================== */
ds_status ds_prefill_attn_chunked(const void *q, const void *k, const void *v, void *out,
                                  const int32_t *cu_seqlens, const int32_t *prefix_lens,
                                  int32_t num_seqs, int32_t total_tokens, int32_t max_chunk_len,
                                  int32_t max_context_len, const ds_kv_cache *cache, int32_t layer,
                                  const int32_t *block_table, int32_t max_blocks_per_seq,
                                  float softmax_scale, void *stream);

/* ======================================================================
 * a7 + a8 — one decode step of one layer ("generates subsequent tokens
 * one at a time"; P:237 batching; P:696-698 memory-bound decode attention).
 * Reading R9: the new token's K/V are appended at position c = cache_lens[b]
 * BEFORE attending, so the step attends c+1 tokens and equals row c of
 * prefill over those c+1 tokens:
 *   (i)  cache[layer][K][bt[b][c/16]][h][c%16] = k_new[b][h]   (and V)
 *   (ii) out[b][h] = sum_{j<=c} softmax_j(scale * q[b][h].k[j]) v[j]
 * q, k_new, v_new, out : bf16 [num_seqs][n_loc][head_dim].
 * block_table : device int32 [num_seqs][max_blocks_per_seq]; row b must already
 *               hold the page for position c (ds_block_table APPEND by 1).
 * cache_lens  : device int32 [num_seqs], c >= 0; max_cache_len >= every c
 *               (host value; sizes the split-K grid).
 * workspace   : device scratch of >= ds_decode_workspace_bytes(...) bytes, 16-B
 *               aligned, caller-owned. It must be ZEROED once before its first
 *               use (e.g. torch.zeros); every call leaves it zeroed again (it
 *               holds split partials and self-resetting merge tickets). Calls
 *               sharing a workspace must be ordered on one stream. The merge
 *               tickets and counters sit in a fixed region at a fixed offset, so
 *               one workspace may serve calls of any batch, head count, head_dim
 *               or length as long as it is large enough for each call.
 * Limits      : num_seqs <= 4096 and num_seqs * n_loc <= 524288 (DS_ERR_INVALID_ARG).
 * Work split: the (seq, head, page) space is cut into equal page ranges, one
 * per warp of a persistent grid; a pair that straddles ranges is merged from
 * its partials (m, l, o) with the log-sum-exp rule (a8), inside the same launch.
 * (Opt-in, environment DS_DEC_PAIRS=k read once per process: from k pairs per SM
 * on, each pair is streamed by one CTA that takes pairs from a counter in the
 * workspace and merges its warps' partials in shared memory; see decode.cu.)
 * Where pages are assigned dynamically (the last 10 % of the pages of big
 * launches; the pair counter) the grouping of pages into partials may differ from
 * call to call, so results agree to fp32 rounding of the merge, not bit for bit;
 * fixed-assignment launches are bitwise reproducible.
 * Errors: DS_ERR_INVALID_ARG, DS_ERR_CUDA. */
size_t ds_decode_workspace_bytes(int32_t num_seqs, int32_t n_loc, int32_t head_dim,
                                 int32_t max_cache_len);
/* ds_decode_kernel — the name of the kernel ds_decode_attn launches for this batch
 * shape on the current device ("decode_pairs_kernel" or "decode_kernel"; a static
 * string, never NULL), for profilers and reports. No device work. */
const char *ds_decode_kernel(int32_t num_seqs, int32_t n_loc);
ds_status ds_decode_attn(const void *q, const void *k_new, const void *v_new, void *out,
                         const ds_kv_cache *cache, int32_t layer,
                         const int32_t *block_table, int32_t max_blocks_per_seq,
                         const int32_t *cache_lens, int32_t num_seqs, int32_t max_cache_len,
                         float softmax_scale, void *workspace, size_t workspace_bytes,
                         void *stream);

/* ds_decode_attn_ex — ds_decode_attn with a flags word (ds_decode_attn == flags 0).
 * DS_DECODE_EARLY_KV: the kernel is launched with programmatic dependent launch
 *   (PDL) and reads cache_lens, block_table and this layer's K/V pages BEFORE the
 *   kernel ahead of it on the stream has finished (its first pages are already in
 *   flight when that kernel drains); q, k_new, v_new, out and workspace are touched
 *   only after it has finished. The CALLER guarantees that the immediately
 *   preceding kernel on the stream writes neither cache_lens, nor block_table, nor
 *   any page of `layer` that this call reads — e.g. a loop of ds_decode_attn over
 *   the layers of one step (each call appends only to its own layer), or a kernel
 *   that only produces q/k_new/v_new. (The kernel before that one has always
 *   finished: an early call lets its successor start only after its own wait.)
 *   A host copy ahead of the call is always safe (it ends the overlap). The
 *   flag changes no arithmetic (results as without it, up to the dynamic
 *   assignment noted above).
 * Errors: as ds_decode_attn; DS_ERR_INVALID_ARG for unknown flag bits. */
#define DS_DECODE_EARLY_KV 1u
ds_status ds_decode_attn_ex(const void *q, const void *k_new, const void *v_new, void *out,
                            const ds_kv_cache *cache, int32_t layer,
                            const int32_t *block_table, int32_t max_blocks_per_seq,
                            const int32_t *cache_lens, int32_t num_seqs, int32_t max_cache_len,
                            float softmax_scale, void *workspace, size_t workspace_bytes,
                            uint32_t flags, void *stream);

/* ======================================================================
 * a4 / a6 — pack and unpack whole pages of a head slice (KV migration, P:363:
 * only between corresponding layers; P:633 head shards; reading R14: whole
 * pages move, slots beyond a sequence's length are unspecified).
 * Staging layout (contiguous, bf16):
 *   staging[layer - layer_begin][kv][i][0:head_count][16][head_dim]
 *     = cache[layer][kv][block_ids[i]][head_begin : head_begin+head_count]
 * for i in [0, num_blocks), layer in [layer_begin, layer_begin+layer_count).
 * Size: ds_kv_staging_bytes(...) = layer_count*2*num_blocks*head_count*16*head_dim*2.
 * block_ids: device int32 [num_blocks] (logical order of the requests' pages).
 * ds_kv_unpack is the inverse scatter into the destination cache's pages.
 * Errors: DS_ERR_INVALID_ARG (ranges, sizes, alignment), DS_ERR_CUDA. */
size_t ds_kv_staging_bytes(const ds_kv_cache *cache, int32_t layer_count,
                           int32_t num_blocks, int32_t head_count);
ds_status ds_kv_pack(const ds_kv_cache *cache, int32_t layer_begin, int32_t layer_count,
                     const int32_t *block_ids, int32_t num_blocks, int32_t head_begin,
                     int32_t head_count, void *staging, size_t staging_bytes, void *stream);
ds_status ds_kv_unpack(const ds_kv_cache *cache, int32_t layer_begin, int32_t layer_count,
                       const int32_t *block_ids, int32_t num_blocks, int32_t head_begin,
                       int32_t head_count, const void *staging, size_t staging_bytes,
                       void *stream);

/* ======================================================================
 * a5 — KV migration prefill rank -> decode rank over NVLink with NCCL p2p
 * ("NCCL ... and asynchronous CudaMemcpy", P:265 sizing, P:382 pull,
 * P:512 transfer time). The communicator is library-owned and bootstrapped
 * by the caller exchanging the 128-byte unique id (e.g. via torch's store).
 * ==================================================================== */
typedef struct ds_comm_s *ds_comm;

/* Writes a 128-byte ncclUniqueId into id_h (host). */
ds_status ds_comm_get_unique_id(void *id_h);
/* Collective over the nranks processes; binds to the current CUDA device. */
ds_status ds_comm_init(const void *id_h, int32_t nranks, int32_t rank, ds_comm *out_h);
ds_status ds_comm_destroy(ds_comm comm);

enum { DS_MIGRATE_SEND = 0, DS_MIGRATE_RECV = 1, DS_MIGRATE_SELF = 2, DS_MIGRATE_LOCAL = 3 };

/* Move whole pages of (layers [layer_begin, +layer_count), head slice
 * [head_begin, +head_count), block_ids[0..num_blocks)) from a prefill rank to
 * a decode rank. Both sides call it with equal layer_count, num_blocks and
 * head_count (their block ids and head offsets may differ):
 *  role SEND (prefill side, `peer` = decode rank): ds_kv_pack into the staging
 *       buffer chunk by chunk, ncclSend each chunk.
 *  role RECV (decode side, `peer` = prefill rank): ncclRecv each chunk into
 *       staging, ds_kv_unpack it into this rank's pages.
 *  role SELF (one rank plays both, N=1 loopback through NCCL): `cache` is the
 *       source, `dst_cache`/`dst_block_ids`/`dst_head_begin` the destination;
 *       the staging buffer holds two halves (send and receive side).
 *  role LOCAL (both instances on one device, "asynchronous CudaMemcpy"):
 *       one kernel copies the pages straight from `cache` to `dst_cache`; no
 *       communicator (comm may be NULL), no staging (may be NULL / 0).
 *  role PULL (decode side, see ds_ipc_*): as LOCAL, but `cache` describes the
 *       prefill rank's pool mapped into this process; the kernel's loads travel
 *       over NVLink (or stay local when both processes share the GPU).
 * For LOCAL / PULL, `dst_layer_begin` may differ from `layer_begin` (pools of
 * different PP stage extents).
 * Chunking: the (layer, kv, block) page-rows are moved in chunks of about
 * 64 MiB (at least one row of head_count pages) through a 2-slot ring in the
 * staging buffer (2 send + 2 receive slots for SELF); the pack of chunk k+1
 * overlaps the transfer of chunk k, the unpack of chunk k the transfer of k+1.
 * The chunking depends only on (head_dim, layer_count, num_blocks, head_count),
 * so both ends agree. staging_bytes must be >= ds_kv_migrate_staging_bytes().
 * The caller's stream is ordered after the whole migration on return of the
 * stream work; NCCL runs on a library-owned side stream.
 * A peer mismatch of counts is undefined behaviour (NCCL hangs or errors).
 * Errors: DS_ERR_INVALID_ARG, DS_ERR_STATE, DS_ERR_NCCL, DS_ERR_CUDA. */
size_t ds_kv_migrate_staging_bytes(const ds_kv_cache *cache, int32_t role, int32_t layer_count,
                                   int32_t num_blocks, int32_t head_count);
ds_status ds_kv_migrate(ds_comm comm, int32_t role, int32_t peer, const ds_kv_cache *cache,
                        int32_t layer_begin, int32_t layer_count, const int32_t *block_ids,
                        int32_t num_blocks, int32_t head_begin, int32_t head_count,
                        const ds_kv_cache *dst_cache, const int32_t *dst_block_ids,
                        int32_t dst_head_begin, int32_t dst_layer_begin, void *staging,
                        size_t staging_bytes, void *stream);

/* a5 zero-copy: when a batch's pages are the consecutive ids [block_begin,
 * block_begin + num_blocks) in the sender's pool and [dst_block_begin, ...) in
 * the receiver's (fresh pools allocate that way: lowest free id first), and the
 * migrated head range is the whole pool (same num_heads at both ends), each
 * (layer, K|V) run is one contiguous region in both pools, so NCCL moves it pool
 * to pool: no staging, no pack / unpack kernels. role SEND (cache = source) or
 * RECV (cache = destination; block_begin = its first id; dst_* ignored) on the
 * two ranks with identical counts, or SELF on one rank (cache -> dst_cache).
 * Stream-ordered on `stream` (NCCL ops enqueued there). Errors as ds_kv_migrate. */
ds_status ds_kv_migrate_contig(ds_comm comm, int32_t role, int32_t peer, const ds_kv_cache *cache,
                               int32_t layer_begin, int32_t layer_count, int32_t block_begin,
                               int32_t num_blocks, const ds_kv_cache *dst_cache,
                               int32_t dst_block_begin, void *stream);

/* ======================================================================
 * a5, one-sided pull: "decoding instances fetch KV cache
 * from prefill instances as needed, using the GPU memory of prefill instances
 * as a queuing buffer", intra-node by asynchronous copies.
 * The prefill rank exports its pool allocation and an inter-process event; the
 * decode rank maps the pool (NVLink peer memory, or the same GPU) and calls
 * ds_kv_migrate(role DS_MIGRATE_PULL) with `cache` = the mapped prefill pool
 * descriptor: ONE kernel gathers the pages straight into its own pool (no
 * staging, no NCCL). Ordering across processes: the prefill side records its
 * event after the prefill; the decode side waits on it (ds_event_wait) before
 * the pull and records its own event after it, which the prefill side waits on
 * before reusing those pages. The host-side handshake (who recorded what) is
 * the caller's (e.g. torch.distributed messages).
 * Handles are 64 opaque bytes (cudaIpcMemHandle_t / cudaIpcEventHandle_t).
 * ==================================================================== */
enum { DS_MIGRATE_PULL = 4 };
typedef struct {
  unsigned char bytes[64];
} ds_ipc_handle;
/* Export the cudaMalloc allocation that contains `ptr` (e.g. a torch tensor inside
 * the caching allocator's segment): handle of the allocation + byte offset of ptr.
 * The importer maps the allocation (ds_ipc_open_mem returns its base) and adds
 * the offset; the exporting process must keep the memory alive while mapped. */
ds_status ds_ipc_export_mem(const void *ptr, ds_ipc_handle *handle_h, size_t *offset_h);
ds_status ds_ipc_open_mem(const ds_ipc_handle *handle_h, void **base_h);
ds_status ds_ipc_close_mem(void *base);

typedef struct ds_event_s *ds_event;
/* an inter-process event of the current device (timing disabled) and its handle */
ds_status ds_event_create_ipc(ds_event *out_h, ds_ipc_handle *handle_h);
ds_status ds_event_open_ipc(const ds_ipc_handle *handle_h, ds_event *out_h);
ds_status ds_event_record(ds_event ev, void *stream);
/* make `stream` wait for the event's most recent record (as seen by this host) */
ds_status ds_event_wait(ds_event ev, void *stream);
ds_status ds_event_destroy(ds_event ev);

#ifdef __cplusplus
}
#endif
#endif /* DS_H_ */
