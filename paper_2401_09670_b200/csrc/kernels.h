// kernels.h — internal launch interface between the C ABI (api.cu) and the
// sm_100a kernels. Not part of the public boundary (include/ds.h is).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace ds {

// a7 + a8
constexpr int kDecodeMaxSeqs = 4096;  // sequences per decode launch (smem page prefix)
constexpr int kDecodeMaxSMs = 160;    // workspace is sized for grids up to this many CTAs
// merge tickets: a fixed region of this many (seq, head) pairs at a fixed offset of
// every decode workspace, so a call with another batch shape or head_dim finds the
// tickets of every pair it can touch at zero (they are reset by their merger)
constexpr int kDecodeMaxPairs = 1 << 19;  // 2 MiB: 4096 sequences x 128 heads
struct DecodeArgs {
  const uint16_t *q, *k_new, *v_new;  // bf16 [B][n][D]
  void *out;                          // bf16 [B][n][D]
  const uint16_t *cache;              // pool base [L][2][NB][n][16][D]
  const int32_t *block_table;         // [B][max_blocks]
  const int32_t *cache_lens;          // [B]
  float *workspace;                   // [warps][2][D+4] straddling-pair partials (o, m, l, pad)
  int32_t *tickets;                   // [kDecodeMaxPairs] merge tickets, pair b*n+h (zero between launches)
  float *chunk_rows;                  // [chunks][2][D+4] partials of the dynamically taken chunks
  int32_t *dyn;                       // [4]: chunk counter, finished CTAs (decode_kernel); pair counter,
                                      // finished CTAs (decode_pairs_kernel) — zero between launches
  int64_t max_chunks;                 // capacity of chunk_rows
  int32_t max_cache_len;              // bound of cache_lens (host-side kernel choice)
  int32_t early_kv;                   // read lengths / table / pages before the PDL wait
  int32_t layer, num_blocks, n_loc, max_blocks, num_seqs;
  float scale_log2;  // softmax_scale * log2(e)
};
struct DecodeLayout {
  size_t dyn_off, rows_off, tickets_off, chunk_off, total;
  int64_t max_chunks;  // dynamic chunks the chunk rows hold
};
DecodeLayout decode_layout(int num_seqs, int n_loc, int head_dim, int num_sms, int max_cache_len);
cudaError_t launch_decode(const DecodeArgs &a, int head_dim, int num_sms, cudaStream_t stream);
bool decode_uses_pairs(int num_seqs, int n_loc, int num_sms);  // decode_pairs_kernel vs decode_kernel

// a4 / a6: page rows <-> staging
struct KvCopyArgs {
  uint16_t *cache;          // pool base
  uint16_t *staging;        // [rows][head_count][16][D]
  const int32_t *block_ids; // [num_blocks]
  int32_t layer_begin, num_blocks_sel, head_begin, head_count;
  int32_t pool_blocks, n_loc, head_dim;
  int64_t row_begin, row_end;  // rows of (layer, kv, i) to copy, staging row r at r - row_begin
};
cudaError_t launch_kv_copy(const KvCopyArgs &a, bool pack, cudaStream_t stream);

// a4+a5+a6 on one device (LOCAL): pool pages -> pool pages
struct KvLocalArgs {
  const uint16_t *src;
  uint16_t *dst;
  const int32_t *src_ids, *dst_ids;  // [num_blocks_sel]
  int32_t layer_begin, dst_layer_begin, layer_count, num_blocks_sel, head_count, head_dim;
  int32_t src_blocks, src_heads, src_head0, dst_blocks, dst_heads, dst_head0;
};
cudaError_t launch_kv_local(const KvLocalArgs &a, cudaStream_t stream);

// a2 + a3
constexpr int kPrefillQRows = 128;  // q rows per CTA (TMA box of Q)
constexpr int kPrefillKVRows = 64;  // keys per kv tile (TMA box of K and V)
struct PrefillArgs {
  void *out;                   // bf16 [T][n][D]
  const int32_t *cu_seqlens;   // [B+1]
  const int32_t *prefix_lens;  // [B] cached tokens before the chunk (chunked prefill) or nullptr
  const int32_t *block_table;  // [B][max_blocks]
  int32_t num_seqs, n_loc, max_blocks, num_q_tiles;
  int32_t compact;             // item space = existing q tiles only (num_seqs <= kPrefillCompactSeqs)
  int64_t grid_items;          // launched items (CTAs before work stealing)
  int32_t layer, num_blocks;   // cache layer / pool pages
  float scale_log2;
  int32_t persistent;          // CTAs take over unlaunched CTAs' items (cluster launch control)
  // fused push migration (ds_prefill_attn_push): every page also goes to the
  // destination pool (tm_dst) at dst_layer / dst_block_table / dst_head0
  const int32_t *dst_block_table;  // [B][dst_max_blocks] or nullptr (no push)
  int32_t dst_max_blocks, dst_layer, dst_num_blocks, dst_head0;
  int32_t write_local;             // also write the source pool (tm_cache)
};
cudaError_t launch_prefill(const PrefillArgs &a, const CUtensorMap &tm_q, const CUtensorMap &tm_k,
                           const CUtensorMap &tm_v, const CUtensorMap &tm_cache, const CUtensorMap &tm_o,
                           const CUtensorMap *tm_dst, int head_dim, cudaStream_t stream);
size_t prefill_smem_bytes(int head_dim);
constexpr int kPrefillCompactSeqs = 1024;  // sequences whose tile prefix fits the prefill CTA's smem
// items to launch: compact = n_loc x an upper bound of sum ceil(len/128) from the
// host-side token total; else num_q_tiles x n_loc x num_seqs
void prefill_set_grid(PrefillArgs &a, int64_t total_tokens);
bool prefill_persistent(int max_len);  // run the prefill CTAs persistently for this length?
// experimental (DS_PREFILL_KERNEL=2q): two 128-row q tiles per CTA, 128-key tiles
cudaError_t launch_prefill2q(const PrefillArgs &a, const CUtensorMap &tm_q, const CUtensorMap &tm_k,
                             const CUtensorMap &tm_v, const CUtensorMap &tm_cache, const CUtensorMap &tm_o,
                             int head_dim, cudaStream_t stream);

// NEXT-3: append the chunk's K/V at positions prefix_lens[r] + t of each sequence
struct KvAppendArgs {
  const uint16_t *k, *v;       // [T][n][D]
  uint16_t *cache;             // pool base
  const int32_t *cu_seqlens, *prefix_lens, *block_table;
  int32_t num_seqs, n_loc, head_dim, max_blocks, layer, num_blocks, total_tokens;
};
cudaError_t launch_kv_append(const KvAppendArgs &a, cudaStream_t stream);

}  // namespace ds
