/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 CPU model of the DistServe KV-cache data
 * path (arXiv 2401.09670). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2401_09670_b200/, libds.so) never includes, links or calls it, and this
 * file includes nothing from there.
 *
 * Citations are PAPER.md lines (P:n) with their section; readings Rn refer to
 * DESIGN.md "Readings of the paper".
 *
 *  - attention (prefill row / decode row): §2.1 (prefill processes the
 *    prompt, decode one token per step reusing the KV cache), App. A
 *    ("attention only operates among the tokens in the same request"),
 *    classic MHA P:454. Written as the plain definition (R1 scale 1/sqrt(s)
 *    passed explicitly, R2 causal j<=i), two-pass softmax in fp64.
 *  - paged pool + block table: PagedAttention P:251; allocation
 *    policy R13 (lowest free id first, argument order, logical order), all-or-
 *    nothing admission R-admit.
 *  - migration: KV moves only between corresponding layers P:363, heads split
 *    by TP P:633 (R11), pull semantics P:382 (bytes identical either way, R10).
 *  - KV bytes: §3.3 ("1.13GB" for OPT-66B, 512 tokens; R7 = GiB).
 *
 * Parity pins (tests/test_oracle_pins.py): every function here is pinned by a
 * brute-force numpy reference, closed forms, invariants or the paper's printed
 * number. Nothing is "parity unpinned".
 *
 * Inputs are bf16 bit patterns (uint16); they are widened exactly to double.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_INVALID 1
#define OR_NO_BLOCKS 3

static double bf16_to_f64(uint16_t b) {
  uint32_t u = ((uint32_t)b) << 16;
  float f;
  memcpy(&f, &u, sizeof f);
  return (double)f;
}

/* ---------------------------------------------------------------------------
 * The definition, one query row:
 *   x_j = scale * sum_d q[d] k_j[d]            (j over the keys given)
 *   m   = max_j x_j ;  p_j = exp(x_j - m) ;  Z = sum_j p_j
 *   o   = sum_j (p_j / Z) v_j
 * keys/values are given as arrays of row pointers (bf16 bits, length d).
 * ------------------------------------------------------------------------- */
static void attend_row(const uint16_t *q, const uint16_t *const *krows,
                       const uint16_t *const *vrows, int nkeys, int d,
                       double scale, double *x /* scratch [nkeys] */,
                       double *out /* [d] */) {
  double m = -INFINITY;
  for (int j = 0; j < nkeys; ++j) {
    double dot = 0.0;
    for (int t = 0; t < d; ++t) dot += bf16_to_f64(q[t]) * bf16_to_f64(krows[j][t]);
    x[j] = scale * dot;
    if (x[j] > m) m = x[j];
  }
  double Z = 0.0;
  for (int j = 0; j < nkeys; ++j) {
    x[j] = exp(x[j] - m);
    Z += x[j];
  }
  for (int t = 0; t < d; ++t) out[t] = 0.0;
  for (int j = 0; j < nkeys; ++j) {
    double w = x[j] / Z;
    for (int t = 0; t < d; ++t) out[t] += w * bf16_to_f64(vrows[j][t]);
  }
}

/* ---------------------------------------------------------------------------
 * Threading helper: plain pthreads over independent work items.
 * ------------------------------------------------------------------------- */
typedef void (*item_fn)(void *ctx, long item);
typedef struct {
  item_fn fn;
  void *ctx;
  long n_items;
  int nthreads;
  int tid;
} worker_arg;

static void *worker_main(void *p) {
  worker_arg *a = (worker_arg *)p;
  for (long i = a->tid; i < a->n_items; i += a->nthreads) a->fn(a->ctx, i);
  return NULL;
}

static void parallel_for(item_fn fn, void *ctx, long n_items, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if (nthreads == 1 || n_items <= 1) {
    for (long i = 0; i < n_items; ++i) fn(ctx, i);
    return;
  }
  pthread_t th[256];
  worker_arg args[256];
  for (int t = 0; t < nthreads; ++t) {
    args[t] = (worker_arg){fn, ctx, n_items, nthreads, t};
    pthread_create(&th[t], NULL, worker_main, &args[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* ---------------------------------------------------------------------------
 * a2: prefill causal attention over a packed varlen batch.
 *   q,k,v: [T][n][d] bf16 bits; cu_seqlens [B+1]; out [T][n][d] fp64.
 * Row i of sequence r attends keys j <= i of the same sequence (R2).
 * `rows_begin/rows_count` optionally restrict the rows computed (per sequence,
 * relative to its start; rows_count < 0 means all) for sampled parity checks.
 * ------------------------------------------------------------------------- */
typedef struct {
  const uint16_t *q, *k, *v;
  const int32_t *cu;
  int n, d;
  double scale;
  double *out;
  int32_t num_seqs;
} prefill_ctx;

static void prefill_item(void *pctx, long item) {
  prefill_ctx *c = (prefill_ctx *)pctx;
  long r = item / c->n;
  int h = (int)(item % c->n);
  int32_t start = c->cu[r], len = c->cu[r + 1] - c->cu[r];
  if (len <= 0) return;
  const uint16_t **kr = malloc(sizeof(*kr) * len);
  const uint16_t **vr = malloc(sizeof(*vr) * len);
  double *x = malloc(sizeof(double) * len);
  long rs = (long)c->n * c->d;
  for (int j = 0; j < len; ++j) {
    kr[j] = c->k + (long)(start + j) * rs + (long)h * c->d;
    vr[j] = c->v + (long)(start + j) * rs + (long)h * c->d;
  }
  for (int i = 0; i < len; ++i) {
    const uint16_t *qi = c->q + (long)(start + i) * rs + (long)h * c->d;
    attend_row(qi, kr, vr, i + 1, c->d, c->scale, x,
               c->out + (long)(start + i) * rs + (long)h * c->d);
  }
  free(kr);
  free(vr);
  free(x);
}

int oracle_prefill(const uint16_t *q, const uint16_t *k, const uint16_t *v,
                   const int32_t *cu_seqlens, int32_t num_seqs, int32_t n_heads,
                   int32_t head_dim, double scale, double *out, int32_t nthreads) {
  if (num_seqs < 0 || n_heads <= 0 || head_dim <= 0) return OR_INVALID;
  prefill_ctx c = {q, k, v, cu_seqlens, n_heads, head_dim, scale, out, num_seqs};
  parallel_for(prefill_item, &c, (long)num_seqs * n_heads, nthreads);
  return OR_OK;
}

/* One row i (0-based within sequence r) for one head: sampled checks at full size. */
int oracle_prefill_row(const uint16_t *q, const uint16_t *k, const uint16_t *v,
                       const int32_t *cu_seqlens, int32_t r, int32_t i, int32_t h,
                       int32_t n_heads, int32_t head_dim, double scale, double *out) {
  int32_t start = cu_seqlens[r], len = cu_seqlens[r + 1] - cu_seqlens[r];
  if (i < 0 || i >= len || h < 0 || h >= n_heads) return OR_INVALID;
  long rs = (long)n_heads * head_dim;
  const uint16_t **kr = malloc(sizeof(*kr) * (i + 1));
  const uint16_t **vr = malloc(sizeof(*vr) * (i + 1));
  double *x = malloc(sizeof(double) * (i + 1));
  for (int j = 0; j <= i; ++j) {
    kr[j] = k + (long)(start + j) * rs + (long)h * head_dim;
    vr[j] = v + (long)(start + j) * rs + (long)h * head_dim;
  }
  attend_row(q + (long)(start + i) * rs + (long)h * head_dim, kr, vr, i + 1, head_dim,
             scale, x, out);
  free(kr);
  free(vr);
  free(x);
  return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Paged pool model (D2).
 * Pages are stored [block][head][layer][kv][slot][d] — deliberately NOT the GPU
 * library's layout; tests map between the two through explicit indexing.
 * Free set: byte-per-block flags; allocation takes the lowest free id (R13).
 * ------------------------------------------------------------------------- */
typedef struct {
  int32_t layers, num_blocks, heads, block_size, head_dim;
  uint16_t *pages;
  uint8_t *is_free;
  int32_t num_free;
} oracle_pool;

oracle_pool *oracle_pool_create(int32_t layers, int32_t num_blocks, int32_t heads,
                                int32_t block_size, int32_t head_dim) {
  if (layers <= 0 || num_blocks <= 0 || heads <= 0 || block_size <= 0 || head_dim <= 0)
    return NULL;
  oracle_pool *p = calloc(1, sizeof *p);
  p->layers = layers;
  p->num_blocks = num_blocks;
  p->heads = heads;
  p->block_size = block_size;
  p->head_dim = head_dim;
  size_t n = (size_t)num_blocks * heads * layers * 2 * block_size * head_dim;
  p->pages = calloc(n, sizeof(uint16_t));
  p->is_free = malloc((size_t)num_blocks);
  memset(p->is_free, 1, (size_t)num_blocks);
  p->num_free = num_blocks;
  if (!p->pages || !p->is_free) return NULL;
  return p;
}

void oracle_pool_destroy(oracle_pool *p) {
  if (!p) return;
  free(p->pages);
  free(p->is_free);
  free(p);
}

int32_t oracle_pool_num_free(const oracle_pool *p) { return p->num_free; }

/* page (layer, kv, block, head) -> pointer to [block_size][head_dim] bits */
uint16_t *oracle_pool_page(oracle_pool *p, int32_t layer, int32_t kv, int32_t block,
                           int32_t head) {
  size_t idx = ((((size_t)block * p->heads + head) * p->layers + layer) * 2 + kv);
  return p->pages + idx * p->block_size * p->head_dim;
}

static int32_t blocks_for(int64_t tokens, int32_t bs) {
  return (int32_t)((tokens + bs - 1) / bs);
}

/* a1 — APPEND (ALLOC is APPEND from cur_len 0): grow seq s from c to c+k tokens;
 * a new page is taken exactly when ceil((c+k)/bs) > ceil(c/bs). All-or-nothing:
 * if the pool cannot satisfy the whole call nothing changes. table is
 * [num_seqs][max_blocks], -1 padded; entries below ceil(c/bs) must already be set. */
int oracle_bt_append(oracle_pool *p, int32_t num_seqs, const int32_t *cur_lens,
                     const int32_t *add_lens, int32_t *table, int32_t max_blocks,
                     int32_t block_size) {
  if (num_seqs < 0 || block_size != p->block_size) return OR_INVALID;
  int64_t need = 0;
  for (int s = 0; s < num_seqs; ++s) {
    if (cur_lens[s] < 0 || add_lens[s] < 0) return OR_INVALID;
    int32_t nb_old = blocks_for(cur_lens[s], block_size);
    int32_t nb_new = blocks_for((int64_t)cur_lens[s] + add_lens[s], block_size);
    if (nb_new > max_blocks) return OR_INVALID;
    need += nb_new - nb_old;
  }
  if (need > p->num_free) return OR_NO_BLOCKS;
  for (int s = 0; s < num_seqs; ++s) {
    int32_t nb_old = blocks_for(cur_lens[s], block_size);
    int32_t nb_new = blocks_for((int64_t)cur_lens[s] + add_lens[s], block_size);
    for (int32_t b = nb_old; b < nb_new; ++b) {
      int32_t id = 0;
      while (!p->is_free[id]) ++id; /* lowest free id (R13) */
      p->is_free[id] = 0;
      p->num_free--;
      table[(size_t)s * max_blocks + b] = id;
    }
  }
  return OR_OK;
}

/* a1 — FREE: return the ceil(cur_len/bs) pages of each row and reset it to -1. */
int oracle_bt_free(oracle_pool *p, int32_t num_seqs, const int32_t *cur_lens,
                   int32_t *table, int32_t max_blocks, int32_t block_size) {
  if (num_seqs < 0 || block_size != p->block_size) return OR_INVALID;
  for (int s = 0; s < num_seqs; ++s) {
    int32_t nb = blocks_for(cur_lens[s], block_size);
    if (cur_lens[s] < 0 || nb > max_blocks) return OR_INVALID;
    for (int32_t b = 0; b < nb; ++b) {
      int32_t id = table[(size_t)s * max_blocks + b];
      if (id < 0 || id >= p->num_blocks || p->is_free[id]) return OR_INVALID;
    }
  }
  for (int s = 0; s < num_seqs; ++s) {
    int32_t nb = blocks_for(cur_lens[s], block_size);
    for (int32_t b = 0; b < nb; ++b) {
      int32_t *e = &table[(size_t)s * max_blocks + b];
      p->is_free[*e] = 1;
      p->num_free++;
      *e = -1;
    }
  }
  return OR_OK;
}

/* a3 — write the prompt K/V of a packed batch into the pages of `layer`:
 *   page(layer, K, bt[r][t/bs], h)[t % bs] = k[start_r + t][h]   (same for V). */
int oracle_pool_write_prefill(oracle_pool *p, int32_t layer, const uint16_t *k,
                              const uint16_t *v, const int32_t *cu_seqlens,
                              int32_t num_seqs, const int32_t *table, int32_t max_blocks) {
  int bs = p->block_size, d = p->head_dim, n = p->heads;
  for (int r = 0; r < num_seqs; ++r) {
    int32_t start = cu_seqlens[r], len = cu_seqlens[r + 1] - cu_seqlens[r];
    for (int t = 0; t < len; ++t) {
      int32_t blk = table[(size_t)r * max_blocks + t / bs];
      if (blk < 0 || blk >= p->num_blocks) return OR_INVALID;
      for (int h = 0; h < n; ++h) {
        memcpy(oracle_pool_page(p, layer, 0, blk, h) + (size_t)(t % bs) * d,
               k + ((size_t)(start + t) * n + h) * d, sizeof(uint16_t) * d);
        memcpy(oracle_pool_page(p, layer, 1, blk, h) + (size_t)(t % bs) * d,
               v + ((size_t)(start + t) * n + h) * d, sizeof(uint16_t) * d);
      }
    }
  }
  return OR_OK;
}

/* ---------------------------------------------------------------------------
 * a7: one decode step for `layer` ("generates subsequent tokens one at a
 * time"; R9: the new token's K/V are appended at position c BEFORE attending,
 * so decode(c) equals row c of prefill over c+1 tokens).
 *   q,k_new,v_new: [B][n][d] bits; cache_lens[b] = c_b; out [B][n][d] fp64.
 * The caller has already grown the block table (APPEND by 1) so that block
 * bt[b][c_b / bs] exists.
 * ------------------------------------------------------------------------- */
typedef struct {
  oracle_pool *p;
  int32_t layer;
  const uint16_t *q;
  const int32_t *table, *cache_lens;
  int32_t max_blocks;
  double scale;
  double *out;
} decode_ctx;

static void decode_item(void *pctx, long item) {
  decode_ctx *c = (decode_ctx *)pctx;
  oracle_pool *p = c->p;
  int n = p->heads, d = p->head_dim, bs = p->block_size;
  long b = item / n;
  int h = (int)(item % n);
  int32_t ctx = c->cache_lens[b] + 1;
  const uint16_t **kr = malloc(sizeof(*kr) * ctx);
  const uint16_t **vr = malloc(sizeof(*vr) * ctx);
  double *x = malloc(sizeof(double) * ctx);
  for (int j = 0; j < ctx; ++j) {
    int32_t blk = c->table[(size_t)b * c->max_blocks + j / bs];
    kr[j] = oracle_pool_page(p, c->layer, 0, blk, h) + (size_t)(j % bs) * d;
    vr[j] = oracle_pool_page(p, c->layer, 1, blk, h) + (size_t)(j % bs) * d;
  }
  attend_row(c->q + ((size_t)b * n + h) * d, kr, vr, ctx, d, c->scale, x,
             c->out + ((size_t)b * n + h) * d);
  free(kr);
  free(vr);
  free(x);
}

int oracle_decode(oracle_pool *p, int32_t layer, const uint16_t *q, const uint16_t *k_new,
                  const uint16_t *v_new, const int32_t *table, int32_t max_blocks,
                  const int32_t *cache_lens, int32_t num_seqs, double scale, double *out,
                  int32_t nthreads) {
  int n = p->heads, d = p->head_dim, bs = p->block_size;
  if (num_seqs < 0 || layer < 0 || layer >= p->layers) return OR_INVALID;
  for (int b = 0; b < num_seqs; ++b) {
    int32_t c = cache_lens[b];
    if (c < 0 || c / bs >= max_blocks) return OR_INVALID;
    int32_t blk = table[(size_t)b * max_blocks + c / bs];
    if (blk < 0 || blk >= p->num_blocks) return OR_INVALID;
    for (int h = 0; h < n; ++h) { /* (i) append at position c */
      memcpy(oracle_pool_page(p, layer, 0, blk, h) + (size_t)(c % bs) * d,
             k_new + ((size_t)b * n + h) * d, sizeof(uint16_t) * d);
      memcpy(oracle_pool_page(p, layer, 1, blk, h) + (size_t)(c % bs) * d,
             v_new + ((size_t)b * n + h) * d, sizeof(uint16_t) * d);
    }
  }
  decode_ctx c = {p, layer, q, table, cache_lens, max_blocks, scale, out};
  parallel_for(decode_item, &c, (long)num_seqs * n, nthreads); /* (ii) attend c+1 */
  return OR_OK;
}

/* ---------------------------------------------------------------------------
 * NEXT-3 chunked prefill ("segmenting long prefill into chunks", P:142:
 * chunk k re-reads the KV of all earlier chunks): sequence r already holds
 * prefix_lens[r] = c tokens in the pool; its next chunk of l tokens (q,k,v
 * packed by cu_seqlens) is appended at positions c..c+l-1 and row i (global
 * position c+i) attends keys 0..c+i. The plain definition, with the keys
 * gathered through the block table.
 * ------------------------------------------------------------------------- */
typedef struct {
  oracle_pool *p;
  int32_t layer;
  const uint16_t *q;
  const int32_t *cu, *prefix, *table;
  int32_t max_blocks;
  double scale;
  double *out;
} chunk_ctx;

static void chunk_item(void *pctx, long item) {
  chunk_ctx *c = (chunk_ctx *)pctx;
  oracle_pool *p = c->p;
  int n = p->heads, d = p->head_dim, bs = p->block_size;
  long r = item / n;
  int h = (int)(item % n);
  int32_t start = c->cu[r], len = c->cu[r + 1] - c->cu[r], c0 = c->prefix[r];
  int32_t total = c0 + len;
  const uint16_t **kr = malloc(sizeof(*kr) * (total > 0 ? total : 1));
  const uint16_t **vr = malloc(sizeof(*vr) * (total > 0 ? total : 1));
  double *x = malloc(sizeof(double) * (total > 0 ? total : 1));
  for (int j = 0; j < total; ++j) {
    int32_t blk = c->table[(size_t)r * c->max_blocks + j / bs];
    kr[j] = oracle_pool_page(p, c->layer, 0, blk, h) + (size_t)(j % bs) * d;
    vr[j] = oracle_pool_page(p, c->layer, 1, blk, h) + (size_t)(j % bs) * d;
  }
  for (int i = 0; i < len; ++i)
    attend_row(c->q + ((size_t)(start + i) * n + h) * d, kr, vr, c0 + i + 1, d, c->scale, x,
               c->out + ((size_t)(start + i) * n + h) * d);
  free(kr);
  free(vr);
  free(x);
}

int oracle_chunked_prefill(oracle_pool *p, int32_t layer, const uint16_t *q, const uint16_t *k,
                           const uint16_t *v, const int32_t *cu_seqlens, const int32_t *prefix_lens,
                           int32_t num_seqs, const int32_t *table, int32_t max_blocks, double scale,
                           double *out, int32_t nthreads) {
  int n = p->heads, d = p->head_dim, bs = p->block_size;
  if (num_seqs < 0 || layer < 0 || layer >= p->layers) return OR_INVALID;
  for (int r = 0; r < num_seqs; ++r) { /* append the chunk's K/V at positions c..c+l-1 */
    int32_t start = cu_seqlens[r], len = cu_seqlens[r + 1] - cu_seqlens[r], c0 = prefix_lens[r];
    if (c0 < 0 || len < 0 || (c0 + len + bs - 1) / bs > max_blocks) return OR_INVALID;
    for (int t = 0; t < len; ++t) {
      int32_t pos = c0 + t, blk = table[(size_t)r * max_blocks + pos / bs];
      if (blk < 0 || blk >= p->num_blocks) return OR_INVALID;
      for (int h = 0; h < n; ++h) {
        memcpy(oracle_pool_page(p, layer, 0, blk, h) + (size_t)(pos % bs) * d,
               k + ((size_t)(start + t) * n + h) * d, sizeof(uint16_t) * d);
        memcpy(oracle_pool_page(p, layer, 1, blk, h) + (size_t)(pos % bs) * d,
               v + ((size_t)(start + t) * n + h) * d, sizeof(uint16_t) * d);
      }
    }
  }
  chunk_ctx c = {p, layer, q, cu_seqlens, prefix_lens, table, max_blocks, scale, out};
  parallel_for(chunk_item, &c, (long)num_seqs * n, nthreads);
  return OR_OK;
}

/* ---------------------------------------------------------------------------
 * a4+a5+a6: migrate whole pages of `num_blocks` logical blocks, layers
 * [layer_begin, layer_begin+layer_count), heads [src_head0, src_head0+head_count)
 * of the source pool into heads [dst_head0, ...) of the destination pool, block
 * src_blocks[i] -> dst_blocks[i] (KV moves only between corresponding layers,
 * P:363; head slices per TP rank). Returns bytes moved (>= 0) or -1.
 * ------------------------------------------------------------------------- */
int64_t oracle_migrate(oracle_pool *src, oracle_pool *dst, int32_t layer_begin,
                       int32_t layer_count, const int32_t *src_blocks,
                       const int32_t *dst_blocks, int32_t num_blocks, int32_t src_head0,
                       int32_t dst_head0, int32_t head_count) {
  if (src->block_size != dst->block_size || src->head_dim != dst->head_dim) return -1;
  if (layer_begin < 0 || layer_begin + layer_count > src->layers ||
      layer_begin + layer_count > dst->layers)
    return -1;
  if (src_head0 < 0 || src_head0 + head_count > src->heads || dst_head0 < 0 ||
      dst_head0 + head_count > dst->heads)
    return -1;
  size_t page_elems = (size_t)src->block_size * src->head_dim;
  int64_t bytes = 0;
  for (int i = 0; i < num_blocks; ++i)
    for (int l = layer_begin; l < layer_begin + layer_count; ++l)
      for (int kv = 0; kv < 2; ++kv)
        for (int h = 0; h < head_count; ++h) {
          memcpy(oracle_pool_page(dst, l, kv, dst_blocks[i], dst_head0 + h),
                 oracle_pool_page(src, l, kv, src_blocks[i], src_head0 + h),
                 page_elems * sizeof(uint16_t));
          bytes += (int64_t)(page_elems * sizeof(uint16_t));
        }
  return bytes;
}

/* KV-cache bytes of `tokens` tokens over `layers` layers, heads x head_dim, at
 * `elem_bytes` per element: K and V per layer per token per head (
 * SPEC kv_cache_bytes). OPT-66B, 512 tokens, 2 B -> 1,207,959,552 ("1.13GB"). */
int64_t oracle_kv_bytes(int32_t layers, int64_t tokens, int32_t heads, int32_t head_dim,
                        int32_t elem_bytes) {
  return 2LL * layers * tokens * heads * head_dim * elem_bytes;
}
