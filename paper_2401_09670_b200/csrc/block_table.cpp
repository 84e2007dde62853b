// block_table.cpp — a1: page allocation and block tables (host, synchronous).
//
// PagedAttention-style fixed-size KV pages with a per-request logical->physical
// block map. The paper gives no allocation
// policy; ours (reading R13) makes tables bit-comparable with the
// oracle: lowest free id first, sequences in argument order, logical blocks in
// order. Admission is all-or-nothing (SPEC S:270 CapacityError).
//
// The free set is a two-level bitmap (64-bit words + a summary of non-empty
// words) so "lowest free id" is O(num_blocks/4096) worst case and O(1) typical.
#include <stdint.h>

#include <mutex>
#include <new>
#include <vector>

#include "../../include/ds.h"
#include "internal.h"

struct ds_pool_s {
  int32_t num_blocks = 0;
  int32_t num_free = 0;
  std::vector<uint64_t> words;    // bit set = free
  std::vector<uint64_t> summary;  // bit w set = words[w] != 0
  std::mutex mu;

  void set_free(int32_t id) {
    const int32_t w = id >> 6;
    words[w] |= 1ull << (id & 63);
    summary[w >> 6] |= 1ull << (w & 63);
  }
  int32_t take_lowest() {  // precondition: num_free > 0
    for (size_t s = 0; s < summary.size(); ++s) {
      if (!summary[s]) continue;
      const int32_t w = (int32_t)(s * 64 + __builtin_ctzll(summary[s]));
      const int32_t bit = __builtin_ctzll(words[w]);
      words[w] &= words[w] - 1;
      if (!words[w]) summary[w >> 6] &= ~(1ull << (w & 63));
      return w * 64 + bit;
    }
    return -1;
  }
  bool is_free(int32_t id) const { return (words[id >> 6] >> (id & 63)) & 1ull; }
  void clear_free(int32_t id) {  // undo set_free (rollback of a rejected call)
    const int32_t w = id >> 6;
    words[w] &= ~(1ull << (id & 63));
    if (!words[w]) summary[w >> 6] &= ~(1ull << (w & 63));
  }
};

static int32_t blocks_for(int64_t tokens, int32_t bs) { return (int32_t)((tokens + bs - 1) / bs); }

extern "C" ds_status ds_pool_create(int32_t num_blocks, ds_pool *out_h) {
  if (!out_h || num_blocks <= 0) return ds::fail(DS_ERR_INVALID_ARG, "ds_pool_create: num_blocks must be > 0");
  ds_pool p = new (std::nothrow) ds_pool_s();
  if (!p) return ds::fail(DS_ERR_INVALID_ARG, "ds_pool_create: out of host memory");
  p->num_blocks = num_blocks;
  const int32_t nw = (num_blocks + 63) / 64;
  p->words.assign(nw, 0);
  p->summary.assign((nw + 63) / 64, 0);
  for (int32_t id = 0; id < num_blocks; ++id) p->set_free(id);
  p->num_free = num_blocks;
  *out_h = p;
  return DS_OK;
}

extern "C" ds_status ds_pool_destroy(ds_pool pool) {
  if (!pool) return ds::fail(DS_ERR_STATE, "ds_pool_destroy: null pool");
  delete pool;
  return DS_OK;
}

extern "C" ds_status ds_pool_num_free(ds_pool pool, int32_t *num_free_h) {
  if (!pool || !num_free_h) return ds::fail(DS_ERR_INVALID_ARG, "ds_pool_num_free: null argument");
  std::lock_guard<std::mutex> g(pool->mu);
  *num_free_h = pool->num_free;
  return DS_OK;
}

extern "C" ds_status ds_block_table(ds_pool pool, int32_t op, int32_t num_seqs,
                                    const int32_t *cur_lens_h, const int32_t *add_lens_h,
                                    int32_t *table_h, int32_t max_blocks_per_seq,
                                    int32_t block_size, int32_t *num_free_h) {
  if (!pool) return ds::fail(DS_ERR_STATE, "ds_block_table: null pool");
  if (block_size != 16) return ds::fail(DS_ERR_INVALID_ARG, "ds_block_table: block_size must be 16");
  if (num_seqs < 0 || max_blocks_per_seq < 0)
    return ds::fail(DS_ERR_INVALID_ARG, "ds_block_table: negative num_seqs/max_blocks_per_seq");
  if (op != DS_BT_APPEND && op != DS_BT_FREE) return ds::fail(DS_ERR_INVALID_ARG, "ds_block_table: bad op");
  std::lock_guard<std::mutex> g(pool->mu);
  if (num_seqs > 0 && (!cur_lens_h || !table_h || (op == DS_BT_APPEND && !add_lens_h)))
    return ds::fail(DS_ERR_INVALID_ARG, "ds_block_table: null array");
  if (op == DS_BT_APPEND) {
    int64_t need = 0;
    for (int32_t s = 0; s < num_seqs; ++s) {
      if (cur_lens_h[s] < 0 || add_lens_h[s] < 0)
        return ds::fail(DS_ERR_INVALID_ARG, "ds_block_table: negative length");
      const int32_t nb_old = blocks_for(cur_lens_h[s], block_size);
      const int32_t nb_new = blocks_for((int64_t)cur_lens_h[s] + add_lens_h[s], block_size);
      if (nb_new > max_blocks_per_seq)
        return ds::fail(DS_ERR_INVALID_ARG, "ds_block_table: sequence needs more than max_blocks_per_seq pages");
      need += nb_new - nb_old;
    }
    if (need > pool->num_free) return ds::fail(DS_ERR_NO_BLOCKS, "ds_block_table: pool exhausted (nothing allocated)");
    std::vector<int64_t> slots;  // table entries written so far (rollback if the free set is inconsistent)
    slots.reserve((size_t)need);
    for (int32_t s = 0; s < num_seqs; ++s) {
      const int32_t nb_old = blocks_for(cur_lens_h[s], block_size);
      const int32_t nb_new = blocks_for((int64_t)cur_lens_h[s] + add_lens_h[s], block_size);
      for (int32_t b = nb_old; b < nb_new; ++b) {
        const int32_t id = pool->take_lowest();
        if (id < 0) {  // cannot happen while num_free is exact; never write -1 into a table
          for (int64_t e : slots) {
            pool->set_free(table_h[e]);
            table_h[e] = -1;
          }
          pool->num_free += (int32_t)slots.size();
          return ds::fail(DS_ERR_STATE, "ds_block_table: free set inconsistent with num_free (nothing allocated)");
        }
        const int64_t e = (int64_t)s * max_blocks_per_seq + b;
        table_h[e] = id;
        slots.push_back(e);
        pool->num_free--;
      }
    }
  } else {
    // validate by freeing tentatively: an id that is out of range, not allocated,
    // or listed twice in this call (already freed a moment ago) rolls the call back
    std::vector<int32_t> freed;
    for (int32_t s = 0; s < num_seqs; ++s) {
      const int32_t nb = blocks_for(cur_lens_h[s], block_size);
      bool bad = cur_lens_h[s] < 0 || nb > max_blocks_per_seq;
      for (int32_t b = 0; !bad && b < nb; ++b) {
        const int32_t id = table_h[(int64_t)s * max_blocks_per_seq + b];
        if (id < 0 || id >= pool->num_blocks || pool->is_free(id)) {
          bad = true;
          break;
        }
        pool->set_free(id);
        freed.push_back(id);
      }
      if (bad) {
        for (int32_t id : freed) pool->clear_free(id);
        return ds::fail(DS_ERR_INVALID_ARG,
                        "ds_block_table: bad length in FREE, or FREE of a page that is not allocated "
                        "(or listed twice); nothing freed");
      }
    }
    pool->num_free += (int32_t)freed.size();
    for (int32_t s = 0; s < num_seqs; ++s) {
      const int32_t nb = blocks_for(cur_lens_h[s], block_size);
      for (int32_t b = 0; b < nb; ++b) table_h[(int64_t)s * max_blocks_per_seq + b] = -1;
    }
  }
  if (num_free_h) *num_free_h = pool->num_free;
  return DS_OK;
}
