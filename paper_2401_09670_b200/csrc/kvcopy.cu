// kvcopy.cu — a4 pack / a6 unpack of whole KV pages for migration.
//
// KV moves only between corresponding layers and TP ranks own
// contiguous head ranges (reading R11), so for every (layer, kv, block)
// the head slice [head_begin, head_begin+head_count) is ONE contiguous run of
// head_count pages (4 KiB each at head_dim 128) in the pool layout
// [L][2][NB][n][16][D]. Pack/unpack is therefore a gather/scatter of
// contiguous rows: staging row r = (layer, kv, i) <-> pool row
// (layer_begin+layer, kv, block_ids[i], head_begin..).
//
// HBM-bound copy: 256-thread CTAs, each thread moves 4 x 16 B per iteration
// (all loads issued before the stores), grid-stride over (row, 16 KiB segment)
// work items; grid = a multiple of the 148 SMs.
#include "common.cuh"
#include "kernels.h"

namespace ds {
namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 4;
constexpr int kSegBytes = kThreads * kUnroll * 16;  // 16 KiB per work item

DS_DEVICE uint4 ld_stream(const uint4 *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <bool kPack>
__global__ void __launch_bounds__(kThreads) kv_copy_kernel(const KvCopyArgs a) {
  const int64_t page_bytes = 16LL * a.head_dim * 2;
  const int64_t row_bytes = page_bytes * a.head_count;
  const int64_t segs_per_row = (row_bytes + kSegBytes - 1) / kSegBytes;
  const int64_t rows = a.row_end - a.row_begin;
  const int64_t items = rows * segs_per_row;
  const int64_t kv_stride = (int64_t)a.pool_blocks * a.n_loc * page_bytes;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t rr = it / segs_per_row, seg = it % segs_per_row;
    const int64_t r = a.row_begin + rr;
    const int64_t i = r % a.num_blocks_sel;
    const int64_t kv = (r / a.num_blocks_sel) & 1;
    const int64_t layer = a.layer_begin + r / (2LL * a.num_blocks_sel);
    const int64_t blk = a.block_ids[i];
    char *pool_row = reinterpret_cast<char *>(a.cache) + (2 * layer + kv) * kv_stride +
                     (blk * a.n_loc + a.head_begin) * page_bytes;
    char *stage_row = reinterpret_cast<char *>(a.staging) + rr * row_bytes;
    const char *src = kPack ? pool_row : stage_row;
    char *dst = kPack ? stage_row : pool_row;
    const int64_t base = seg * kSegBytes;
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t off = base + ((int64_t)u * kThreads + threadIdx.x) * 16;
      if (off < row_bytes) v[u] = ld_stream(reinterpret_cast<const uint4 *>(src + off));
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t off = base + ((int64_t)u * kThreads + threadIdx.x) * 16;
      if (off < row_bytes) *reinterpret_cast<uint4 *>(dst + off) = v[u];
    }
  }
}

// LOCAL / PULL migration: pool row -> pool row directly, no staging buffer and
// no NCCL ("asynchronous CudaMemcpy"). For PULL the source pool is a
// peer GPU's allocation mapped through CUDA IPC, so the loads cross NVLink.
__global__ void __launch_bounds__(kThreads) kv_local_kernel(const KvLocalArgs a) {
  const int64_t page_bytes = 16LL * a.head_dim * 2;
  const int64_t row_bytes = page_bytes * a.head_count;
  const int64_t segs_per_row = (row_bytes + kSegBytes - 1) / kSegBytes;
  const int64_t rows = 2LL * a.layer_count * a.num_blocks_sel;
  const int64_t items = rows * segs_per_row;
  const int64_t src_kv = (int64_t)a.src_blocks * a.src_heads * page_bytes;
  const int64_t dst_kv = (int64_t)a.dst_blocks * a.dst_heads * page_bytes;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t r = it / segs_per_row, seg = it % segs_per_row;
    const int64_t i = r % a.num_blocks_sel;
    const int64_t kv = (r / a.num_blocks_sel) & 1;
    const int64_t l = r / (2LL * a.num_blocks_sel);
    const char *src = reinterpret_cast<const char *>(a.src) + (2 * (a.layer_begin + l) + kv) * src_kv +
                      ((int64_t)a.src_ids[i] * a.src_heads + a.src_head0) * page_bytes;
    char *dst = reinterpret_cast<char *>(a.dst) + (2 * (a.dst_layer_begin + l) + kv) * dst_kv +
                ((int64_t)a.dst_ids[i] * a.dst_heads + a.dst_head0) * page_bytes;
    const int64_t base = seg * kSegBytes;
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t off = base + ((int64_t)u * kThreads + threadIdx.x) * 16;
      if (off < row_bytes) v[u] = ld_stream(reinterpret_cast<const uint4 *>(src + off));
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t off = base + ((int64_t)u * kThreads + threadIdx.x) * 16;
      if (off < row_bytes) *reinterpret_cast<uint4 *>(dst + off) = v[u];
    }
  }
}

// NEXT-3: scatter the chunk's K/V rows to their pages (position prefix + t);
// one thread per 16-B vector of (token, kv, head) rows, coalesced along head_dim.
__global__ void __launch_bounds__(kThreads) kv_append_kernel(const KvAppendArgs a) {
  const int vec_per_row = a.head_dim / 8;
  const int64_t per_token = 2LL * a.n_loc * vec_per_row;
  const int64_t total = (int64_t)a.total_tokens * per_token;
  const int64_t page_elems = 16LL * a.head_dim;
  const int64_t kv_stride = (int64_t)a.num_blocks * a.n_loc * page_elems;
  for (int64_t x = (int64_t)blockIdx.x * kThreads + threadIdx.x; x < total; x += (int64_t)gridDim.x * kThreads) {
    const int t = (int)(x / per_token);
    const int64_t rem = x % per_token;
    const int kv = (int)(rem / (a.n_loc * vec_per_row));
    const int h = (int)(rem / vec_per_row % a.n_loc), vec = (int)(rem % vec_per_row);
    int lo = 0, hi = a.num_seqs - 1;  // sequence r with cu[r] <= t < cu[r+1]
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (a.cu_seqlens[mid] <= t) lo = mid;
      else hi = mid - 1;
    }
    const int pos = a.prefix_lens[lo] + (t - a.cu_seqlens[lo]);
    const int blk = a.block_table[(int64_t)lo * a.max_blocks + (pos >> 4)];
    const uint16_t *src = (kv ? a.v : a.k) + ((int64_t)t * a.n_loc + h) * a.head_dim + vec * 8;
    uint16_t *dst = a.cache + (2LL * a.layer + kv) * kv_stride + ((int64_t)blk * a.n_loc + h) * page_elems +
                    (int64_t)(pos & 15) * a.head_dim + vec * 8;
    *reinterpret_cast<uint4 *>(dst) = *reinterpret_cast<const uint4 *>(src);
  }
}

}  // namespace

cudaError_t launch_kv_append(const KvAppendArgs &a, cudaStream_t stream) {
  const int64_t total = (int64_t)a.total_tokens * 2 * a.n_loc * (a.head_dim / 8);
  if (total <= 0) return cudaSuccess;
  const int64_t blocks = (total + kThreads - 1) / kThreads;
  kv_append_kernel<<<(int)(blocks < 148LL * 16 ? blocks : 148LL * 16), kThreads, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_kv_local(const KvLocalArgs &a, cudaStream_t stream) {
  const int64_t row_bytes = 16LL * a.head_dim * 2 * a.head_count;
  const int64_t items = 2LL * a.layer_count * a.num_blocks_sel * ((row_bytes + kSegBytes - 1) / kSegBytes);
  if (items <= 0) return cudaSuccess;
  const int grid = (int)(items < 148LL * 8 ? items : 148LL * 8);
  kv_local_kernel<<<grid, kThreads, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_kv_copy(const KvCopyArgs &a, bool pack, cudaStream_t stream) {
  const int64_t row_bytes = 16LL * a.head_dim * 2 * a.head_count;
  const int64_t items = (a.row_end - a.row_begin) * ((row_bytes + kSegBytes - 1) / kSegBytes);
  if (items <= 0) return cudaSuccess;
  int grid = (int)(items < 148LL * 8 ? items : 148LL * 8);
  if (pack)
    kv_copy_kernel<true><<<grid, kThreads, 0, stream>>>(a);
  else
    kv_copy_kernel<false><<<grid, kThreads, 0, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace ds
