// migrate.cu — a5: KV migration prefill rank -> decode rank with NCCL p2p.
//
// PAPER.md P:407 (NCCL across nodes, asynchronous cudaMemcpy within a node —
// "avoids blocking the GPU computation during transmission"), P:265 (1.13 GB per
// OPT-66B 512-token request), P:382 (decode instances *pull* KV when they have
// memory; the prefill GPU's memory is the queue buffer), P:363 (only between
// corresponding layers), P:633 (TP head shards).
//
// On B200 every GPU of the node reaches every peer at full NVLink-5 bandwidth
// through NVSwitch, so one two-sided ncclSend/ncclRecv per chunk is the whole
// protocol. Pages are gathered (a4) into a chunk ring in the staging buffer on
// the caller's stream while NCCL moves the previous chunk on a library-owned
// side stream; the receiver scatters (a6) chunk k while chunk k+1 is in flight.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdio.h>
#include <string.h>

#include <new>

#include "../../include/ds.h"
#include "internal.h"
#include "kernels.h"

namespace ds {
ds_status kv_copy_checked(const ds_kv_cache *cache, int32_t layer_begin, int32_t layer_count,
                          const int32_t *block_ids, int32_t num_blocks, int32_t head_begin,
                          int32_t head_count, void *staging, size_t staging_bytes,
                          int64_t row_begin, int64_t row_end, bool pack, cudaStream_t stream,
                          const char *W, bool dry_run = false);
}  // namespace ds

using namespace ds;

struct ds_comm_s {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 0, device = -1;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_start = nullptr;
  cudaEvent_t ev_a[2] = {nullptr, nullptr};  // recorded on the caller's stream
  cudaEvent_t ev_b[2] = {nullptr, nullptr};  // recorded on the side (NCCL) stream
};

namespace {
constexpr int64_t kChunkTarget = 64ll << 20;  // bytes per transfer chunk

#define DS_CUDA(call, W)                                        \
  do {                                                          \
    cudaError_t e_ = (call);                                    \
    if (e_ != cudaSuccess)                                      \
      return fail(DS_ERR_CUDA, "%s: %s", W, cudaGetErrorString(e_)); \
  } while (0)
#define DS_NCCL(call, W)                                        \
  do {                                                          \
    ncclResult_t r_ = (call);                                   \
    if (r_ != ncclSuccess)                                      \
      return fail(DS_ERR_NCCL, "%s: %s", W, ncclGetErrorString(r_)); \
  } while (0)

int64_t chunk_rows_for(int64_t row_bytes, int64_t rows) {
  int64_t c = kChunkTarget / row_bytes;
  if (c < 1) c = 1;
  if (c > rows) c = rows;
  return c;
}
}  // namespace

extern "C" const char *ds_build_info(void) {
  static char buf[128];
  int v = 0;
  ncclGetVersion(&v);
  snprintf(buf, sizeof buf, "libds sm_100a nccl %d.%d.%d", v / 10000, (v / 100) % 100, v % 100);
  return buf;
}

extern "C" size_t ds_kv_migrate_staging_bytes(const ds_kv_cache *cache, int32_t role,
                                              int32_t layer_count, int32_t num_blocks,
                                              int32_t head_count) {
  if (!cache || layer_count <= 0 || num_blocks <= 0 || head_count <= 0) return 0;
  const int64_t row_bytes = (int64_t)head_count * 16 * cache->head_dim * 2;
  const int64_t rows = (int64_t)layer_count * 2 * num_blocks;
  if (role == DS_MIGRATE_LOCAL || role == DS_MIGRATE_PULL) return 0;
  const int64_t slots = role == DS_MIGRATE_SELF ? 4 : 2;
  return (size_t)(slots * chunk_rows_for(row_bytes, rows) * row_bytes);
}

extern "C" ds_status ds_comm_get_unique_id(void *id_h) {
  if (!id_h) return fail(DS_ERR_INVALID_ARG, "ds_comm_get_unique_id: NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  DS_NCCL(ncclGetUniqueId(&id), "ds_comm_get_unique_id");
  memcpy(id_h, &id, sizeof id);
  return DS_OK;
}

extern "C" ds_status ds_comm_init(const void *id_h, int32_t nranks, int32_t rank, ds_comm *out_h) {
  const char *W = "ds_comm_init";
  if (!id_h || !out_h || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(DS_ERR_INVALID_ARG, "%s: bad arguments", W);
  ds_comm c = new (std::nothrow) ds_comm_s();
  if (!c) return fail(DS_ERR_INVALID_ARG, "%s: out of host memory", W);
  ncclUniqueId id;
  memcpy(&id, id_h, sizeof id);
  c->rank = rank;
  c->nranks = nranks;
  cudaGetDevice(&c->device);
  ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(DS_ERR_NCCL, "%s: %s", W, ncclGetErrorString(r));
  }
  cudaError_t e = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&c->ev_a[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_b[i], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) {
    ds_comm_destroy(c);
    return fail(DS_ERR_CUDA, "%s: %s", W, cudaGetErrorString(e));
  }
  *out_h = c;
  return DS_OK;
}

extern "C" ds_status ds_comm_destroy(ds_comm c) {
  if (!c) return fail(DS_ERR_STATE, "ds_comm_destroy: NULL");
  if (c->side) cudaStreamSynchronize(c->side);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->ev_start) cudaEventDestroy(c->ev_start);
  for (int i = 0; i < 2; ++i) {
    if (c->ev_a[i]) cudaEventDestroy(c->ev_a[i]);
    if (c->ev_b[i]) cudaEventDestroy(c->ev_b[i]);
  }
  delete c;
  return DS_OK;
}

static ds_status migrate_local(const ds_kv_cache *src, int32_t layer_begin, int32_t layer_count,
                               const int32_t *src_ids, int32_t num_blocks, int32_t src_h0,
                               int32_t head_count, const ds_kv_cache *dst, const int32_t *dst_ids,
                               int32_t dst_h0, int32_t dst_layer_begin, void *stream) {
  const char *W = "ds_kv_migrate(LOCAL/PULL)";
  if (!src || !dst) return fail(DS_ERR_INVALID_ARG, "%s: NULL cache", W);
  if (layer_count < 0 || num_blocks < 0 || head_count < 0)
    return fail(DS_ERR_INVALID_ARG, "%s: negative count", W);
  const ds_kv_cache *ends[2] = {src, dst};
  const int32_t h0s[2] = {src_h0, dst_h0};
  const int32_t l0s[2] = {layer_begin, dst_layer_begin};
  for (int e = 0; e < 2; ++e) {
    const ds_kv_cache *c = ends[e];
    if (!c->base || c->block_size != 16 || (c->head_dim != 64 && c->head_dim != 128))
      return fail(DS_ERR_INVALID_ARG, "%s: bad cache descriptor", W);
    if (l0s[e] < 0 || l0s[e] + layer_count > c->num_layers)
      return fail(DS_ERR_INVALID_ARG, "%s: layer range outside the pool", W);
    if (h0s[e] < 0 || h0s[e] + head_count > c->num_heads)
      return fail(DS_ERR_INVALID_ARG, "%s: head slice outside n_loc", W);
  }
  if (src->head_dim != dst->head_dim) return fail(DS_ERR_INVALID_ARG, "%s: head_dim differs", W);
  if ((int64_t)layer_count * num_blocks * head_count == 0) return DS_OK;
  if (!src_ids || !dst_ids) return fail(DS_ERR_INVALID_ARG, "%s: NULL block ids", W);
  KvLocalArgs a{};
  a.src = static_cast<const uint16_t *>(src->base);
  a.dst = static_cast<uint16_t *>(dst->base);
  a.src_ids = src_ids;
  a.dst_ids = dst_ids;
  a.layer_begin = layer_begin;
  a.dst_layer_begin = dst_layer_begin;
  a.layer_count = layer_count;
  a.num_blocks_sel = num_blocks;
  a.head_count = head_count;
  a.head_dim = src->head_dim;
  a.src_blocks = src->num_blocks;
  a.src_heads = src->num_heads;
  a.src_head0 = src_h0;
  a.dst_blocks = dst->num_blocks;
  a.dst_heads = dst->num_heads;
  a.dst_head0 = dst_h0;
  cudaError_t e = launch_kv_local(a, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(DS_ERR_CUDA, "%s: %s", W, cudaGetErrorString(e));
  return DS_OK;
}

extern "C" ds_status ds_kv_migrate(ds_comm comm, int32_t role, int32_t peer,
                                   const ds_kv_cache *cache, int32_t layer_begin,
                                   int32_t layer_count, const int32_t *block_ids,
                                   int32_t num_blocks, int32_t head_begin, int32_t head_count,
                                   const ds_kv_cache *dst_cache, const int32_t *dst_block_ids,
                                   int32_t dst_head_begin, int32_t dst_layer_begin, void *staging,
                                   size_t staging_bytes, void *stream) {
  const char *W = "ds_kv_migrate";
  if (role == DS_MIGRATE_LOCAL || role == DS_MIGRATE_PULL)
    return migrate_local(cache, layer_begin, layer_count, block_ids, num_blocks, head_begin, head_count, dst_cache,
                         dst_block_ids, dst_head_begin, dst_layer_begin, stream);
  if (!comm || !comm->comm) return fail(DS_ERR_STATE, "%s: invalid communicator", W);
  if (role != DS_MIGRATE_SEND && role != DS_MIGRATE_RECV && role != DS_MIGRATE_SELF)
    return fail(DS_ERR_INVALID_ARG, "%s: bad role", W);
  if (role == DS_MIGRATE_SELF) peer = comm->rank;
  if (peer < 0 || peer >= comm->nranks) return fail(DS_ERR_INVALID_ARG, "%s: peer out of range", W);
  if (role != DS_MIGRATE_SELF && peer == comm->rank)
    return fail(DS_ERR_INVALID_ARG, "%s: SEND/RECV to self; use DS_MIGRATE_SELF", W);
  if (!cache) return fail(DS_ERR_INVALID_ARG, "%s: NULL cache", W);
  if (layer_count < 0 || num_blocks < 0 || head_count < 0)
    return fail(DS_ERR_INVALID_ARG, "%s: negative count", W);
  if (role == DS_MIGRATE_SELF) {
    if (!dst_cache || !dst_block_ids) return fail(DS_ERR_INVALID_ARG, "%s: SELF needs dst_cache/dst_block_ids", W);
    if (dst_cache->head_dim != cache->head_dim)
      return fail(DS_ERR_INVALID_ARG, "%s: head_dim differs between source and destination", W);
  }
  {  // validate both ends up front so a rejected call launches nothing
    const ds_kv_cache *ends[2] = {cache, role == DS_MIGRATE_SELF ? dst_cache : cache};
    const int32_t h0s[2] = {head_begin, role == DS_MIGRATE_SELF ? dst_head_begin : head_begin};
    for (int e = 0; e < 2; ++e) {
      const ds_kv_cache *c = ends[e];
      if (!c->base || c->block_size != 16 || (c->head_dim != 64 && c->head_dim != 128))
        return fail(DS_ERR_INVALID_ARG, "%s: bad cache descriptor", W);
      if (layer_begin < 0 || layer_begin + layer_count > c->num_layers)
        return fail(DS_ERR_INVALID_ARG, "%s: layer range outside the pool", W);
      if (h0s[e] < 0 || h0s[e] + head_count > c->num_heads)
        return fail(DS_ERR_INVALID_ARG, "%s: head slice outside n_loc", W);
    }
    if (num_blocks > 0 && !block_ids) return fail(DS_ERR_INVALID_ARG, "%s: NULL block_ids", W);
  }
  const int64_t rows = (int64_t)layer_count * 2 * num_blocks;
  if (rows == 0 || head_count == 0) return DS_OK;
  const int64_t row_bytes = (int64_t)head_count * 16 * cache->head_dim * 2;
  const int64_t crows = chunk_rows_for(row_bytes, rows);
  const size_t need = ds_kv_migrate_staging_bytes(cache, role, layer_count, num_blocks, head_count);
  if (!staging || staging_bytes < need)
    return fail(DS_ERR_INVALID_ARG, "%s: staging must be >= %zu bytes", W, need);
  cudaStream_t A = static_cast<cudaStream_t>(stream), B = comm->side;
  char *stg = static_cast<char *>(staging);
  const int64_t slot_bytes = crows * row_bytes;
  const int64_t nchunks = (rows + crows - 1) / crows;
  const bool send_side = role != DS_MIGRATE_RECV;
  const ds_kv_cache *src = cache;
  const ds_kv_cache *dst = role == DS_MIGRATE_SELF ? dst_cache : cache;
  const int32_t *dst_ids = role == DS_MIGRATE_SELF ? dst_block_ids : block_ids;
  const int32_t dst_h0 = role == DS_MIGRATE_SELF ? dst_head_begin : head_begin;
  char *recv_base = role == DS_MIGRATE_SELF ? stg + 2 * slot_bytes : stg;

  // every pack / unpack launch of the loop below is checked once up front (device,
  // pool, ranges, staging), so a rejected call posts no send or receive and leaves
  // both streams and the peer untouched
  if (send_side)
    if (ds_status s = kv_copy_checked(src, layer_begin, layer_count, block_ids, num_blocks, head_begin,
                                      head_count, stg, slot_bytes, 0, crows, true, A, W, true))
      return s;
  if (role != DS_MIGRATE_SEND)
    if (ds_status s = kv_copy_checked(dst, layer_begin, layer_count, dst_ids, num_blocks, dst_h0, head_count,
                                      recv_base, slot_bytes, 0, crows, false, A, W, true))
      return s;
  DS_CUDA(cudaEventRecord(comm->ev_start, A), W);
  DS_CUDA(cudaStreamWaitEvent(B, comm->ev_start, 0), W);
  for (int64_t k = 0; k < nchunks; ++k) {
    const int slot = (int)(k & 1);
    const int64_t r0 = k * crows, r1 = r0 + crows < rows ? r0 + crows : rows;
    const size_t bytes = (size_t)((r1 - r0) * row_bytes);
    char *sbuf = stg + slot * slot_bytes;
    char *rbuf = recv_base + slot * slot_bytes;
    if (send_side) {
      // slot is free once the transfer of chunk k-2 has completed
      if (k >= 2) DS_CUDA(cudaStreamWaitEvent(A, comm->ev_b[slot], 0), W);
      if (ds_status s = kv_copy_checked(src, layer_begin, layer_count, block_ids, num_blocks,
                                        head_begin, head_count, sbuf, slot_bytes, r0, r1, true, A, W))
        return s;
      DS_CUDA(cudaEventRecord(comm->ev_a[slot], A), W);
      DS_CUDA(cudaStreamWaitEvent(B, comm->ev_a[slot], 0), W);  // packed (and, SELF: k-2 unpacked)
    } else if (k >= 2) {
      DS_CUDA(cudaStreamWaitEvent(B, comm->ev_a[slot], 0), W);  // unpack of chunk k-2 done
    }
    DS_NCCL(ncclGroupStart(), W);
    if (role != DS_MIGRATE_RECV) DS_NCCL(ncclSend(sbuf, bytes, ncclUint8, peer, comm->comm, B), W);
    if (role != DS_MIGRATE_SEND) DS_NCCL(ncclRecv(rbuf, bytes, ncclUint8, peer, comm->comm, B), W);
    DS_NCCL(ncclGroupEnd(), W);
    DS_CUDA(cudaEventRecord(comm->ev_b[slot], B), W);
    if (role != DS_MIGRATE_SEND) {
      DS_CUDA(cudaStreamWaitEvent(A, comm->ev_b[slot], 0), W);
      // staging row r0 of the chunk sits at the start of the receive slot
      if (ds_status s = kv_copy_checked(dst, layer_begin, layer_count, dst_ids, num_blocks,
                                        dst_h0, head_count, rbuf, slot_bytes, r0, r1, false, A, W))
        return s;
      if (role == DS_MIGRATE_RECV) DS_CUDA(cudaEventRecord(comm->ev_a[slot], A), W);
    }
  }
  // the caller's stream is ordered after every transfer of this call
  DS_CUDA(cudaEventRecord(comm->ev_start, B), W);
  DS_CUDA(cudaStreamWaitEvent(A, comm->ev_start, 0), W);
  return DS_OK;
}

// a5 without a4 / a6: consecutive page ids on both ends and the whole head range
// make every (layer, K|V) run of the batch one contiguous region of both pools,
// so NCCL moves it pool to pool — no staging ring, no pack / unpack kernels (whose
// HBM passes would compete with the prefill and decode kernels running beside the
// transfer). One ncclGroup per layer (its K and V runs) on the caller's stream.
extern "C" ds_status ds_kv_migrate_contig(ds_comm comm, int32_t role, int32_t peer, const ds_kv_cache *cache,
                                          int32_t layer_begin, int32_t layer_count, int32_t block_begin,
                                          int32_t num_blocks, const ds_kv_cache *dst_cache,
                                          int32_t dst_block_begin, void *stream) {
  const char *W = "ds_kv_migrate_contig";
  if (!comm || !comm->comm) return fail(DS_ERR_STATE, "%s: invalid communicator", W);
  if (role != DS_MIGRATE_SEND && role != DS_MIGRATE_RECV && role != DS_MIGRATE_SELF)
    return fail(DS_ERR_INVALID_ARG, "%s: bad role (SEND, RECV or SELF)", W);
  if (role == DS_MIGRATE_SELF) peer = comm->rank;
  if (peer < 0 || peer >= comm->nranks) return fail(DS_ERR_INVALID_ARG, "%s: peer out of range", W);
  if (role != DS_MIGRATE_SELF && peer == comm->rank)
    return fail(DS_ERR_INVALID_ARG, "%s: SEND/RECV to self; use DS_MIGRATE_SELF", W);
  if (!cache || (role == DS_MIGRATE_SELF && !dst_cache)) return fail(DS_ERR_INVALID_ARG, "%s: NULL cache", W);
  if (layer_count < 0 || num_blocks < 0) return fail(DS_ERR_INVALID_ARG, "%s: negative count", W);
  const ds_kv_cache *ends[2] = {cache, role == DS_MIGRATE_SELF ? dst_cache : cache};
  const int32_t b0s[2] = {block_begin, role == DS_MIGRATE_SELF ? dst_block_begin : block_begin};
  for (int e = 0; e < 2; ++e) {
    const ds_kv_cache *c = ends[e];
    if (!c->base || c->block_size != 16 || (c->head_dim != 64 && c->head_dim != 128))
      return fail(DS_ERR_INVALID_ARG, "%s: bad cache descriptor", W);
    if (layer_begin < 0 || layer_begin + layer_count > c->num_layers)
      return fail(DS_ERR_INVALID_ARG, "%s: layer range outside the pool", W);
    if (b0s[e] < 0 || (int64_t)b0s[e] + num_blocks > c->num_blocks)
      return fail(DS_ERR_INVALID_ARG, "%s: block range outside the pool", W);
  }
  if (ends[1]->head_dim != cache->head_dim || ends[1]->num_heads != cache->num_heads)
    return fail(DS_ERR_INVALID_ARG, "%s: source and destination geometry differ", W);
  if ((int64_t)layer_count * num_blocks == 0) return DS_OK;
  const int64_t blk_bytes = (int64_t)cache->num_heads * 16 * cache->head_dim * 2;
  const size_t run = (size_t)(num_blocks * blk_bytes);
  cudaStream_t A = static_cast<cudaStream_t>(stream);
  for (int32_t l = layer_begin; l < layer_begin + layer_count; ++l) {
    DS_NCCL(ncclGroupStart(), W);
    for (int kv = 0; kv < 2; ++kv) {
      if (role != DS_MIGRATE_RECV) {
        const char *src = static_cast<const char *>(cache->base) +
                          ((int64_t)(2 * l + kv) * cache->num_blocks + block_begin) * blk_bytes;
        DS_NCCL(ncclSend(src, run, ncclUint8, peer, comm->comm, A), W);
      }
      if (role != DS_MIGRATE_SEND) {
        const ds_kv_cache *d = ends[1];
        char *dst = static_cast<char *>(d->base) + ((int64_t)(2 * l + kv) * d->num_blocks + b0s[1]) * blk_bytes;
        DS_NCCL(ncclRecv(dst, run, ncclUint8, peer, comm->comm, A), W);
      }
    }
    DS_NCCL(ncclGroupEnd(), W);
  }
  return DS_OK;
}

// ---------------------------------------------------------------- CUDA IPC (PULL)
struct ds_event_s {
  cudaEvent_t ev = nullptr;
};

typedef CUresult (*PFN_getAddressRange)(CUdeviceptr *, size_t *, CUdeviceptr);

extern "C" ds_status ds_ipc_export_mem(const void *ptr, ds_ipc_handle *handle_h, size_t *offset_h) {
  const char *W = "ds_ipc_export_mem";
  if (!ptr || !handle_h || !offset_h) return fail(DS_ERR_INVALID_ARG, "%s: NULL argument", W);
  static_assert(sizeof(cudaIpcMemHandle_t) == sizeof(ds_ipc_handle), "IPC handle size");
  // the handle names the whole cudaMalloc allocation; report where `ptr` sits in it
  static PFN_getAddressRange range_fn = nullptr;
  if (!range_fn) {
    void *fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return fail(DS_ERR_CUDA, "%s: cuMemGetAddressRange unavailable", W);
    range_fn = reinterpret_cast<PFN_getAddressRange>(fp);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range_fn(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
    return fail(DS_ERR_CUDA, "%s: pointer is not device memory", W);
  cudaIpcMemHandle_t h;
  DS_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base)), W);
  memcpy(handle_h->bytes, &h, sizeof h);
  *offset_h = (size_t)(reinterpret_cast<CUdeviceptr>(ptr) - base);
  return DS_OK;
}

extern "C" ds_status ds_ipc_open_mem(const ds_ipc_handle *handle_h, void **base_h) {
  const char *W = "ds_ipc_open_mem";
  if (!handle_h || !base_h) return fail(DS_ERR_INVALID_ARG, "%s: NULL argument", W);
  cudaIpcMemHandle_t h;
  memcpy(&h, handle_h->bytes, sizeof h);
  DS_CUDA(cudaIpcOpenMemHandle(base_h, h, cudaIpcMemLazyEnablePeerAccess), W);
  return DS_OK;
}

extern "C" ds_status ds_ipc_close_mem(void *base) {
  if (!base) return fail(DS_ERR_INVALID_ARG, "ds_ipc_close_mem: NULL");
  DS_CUDA(cudaIpcCloseMemHandle(base), "ds_ipc_close_mem");
  return DS_OK;
}

extern "C" ds_status ds_event_create_ipc(ds_event *out_h, ds_ipc_handle *handle_h) {
  const char *W = "ds_event_create_ipc";
  if (!out_h || !handle_h) return fail(DS_ERR_INVALID_ARG, "%s: NULL argument", W);
  static_assert(sizeof(cudaIpcEventHandle_t) == sizeof(ds_ipc_handle), "IPC event handle size");
  ds_event e = new (std::nothrow) ds_event_s();
  if (!e) return fail(DS_ERR_INVALID_ARG, "%s: out of host memory", W);
  cudaError_t err = cudaEventCreateWithFlags(&e->ev, cudaEventInterprocess | cudaEventDisableTiming);
  cudaIpcEventHandle_t h;
  if (err == cudaSuccess) err = cudaIpcGetEventHandle(&h, e->ev);
  if (err != cudaSuccess) {
    if (e->ev) cudaEventDestroy(e->ev);
    delete e;
    return fail(DS_ERR_CUDA, "%s: %s", W, cudaGetErrorString(err));
  }
  memcpy(handle_h->bytes, &h, sizeof h);
  *out_h = e;
  return DS_OK;
}

extern "C" ds_status ds_event_open_ipc(const ds_ipc_handle *handle_h, ds_event *out_h) {
  const char *W = "ds_event_open_ipc";
  if (!out_h || !handle_h) return fail(DS_ERR_INVALID_ARG, "%s: NULL argument", W);
  ds_event e = new (std::nothrow) ds_event_s();
  if (!e) return fail(DS_ERR_INVALID_ARG, "%s: out of host memory", W);
  cudaIpcEventHandle_t h;
  memcpy(&h, handle_h->bytes, sizeof h);
  cudaError_t err = cudaIpcOpenEventHandle(&e->ev, h);
  if (err != cudaSuccess) {
    delete e;
    return fail(DS_ERR_CUDA, "%s: %s", W, cudaGetErrorString(err));
  }
  *out_h = e;
  return DS_OK;
}

extern "C" ds_status ds_event_record(ds_event e, void *stream) {
  if (!e || !e->ev) return fail(DS_ERR_STATE, "ds_event_record: invalid event");
  DS_CUDA(cudaEventRecord(e->ev, static_cast<cudaStream_t>(stream)), "ds_event_record");
  return DS_OK;
}

extern "C" ds_status ds_event_wait(ds_event e, void *stream) {
  if (!e || !e->ev) return fail(DS_ERR_STATE, "ds_event_wait: invalid event");
  DS_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), e->ev, 0), "ds_event_wait");
  return DS_OK;
}

extern "C" ds_status ds_event_destroy(ds_event e) {
  if (!e) return fail(DS_ERR_STATE, "ds_event_destroy: NULL");
  if (e->ev) cudaEventDestroy(e->ev);
  delete e;
  return DS_OK;
}
