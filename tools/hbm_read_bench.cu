// Microbenchmark: achievable HBM bandwidth on this GPU for (a) a pure streaming
// read (what decode attention does: every cached K/V byte read once) with 16-B
// vector loads and with 1-D TMA bulk copies into smem, and (b) device-to-device
// copy (read + write, the MEASURED_PEAKS "copy" figure). 4 GiB buffers, > L2.
// Usage: hbm_read_bench [MiB] [sustain_seconds] — with a second argument each pattern is
// also timed after that many seconds back to back (the power-capped steady state).
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void read_ld(const uint4 *__restrict__ p, size_t n, unsigned long long *sink) {
  uint32_t acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint4 a = __ldcs(p + i), b = __ldcs(p + i + stride), c = __ldcs(p + i + 2 * stride), d = __ldcs(p + i + 3 * stride);
    acc ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  for (; i < n; i += stride) acc ^= __ldcs(p + i).x;
  if (acc == 0x12345678u) *sink = acc;
}

// each CTA streams kChunk-byte chunks through a kSlots-slot smem ring with cp.async.bulk;
// kScatter visits the chunks in a pseudo-random order (like pages behind a block table)
template <uint32_t kChunk, uint32_t kSlots, bool kScatter>
__global__ void read_bulk(const uint8_t *__restrict__ p, size_t bytes, unsigned long long *sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[kSlots];
  const size_t nchunks = bytes / kChunk;
  if (threadIdx.x == 0) {
    for (int s = 0; s < (int)kSlots; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t acc = 0;
  size_t c = blockIdx.x;
  uint32_t issued = 0, done = 0;
  auto issue = [&](size_t chunk, uint32_t slot) {
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[slot]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kChunk));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(sm + slot * kChunk)),
                 "l"(p + (kScatter ? (chunk * 2654435761ull) % nchunks : chunk) * kChunk), "r"(kChunk), "r"(b)
                 : "memory");
  };
  for (; issued < kSlots && c + (size_t)issued * gridDim.x < nchunks; ++issued) issue(c + (size_t)issued * gridDim.x, issued);
  while (done < issued) {
    const uint32_t slot = done % kSlots, ph = (done / kSlots) & 1;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.b32 %0,1,0,P;}"
                   : "=r"(ok)
                   : "r"((uint32_t)__cvta_generic_to_shared(&bar[slot])), "r"(ph)
                   : "memory");
    acc ^= sm[slot * kChunk];
    const size_t nxt = c + (size_t)issued * gridDim.x;
    if (nxt < nchunks) {
      issue(nxt, issued % kSlots);
      ++issued;
    }
    ++done;
  }
  if (acc == 0x12345678u) *sink = acc;
}

// decode-like: 16 warps per CTA, each with its own 3-slot ring of 4 KiB pages filled by
// one lane; page k of a warp's range lives at (k % run) * stride_pages + k / run (pages)
// so stride_pages = 1 is sequential and stride_pages = 40 mimics one head of a
// [blocks][40 heads][16][128] pool walked block by block
template <int kSlotsPerWarp>
__global__ void read_warps(const uint8_t *__restrict__ p, size_t bytes, int stride_pages, unsigned long long *sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[16 * kSlotsPerWarp];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t npages = bytes / 4096;
  const size_t per_warp = npages / (gridDim.x * 16);
  const size_t w = (size_t)blockIdx.x * 16 + warp;
  uint8_t *ring = sm + warp * kSlotsPerWarp * 4096;
  uint64_t *wb = bar + warp * kSlotsPerWarp;
  if (lane == 0)
    for (int s = 0; s < kSlotsPerWarp; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&wb[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncwarp();
  // the warp's pages: a contiguous range of "logical" pages, mapped through the stride
  const size_t run = npages / stride_pages;  // pages per "head"
  auto addr = [&](size_t k) {
    const size_t lp = w * per_warp + k;  // logical page: head-major (head = lp / run, block = lp % run)
    const size_t head = lp / run, blk = lp % run;
    return p + (blk * stride_pages + head) * 4096;
  };
  auto issue = [&](size_t k, int slot) {
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&wb[slot]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(4096));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(ring + slot * 4096)),
                 "l"(addr(k)), "r"(4096), "r"(b)
                 : "memory");
  };
  uint32_t acc = 0;
  if (lane == 0)
    for (int s = 0; s < kSlotsPerWarp && s < (int)per_warp; ++s) issue(s, s);
  for (size_t k = 0; k < per_warp; ++k) {
    const int slot = k % kSlotsPerWarp;
    const uint32_t ph = (k / kSlotsPerWarp) & 1;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.b32 %0,1,0,P;}"
                   : "=r"(ok)
                   : "r"((uint32_t)__cvta_generic_to_shared(&wb[slot])), "r"(ph)
                   : "memory");
    acc ^= reinterpret_cast<const uint32_t *>(ring + slot * 4096)[lane * 32];  // touch the page
    __syncwarp();
    if (lane == 0 && k + kSlotsPerWarp < per_warp) issue(k + kSlotsPerWarp, slot);
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main(int argc, char **argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = argc > 1 ? (size_t)atoll(argv[1]) << 20 : 4ull << 30;  // MiB
  const double sustain_s = argc > 2 ? atof(argv[2]) : 0.0;  // also time each pattern after this long under load
  uint8_t *a, *b;
  unsigned long long *sink;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMalloc(&sink, 8);
  cudaMemset(a, 1, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaFuncSetAttribute(read_bulk<16384, 8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
  cudaFuncSetAttribute(read_bulk<4096, 48, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 4096);
  cudaFuncSetAttribute(read_bulk<4096, 48, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 4096);
  cudaFuncSetAttribute(read_bulk<4096, 24, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 24 * 4096);
  const char *names[] = {"read, 16-B loads (8 CTA/SM)", "read, TMA bulk 8x16K (1 CTA/SM)", "read, TMA bulk 8x16K (2 CTA/SM)",
                         "D2D copy (read+write bytes)", "read, bulk 48x4K seq (1 CTA/SM)", "read, bulk 48x4K scattered",
                         "read, bulk 24x4K scattered x2 CTA", "decode-like 16 warps x 3 x 4K, seq",
                         "decode-like, 40-page stride (1 head)"};
  cudaFuncSetAttribute(read_warps<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 3 * 4096);
  for (int k = 0; k < 9; ++k) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (k == 0) read_ld<<<sms * 8, 512>>>((const uint4 *)a, bytes / 16, sink);
      else if (k == 1) read_bulk<16384, 8, false><<<sms, 32, 8 * 16384>>>(a, bytes, sink);
      else if (k == 2) read_bulk<16384, 8, false><<<sms * 2, 32, 8 * 16384>>>(a, bytes, sink);
      else if (k == 3) cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice);
      else if (k == 4) read_bulk<4096, 48, false><<<sms, 32, 48 * 4096>>>(a, bytes, sink);
      else if (k == 5) read_bulk<4096, 48, true><<<sms, 32, 48 * 4096>>>(a, bytes, sink);
      else if (k == 6) read_bulk<4096, 24, true><<<sms * 2, 32, 24 * 4096>>>(a, bytes, sink);
      else if (k == 7) read_warps<3><<<sms, 512, 16 * 3 * 4096>>>(a, bytes, 1, sink);
      else read_warps<3><<<sms, 512, 16 * 3 * 4096>>>(a, bytes, 40, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double moved = (k == 3 ? 2.0 : 1.0) * bytes;
    printf("%-34s %8.3f ms  %7.1f GB/s", names[k], best, moved / best / 1e6);
    if (sustain_s > 0) {  // the same launch back to back for sustain_s seconds; average of the last half
      const int n = (int)(sustain_s * 1e3 / best);
      for (int rep = 0; rep < n; ++rep) {
        if (rep == n / 2) cudaEventRecord(e0);
        if (k == 0) read_ld<<<sms * 8, 512>>>((const uint4 *)a, bytes / 16, sink);
        else if (k == 1) read_bulk<16384, 8, false><<<sms, 32, 8 * 16384>>>(a, bytes, sink);
        else if (k == 2) read_bulk<16384, 8, false><<<sms * 2, 32, 8 * 16384>>>(a, bytes, sink);
        else if (k == 3) cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice);
        else if (k == 4) read_bulk<4096, 48, false><<<sms, 32, 48 * 4096>>>(a, bytes, sink);
        else if (k == 5) read_bulk<4096, 48, true><<<sms, 32, 48 * 4096>>>(a, bytes, sink);
        else if (k == 6) read_bulk<4096, 24, true><<<sms * 2, 32, 24 * 4096>>>(a, bytes, sink);
        else if (k == 7) read_warps<3><<<sms, 512, 16 * 3 * 4096>>>(a, bytes, 1, sink);
        else read_warps<3><<<sms, 512, 16 * 3 * 4096>>>(a, bytes, 40, sink);
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double per = ms / (n - n / 2);
      printf("   sustained %.0f s: %8.3f ms  %7.1f GB/s", sustain_s, per, moved / per / 1e6);
    }
    printf("\n");
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
