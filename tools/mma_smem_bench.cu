// Microbenchmark: how fast does the tensor pipe run an attention-shaped
// tcgen05.mma stream, and what does shared memory traffic cost it?
//   * SS (A and B from smem) vs TS (A from TMEM) at N = 64 / 128 / 256, K = 128
//     (8 instructions of K = 16, like the S = Q K^T MMA of prefill.cu);
//   * optionally with a second warp streaming TMA bulk copies (L2 -> smem) into a
//     separate smem region at full speed — the K/V tile fill of the prefill kernel;
//   * one or two CTAs per SM.
// Prints cycles per MMA instruction (clock64 on the issuing thread, from the
// first issue to the commit's mbarrier completion) next to the math-only ideal
// (M*N*K*2 / 8192 flop per clock per SM) and the fill bytes per clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2401_09670_b200/csrc \
//        tools/mma_smem_bench.cu -o tools/mma_smem_bench -lcuda
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

using namespace ds;

constexpr uint32_t kA = 0;              // A: 128 rows x 128 dims bf16, SW128 (2 x 16 KiB column blocks)
constexpr uint32_t kB = 32768;          // B: N rows x 128 dims (2 x N*128 B column blocks)
constexpr uint32_t kFill = kB + 65536;  // fill ring: 2 x 16 KiB
constexpr uint32_t kBar = kFill + 32768;
constexpr uint32_t kSmem = kBar + 64 + 1024;
constexpr uint32_t kSmemSmall = 32768 + 16384 + 32768 + 64 + 1024;  // N = 64 layout for 2 CTAs/SM

struct Out {
  long long cycles;
  long long fill_bytes;
  long long fill_cycles;
};

template <int N, bool kTS, bool kFillOn>
__global__ void __launch_bounds__(128) mma_kernel(Out *out, const uint8_t *gbuf, int iters, int small) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t *smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t B_OFF = kB, FILL = small ? kB + 16384 : kFill, BAR = small ? kB + 16384 + 32768 : kBar;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + BAR);  // [0] mma done, [1..2] fill slots
  volatile uint32_t *flag = reinterpret_cast<volatile uint32_t *>(smem + BAR + 32);
  uint32_t *tslot = reinterpret_cast<uint32_t *>(smem + BAR + 40);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 3; ++b) mbar_init(&bars[b], 1);
    *flag = 0;
    fence_barrier_init();
  }
  // finite operands (values do not matter for timing)
  for (uint32_t o = threadIdx.x * 16; o < B_OFF + N * 256; o += 128 * 16)
    *reinterpret_cast<uint4 *>(smem + o) = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);
  fence_proxy_async_smem();
  if (warp == 0) {
    tmem_alloc<256>(tslot);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t tD = tmem, tA = tmem + (N <= 128 ? 128 : 0);
  if (kTS && warp >= 0 && warp < 4) {  // A (128 x 128 bf16) into TMEM columns [tA, tA+64): all 4 warps
    uint32_t v[32];
    for (int e = 0; e < 32; ++e) v[e] = 0x3f803f80u;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    tmem_st32(tA + lane_off, v);
    tmem_st32(tA + lane_off + 32, v);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == 0) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, N, 0, 0);
      const long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t bd = smem_desc_sw128(sbase + B_OFF + (kk >> 2) * (N * 128) + (kk & 3) * 32, 16, 1024);
          if (kTS)
            umma_ts(tD, tA + kk * 8, bd, idesc, kk > 0);
          else
            umma_ss(tD, smem_desc_sw128(sbase + kA + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), bd, idesc,
                    kk > 0);
        }
      }
      umma_commit(&bars[0]);
      mbar_wait(&bars[0], 0);
      const long long t1 = clock64();
      out[blockIdx.x].cycles = t1 - t0;
      *flag = 1;
    }
    __syncwarp();
  } else if (warp == 1 && kFillOn) {
    if (elect_one()) {
      const long long t0 = clock64();
      long long bytes = 0;
      uint32_t n = 0;
      const uint8_t *src = gbuf + (size_t)(blockIdx.x % 64) * 65536;
      while (*flag == 0) {
        const int s = n & 1;
        if (n >= 2) mbar_wait(&bars[1 + s], ((n >> 1) - 1) & 1);
        mbar_arrive_expect_tx(&bars[1 + s], 16384);
        bulk_g2s(smem + FILL + s * 16384, src + (n & 3) * 16384, 16384, &bars[1 + s]);
        bytes += 16384;
        ++n;
      }
      for (uint32_t t = n >= 2 ? n - 2 : 0; t < n; ++t) mbar_wait(&bars[1 + (t & 1)], (t >> 1) & 1);
      out[blockIdx.x].fill_bytes = bytes;
      out[blockIdx.x].fill_cycles = clock64() - t0;
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

template <int N, bool TS, bool F>
void run(const char *name, int ctas_per_sm, uint8_t *gbuf, Out *dout, int sms) {
  const int small = ctas_per_sm > 1;
  const uint32_t smem = small ? kSmemSmall : kSmem;
  cudaFuncSetAttribute(mma_kernel<N, TS, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int iters = 2000, grid = sms * ctas_per_sm;
  cudaMemset(dout, 0, sizeof(Out) * grid);
  mma_kernel<N, TS, F><<<grid, 128, smem>>>(dout, gbuf, 50, small);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_kernel<N, TS, F><<<grid, 128, smem>>>(dout, gbuf, iters, small);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  if (err != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(err));
    exit(1);
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  Out *h = (Out *)malloc(sizeof(Out) * grid);
  cudaMemcpy(h, dout, sizeof(Out) * grid, cudaMemcpyDeviceToHost);
  double cyc = 0, fb = 0, fc = 0;
  for (int i = 0; i < grid; ++i) {
    cyc += h[i].cycles;
    fb += h[i].fill_bytes;
    fc += h[i].fill_cycles;
  }
  cyc /= grid;
  const double per_instr = cyc / (iters * 8.0);
  const double ideal = 128.0 * N * 16 * 2 / 8192.0;
  const double flops = 2.0 * 128 * N * 128 * iters * (double)grid;
  printf("%-34s ctas/SM %d  cycles/instr %7.1f (math ideal %5.1f, x%.2f per SM with %d CTAs)  %7.1f TF/s", name,
         ctas_per_sm, per_instr, ideal, per_instr / ideal / ctas_per_sm, ctas_per_sm, flops / (ms * 1e-3) / 1e12);
  if (F) printf("  fill %.1f B/clk/CTA", fb / fc);
  printf("\n");
  free(h);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint8_t *gbuf;
  cudaMalloc(&gbuf, 64 * 65536);
  cudaMemset(gbuf, 0, 64 * 65536);
  Out *dout;
  cudaMalloc(&dout, sizeof(Out) * sms * 2);
  for (int rep = 0; rep < 2; ++rep) {
    run<64, false, false>("SS N=64", 1, gbuf, dout, sms);
    run<128, false, false>("SS N=128", 1, gbuf, dout, sms);
    run<256, false, false>("SS N=256", 1, gbuf, dout, sms);
    run<64, true, false>("TS N=64", 1, gbuf, dout, sms);
    run<128, true, false>("TS N=128", 1, gbuf, dout, sms);
    run<64, false, true>("SS N=64 + TMA fill", 1, gbuf, dout, sms);
    run<128, false, true>("SS N=128 + TMA fill", 1, gbuf, dout, sms);
    run<256, false, true>("SS N=256 + TMA fill", 1, gbuf, dout, sms);
    run<64, true, true>("TS N=64 + TMA fill", 1, gbuf, dout, sms);
    run<128, true, true>("TS N=128 + TMA fill", 1, gbuf, dout, sms);
    run<64, false, false>("SS N=64", 2, gbuf, dout, sms);
    run<64, true, false>("TS N=64", 2, gbuf, dout, sms);
    run<64, false, true>("SS N=64 + TMA fill", 2, gbuf, dout, sms);
    run<64, true, true>("TS N=64 + TMA fill", 2, gbuf, dout, sms);
  }
  return 0;
}
