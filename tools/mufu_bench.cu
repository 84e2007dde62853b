// Microbenchmark: MUFU ex2.approx.f32 vs FFMA throughput per SM on this GPU.
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__global__ void ex2_kernel(float *out, int iters, float seed) {
  float a0 = seed + threadIdx.x * 1e-6f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  float a4 = a0 + 0.4f, a5 = a0 + 0.5f, a6 = a0 + 0.6f, a7 = a0 + 0.7f;
  for (int i = 0; i < iters; ++i) {
#define EX(a) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a));
    EX(a0) EX(a1) EX(a2) EX(a3) EX(a4) EX(a5) EX(a6) EX(a7)
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void ex2h2_kernel(float *out, int iters, float seed) {
  // ex2.approx.f16x2: two exponentials per lane per instruction
  unsigned a[8];
  for (int j = 0; j < 8; ++j) {
    __half2 h = __floats2half2_rn(-0.01f * (j + 1) + seed * 1e-3f, -0.02f * (j + 1));
    a[j] = *reinterpret_cast<unsigned *>(&h);
  }
  for (int i = 0; i < iters; ++i) {
#define EH(x) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x));
    EH(a[0]) EH(a[1]) EH(a[2]) EH(a[3]) EH(a[4]) EH(a[5]) EH(a[6]) EH(a[7])
  }
  unsigned s = 0;
  for (int j = 0; j < 8; ++j) s ^= a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float(s);
}
__global__ void ex2bh2_kernel(float *out, int iters, float seed) {
  // ex2.approx.ftz.bf16x2: two exponentials per lane per instruction
  unsigned a[8];
  for (int j = 0; j < 8; ++j) a[j] = 0xbc00bc00u + j + (unsigned)(seed * 16);
  for (int i = 0; i < iters; ++i) {
#define EB(x) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(x));
    EB(a[0]) EB(a[1]) EB(a[2]) EB(a[3]) EB(a[4]) EB(a[5]) EB(a[6]) EB(a[7])
  }
  unsigned s = 0;
  for (int j = 0; j < 8; ++j) s ^= a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float(s);
}
__global__ void ffma_kernel(float *out, int iters, float seed) {
  float a0 = seed + threadIdx.x * 1e-6f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  float a4 = a0 + 0.4f, a5 = a0 + 0.5f, a6 = a0 + 0.6f, a7 = a0 + 0.7f;
  for (int i = 0; i < iters; ++i) {
#define FM(a) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f33800000;" : "+f"(a));
    FM(a0) FM(a1) FM(a2) FM(a3) FM(a4) FM(a5) FM(a6) FM(a7)
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *out;
  cudaMalloc(&out, sms * 8 * 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000, blocks = sms * 4, threads = 512;
  for (int k = 0; k < 4; ++k) {
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(e0);
      if (k == 0) ex2_kernel<<<blocks, threads>>>(out, iters, 0.5f);
      else if (k == 1) ffma_kernel<<<blocks, threads>>>(out, iters, 0.5f);
      else if (k == 2) ex2h2_kernel<<<blocks, threads>>>(out, iters, 0.5f);
      else ex2bh2_kernel<<<blocks, threads>>>(out, iters, 0.5f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = double(blocks) * threads * iters * 8;
    double per_s = ops / (ms * 1e-3);
    // per SM per clock at the *current* clock is unknown; report per SM per ns and per clk at max clock
    printf("%s: %.3f ms, %.1f Gop/s, %.2f op/clk/SM at max clock %d MHz\n", k == 0 ? "ex2.approx.f32" : k == 1 ? "ffma" : k == 2 ? "ex2.approx.f16x2 (instr; x2 values)" : "ex2.approx.ftz.bf16x2 (instr; x2 values)", ms,
           per_s / 1e9, per_s / sms / (clk * 1e3), clk / 1000);
  }
  return 0;
}
