// Which not-yet-launched CTA does clusterlaunchcontrol.try_cancel hand over?
// Each CTA (one warp, big smem so only 2 fit per SM) processes its own blockIdx
// and then cancelled ones; every processed index is stamped with a global
// sequence number. Prints the processing order.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ unsigned g_seq;

__global__ void k(int *order, int *who) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint4 *resp = reinterpret_cast<uint4 *>(sm);
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + 64);
  const unsigned bar_a = (unsigned)__cvta_generic_to_shared(bar);
  const unsigned resp_a = (unsigned)__cvta_generic_to_shared(resp);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  int item = blockIdx.x;
  for (unsigned q = 0;; ++q) {
    if (threadIdx.x == 0) {
      unsigned s = atomicAdd(&g_seq, 1);
      order[item] = (int)s;
      who[item] = blockIdx.x;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;" ::"r"(bar_a) : "memory");
      asm volatile("clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 [%0], [%1];"
                   ::"r"(resp_a), "r"(bar_a) : "memory");
    }
    __syncwarp();
    unsigned done = 0;
    for (long spin = 0; !done && spin < 4000000; ++spin)
      asm volatile("{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\nselp.u32 %0, 1, 0, P;\n}"
                   : "=r"(done) : "r"(bar_a), "r"(q & 1) : "memory");
    if (!done) {
      if (threadIdx.x == 0) order[item] = -2;
      break;
    }
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(resp_a) : "memory");
    unsigned ok, x = 0, y = 0, z = 0;
    asm volatile("{\n.reg .b128 R;\n.reg .pred P;\nmov.b128 R, {%4, %5};\n"
                 "clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 P, R;\nselp.u32 %0, 1, 0, P;\n"
                 "@P clusterlaunchcontrol.query_cancel.get_first_ctaid.v4.b32.b128 {%1, %2, %3, _}, R;\n}"
                 : "=r"(ok), "+r"(x), "+r"(y), "+r"(z)
                 : "l"((uint64_t)r.x | ((uint64_t)r.y << 32)), "l"((uint64_t)r.z | ((uint64_t)r.w << 32)) : "memory");
    __syncwarp();
    if (!ok) break;
    item = (int)x;
  }
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  printf("start\n");
  const int N = 4000;
  int *order, *who;
  cudaMalloc(&order, N * 4);
  cudaMalloc(&who, N * 4);
  cudaMemset(order, 0xff, N * 4);
  printf("set attr: %s\n", cudaGetErrorString(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024)));
  k<<<N, 32, 100 * 1024>>>(order, who);
  printf("launch: %s\n", cudaGetErrorString(cudaGetLastError()));
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  std::vector<int> o(N), w(N);
  cudaMemcpy(o.data(), order, N * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(w.data(), who, N * 4, cudaMemcpyDeviceToHost);
  std::vector<int> by_seq(N, -1);
  int missing = 0, stolen = 0, timeouts = 0;
  for (int i = 0; i < N; ++i) {
    if (o[i] == -2) ++timeouts;
    if (o[i] < 0 || o[i] >= N) { ++missing; continue; }
    by_seq[o[i]] = i;
    stolen += w[i] != i;
  }
  printf("missing %d stolen %d timeouts %d\nprocessing order (item index by sequence number):\n", missing, stolen, timeouts);
  for (int s = 0; s < N; s += (s < 400 ? 1 : 97)) printf("%d ", by_seq[s]);
  printf("\nlast 20: ");
  for (int s = N - 20; s < N; ++s) printf("%d ", by_seq[s]);
  printf("\n");
  return 0;
}
