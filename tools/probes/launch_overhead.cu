// Launch-overhead probe: event-timed back-to-back launches of empty kernels with
// and without a large dynamic smem carve-out and a TMEM alloc/dealloc.
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/lo tools/probes/launch_overhead.cu && /tmp/lo
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_empty(int* p) {
  if (p && threadIdx.x == 1000) *p = 1;
}
__global__ void k_smem(int* p) {
  extern __shared__ int s[];
  if (p && threadIdx.x == 1000) *p = s[0];
}
__global__ void k_tmem(int* p) {
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512));
}

template <typename F>
float timeit(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 5; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return 1e3f * ms / reps;
}

int main() {
  const int smem = 206 * 1024;
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  printf("empty 148x192            %.2f us\n", timeit([] { k_empty<<<148, 192>>>(nullptr); }, 200));
  printf("smem206K 148x192         %.2f us\n", timeit([&] { k_smem<<<148, 192, smem>>>(nullptr); }, 200));
  printf("smem206K+tmem512 148x192 %.2f us\n", timeit([&] { k_tmem<<<148, 192, smem>>>(nullptr); }, 200));
  printf("tmem512 no smem 148x192  %.2f us\n", timeit([&] { k_tmem<<<148, 192, 0>>>(nullptr); }, 200));
  printf("alternating empty/smem   %.2f us\n", timeit([&] {
    k_empty<<<148, 192>>>(nullptr);
    k_smem<<<148, 192, smem>>>(nullptr);
  }, 200));
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
