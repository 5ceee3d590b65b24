// Probe: TMA (cp.async.bulk.tensor 2-D, 128B swizzle) ingress rate per SM.
// Each CTA streams `iters` boxes of {64 cols x box_rows} bf16 from a large matrix through a `stages`-deep
// mbarrier ring (consumer = the same thread re-arming), for grid CTAs; reports aggregate and per-SM GB/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probes/tma_rate tools/probes/tma_rate.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_stream(const __grid_constant__ CUtensorMap map, int rows_total, int box_rows, int stages,
                         int iters, int nthr) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = (uint64_t*)(base + stages * box_rows * 128);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // nthr issuing threads (one per warp), thread t owns stages t, t + nthr, ...
  const int tw = threadIdx.x >> 5;
  if ((threadIdx.x & 31) != 0 || tw >= nthr) return;
  const uint32_t bytes = box_rows * 128;
  const int nrb = rows_total / box_rows;
  int rb = (blockIdx.x * 7919) % nrb;
  // prime
  for (int i = tw; i < iters + stages; i += nthr) {
    const int s = i % stages;
    if (i >= stages) {  // wait for the load issued `stages` ago
      const uint32_t ph = ((i - stages) / stages) & 1;
      uint32_t ok = 0;
      do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}"
                     : "=r"(ok) : "r"(su32(&bar[s])), "r"(ph) : "memory");
      } while (!ok);
    }
    if (i < iters) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(bytes) : "memory");
      const int x = (i % 8) * 64;
      const int y = ((rb + i / 8) % nrb) * box_rows;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
              su32(base + s * bytes)),
          "l"((uint64_t)&map), "r"(su32(&bar[s])), "r"(x), "r"(y)
          : "memory");
    }
  }
}

int main() {
  const int64_t rows = 1 << 16, cols = 512;  // 64 MB bf16 (L2-resident-ish: 126 MB L2)
  void* buf;
  cudaMalloc(&buf, rows * cols * 2);
  cudaMemset(buf, 1, rows * cols * 2);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int nthr : {1, 2, 4})
  for (int box_rows : {32, 128, 256}) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(cols * 2)};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    const int bytes = box_rows * 128;
    for (int inflight_kb : {128}) {
      const int stages = inflight_kb * 1024 / bytes;
      if (stages < 1 || stages > 64) continue;
      for (int grid : {sms}) {
        const int per_sm = grid > sms ? 2 : 1;
        const int smem = stages * bytes + 1024 + 64 * 8;
        if (smem * per_sm > 228 * 1024) continue;
        const int iters = (int)(((int64_t)8 << 20) / bytes);  // 8 MB per CTA
        k_stream<<<grid, 128, smem>>>(map, (int)rows, box_rows, stages, iters, nthr);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        k_stream<<<grid, 128, smem>>>(map, (int)rows, box_rows, stages, iters, nthr);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double tot = (double)grid * iters * bytes;
        printf("threads %d box %3d rows (%5d B)  in-flight %3d KB/CTA  grid %3d : %7.0f GB/s total, %5.1f GB/s per CTA\n", nthr, box_rows,
               bytes, inflight_kb, grid, tot / ms / 1e6, tot / ms / 1e6 / grid);
      }
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
