// Probe: per-kernel cost of back-to-back kernels replayed from a CUDA graph, with and
// without programmatic dependent launch (PDL), for an empty kernel and a "small" kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probes/graph_gap tools/probes/graph_gap.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_small(float* p, int n, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = p[i] * 1.0001f + 1.f;
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
}

float run(int grid, int block, int n, bool pdl, float* buf) {
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  const int K = 256;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int k = 0; k < K; ++k) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k_small, buf, n, pdl ? 1 : 0);
  }
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return 1e3f * ms / (10 * K);
}

int main() {
  float* buf;
  cudaMalloc(&buf, 64 << 20);
  for (int pdl = 0; pdl < 2; ++pdl) {
    printf("pdl=%d  1 CTA x 32       : %.2f us/kernel\n", pdl, run(1, 32, 32, pdl, buf));
    printf("pdl=%d  148 CTA x 256    : %.2f us/kernel\n", pdl, run(148, 256, 148 * 256, pdl, buf));
    printf("pdl=%d  1024 CTA x 256 (1 MB rw): %.2f us/kernel\n", pdl, run(1024, 256, 1024 * 256, pdl, buf));
    printf("pdl=%d  8192 CTA x 256 (8 MB rw): %.2f us/kernel\n", pdl, run(8192, 256, 8192 * 256, pdl, buf));
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
