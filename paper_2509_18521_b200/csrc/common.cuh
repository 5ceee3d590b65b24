// Shared device/host helpers for the APRIL B200 engine.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "../../include/april_b200.h"

namespace ab {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define AB_CUDA(x)                                                                                   \
  do {                                                                                               \
    cudaError_t err__ = (x);                                                                         \
    if (err__ != cudaSuccess)                                                                        \
      throw ::ab::Error(AB_ERR_CUDA, std::string(#x " failed: ") + cudaGetErrorString(err__) + " at " + \
                                         __FILE__ + ":" + std::to_string(__LINE__));                  \
  } while (0)

#define AB_REQUIRE(cond, code, msg)                  \
  do {                                               \
    if (!(cond)) throw ::ab::Error((code), (msg));   \
  } while (0)

// ---------------------------------------------------------------------------
// Philox4x64-10 exactly as numpy's bit generator:
// word t of a stream keyed (k0, k1) is lane t&3 of the block at counter
// ((t >> 2) + 1, 0, 0, 0); the draw is (word >> 11) * 2^-53.
// Reference: src/april_sim/rng.py:50-55 (numpy Philox, counter pre-incremented).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

__host__ __device__ __forceinline__ uint64_t philox_word(uint64_t k0, uint64_t k1, uint64_t t) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
  uint64_t x0 = (t >> 2) + 1, x1 = 0, x2 = 0, x3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += W0;
      k1 += W1;
    }
    uint64_t lo0 = M0 * x0, hi0 = mulhi64(M0, x0);
    uint64_t lo1 = M1 * x2, hi1 = mulhi64(M1, x2);
    uint64_t n0 = hi1 ^ x1 ^ k0, n2 = hi0 ^ x3 ^ k1;
    x0 = n0;
    x1 = lo1;
    x2 = n2;
    x3 = lo0;
  }
  switch (t & 3) {
    case 0: return x0;
    case 1: return x1;
    case 2: return x2;
    default: return x3;
  }
}

__host__ __device__ __forceinline__ double philox_uniform(uint64_t k0, uint64_t k1, uint64_t t) {
  return (double)(philox_word(k0, k1, t) >> 11) * 0x1.0p-53;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_min_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// numpy float64 add.reduce: pairwise summation, 8 accumulators below 128
// elements, sequential below 8 (numpy/core/src/umath/loops_utils.h.src).
__host__ __device__ inline double np_pairwise_sum(const double* a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}


void set_last_error(const char* msg);  // engine.cu

// Programmatic dependent launch: kernels of the decode iteration are launched with programmatic
// stream serialization, so a kernel's CTAs are scheduled while its predecessor's last CTAs are
// still running; each such kernel calls pdl_wait() before it touches anything the predecessor
// writes, and pdl_launch() once it no longer needs to delay its own successor.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  AB_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

}  // namespace ab
