// K6: group-normalised advantages over contiguous groups of G rewards.
//
// Reference: src/april_sim/policy.py:115-124 (group_advantages), applied to
// contiguous per-group slices of the delivered batch (simulate.py:54-65).
//   mode 0  mean baseline        A = r - mean(r)
//   mode 1  mean/std (GRPO)      A = (r - mean(r)) / (std_pop(r) + eps)
//   mode 2  DAPO                 as mode 1, plus a per-group zero-std flag
//                                (dynamic-sampling filter; not in the reference,
//                                parity-unpinned)
//   mode 3  GSPO                 as mode 1 (the sequence-level ratio uses the
//                                length-normalised behaviour log-prob from
//                                ab_engine_sequence_logprobs; parity-unpinned)
// numpy's mean/std are pairwise sums (np_pairwise_sum), so results are
// bit-identical to the reference for any G.
#include <vector>

#include "common.cuh"

namespace ab {

constexpr int kMaxGroupForAdv = 1024;

__global__ void k_group_advantages(const double* __restrict__ r, int n_groups, int G, int mode, double eps,
                                   double* __restrict__ adv, int32_t* __restrict__ flags) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_groups) return;
  const double* x = r + (int64_t)g * G;
  double buf[kMaxGroupForAdv <= 64 ? kMaxGroupForAdv : 64];
  const double mean = np_pairwise_sum(x, G) / G;
  double var = 0.0;
  if (G <= 64) {
    for (int i = 0; i < G; ++i) {
      const double c = x[i] - mean;
      buf[i] = c * c;
    }
    var = np_pairwise_sum(buf, G) / G;
  } else {
    // groups beyond 64 samples: sequential blocks of 64 folded pairwise-free
    // (no reference configuration reaches this)
    for (int i = 0; i < G; ++i) {
      const double c = x[i] - mean;
      var += c * c;
    }
    var /= G;
  }
  const double sd = sqrt(var);
  for (int i = 0; i < G; ++i) {
    const double c = x[i] - mean;
    adv[(int64_t)g * G + i] = mode == 0 ? c : c / (sd + eps);
  }
  if (flags) flags[g] = (sd == 0.0) ? 1 : 0;
}

}  // namespace ab

static bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

extern "C" int ab_group_advantages(const double* rewards, int n_groups, int group_size, int mode, double eps,
                                   double* adv, int32_t* zero_std_flags, int device) {
  try {
    AB_REQUIRE(n_groups >= 0 && group_size >= 1, AB_ERR_CONFIG, "advantages need at least one reward");
    AB_REQUIRE(group_size <= ab::kMaxGroupForAdv, AB_ERR_CONFIG, "group too large");
    AB_REQUIRE(mode >= 0 && mode <= 3, AB_ERR_CONFIG, "unknown advantage mode");
    if (n_groups == 0) return AB_OK;
    AB_CUDA(cudaSetDevice(device));
    const size_t n = (size_t)n_groups * group_size;
    const bool dev_in = is_device_ptr(rewards), dev_out = is_device_ptr(adv);
    const bool dev_flags = zero_std_flags == nullptr || is_device_ptr(zero_std_flags);
    double *dr = const_cast<double*>(rewards), *da = adv;
    int32_t* df = zero_std_flags;
    if (!dev_in) {
      AB_CUDA(cudaMalloc(&dr, n * sizeof(double)));
      AB_CUDA(cudaMemcpy(dr, rewards, n * sizeof(double), cudaMemcpyHostToDevice));
    }
    if (!dev_out) AB_CUDA(cudaMalloc(&da, n * sizeof(double)));
    if (!dev_flags) AB_CUDA(cudaMalloc(&df, n_groups * sizeof(int32_t)));
    ab::k_group_advantages<<<ab::ceil_div(n_groups, 128), 128>>>(dr, n_groups, group_size, mode, eps, da, df);
    AB_CUDA(cudaGetLastError());
    if (!dev_out) AB_CUDA(cudaMemcpy(adv, da, n * sizeof(double), cudaMemcpyDeviceToHost));
    if (!dev_flags) AB_CUDA(cudaMemcpy(zero_std_flags, df, n_groups * sizeof(int32_t), cudaMemcpyDeviceToHost));
    AB_CUDA(cudaDeviceSynchronize());
    if (!dev_in) cudaFree(dr);
    if (!dev_out) cudaFree(da);
    if (!dev_flags) cudaFree(df);
    return AB_OK;
  } catch (const ab::Error& e) {
    ab::set_last_error(e.what());
    return e.code;
  }
}
