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
// numpy's mean/std are pairwise sums (np_pairwise_sum; the squared deviations are
// summed by the same recursion, generated on the fly), so results are bit-identical to
// the reference's numpy for any G.
//
// K7 (trainer-side consumption): the clipped-ratio terms of a mixed-policy
// batch -- per token r = exp(logp_now - logp_behaviour), the clip mask of the DAPO
// clip-higher surrogate (policy.py:153-177: clipped iff A > 0 and r > 1 + eps_high, or
// A < 0 and r < 1 - eps) and per response sum_t min(r A, clip(r, 1 - eps, 1 + eps_high) A);
// sequence_level: GSPO's length-normalised ratio exp(mean_t(logp_now - logp_behaviour)).
#include <mutex>
#include <vector>

#include "common.cuh"

namespace ab {

// numpy pairwise add.reduce over f(0..n) (same blocking as np_pairwise_sum)
template <typename F>
__device__ double np_pairwise_sum_f(const F& f, int off, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r += f(off + i);
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = f(off + j);
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += f(off + i + j);
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += f(off + i);
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise_sum_f(f, off, n2) + np_pairwise_sum_f(f, off + n2, n - n2);
}

__global__ void k_group_advantages(const double* __restrict__ r, int n_groups, int G, int mode, double eps,
                                   double* __restrict__ adv, int32_t* __restrict__ flags) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_groups) return;
  const double* x = r + (int64_t)g * G;
  const double mean = np_pairwise_sum(x, G) / G;
  auto sq = [&](int i) {
    const double c = x[i] - mean;
    return __dmul_rn(c, c);  // rounded product, never contracted into the sum's FMA (numpy rounds it)
  };
  const double sd = sqrt(np_pairwise_sum_f(sq, 0, G) / G);
  for (int i = 0; i < G; ++i) {
    const double c = x[i] - mean;
    adv[(int64_t)g * G + i] = mode == 0 ? c : c / (sd + eps);
  }
  if (flags) flags[g] = (sd == 0.0) ? 1 : 0;
}

// one warp per response; lane-strided partial sums folded by a fixed xor tree (deterministic)
__global__ void k_clipped_ratio(const double* __restrict__ now, const double* __restrict__ beh,
                                const int64_t* __restrict__ offs, int n, const double* __restrict__ adv, double lo,
                                double hi, int seq_level, double* __restrict__ ratios, int32_t* __restrict__ clipped,
                                double* __restrict__ surrogate) {
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (k >= n) return;
  const int64_t o0 = offs[k], o1 = offs[k + 1];
  const double a = adv[k];
  auto term = [&](double r) { return fmin(r * a, fmin(fmax(r, lo), hi) * a); };
  auto is_clipped = [&](double r) { return (a > 0.0 && r > hi) || (a < 0.0 && r < lo); };
  if (seq_level) {
    double d = 0.0;
    for (int64_t t = o0 + lane; t < o1; t += 32) d += now[t] - beh[t];
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) d += __shfl_xor_sync(0xffffffffu, d, s);
    if (lane == 0) {
      const double r = o1 > o0 ? exp(d / (double)(o1 - o0)) : 0.0;
      ratios[k] = r;
      clipped[k] = o1 > o0 && is_clipped(r);
      surrogate[k] = o1 > o0 ? term(r) : 0.0;
    }
    return;
  }
  double acc = 0.0;
  for (int64_t t = o0 + lane; t < o1; t += 32) {
    const double r = exp(now[t] - beh[t]);
    ratios[t] = r;
    clipped[t] = is_clipped(r);
    acc += term(r);
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if (lane == 0) surrogate[k] = acc;
}

// Per-device scratch reused across calls (grown on demand, stream-ordered) and a private
// non-blocking stream: no allocation per call, and no device-wide synchronisation, so a call never
// waits on an engine's decode loop running on the same device (several engines per process in the
// data-parallel tests).  The mutex serialises callers that share a device.
struct Scratch {
  std::mutex mu;
  cudaStream_t stream = nullptr;
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes) {
    if (!stream) AB_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    if (bytes > cap) {
      if (p) AB_CUDA(cudaFreeAsync(p, stream));
      cap = bytes + (bytes >> 1);
      AB_CUDA(cudaMallocAsync(&p, cap, stream));
    }
    return p;
  }
};
static Scratch g_scratch[16];

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
    AB_REQUIRE(mode >= 0 && mode <= 3, AB_ERR_CONFIG, "unknown advantage mode");
    AB_REQUIRE(device >= 0 && device < 16, AB_ERR_CONFIG, "device index out of range");
    if (n_groups == 0) return AB_OK;
    AB_CUDA(cudaSetDevice(device));
    const size_t n = (size_t)n_groups * group_size;
    const bool dev_in = is_device_ptr(rewards), dev_out = is_device_ptr(adv);
    const bool dev_flags = zero_std_flags == nullptr || is_device_ptr(zero_std_flags);
    // host arrays are staged through one reusable device buffer: [rewards | advantages | flags]
    ab::Scratch& sc = ab::g_scratch[device];
    std::lock_guard<std::mutex> lock(sc.mu);
    uint8_t* scratch = (uint8_t*)sc.get(2 * n * sizeof(double) + n_groups * sizeof(int32_t));
    cudaStream_t st = sc.stream;
    const double* dr = dev_in ? rewards : (const double*)scratch;
    double* da = dev_out ? adv : (double*)(scratch + n * sizeof(double));
    int32_t* df = dev_flags ? zero_std_flags : (int32_t*)(scratch + 2 * n * sizeof(double));
    if (!dev_in) AB_CUDA(cudaMemcpyAsync((void*)dr, rewards, n * sizeof(double), cudaMemcpyHostToDevice, st));
    ab::k_group_advantages<<<ab::ceil_div(n_groups, 128), 128, 0, st>>>(dr, n_groups, group_size, mode, eps, da, df);
    AB_CUDA(cudaGetLastError());
    if (!dev_out) AB_CUDA(cudaMemcpyAsync(adv, da, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (!dev_flags)
      AB_CUDA(cudaMemcpyAsync(zero_std_flags, df, n_groups * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    AB_CUDA(cudaStreamSynchronize(st));
    return AB_OK;
  } catch (const ab::Error& e) {
    ab::set_last_error(e.what());
    return e.code;
  }
}

extern "C" int ab_clipped_ratio_terms(const double* logp_now, const double* logp_beh, const int64_t* offs, int n,
                                      const double* adv, double eps_clip, double eps_clip_high, int sequence_level,
                                      double* ratios, int32_t* clipped, double* surrogate, int device) {
  try {
    AB_REQUIRE(n >= 0 && offs != nullptr, AB_ERR_CONTRACT, "clipped ratio: bad arguments");
    AB_REQUIRE(device >= 0 && device < 16, AB_ERR_CONFIG, "device index out of range");
    if (n == 0) return AB_OK;
    const int64_t T = offs[n];
    for (int k = 0; k < n; ++k) AB_REQUIRE(offs[k] <= offs[k + 1], AB_ERR_CONTRACT, "offsets must not decrease");
    AB_CUDA(cudaSetDevice(device));
    const int64_t nr = sequence_level ? n : T;
    // host in / host out through one reusable device buffer
    const size_t bytes = (size_t)(2 * T + n) * 8 + (size_t)(n + 1) * 8 + (size_t)nr * 12 + (size_t)n * 8;
    ab::Scratch& sc = ab::g_scratch[device];
    std::lock_guard<std::mutex> lock(sc.mu);
    uint8_t* p = (uint8_t*)sc.get(bytes);
    cudaStream_t st = sc.stream;
    double* d_now = (double*)p;
    double* d_beh = d_now + T;
    double* d_adv = d_beh + T;
    int64_t* d_offs = (int64_t*)(d_adv + n);
    double* d_rat = (double*)(d_offs + n + 1);
    double* d_sur = d_rat + nr;
    int32_t* d_clip = (int32_t*)(d_sur + n);
    if (T) {
      AB_CUDA(cudaMemcpyAsync(d_now, logp_now, T * 8, cudaMemcpyHostToDevice, st));
      AB_CUDA(cudaMemcpyAsync(d_beh, logp_beh, T * 8, cudaMemcpyHostToDevice, st));
    }
    AB_CUDA(cudaMemcpyAsync(d_adv, adv, n * 8, cudaMemcpyHostToDevice, st));
    AB_CUDA(cudaMemcpyAsync(d_offs, offs, (n + 1) * 8, cudaMemcpyHostToDevice, st));
    ab::k_clipped_ratio<<<ab::ceil_div(n, 8), 256, 0, st>>>(d_now, d_beh, d_offs, n, d_adv, 1.0 - eps_clip,
                                                            1.0 + eps_clip_high, sequence_level, d_rat, d_clip,
                                                            d_sur);
    AB_CUDA(cudaGetLastError());
    if (nr) {
      AB_CUDA(cudaMemcpyAsync(ratios, d_rat, nr * 8, cudaMemcpyDeviceToHost, st));
      AB_CUDA(cudaMemcpyAsync(clipped, d_clip, nr * 4, cudaMemcpyDeviceToHost, st));
    }
    AB_CUDA(cudaMemcpyAsync(surrogate, d_sur, n * 8, cudaMemcpyDeviceToHost, st));
    AB_CUDA(cudaStreamSynchronize(st));
    return AB_OK;
  } catch (const ab::Error& e) {
    ab::set_last_error(e.what());
    return e.code;
  }
}
