// K1 (transformer path): fused sampler over the lm_head logits.
//
// One CTA per live row.  A single pass over the row keeps, per thread and
// for a fixed contiguous chunk of the vocabulary, an online (max, sum of
// 2^((z - max) * invT * log2 e)) pair; a block reduction gives the row max
// M and the fp64 partition sum S (chunk sums rescaled to M, in fixed chunk
// order, so the result is deterministic).  The Philox draw u at position =
// generated tokens selects the first index whose running sum exceeds u*S
// (index-order inverse CDF, SURVEY.md Appendix A.7 / policy.py:93-94): a block
// exclusive scan over chunk sums finds the owning chunk and one thread rescans
// it.  Greedy = argmax, lowest index on ties.  logp = (z_tok - M)*invT - ln S.
// The epilogue is the engine's growth step (engine.py:274-289 semantics):
// payload write, gen += 1, stop rules (trace length, or EOS then l_max).
#include <cfloat>

#include "model.cuh"

namespace ab {

namespace {

constexpr int kSampThreads = 1024;
constexpr float kLog2e = 1.4426950408889634f;
constexpr double kLn2 = 0.6931471805599453;

__global__ void __launch_bounds__(kSampThreads) k_sample(EngineDev e, ModelDev m, const float* __restrict__ logits,
                                                         float inv_temp, int greedy) {
  Ctl* c = e.ctl;
  if (c->stop) return;
  const int i = blockIdx.x;
  if (i >= c->b) return;
  const int V = m.V;
  const float* z = logits + (size_t)i * V;
  const int cs = ((V + kSampThreads - 1) / kSampThreads + 3) & ~3;
  const int b0 = min(V, (int)threadIdx.x * cs), b1 = min(V, b0 + cs);
  const float k2 = inv_temp * kLog2e;

  // pass 1: online max / scaled sum over this thread's chunk, plus argmax
  float mx = -FLT_MAX;
  int am = 0x7fffffff;
  double sum = 0.0;  // sum of 2^((z - mx) * k2)
  for (int j = b0; j < b1; j += 4) {
    float4 v;
    if (j + 4 <= b1) {
      v = *reinterpret_cast<const float4*>(z + j);
    } else {
      v.x = z[j];
      v.y = j + 1 < b1 ? z[j + 1] : -FLT_MAX;
      v.z = j + 2 < b1 ? z[j + 2] : -FLT_MAX;
      v.w = j + 3 < b1 ? z[j + 3] : -FLT_MAX;
    }
    const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (j + q >= b1) break;
      const float x = vv[q];
      if (x > mx) {
        sum = sum * (double)exp2f((mx - x) * k2);
        mx = x;
        am = j + q;
      }
      sum += (double)exp2f((x - mx) * k2);
    }
  }
  // block max + lowest argmax
  __shared__ float s_m[32];
  __shared__ int s_a[32];
  __shared__ double s_d[32];
  __shared__ float s_M;
  __shared__ int s_tok;
  __shared__ double s_S, s_target;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float wm = mx;
  int wa = am;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, wm, o);
    const int oa = __shfl_xor_sync(0xffffffffu, wa, o);
    if (om > wm || (om == wm && oa < wa)) {
      wm = om;
      wa = oa;
    }
  }
  if (lane == 0) {
    s_m[w] = wm;
    s_a[w] = wa;
  }
  __syncthreads();
  if (w == 0) {
    wm = s_m[lane];
    wa = s_a[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, wm, o);
      const int oa = __shfl_xor_sync(0xffffffffu, wa, o);
      if (om > wm || (om == wm && oa < wa)) {
        wm = om;
        wa = oa;
      }
    }
    if (lane == 0) {
      s_M = wm;
      s_tok = wa;
    }
  }
  __syncthreads();
  const float M = s_M;
  // chunk sum rescaled to the row max; block exclusive scan in fixed order
  const double mine = (b0 < b1 && mx > -FLT_MAX) ? sum * (double)exp2f((mx - M) * k2) : 0.0;
  double incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_d[w] = incl;
  __syncthreads();
  if (w == 0) {
    double v = s_d[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    s_d[lane] = v;
    if (lane == 31) s_S = v;
  }
  __syncthreads();
  const double prefix = (w ? s_d[w - 1] : 0.0) + incl - mine;
  const double S = s_S;
  const int h = e.slot_handle[i];
  const int g = e.h_gen[h];
  if (!greedy) {
    if (threadIdx.x == 0) {
      const ulonglong2 k = e.h_key[h];
      s_target = philox_uniform(k.x, k.y, (uint64_t)g) * S;
      s_tok = -1;
    }
    __syncthreads();
    const double target = s_target;
    if (mine > 0.0 && prefix <= target && target < prefix + mine) {
      double run = prefix;
      int tok = b1 - 1;
      for (int j = b0; j < b1; ++j) {
        run += (double)exp2f((z[j] - M) * k2);
        if (run > target) {
          tok = j;
          break;
        }
      }
      s_tok = tok;
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_tok < 0) {  // u*S rounded past the last chunk: last token with mass
      int t = V - 1;
      while (t > 0 && z[t] == -FLT_MAX) --t;
      s_tok = t;
    }
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  const int tok = s_tok;
  const double logp = (double)((z[tok] - M) * inv_temp) - log2(S) * kLn2;
  if (e.record) {
    e.h_tokens[(size_t)h * e.L + g] = tok;
    e.h_logp[(size_t)h * e.L + g] = logp;
  }
  const int g1 = g + 1;
  e.h_gen[h] = g1;
  m.h_ctx[h] += 1;
  m.h_last_tok[h] = tok;
  int reason = -1;
  if (e.stop_mode == AB_STOP_TRACE) {
    const int stop_at = e.h_stop[h];
    if (g1 == stop_at) reason = stop_at >= e.l_max ? AB_REASON_MAX_LENGTH : AB_REASON_TARGET_LENGTH;
  } else {
    bool eos = false;
    for (int k = 0; k < e.n_eos; ++k) eos |= (tok == e.eos[k]);
    if (eos)
      reason = AB_REASON_STOP_TOKEN;
    else if (g1 >= e.l_max)
      reason = AB_REASON_MAX_LENGTH;
  }
  e.slot_token[i] = tok;
  e.slot_finish[i] = reason + 1;
}

}  // namespace

void launch_sampler(const EngineDev& e, const ModelDev& m, const float* logits, float inv_temp, int greedy,
                    float top_p, cudaStream_t s) {
  AB_REQUIRE(top_p >= 1.f, AB_ERR_CONFIG, "top_p < 1 is not supported by this build");
  k_sample<<<e.S, kSampThreads, 0, s>>>(e, m, logits, inv_temp, greedy);
}

}  // namespace ab
