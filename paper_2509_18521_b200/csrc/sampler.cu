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
constexpr double kMassScale = 1099511627776.0;  // 2^40: fixed-point token mass for the nucleus search
constexpr int kHistCopies = 8;

// Monotone map float -> uint32 (larger logit <=> larger key).
__device__ __forceinline__ uint32_t fkey(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

struct RowSmem {
  float m[32];
  int a[32];
  double d[32];
  float M;
  int tok;
  double S, target;
  unsigned long long hist[kHistCopies][256];  // radix histograms (nucleus search), one per 4 warps
  unsigned long long tot;
  uint32_t prefix;
  unsigned long long remaining;
};

// One row of the fused sampler, executed by the whole CTA (kSampThreads threads).
// Pass 1: per-thread online (max, sum of 2^((z - max) * k2)) over a fixed contiguous chunk of
// the vocabulary + argmax (lowest index on ties); block max; chunk sums rescaled to the row max
// and combined by a fixed-order block scan (fp64): deterministic.
// top_p < 1 (nucleus): the kept set is every token whose logit is >= the largest threshold
// z* with  mass{z >= z*} >= top_p * mass(all); it is found exactly by a 4-pass radix select on
// the orderable key of the logit, weighting each token by its fixed-point mass
// floor(2^((z - max) * k2) * 2^40) (integer atomics: order independent).  The draw u then
// selects the first kept index whose running kept mass exceeds u * S_kept (index-order inverse
// CDF), and logp is the log-probability under the truncated
// distribution.  Greedy = argmax (always in the nucleus).  Returns the token on thread 0 (and
// in sm.tok) and its logp on thread 0.
__device__ void sample_row(const float* __restrict__ z, int V, float inv_temp, int greedy, float top_p, double u,
                           RowSmem& sm, int& tok_out, double& logp_out) {
  const int cs = ((V + kSampThreads - 1) / kSampThreads + 3) & ~3;
  const int b0 = min(V, (int)threadIdx.x * cs), b1 = min(V, b0 + cs);
  const float k2 = inv_temp * kLog2e;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;

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
    sm.m[w] = wm;
    sm.a[w] = wa;
  }
  __syncthreads();
  if (w == 0) {
    wm = sm.m[lane];
    wa = sm.a[lane];
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
      sm.M = wm;
      sm.tok = wa;
    }
  }
  __syncthreads();
  const float M = sm.M;
  const bool nucleus = !greedy && top_p < 1.f;
  uint32_t kmin = 0;  // kept: fkey(z) >= kmin
  if (nucleus) {
    // ---- exact nucleus threshold by radix select over the logit keys ----
    unsigned long long* hist = &sm.hist[w & (kHistCopies - 1)][0];
    uint32_t prefix = 0, pmask = 0;
    for (int pass = 0; pass < 4; ++pass) {
      const int shift = 24 - 8 * pass;
      for (int i = threadIdx.x; i < kHistCopies * 256; i += kSampThreads) (&sm.hist[0][0])[i] = 0ull;
      __syncthreads();
      for (int j = b0; j < b1; ++j) {
        const float x = z[j];
        const uint32_t key = fkey(x);
        if ((key & pmask) != prefix) continue;
        const unsigned long long q = (unsigned long long)((double)exp2f((x - M) * k2) * kMassScale);
        atomicAdd(&hist[(key >> shift) & 255], q);
      }
      __syncthreads();
      if (w == 0) {
        // bin totals over the warps (fixed order), then the top-down walk by lane 0
        for (int bin = lane; bin < 256; bin += 32) {
          unsigned long long t = 0ull;
          for (int ww = 0; ww < kHistCopies; ++ww) t += sm.hist[ww][bin];
          sm.hist[0][bin] = t;
        }
        __syncwarp();
        if (lane == 0) {
          if (pass == 0) {
            unsigned long long tot = 0ull;
            for (int bin = 0; bin < 256; ++bin) tot += sm.hist[0][bin];
            sm.tot = tot;
            sm.remaining = (unsigned long long)ceil((double)top_p * (double)tot);
            if (sm.remaining == 0ull) sm.remaining = 1ull;
          }
          unsigned long long cum = 0ull, rem = sm.remaining;
          int chosen = 0;
          for (int bin = 255; bin >= 0; --bin) {
            const unsigned long long h = sm.hist[0][bin];
            if (cum + h >= rem && h > 0ull) {
              chosen = bin;
              rem -= cum;
              break;
            }
            cum += h;
          }
          sm.remaining = rem;
          sm.prefix = prefix | ((uint32_t)chosen << shift);
        }
      }
      __syncthreads();
      prefix = sm.prefix;
      pmask |= 0xFFu << shift;
      __syncthreads();
    }
    kmin = prefix;
  }
  // chunk sums rescaled to the row max (nucleus: kept tokens only); block exclusive scan in fixed order
  double mine;
  if (!nucleus) {
    mine = (b0 < b1 && mx > -FLT_MAX) ? sum * (double)exp2f((mx - M) * k2) : 0.0;
  } else {
    mine = 0.0;
    for (int j = b0; j < b1; ++j)
      if (fkey(z[j]) >= kmin) mine += (double)exp2f((z[j] - M) * k2);
  }
  double incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) sm.d[w] = incl;
  __syncthreads();
  if (w == 0) {
    double v = sm.d[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    sm.d[lane] = v;
    if (lane == 31) sm.S = v;
  }
  __syncthreads();
  const double prefix_sum = (w ? sm.d[w - 1] : 0.0) + incl - mine;
  const double S = sm.S;
  if (!greedy) {
    if (threadIdx.x == 0) {
      sm.target = u * S;
      sm.tok = -1;
    }
    __syncthreads();
    const double target = sm.target;
    if (mine > 0.0 && prefix_sum <= target && target < prefix_sum + mine) {
      double run = prefix_sum;
      int t = -1, last_kept = -1;
      for (int j = b0; j < b1; ++j) {
        if (nucleus && fkey(z[j]) < kmin) continue;
        last_kept = j;
        run += (double)exp2f((z[j] - M) * k2);
        if (run > target) {
          t = j;
          break;
        }
      }
      sm.tok = t >= 0 ? t : last_kept;
    }
    __syncthreads();
    if (threadIdx.x == 0 && sm.tok < 0) {  // u*S rounded past the last chunk: last token with mass
      int t = V - 1;
      while (t > 0 && (z[t] == -FLT_MAX || (nucleus && fkey(z[t]) < kmin))) --t;
      sm.tok = t;
    }
    __syncthreads();
  }
  tok_out = sm.tok;
  logp_out = 0.0;
  if (threadIdx.x == 0) logp_out = (double)((z[tok_out] - M) * inv_temp) - log2(S) * kLn2;
}

__global__ void __launch_bounds__(kSampThreads) k_sample(EngineDev e, ModelDev m, const float* __restrict__ logits,
                                                         float inv_temp, int greedy, float top_p) {
  pdl_wait();
  // (no early launch_dependents: the successor pre-launches when this grid drains)
  Ctl* c = e.ctl;
  if (c->stop) return;
  const int i = blockIdx.x;
  if (i >= c->b) return;
  __shared__ RowSmem sm;
  const int h = e.slot_handle[i];
  const int g = e.h_gen[h];
  double u = 0.0;
  if (!greedy) {
    const ulonglong2 k = e.h_key[h];
    u = philox_uniform(k.x, k.y, (uint64_t)g);
  }
  int tok;
  double logp;
  sample_row(logits + (size_t)i * m.V, m.V, inv_temp, greedy, top_p, u, sm, tok, logp);
  if (threadIdx.x != 0) return;
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

// Test entry kernel: the same per-row routine on caller-provided logits and draws.
__global__ void __launch_bounds__(kSampThreads) k_sample_rows(const float* __restrict__ logits, int V,
                                                               float inv_temp, int greedy, float top_p,
                                                               const double* __restrict__ u, int* __restrict__ tok,
                                                               double* __restrict__ logp) {
  __shared__ RowSmem sm;
  int t;
  double lp;
  sample_row(logits + (size_t)blockIdx.x * V, V, inv_temp, greedy, top_p, u[blockIdx.x], sm, t, lp);
  if (threadIdx.x == 0) {
    tok[blockIdx.x] = t;
    logp[blockIdx.x] = lp;
  }
}

}  // namespace

void launch_sampler(const EngineDev& e, const ModelDev& m, const float* logits, float inv_temp, int greedy,
                    float top_p, cudaStream_t s) {
  AB_REQUIRE(top_p > 0.f && top_p <= 1.f, AB_ERR_CONFIG, "top_p must lie in (0, 1]");
  launch_pdl(k_sample, dim3(e.S), dim3(kSampThreads), 0, s, e, m, logits, inv_temp, greedy, top_p);
}

}  // namespace ab

// Test entry: the fused sampler's per-row routine on device buffers (logits [rows, V] fp32,
// draws u [rows] fp64) -> token [rows] int32, logp [rows] fp64.
extern "C" int ab_debug_sample_rows(const float* logits, int rows, int V, float temperature, int greedy, float top_p,
                                    const double* u, int* tok, double* logp) {
  try {
    AB_REQUIRE(top_p > 0.f && top_p <= 1.f, AB_ERR_CONFIG, "top_p must lie in (0, 1]");
    const float inv_temp = temperature > 0.f ? 1.f / temperature : 1.f;
    ab::k_sample_rows<<<rows, ab::kSampThreads>>>(logits, V, inv_temp, greedy, top_p, u, tok, logp);
    AB_CUDA(cudaGetLastError());
    AB_CUDA(cudaDeviceSynchronize());
    return AB_OK;
  } catch (const ab::Error& e) {
    ab::set_last_error(e.what());
    return e.code;
  }
}
