// K1 (transformer path): fused sampler over the lm_head logits.
//
// Two paths share the row rule.  Temperature / greedy (top_p = 1, the decode default) runs two
// kernels: `k_sample_pieces` splits every row into fixed 1024-logit pieces, one warp per piece, so
// all SMs stream the logits whatever the live batch (a persistent grid of warps pulls (row, piece)
// items and writes each piece's (max, argmax, sum of 2^((z - max) * k2))), then `k_sample_finish`
// (one warp per row) combines the row in fixed piece order and finishes it (draw, owning-piece
// rescan, growth step).  Piece boundaries do not depend on the batch size, so a row's result does
// not either.  `k_sample` below (nucleus top_p < 1) keeps one CTA per row:
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
  const bool vec_ok = (V & 3) == 0;  // rows 16-byte aligned: float4 loads
  for (int j = b0; j < b1; j += 4) {
    float4 v;
    if (vec_ok && j + 4 <= b1) {
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

// ---------------------------------------------------------------------------------------------
// split sampler (top_p = 1)

constexpr int kPiece = 1024;        // logits per piece: one warp, 8 float4 per lane
constexpr int kSplitWarps = 8;      // warps per CTA
constexpr int kSplitCtasPerSm = 4;

__device__ __forceinline__ void am_merge(float& m, int& a, float om, int oa) {
  if (om > m || (om == m && oa < a)) {
    m = om;
    a = oa;
  }
}

// The growth step of the engine (engine.py:274-289 semantics) for live row i: payload write,
// gen += 1, stop rules (trace length, or EOS then l_max).
__device__ __forceinline__ void grow_row(const EngineDev& e, const ModelDev& m, int i, int h, int g, int tok,
                                        double logp) {
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

struct SplitDebug {  // test entry: caller rows / draws / outputs instead of the engine
  int rows;
  const double* u;
  int* tok;
  double* logp;
};

// One warp combines a row from its P piece partials (fixed piece order: deterministic) and returns
// the token / logp on every lane.  target = u * S selects the first index whose running mass
// exceeds it: the owning piece is found from the piece sums, then that piece (1024 logits, L2
// resident) is reloaded in one round (8 float4 per lane, the pass-1 layout: element
// 128 k + 4 lane + q) and located with per-tile lane sums, tile totals and one warp scan.
constexpr int kMaxPpl = 8;  // pieces per lane: P <= 256 (V <= 262,144)
// draw(): the row's uniform (Philox at the current position, or the test's); evaluated after the
// partial loads are issued so its dependent loads and the Philox rounds overlap them
template <typename Draw>
__device__ void split_finish_row(const float* __restrict__ z, int V, int P, const float4* __restrict__ part,
                                 float k2, float inv_temp, int greedy, Draw draw, int& tok, double& logp) {
  const int lane = threadIdx.x & 31;
  const int ppl = (P + 31) / 32;  // pieces per lane (contiguous)
  const int p0 = lane * ppl;
  float pm[kMaxPpl];
  int pa[kMaxPpl];
  double ps[kMaxPpl];
#pragma unroll
  for (int t = 0; t < kMaxPpl; ++t) {
    pm[t] = -FLT_MAX;
    pa[t] = 0x7fffffff;
    ps[t] = 0.0;
    if (t < ppl && p0 + t < P) {
      const float4 q = __ldcg(part + p0 + t);
      pm[t] = q.x;
      pa[t] = __float_as_int(q.y);
      ps[t] = __hiloint2double(__float_as_int(q.w), __float_as_int(q.z));
    }
  }
  const double u = draw();
  float M = -FLT_MAX;
  int A = 0x7fffffff;
#pragma unroll
  for (int t = 0; t < kMaxPpl; ++t) am_merge(M, A, pm[t], pa[t]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) am_merge(M, A, __shfl_xor_sync(0xffffffffu, M, o), __shfl_xor_sync(0xffffffffu, A, o));
  double mine = 0.0;
#pragma unroll
  for (int t = 0; t < kMaxPpl; ++t) {
    ps[t] = pm[t] > -FLT_MAX ? ps[t] * (double)exp2f((pm[t] - M) * k2) : 0.0;  // rescaled to the row max
    mine += ps[t];
  }
  double incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const double S = __shfl_sync(0xffffffffu, incl, 31);
  tok = A;
  if (!greedy) {
    const double target = u * S;
    const double before = incl - mine;
    const unsigned own = __ballot_sync(0xffffffffu, mine > 0.0 && before <= target && target < incl);
    int piece = -1;
    double base = 0.0;
    if (own) {
      const int ol = __ffs(own) - 1;
      double run = before, pb = 0.0;
      int pc = -1;
#pragma unroll
      for (int t = 0; t < kMaxPpl; ++t) {
        if (pc >= 0 && run > target) break;  // (found in an earlier piece)
        if (ps[t] > 0.0) {
          pc = p0 + t;  // (rounding: the last massive piece of the lane)
          pb = run;
        }
        run += ps[t];
      }
      piece = __shfl_sync(0xffffffffu, pc, ol);
      base = __shfl_sync(0xffffffffu, pb, ol);
    }
    int found = -1;
    if (piece >= 0) {
      const int j0 = piece * kPiece, j1 = min(V, j0 + kPiece);
      float x[32];
#pragma unroll
      for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = j0 + 4 * (lane + 32 * k) + q;
          x[4 * k + q] = j < j1 ? __ldcg(z + j) : -FLT_MAX;
        }
      double ls[8];  // this lane's mass in tile k (elements 128 k + 4 lane + q)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        ls[k] = 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (x[4 * k + q] > -FLT_MAX) ls[k] += (double)exp2f((x[4 * k + q] - M) * k2);
      }
      double tt[8];  // tile totals (fixed xor tree)
#pragma unroll
      for (int k = 0; k < 8; ++k) tt[k] = ls[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int k = 0; k < 8; ++k) tt[k] += __shfl_xor_sync(0xffffffffu, tt[k], o);
      int kt = -1;
      double tb = base;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (kt < 0 && tt[k] > 0.0) {
          if (tb + tt[k] > target) kt = k;
          else tb += tt[k];
        }
      }
      int last = -1;
      if (kt < 0) {  // u * S rounded past the piece: its last index with mass
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (x[4 * k + q] > -FLT_MAX) last = max(last, j0 + 4 * (lane + 32 * k) + q);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
        found = last;
      } else {
        double lsk = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k == kt) lsk = ls[k];
        double li = lsk;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double y = __shfl_up_sync(0xffffffffu, li, o);
          if (lane >= o) li += y;
        }
        const unsigned hit = __ballot_sync(0xffffffffu, lsk > 0.0 && tb + li > target);
        const int hl = hit ? __ffs(hit) - 1 : 31;
        int fq = -1;
        if (lane == hl) {
          double run = tb + li - lsk;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (k == kt)
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float xv = x[4 * k + q];
                if (xv <= -FLT_MAX || fq >= 0 && run > target) continue;
                run += (double)exp2f((xv - M) * k2);
                fq = j0 + 4 * (lane + 32 * k) + q;  // the first index whose running mass exceeds target
              }
        }
        found = __shfl_sync(0xffffffffu, fq, hl);
      }
    }
    if (found < 0) {  // u * S rounded past every piece: the last token with mass
      int t = V - 1;
      while (t > 0 && z[t] == -FLT_MAX) --t;
      found = t;
    }
    tok = found;
  }
  logp = (double)((__ldcg(z + tok) - M) * inv_temp) - log2(S) * kLn2;
}

// Pass 1: a persistent grid of warps streams (row, piece) items: per piece its max, lowest argmax
// and fp64 sum of 2^((z - max) * k2) (8 float4 per lane, one coalesced 4 KB read), written to
// part[row][piece].  No fences or atomics on the streaming path: pass 2 is the next kernel.
__global__ void __launch_bounds__(kSplitWarps * 32, kSplitCtasPerSm)
    k_sample_pieces(const Ctl* __restrict__ ctl, int dbg_rows, const float* __restrict__ logits, int V, float inv_temp,
                    float4* __restrict__ part) {
  pdl_wait();
  int b;
  if (ctl) {
    if (ctl->stop) return;
    b = ctl->b;
  } else {
    b = dbg_rows;
  }
  pdl_launch();  // pass 2 launches and waits for this grid
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int P = (V + kPiece - 1) / kPiece;
  const float k2 = inv_temp * kLog2e;
  const int items = b * P;
  const bool vec_ok = (V & 3) == 0;  // rows 16-byte aligned: float4 loads
  for (int it = (int)blockIdx.x * kSplitWarps + w; it < items; it += (int)gridDim.x * kSplitWarps) {
    const int row = it / P, piece = it - row * P;
    const float* z = logits + (size_t)row * V;
    const int j0 = piece * kPiece, j1 = min(V, j0 + kPiece);
    float x[32];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int j = j0 + 4 * (lane + 32 * k);
      if (vec_ok && j + 4 <= j1) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(z + j));
        x[4 * k] = v.x;
        x[4 * k + 1] = v.y;
        x[4 * k + 2] = v.z;
        x[4 * k + 3] = v.w;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) x[4 * k + q] = j + q < j1 ? z[j + q] : -FLT_MAX;
      }
    }
    float mx = -FLT_MAX;
    int am = 0x7fffffff;
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (x[4 * k + q] > mx) {  // strictly greater: the lowest index of a lane wins ties
          mx = x[4 * k + q];
          am = j0 + 4 * (lane + 32 * k) + q;
        }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) am_merge(mx, am, __shfl_xor_sync(0xffffffffu, mx, o), __shfl_xor_sync(0xffffffffu, am, o));
    // lane sum in fp32 over 32 values (each <= 1), then fp64 across lanes (fixed xor tree)
    float fs = 0.f;
    if (mx > -FLT_MAX) {
#pragma unroll
      for (int k = 0; k < 32; ++k)
        if (x[k] > -FLT_MAX) fs += exp2f((x[k] - mx) * k2);
    }
    double sum = (double)fs;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0)
      part[(size_t)row * P + piece] =
          make_float4(mx, __int_as_float(am), __int_as_float(__double2loint(sum)), __int_as_float(__double2hiint(sum)));
  }
}

// Pass 2: one warp per live row combines its piece partials in fixed order, draws, rescans the
// owning piece and runs the growth step (engine) or writes the test outputs.
__global__ void __launch_bounds__(256) k_sample_finish(EngineDev e, ModelDev m, const float* __restrict__ logits,
                                                      int V, float inv_temp, int greedy,
                                                      const float4* __restrict__ part, SplitDebug dbg) {
  pdl_wait();
  int b;
  if (dbg.tok) {
    b = dbg.rows;
  } else {
    const Ctl* c = e.ctl;
    if (c->stop) return;
    b = c->b;
  }
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= b) return;
  const int P = (V + kPiece - 1) / kPiece;
  const float k2 = inv_temp * kLog2e;
  int h = -1, g = 0;
  auto draw = [&]() -> double {
    if (dbg.tok) return dbg.u[row];
    h = e.slot_handle[row];
    g = e.h_gen[h];
    if (greedy) return 0.0;
    const ulonglong2 key = e.h_key[h];
    return philox_uniform(key.x, key.y, (uint64_t)g);
  };
  int tok;
  double logp;
  split_finish_row(logits + (size_t)row * V, V, P, part + (size_t)row * P, k2, inv_temp, greedy, draw, tok, logp);
  if (lane != 0) return;
  if (dbg.tok) {
    dbg.tok[row] = tok;
    dbg.logp[row] = logp;
  } else {
    grow_row(e, m, row, h, g, tok, logp);
  }
}

int split_grid() {
  static int grid = 0;
  if (!grid) {
    int dev = 0, sms = 0;
    AB_CUDA(cudaGetDevice(&dev));
    AB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    grid = sms * kSplitCtasPerSm;
  }
  return grid;
}

}  // namespace

size_t sampler_scratch_bytes(int rows, int V) { return (size_t)rows * ((V + kPiece - 1) / kPiece) * sizeof(float4); }

bool sampler_uses_split(int greedy, float top_p) { return greedy || top_p >= 1.f; }

void launch_sampler(const EngineDev& e, const ModelDev& m, const float* logits, float inv_temp, int greedy,
                    float top_p, void* part, cudaStream_t s) {
  AB_REQUIRE(top_p > 0.f && top_p <= 1.f, AB_ERR_CONFIG, "top_p must lie in (0, 1]");
  if (sampler_uses_split(greedy, top_p)) {
    SplitDebug no{0, nullptr, nullptr, nullptr};
    launch_pdl(k_sample_pieces, dim3(split_grid()), dim3(kSplitWarps * 32), 0, s, (const Ctl*)e.ctl, 0, logits, m.V,
               inv_temp, (float4*)part);
    launch_pdl(k_sample_finish, dim3(ceil_div(e.S, 8)), dim3(256), 0, s, e, m, logits, m.V, inv_temp, greedy,
               (const float4*)part, no);
  } else {
    launch_pdl(k_sample, dim3(e.S), dim3(kSampThreads), 0, s, e, m, logits, inv_temp, greedy, top_p);
  }
}

}  // namespace ab

// Test entry: the fused sampler's per-row routine on device buffers (logits [rows, V] fp32,
// draws u [rows] fp64) -> token [rows] int32, logp [rows] fp64.
extern "C" int ab_debug_sample_rows(const float* logits, int rows, int V, float temperature, int greedy, float top_p,
                                    const double* u, int* tok, double* logp) {
  try {
    AB_REQUIRE(top_p > 0.f && top_p <= 1.f, AB_ERR_CONFIG, "top_p must lie in (0, 1]");
    const float inv_temp = temperature > 0.f ? 1.f / temperature : 1.f;
    if (rows <= 0) return AB_OK;
    if (ab::sampler_uses_split(greedy, top_p)) {
      // the decode path's split kernel (fixed 1024-logit pieces) on caller rows
      void* part = nullptr;
      AB_CUDA(cudaMalloc(&part, ab::sampler_scratch_bytes(rows, V)));
      ab::SplitDebug dbg{rows, u, tok, logp};
      ab::EngineDev e{};
      ab::ModelDev m{};
      ab::k_sample_pieces<<<ab::split_grid(), ab::kSplitWarps * 32>>>(nullptr, rows, logits, V, inv_temp,
                                                                      (float4*)part);
      ab::k_sample_finish<<<ab::ceil_div(rows, 8), 256>>>(e, m, logits, V, inv_temp, greedy, (const float4*)part,
                                                           dbg);
      AB_CUDA(cudaGetLastError());
      AB_CUDA(cudaDeviceSynchronize());
      cudaFree(part);
    } else {
      ab::k_sample_rows<<<rows, ab::kSampThreads>>>(logits, V, inv_temp, greedy, top_p, u, tok, logp);
      AB_CUDA(cudaGetLastError());
      AB_CUDA(cudaDeviceSynchronize());
    }
    return AB_OK;
  } catch (const ab::Error& e) {
    ab::set_last_error(e.what());
    return e.code;
  }
}
