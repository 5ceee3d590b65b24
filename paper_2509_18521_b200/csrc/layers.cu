// Decoder kernels around the tcgen05 GEMMs and the paged attention
// (attention.cu): weight init, per-iteration row preparation + KV page
// allocation + attention work list, embedding, RMSNorm, q/k-norm + RoPE +
// paged KV write, causal prefill attention for prompt groups, and KV page
// management.
//
// None of this has a reference counterpart (the reference decode engine is a
// cost model, src/april_sim/engine.py:167-171); numerics are pinned by the
// torch-CPU oracle in oracle/cpu_model.py.
#include <cuda_bf16.h>

#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <map>
#include <mutex>

#include "model.cuh"

namespace ab {

namespace {

constexpr float kLog2e = 1.4426950408889634f;
__constant__ int c_pdl_mask = 6;  // see gemm.cu
__constant__ int c_rope_zero = 1;  // debug timing only (AB_ROPE_NOZERO): 0 skips the workspace re-zero

__device__ __forceinline__ bool stopped(const int* stop) { return stop != nullptr && *stop != 0; }

// ---------------------------------------------------------------------------
// weights
// ---------------------------------------------------------------------------

__global__ void k_init_weights(bf16* w, size_t n, uint64_t k0, uint64_t k1, float std, float constant, int mode) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    if (mode == 1) {
      w[i] = __float2bfloat16(constant);
      continue;
    }
    const uint64_t a = philox_word(k0, k1, 2 * i), b = philox_word(k0, k1, 2 * i + 1);
    const double u1 = ((double)(a >> 11) + 1.0) * 0x1.0p-53;  // (0, 1]
    const double u2 = (double)(b >> 11) * 0x1.0p-53;
    const double z = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    w[i] = __float2bfloat16((float)(z * std));
  }
}

__global__ void k_rope_table(float2* rope, int max_pos, int hd, float theta) {
  const int half = hd / 2;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < max_pos * half; idx += gridDim.x * blockDim.x) {
    const int p = idx / half, i = idx % half;
    const float inv = 1.0f / powf(theta, (float)(2 * i) / (float)hd);
    const float ang = (float)p * inv;
    float s, c;
    sincosf(ang, &s, &c);
    rope[idx] = make_float2(c, s);
  }
}

// ---------------------------------------------------------------------------
// per-iteration row preparation + KV page allocation
// ---------------------------------------------------------------------------

// Pop one page index off the free-page stack; on an empty stack fail WITHOUT side effects (the
// top never goes negative, so later releases push to valid slots and no page is lost).
__device__ __forceinline__ int pop_page(Ctl* c) {
  unsigned long long* top = reinterpret_cast<unsigned long long*>(&c->kv_free_top);
  long long cur = *reinterpret_cast<volatile long long*>(top);
  while (cur > 0) {
    const long long prev = (long long)atomicCAS(top, (unsigned long long)cur, (unsigned long long)(cur - 1));
    if (prev == cur) return (int)(cur - 1);
    cur = prev;
  }
  return -1;
}

// Push one page back (error paths: undo a pop whose allocation is abandoned).
__device__ __forceinline__ void push_page(Ctl* c, ModelDev& m, int page) {
  const long long base =
      (long long)atomicAdd(reinterpret_cast<unsigned long long*>(&c->kv_free_top), 1ull);
  m.free_pages[base] = page;
}

// Single block: per live row, gather (token, position, block-table row),
// allocate a KV page when the row crosses a page boundary, and build the
// attention work list (exclusive prefix of KV splits per row).
constexpr int kPrepThreads = 1024;
// attention work items per persistent CTA (dynamic cursor); AB_ATT_ITEMS overrides (tuning).
// Each item costs about one 64-token tile of DRAM time on top of its tiles (end-of-item merge with
// the stage held, start-up), so rows are split only when there are fewer (row, kv head) units
// than CTAs or a row is longer than its share: measured 1 vs 3 at the bench operating points,
// C2 +1.7 % (attention 0.85 -> 0.90 of the copy peak), C3 +1.6 % (0.93 -> 0.96).
__constant__ unsigned long long c_items_per_cta = 1;

// Per-iteration decode prologue: gather the live rows, allocate KV pages for the
// token about to be written, and build the attention work list.  The KV split
// size is picked here from the iteration's total context so that the work list
// has about 4 items per attention CTA (long rows split, short rows whole; the
// attention CTAs then pull items dynamically), never below `min_chunk` tokens.
__global__ void __launch_bounds__(kPrepThreads) k_prep_decode(EngineDev e, ModelDev m, int min_chunk, int att_ctas) {
  Ctl* c = e.ctl;
  if (c->stop) return;
  const int b = c->b;
  const int ipt = (b + kPrepThreads - 1) / kPrepThreads;
  const int beg = min(b, (int)threadIdx.x * ipt), end = min(b, beg + ipt);
  unsigned long long ctx_sum = 0;
  bool fail = false;
  int popped[4], n_popped = 0;  // ipt <= 4 (S <= 4096)
  for (int i = beg; i < end; ++i) {
    const int h = e.slot_handle[i];
    const int pos = m.h_ctx[h];
    m.row_tok[i] = m.h_last_tok[h];
    m.row_pos[i] = pos;
    m.row_btrow[i] = h;
    ctx_sum += (unsigned long long)(pos + 1);
    int page = 0;
    if (pos % m.P == 0) {
      const int idx = pos / m.P < m.MP ? pop_page(c) : -1;
      if (idx < 0) {
        fail = true;
      } else {
        page = m.free_pages[idx];
        m.bt[(size_t)h * m.MP + pos / m.P] = page;
        popped[n_popped++] = page;
      }
    } else {
      page = m.bt[(size_t)h * m.MP + pos / m.P];
    }
    m.row_pslot[i] = page * m.P + pos % m.P;  // KV page and slot of the token written this iteration
  }
  __shared__ int s_w[32];
  __shared__ unsigned long long s_u[32];
  __shared__ int s_chunk;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long cs = ctx_sum;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o);
  if (lane == 0) s_u[w] = cs;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long tot = 0;
    for (int k = 0; k < kPrepThreads / 32; ++k) tot += s_u[k];
    const unsigned long long ipc = c_items_per_cta;
    const unsigned long long per = (tot * (unsigned long long)m.hk + ipc * att_ctas - 1) / (ipc * att_ctas);
    int ch = (int)min(per, (unsigned long long)(1 << 30));
    ch = (ch + 63) & ~63;
    s_chunk = max(ch, min_chunk);
    m.att_ctl[0] = s_chunk;
  }
  for (int l = threadIdx.x; l < m.L; l += kPrepThreads) m.att_ctl[1 + l] = 0;  // per-layer item cursors
  __syncthreads();
  const int chunk = s_chunk;
  int nsp = 0;
  for (int i = beg; i < end; ++i) nsp += (m.row_pos[i] + chunk) / chunk;  // ceil((pos + 1) / chunk)
  // exclusive scan of split counts
  int x = nsp;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[w] = x;
  __syncthreads();
  if (w == 0) {
    int v = s_w[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    s_w[lane] = v;
  }
  __syncthreads();
  int run = (w ? s_w[w - 1] : 0) + x - nsp;
  for (int i = beg; i < end; ++i) {
    m.split_prefix[i] = run;
    const int ns = (m.row_pos[i] + chunk) / chunk;
    for (int s = 0; s < ns; ++s) m.att_items[run + s] = i | (s << 16);  // explicit (row, split) work list
    run += ns;
  }
  if (threadIdx.x == kPrepThreads - 1) m.split_prefix[b] = s_w[31];
  if (c->run_iters < e.it_cap && ctx_sum)
    atomicAdd(reinterpret_cast<unsigned long long*>(&e.it_ctx[c->run_iters]), ctx_sum);
  // out of pages: the iteration is abandoned (every later kernel sees stop), so the pages this
  // prep did pop go back to the stack (h_ctx did not advance; a retry pops them again)
  if (__syncthreads_or(fail)) {
    for (int k = 0; k < n_popped; ++k) push_page(c, m, popped[k]);
    if (threadIdx.x == 0) {
      atomicCAS(&c->error, kErrNone, kErrOutOfKV);
      c->stop = 1;
      c->stop_reason = -2;
    }
  }
}

// ---------------------------------------------------------------------------
// embedding / RMSNorm
// ---------------------------------------------------------------------------

__global__ void k_embed(ModelDev m, const bf16* __restrict__ emb, float* __restrict__ x, const int* rows_dev,
                        int rows_cap, const int* stop) {
  if (stopped(stop)) return;
  const int rows = rows_dev ? min(*rows_dev, rows_cap) : rows_cap;
  const int r = blockIdx.x;
  if (r >= rows) return;
  const bf16* src = emb + (size_t)m.row_tok[r] * m.d;
  float* dst = x + (size_t)r * m.d;
  for (int j = threadIdx.x * 8; j < m.d; j += blockDim.x * 8) {
    const uint4 v = *reinterpret_cast<const uint4*>(src + j);
    const bf16* b = reinterpret_cast<const bf16*>(&v);
    float4 lo = make_float4(__bfloat162float(b[0]), __bfloat162float(b[1]), __bfloat162float(b[2]),
                            __bfloat162float(b[3]));
    float4 hi = make_float4(__bfloat162float(b[4]), __bfloat162float(b[5]), __bfloat162float(b[6]),
                            __bfloat162float(b[7]));
    *reinterpret_cast<float4*>(dst + j) = lo;
    *reinterpret_cast<float4*>(dst + j + 4) = hi;
  }
}

// one warp per row: y = bf16(x * rsqrt(mean(x^2) + eps) * w)
__global__ void k_rmsnorm(const float* __restrict__ x, const bf16* __restrict__ w, bf16* __restrict__ out, int d,
                          float eps, const int* rows_dev, int rows_cap, const int* stop) {
  pdl_wait();
  // (no early launch_dependents: the successor pre-launches when this grid drains)
  if (stopped(stop)) return;
  const int rows = rows_dev ? min(*rows_dev, rows_cap) : rows_cap;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + warp;
  if (r >= rows) return;
  const float* xr = x + (size_t)r * d;
  float ss = 0.f;
  for (int j = lane * 4; j < d; j += 128) {
    const float4 v = *reinterpret_cast<const float4*>(xr + j);
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  ss = warp_sum(ss);
  const float rs = rsqrtf(ss / (float)d + eps);
  bf16* o = out + (size_t)r * d;
  for (int j = lane * 4; j < d; j += 128) {
    const float4 v = *reinterpret_cast<const float4*>(xr + j);
    o[j + 0] = __float2bfloat16(v.x * rs * __bfloat162float(w[j + 0]));
    o[j + 1] = __float2bfloat16(v.y * rs * __bfloat162float(w[j + 1]));
    o[j + 2] = __float2bfloat16(v.z * rs * __bfloat162float(w[j + 2]));
    o[j + 3] = __float2bfloat16(v.w * rs * __bfloat162float(w[j + 3]));
  }
}

// One warp per row, the whole row in registers (NV float4 per lane, d = 128 * NV): one
// coalesced read of x, 8-byte bf16 stores.  Same arithmetic as k_rmsnorm (fp32 sum of
// squares in the same per-lane order, warp_sum, x * rs * w rounded once to bf16).
template <int NV>
__global__ void __launch_bounds__(256) k_rmsnorm_v(const float* __restrict__ x, const bf16* __restrict__ w,
                                                   bf16* __restrict__ out, float eps, const int* rows_dev,
                                                   int rows_cap, const int* stop) {
  pdl_wait();
  if (c_pdl_mask & 4) pdl_launch();  // the next GEMM's CTAs start their prologue alongside
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + warp;
  if (r >= rows_cap) return;
  constexpr int D = NV * 128;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)r * D);
  const uint2* wv = reinterpret_cast<const uint2*>(w);
  float4 v[NV];
  uint2 wr[NV];
  // the row, the norm weights, the stop flag and the live row count are all loaded in one memory
  // round trip (the row is in bounds for any count <= rows_cap; it is discarded if not live)
  const int st = stop ? *stop : 0;
  const int rows = rows_dev ? *rows_dev : rows_cap;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    v[i] = xr[i * 32 + lane];
    wr[i] = __ldg(wv + i * 32 + lane);
  }
  if (st || r >= min(rows, rows_cap)) return;
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
  ss = warp_sum(ss);
  const float rs = rsqrtf(ss / (float)D + eps);
  uint2* o = reinterpret_cast<uint2*>(out + (size_t)r * D);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const uint2 ww = wr[i];
    const __nv_bfloat162 w01 = *reinterpret_cast<const __nv_bfloat162*>(&ww.x);
    const __nv_bfloat162 w23 = *reinterpret_cast<const __nv_bfloat162*>(&ww.y);
    const __nv_bfloat162 o01 = __floats2bfloat162_rn(v[i].x * rs * __low2float(w01), v[i].y * rs * __high2float(w01));
    const __nv_bfloat162 o23 = __floats2bfloat162_rn(v[i].z * rs * __low2float(w23), v[i].w * rs * __high2float(w23));
    uint2 ov;
    ov.x = *reinterpret_cast<const uint32_t*>(&o01);
    ov.y = *reinterpret_cast<const uint32_t*>(&o23);
    o[i * 32 + lane] = ov;
  }
}

// the GEMM's SwiGLU epilogue activation (gemm.cu silu), bit for bit
__device__ __forceinline__ float swiglu_silu(float x) { return __fdividef(x, 1.f + __expf(-x)); }

// SwiGLU over the gate-up reduce-add workspace: 128-column tile T holds gate features
// [64T, 64T + 64) in columns [128T, 128T + 64) and the matching up features in the next 64 (the
// interleaved weight layout).  h = bf16(silu(gate) * up), the same expression as the GEMM's SwiGLU
// epilogue; the consumed workspace is zeroed for the next reduce-add.
__global__ void __launch_bounds__(256) k_swiglu_ws(float* __restrict__ ws, bf16* __restrict__ h, int f,
                                                   const int* __restrict__ sched, const int* rows_dev, int rows_cap,
                                                   const int* stop) {
  pdl_wait();
  if (c_pdl_mask & 4) pdl_launch();
  if (stopped(stop)) return;
  const int rows = min(*rows_dev, rows_cap);
  if (rows <= 0 || sched[rows] == 0) return;  // the workspace plan did not run at this row count
  const int per_row = f / 4;                   // 4 features per thread
  const int64_t n = (int64_t)rows * per_row;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / per_row), j = (int)(i - (int64_t)r * per_row) * 4;
    float* g = ws + (size_t)r * 2 * f + (j >> 6) * 128 + (j & 63);
    const float4 gv = *reinterpret_cast<const float4*>(g);
    const float4 uv = *reinterpret_cast<const float4*>(g + 64);
    const float z[4] = {0.f, 0.f, 0.f, 0.f};
    *reinterpret_cast<float4*>(g) = *reinterpret_cast<const float4*>(z);
    *reinterpret_cast<float4*>(g + 64) = *reinterpret_cast<const float4*>(z);
    const __nv_bfloat162 o01 = __floats2bfloat162_rn(swiglu_silu(gv.x) * uv.x, swiglu_silu(gv.y) * uv.y);
    const __nv_bfloat162 o23 = __floats2bfloat162_rn(swiglu_silu(gv.z) * uv.z, swiglu_silu(gv.w) * uv.w);
    uint2 ov;
    ov.x = *reinterpret_cast<const uint32_t*>(&o01);
    ov.y = *reinterpret_cast<const uint32_t*>(&o23);
    *reinterpret_cast<uint2*>(h + (size_t)r * f + j) = ov;
  }
}

// ---------------------------------------------------------------------------
// q/k-norm + RoPE (rotate-half) + KV write into the row's page
// ---------------------------------------------------------------------------

// NP consecutive bf16 <-> fp32 (NP = 2: one 4-byte access)
template <int NP>
__device__ __forceinline__ void load_pairs(const bf16* p, float (&v)[NP]) {
  if constexpr (NP == 2) {
    const __nv_bfloat162 t = *reinterpret_cast<const __nv_bfloat162*>(p);
    v[0] = __low2float(t);
    v[1] = __high2float(t);
  } else {
#pragma unroll
    for (int j = 0; j < NP; ++j) v[j] = __bfloat162float(p[j]);
  }
}
template <int NP>
__device__ __forceinline__ void store_pairs(bf16* p, const float (&v)[NP]) {
  if constexpr (NP == 2) {
    *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(v[0], v[1]);
  } else {
#pragma unroll
    for (int j = 0; j < NP; ++j) p[j] = __float2bfloat16(v[j]);
  }
}

template <int HD>
__global__ void k_rope_kv(ModelDev m, int layer, const bf16* __restrict__ qkv, const bf16* __restrict__ qn,
                          const bf16* __restrict__ kn, bf16* __restrict__ qout, const int* rows_dev, int rows_cap,
                          const int* stop) {
  pdl_wait();
  // (no early launch_dependents: the successor pre-launches when this grid drains)
  if (stopped(stop)) return;
  const int rows = rows_dev ? min(*rows_dev, rows_cap) : rows_cap;
  const int r = blockIdx.x;
  if (r >= rows) return;
  constexpr int NP = HD / 64;  // rotation pairs per lane
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int pos = m.row_pos[r];
  const int page = m.bt[(size_t)m.row_btrow[r] * m.MP + pos / m.P], slot = pos % m.P;
  const float2* rp = m.rope + (size_t)pos * (HD / 2);
  const bf16* src = qkv + (size_t)r * m.qkv_dim;
  for (int head = warp + blockIdx.y * nw; head < m.hq + 2 * m.hk; head += nw * gridDim.y) {
    const bf16* hv = src + head * HD;
    float a[NP], b[NP];
    load_pairs<NP>(hv + lane * NP, a);
    load_pairs<NP>(hv + lane * NP + HD / 2, b);
    if (head >= m.hq + m.hk) {  // V: straight into the page
      const int kvh = head - m.hq - m.hk;
      bf16* dst = m.kv + m.kv_off(layer, page, 1, kvh, slot);
      store_pairs<NP>(dst + lane * NP, a);
      store_pairs<NP>(dst + lane * NP + HD / 2, b);
      continue;
    }
    const bool is_q = head < m.hq;
    if (m.qk_norm) {
      float ss = 0.f;
#pragma unroll
      for (int j = 0; j < NP; ++j) ss += a[j] * a[j] + b[j] * b[j];
      ss = warp_sum(ss);
      const float rs = rsqrtf(ss / (float)HD + m.eps);
      const bf16* nw_ = is_q ? qn : kn;
      float wa[NP], wb[NP];
      load_pairs<NP>(nw_ + lane * NP, wa);
      load_pairs<NP>(nw_ + lane * NP + HD / 2, wb);
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        a[j] = __bfloat162float(__float2bfloat16(a[j] * rs * wa[j]));
        b[j] = __bfloat162float(__float2bfloat16(b[j] * rs * wb[j]));
      }
    }
    float oa[NP], ob[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const float2 cs = rp[lane * NP + j];
      oa[j] = a[j] * cs.x - b[j] * cs.y;
      ob[j] = b[j] * cs.x + a[j] * cs.y;
    }
    bf16* dst = is_q ? qout + (size_t)r * m.qd + head * HD : m.kv + m.kv_off(layer, page, 0, head - m.hq, slot);
    store_pairs<NP>(dst + lane * NP, oa);
    store_pairs<NP>(dst + lane * NP + HD / 2, ob);
  }
}

// Decode variant: the QKV GEMM reduce-adds its fp32 accumulator into a zeroed workspace (so it can
// split K); this kernel adds the bias, rounds to bf16 exactly where the bf16 GEMM epilogue would
// have (bf16(acc + bias)), runs the same q/k-norm + RoPE + paged KV write, and zeroes the rows it
// consumed for the next layer's GEMM.
template <int HD>
__global__ void k_rope_kv_f32(ModelDev m, int layer, float* __restrict__ qkv, const bf16* __restrict__ bias,
                              const bf16* __restrict__ qn, const bf16* __restrict__ kn, bf16* __restrict__ qout,
                              const int* rows_dev, int rows_cap, const int* stop) {
  pdl_wait();
  // every per-row index is loaded up front in parallel (the prep kernel resolved the KV page)
  const int r = blockIdx.x;
  const int st = stop ? *stop : 0;
  const int rows = rows_dev ? min(*rows_dev, rows_cap) : rows_cap;
  const int pos = m.row_pos[r];
  const int ps = m.row_pslot[r];
  if (st || r >= rows) return;
  constexpr int NP = HD / 64;  // rotation pairs per lane
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int page = ps / m.P, slot = ps - page * m.P;
  const float2* rp = m.rope + (size_t)pos * (HD / 2);
  float* src = qkv + (size_t)r * m.qkv_dim;
  static_assert(NP == 1 || NP == 2, "rotation pairs per lane");
  for (int head = warp + blockIdx.y * nw; head < m.hq + 2 * m.hk; head += nw * gridDim.y) {
    // every load of the head is issued before any store (the zeroing stores would otherwise
    // order the rotation-table and norm-weight loads behind them: one memory round trip)
    const bool is_v = head >= m.hq + m.hk, is_q = head < m.hq;
    float* hv = src + head * HD;
    float* pa = hv + lane * NP;
    float* pb = hv + lane * NP + HD / 2;
    float a[NP], b[NP], ba[NP] = {}, bb[NP] = {}, wa[NP] = {}, wb[NP] = {};
    float2 cs[NP];
    if constexpr (NP == 2) {
      const float2 va = *reinterpret_cast<const float2*>(pa), vb = *reinterpret_cast<const float2*>(pb);
      a[0] = va.x;
      a[1] = va.y;
      b[0] = vb.x;
      b[1] = vb.y;
    } else {
      a[0] = *pa;
      b[0] = *pb;
    }
    if (bias) {
      load_pairs<NP>(bias + head * HD + lane * NP, ba);
      load_pairs<NP>(bias + head * HD + lane * NP + HD / 2, bb);
    }
#pragma unroll
    for (int j = 0; j < NP; ++j) cs[j] = __ldg(rp + lane * NP + j);  // (unconditional: issued with the rest)
    if (!is_v) {
      if (m.qk_norm) {
        const bf16* nw_ = is_q ? qn : kn;
        load_pairs<NP>(nw_ + lane * NP, wa);
        load_pairs<NP>(nw_ + lane * NP + HD / 2, wb);
      }
    }
    if (c_rope_zero) {
      if constexpr (NP == 2) {
        *reinterpret_cast<float2*>(pa) = make_float2(0.f, 0.f);
        *reinterpret_cast<float2*>(pb) = make_float2(0.f, 0.f);
      } else {
        *pa = 0.f;
        *pb = 0.f;
      }
    }
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      a[j] = __bfloat162float(__float2bfloat16(a[j] + ba[j]));
      b[j] = __bfloat162float(__float2bfloat16(b[j] + bb[j]));
    }
    if (is_v) {  // V: straight into the page
      const int kvh = head - m.hq - m.hk;
      bf16* dst = m.kv + m.kv_off(layer, page, 1, kvh, slot);
      store_pairs<NP>(dst + lane * NP, a);
      store_pairs<NP>(dst + lane * NP + HD / 2, b);
      continue;
    }
    if (m.qk_norm) {
      float ss = 0.f;
#pragma unroll
      for (int j = 0; j < NP; ++j) ss += a[j] * a[j] + b[j] * b[j];
      ss = warp_sum(ss);
      const float rs = rsqrtf(ss / (float)HD + m.eps);
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        a[j] = __bfloat162float(__float2bfloat16(a[j] * rs * wa[j]));
        b[j] = __bfloat162float(__float2bfloat16(b[j] * rs * wb[j]));
      }
    }
    float oa[NP], ob[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      oa[j] = a[j] * cs[j].x - b[j] * cs[j].y;
      ob[j] = b[j] * cs[j].x + a[j] * cs[j].y;
    }
    bf16* dst = is_q ? qout + (size_t)r * m.qd + head * HD : m.kv + m.kv_off(layer, page, 0, head - m.hq, slot);
    store_pairs<NP>(dst + lane * NP, oa);
    store_pairs<NP>(dst + lane * NP + HD / 2, ob);
  }
}

// ---------------------------------------------------------------------------
// page management
// ---------------------------------------------------------------------------

// fresh samples inherit their group's prompt pages; the partial tail page is copied
__global__ void k_fork_meta(EngineDev e, ModelDev m, const ab_sample_desc* descs, int n, int32_t* tail_src,
                            int32_t* tail_dst) {
  Ctl* c = e.ctl;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  tail_src[k] = -1;
  const ab_sample_desc s = descs[k];
  if (s.gen_len != 0) return;
  const int h = s.handle, g = s.group_slot;
  const int ctx = m.g_ctx[g];
  const int nfull = ctx / m.P;
  const int32_t* gb = m.bt + (size_t)(m.H + g) * m.MP;
  int32_t* hb = m.bt + (size_t)h * m.MP;
  for (int j = 0; j < nfull; ++j) hb[j] = gb[j];
  m.h_ctx[h] = ctx;
  m.h_last_tok[h] = m.g_last_tok[g];
  m.h_shared[h] = nfull;
  if (ctx % m.P) {
    const int idx = pop_page(c);
    if (idx < 0) {
      atomicCAS(&c->error, kErrNone, kErrOutOfKV);
      return;
    }
    hb[nfull] = m.free_pages[idx];
    tail_src[k] = gb[nfull];
    tail_dst[k] = hb[nfull];
  }
}

__global__ void k_fork_copy(ModelDev m, const int32_t* tail_src, const int32_t* tail_dst) {
  const int k = blockIdx.x, layer = blockIdx.y;
  const int src = tail_src[k];
  if (src < 0) return;
  const int dst = tail_dst[k];
  const size_t n = (size_t)2 * m.hk * m.P * m.hd / 8;  // uint4 chunks (K and V are adjacent)
  const uint4* s = reinterpret_cast<const uint4*>(m.kv + m.kv_off(layer, src, 0, 0, 0));
  uint4* d = reinterpret_cast<uint4*>(m.kv + m.kv_off(layer, dst, 0, 0, 0));
  for (size_t j = threadIdx.x; j < n; j += blockDim.x) d[j] = s[j];
}

// Re-prefill resume (§8 f1): a paused sample whose private KV was dropped at the abort
// re-forks its group's prompt pages (full pages shared, the partial tail page copied) and
// gets fresh pages for every position up to its context; the rows for positions
// g_ctx .. g_ctx + gen - 1 are then recomputed by the prefill pass.  items[k] = {handle,
// group slot, generated tokens, -}.
__global__ void k_resume_fork(EngineDev e, ModelDev m, const int4* items, int n, int32_t* tail_src,
                              int32_t* tail_dst) {
  Ctl* c = e.ctl;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  tail_src[k] = -1;
  const int4 it = items[k];
  const int h = it.x, g = it.y, gen = it.z;
  const int ctx_g = m.g_ctx[g];
  const int nfull = ctx_g / m.P;
  const int ctx = ctx_g + gen;
  const int need = (ctx + m.P - 1) / m.P;
  const int32_t* gb = m.bt + (size_t)(m.H + g) * m.MP;
  int32_t* hb = m.bt + (size_t)h * m.MP;
  for (int j = 0; j < nfull; ++j) hb[j] = gb[j];
  m.h_shared[h] = nfull;
  for (int j = nfull; j < need; ++j) {
    const int idx = j < m.MP ? pop_page(c) : -1;
    if (idx < 0) {
      atomicCAS(&c->error, kErrNone, kErrOutOfKV);
      m.h_ctx[h] = j * m.P;  // what is allocated, so a release frees exactly it
      return;
    }
    hb[j] = m.free_pages[idx];
  }
  m.h_ctx[h] = ctx;
  m.h_last_tok[h] = e.h_tokens[(size_t)h * e.L + gen - 1];
  if (ctx_g % m.P) {
    tail_src[k] = gb[nfull];
    tail_dst[k] = hb[nfull];
  }
}

// Prefill rows of resumed samples: pieces[k] = {handle, group slot, first generated index j0,
// first row}; piece k covers rows [pieces[k].w, pieces[k+1].w).  Row for generated index j
// sits at position g_ctx + j and feeds token j - 1 (j = 0: the prompt's last token).
__global__ void k_extend_rows(EngineDev e, ModelDev m, const int4* pieces, int n_pieces) {
  const int k = blockIdx.x;
  if (k >= n_pieces) return;
  const int4 p = pieces[k];
  const int rend = pieces[k + 1].w;
  const int ctx_g = m.g_ctx[p.y];
  for (int r = p.w + threadIdx.x; r < rend; r += blockDim.x) {
    const int j = p.z + (r - p.w);
    m.row_tok[r] = j == 0 ? m.g_last_tok[p.y] : e.h_tokens[(size_t)p.x * e.L + j - 1];
    m.row_pos[r] = ctx_g + j;
    m.row_btrow[r] = p.x;
  }
}

// Log-prob scoring: scratch block-table rows get pages for `len` positions each
// (items[k] = {bt row, positions}), released afterwards by k_score_release.
__global__ void k_score_alloc(EngineDev e, ModelDev m, const int2* items, int n) {
  Ctl* c = e.ctl;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int2 it = items[k];
  int32_t* row = m.bt + (size_t)it.x * m.MP;
  const int need = (it.y + m.P - 1) / m.P;
  for (int j = 0; j < need; ++j) {
    const int idx = j < m.MP ? pop_page(c) : -1;
    if (idx < 0) {
      atomicCAS(&c->error, kErrNone, kErrOutOfKV);
      for (int q = j; q < need; ++q) row[q] = -1;
      return;
    }
    row[j] = m.free_pages[idx];
  }
}

__global__ void k_score_release(EngineDev e, ModelDev m, const int2* items, int n) {
  Ctl* c = e.ctl;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int2 it = items[k];
  const int32_t* row = m.bt + (size_t)it.x * m.MP;
  int need = (it.y + m.P - 1) / m.P;
  while (need > 0 && row[need - 1] < 0) --need;  // (a failed allocation left -1 entries)
  const long long base =
      (long long)atomicAdd(reinterpret_cast<unsigned long long*>(&c->kv_free_top), (unsigned long long)need);
  for (int j = 0; j < need; ++j) m.free_pages[base + j] = row[j];
}

// dst[i] = src[rows[i]] for bf16 rows of width d (d % 8 == 0)
__global__ void k_gather_rows(const bf16* __restrict__ src, bf16* __restrict__ dst, const int* __restrict__ rows,
                              int n, int d) {
  const int i = blockIdx.x;
  if (i >= n) return;
  const uint4* s = reinterpret_cast<const uint4*>(src + (size_t)rows[i] * d);
  uint4* o = reinterpret_cast<uint4*>(dst + (size_t)i * d);
  for (int j = threadIdx.x; j < d / 8; j += blockDim.x) o[j] = s[j];
}

// out[i] = log softmax(logits[i] / T)[target[i]]   (one block per row, fp64 reduction)
__global__ void __launch_bounds__(256) k_logp_rows(const float* __restrict__ logits, int V,
                                                   const int* __restrict__ target, int n, float inv_temp,
                                                   double* __restrict__ out) {
  const int i = blockIdx.x;
  if (i >= n) return;
  const float* z = logits + (size_t)i * V;
  __shared__ float s_m[8];
  __shared__ double s_s[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float mx = -FLT_MAX;
  for (int j = threadIdx.x; j < V; j += blockDim.x) mx = fmaxf(mx, z[j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) s_m[w] = mx;
  __syncthreads();
  mx = s_m[0];
  for (int k = 1; k < 8; ++k) mx = fmaxf(mx, s_m[k]);
  double sum = 0.0;
  for (int j = threadIdx.x; j < V; j += blockDim.x) sum += (double)__expf((z[j] - mx) * inv_temp);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) s_s[w] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double S = 0.0;
    for (int k = 0; k < 8; ++k) S += s_s[k];
    out[i] = (double)((z[target[i]] - mx) * inv_temp) - log(S);
  }
}

__global__ void k_release(EngineDev e, ModelDev m, const int32_t* handles, int n) {
  Ctl* c = e.ctl;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int h = handles[k];
  const int have = (m.h_ctx[h] + m.P - 1) / m.P;
  const int own0 = m.h_shared[h];
  const int cnt = have - own0;
  if (cnt > 0) {
    const long long base =
        (long long)atomicAdd(reinterpret_cast<unsigned long long*>(&c->kv_free_top), (unsigned long long)cnt);
    for (int j = 0; j < cnt; ++j) m.free_pages[base + j] = m.bt[(size_t)h * m.MP + own0 + j];
  }
  m.h_ctx[h] = 0;
  m.h_shared[h] = 0;
}

__global__ void k_group_alloc(EngineDev e, ModelDev m, const int* groups, const int* lens, const int* last_tok,
                              int n) {
  Ctl* c = e.ctl;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int g = groups[k], len = lens[k];
  const int np = (len + m.P - 1) / m.P;
  int32_t* gb = m.bt + (size_t)(m.H + g) * m.MP;
  for (int j = 0; j < np; ++j) {
    const int idx = pop_page(c);
    if (idx < 0) {
      atomicCAS(&c->error, kErrNone, kErrOutOfKV);
      m.g_npages[g] = j;
      return;
    }
    gb[j] = m.free_pages[idx];
  }
  m.g_npages[g] = np;
  m.g_ctx[g] = len;
  m.g_last_tok[g] = last_tok[k];
}

__global__ void k_group_release(EngineDev e, ModelDev m, int g) {
  Ctl* c = e.ctl;
  const int np = m.g_npages[g];
  if (threadIdx.x != 0 || np <= 0) return;
  const long long base =
      (long long)atomicAdd(reinterpret_cast<unsigned long long*>(&c->kv_free_top), (unsigned long long)np);
  for (int j = 0; j < np; ++j) m.free_pages[base + j] = m.bt[(size_t)(m.H + g) * m.MP + j];
  m.g_npages[g] = 0;
  m.g_ctx[g] = 0;
}

}  // namespace

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

int attention_items_per_cta() {
  const char* ai = getenv("AB_ATT_ITEMS");
  return ai ? std::max(1, atoi(ai)) : 1;
}

void set_pdl_mask_layers(int mask) {
  AB_CUDA(cudaMemcpyToSymbol(c_pdl_mask, &mask, sizeof(int)));
  const int z = getenv("AB_ROPE_NOZERO") ? 0 : 1;  // timing experiments only: results are then wrong
  AB_CUDA(cudaMemcpyToSymbol(c_rope_zero, &z, sizeof(int)));
  const unsigned long long items = (unsigned long long)attention_items_per_cta();
  AB_CUDA(cudaMemcpyToSymbol(c_items_per_cta, &items, sizeof(items)));
}

void launch_init_weights(bf16* w, size_t n, uint64_t seed, uint64_t tensor_id, float std, float constant,
                         cudaStream_t s) {
  const int mode = std > 0.f ? 0 : 1;
  k_init_weights<<<4 * 148, 256, 0, s>>>(w, n, seed ^ 0x5DEECE66Dull, tensor_id, std, constant, mode);
  AB_CUDA(cudaGetLastError());
}

void launch_rope_table(float2* rope, int max_pos, int hd, float theta, cudaStream_t s) {
  k_rope_table<<<4 * 148, 256, 0, s>>>(rope, max_pos, hd, theta);
  AB_CUDA(cudaGetLastError());
}

void launch_prep_decode(const EngineDev& e, const ModelDev& m, int chunk, cudaStream_t s) {
  static int att_ctas = 0;
  if (!att_ctas) att_ctas = decode_attention_ctas(m);
  k_prep_decode<<<1, kPrepThreads, 0, s>>>(e, m, chunk, att_ctas);
}

void launch_embed(const ModelDev& m, const bf16* emb, float* x, const int* rows_dev, int rows_cap, const int* stop,
                  cudaStream_t s) {
  k_embed<<<rows_cap, 128, 0, s>>>(m, emb, x, rows_dev, rows_cap, stop);
}

void launch_swiglu_ws(float* ws, bf16* h, int f, const int* sched, const int* rows_dev, int rows_cap, const int* stop,
                      cudaStream_t s) {
  static int grid = 0;
  if (!grid) {
    int dev = 0, sms = 0;
    AB_CUDA(cudaGetDevice(&dev));
    AB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    grid = 2 * sms;
  }
  launch_pdl(k_swiglu_ws, dim3(grid), dim3(256), 0, s, ws, h, f, sched, rows_dev, rows_cap, stop);
}

void launch_rmsnorm(const float* x, const bf16* w, bf16* out, int d, float eps, const int* rows_dev, int rows_cap,
                    const int* stop, cudaStream_t s) {
  const dim3 g(ceil_div(rows_cap, 8)), t(256);
  switch (d % 128 ? 0 : d / 128) {
    case 2: launch_pdl(k_rmsnorm_v<2>, g, t, 0, s, x, w, out, eps, rows_dev, rows_cap, stop); break;
    case 4: launch_pdl(k_rmsnorm_v<4>, g, t, 0, s, x, w, out, eps, rows_dev, rows_cap, stop); break;
    case 8: launch_pdl(k_rmsnorm_v<8>, g, t, 0, s, x, w, out, eps, rows_dev, rows_cap, stop); break;
    case 12: launch_pdl(k_rmsnorm_v<12>, g, t, 0, s, x, w, out, eps, rows_dev, rows_cap, stop); break;
    case 16: launch_pdl(k_rmsnorm_v<16>, g, t, 0, s, x, w, out, eps, rows_dev, rows_cap, stop); break;
    case 20: launch_pdl(k_rmsnorm_v<20>, g, t, 0, s, x, w, out, eps, rows_dev, rows_cap, stop); break;
    case 24: launch_pdl(k_rmsnorm_v<24>, g, t, 0, s, x, w, out, eps, rows_dev, rows_cap, stop); break;
    case 28: launch_pdl(k_rmsnorm_v<28>, g, t, 0, s, x, w, out, eps, rows_dev, rows_cap, stop); break;
    case 32: launch_pdl(k_rmsnorm_v<32>, g, t, 0, s, x, w, out, eps, rows_dev, rows_cap, stop); break;
    default: launch_pdl(k_rmsnorm, g, t, 0, s, x, w, out, d, eps, rows_dev, rows_cap, stop); break;
  }
}

// q / k / v heads per row spread over blockIdx.y so that each warp owns one head (a latency-bound
// kernel: a short dependent chain per warp, many warps)
static int rope_hy(const ModelDev& m) { return ceil_div(m.hq + 2 * m.hk, 8); }

void launch_rope_kv(const ModelDev& m, int layer, const bf16* qkv, const bf16* q_norm, const bf16* k_norm, bf16* q_out,
                    const int* rows_dev, int rows_cap, const int* stop, cudaStream_t s) {
  if (m.hd == 128)
    launch_pdl(k_rope_kv<128>, dim3(rows_cap, rope_hy(m)), dim3(256), 0, s, m, layer, qkv, q_norm, k_norm, q_out, rows_dev, rows_cap,
               stop);
  else
    launch_pdl(k_rope_kv<64>, dim3(rows_cap, rope_hy(m)), dim3(256), 0, s, m, layer, qkv, q_norm, k_norm, q_out, rows_dev, rows_cap,
               stop);
}

void launch_rope_kv_f32(const ModelDev& m, int layer, float* qkv, const bf16* bias, const bf16* q_norm,
                        const bf16* k_norm, bf16* q_out, const int* rows_dev, int rows_cap, const int* stop,
                        cudaStream_t s) {
  if (m.hd == 128)
    launch_pdl(k_rope_kv_f32<128>, dim3(rows_cap, rope_hy(m)), dim3(256), 0, s, m, layer, qkv, bias, q_norm, k_norm, q_out,
               rows_dev, rows_cap, stop);
  else
    launch_pdl(k_rope_kv_f32<64>, dim3(rows_cap, rope_hy(m)), dim3(256), 0, s, m, layer, qkv, bias, q_norm, k_norm, q_out,
               rows_dev, rows_cap, stop);
}

// Fork metadata scratch, one per engine stream (several engines may share a process), grown
// stream-ordered so a growth never synchronises the device.
static int32_t* fork_scratch(cudaStream_t s, int n, int* cap_out) {
  static std::mutex mu;
  static std::map<cudaStream_t, std::pair<int32_t*, int>> bufs;
  std::lock_guard<std::mutex> lock(mu);
  auto& b = bufs[s];
  if (n > b.second) {
    if (b.first) AB_CUDA(cudaFreeAsync(b.first, s));
    b.second = n + 1024;
    AB_CUDA(cudaMallocAsync(&b.first, sizeof(int32_t) * 2 * b.second, s));
  }
  *cap_out = b.second;
  return b.first;
}

void launch_fork_groups(const EngineDev& e, const ModelDev& m, const ab_sample_desc* descs, int n, cudaStream_t s) {
  int cap = 0;
  int32_t* buf = fork_scratch(s, n, &cap);
  k_fork_meta<<<ceil_div(n, 128), 128, 0, s>>>(e, m, descs, n, buf, buf + cap);
  k_fork_copy<<<dim3(n, m.L), 256, 0, s>>>(m, buf, buf + cap);
}

void launch_resume_fork(const EngineDev& e, const ModelDev& m, const int4* items, int n, cudaStream_t s) {
  int cap = 0;
  int32_t* buf = fork_scratch(s, n, &cap);
  k_resume_fork<<<ceil_div(n, 128), 128, 0, s>>>(e, m, items, n, buf, buf + cap);
  k_fork_copy<<<dim3(n, m.L), 256, 0, s>>>(m, buf, buf + cap);
}

void launch_extend_rows(const EngineDev& e, const ModelDev& m, const int4* pieces, int n_pieces, cudaStream_t s) {
  k_extend_rows<<<n_pieces, 256, 0, s>>>(e, m, pieces, n_pieces);
}

void launch_score_alloc(const EngineDev& e, const ModelDev& m, const int2* items, int n, cudaStream_t s) {
  k_score_alloc<<<ceil_div(n, 64), 64, 0, s>>>(e, m, items, n);
}
void launch_score_release(const EngineDev& e, const ModelDev& m, const int2* items, int n, cudaStream_t s) {
  k_score_release<<<ceil_div(n, 64), 64, 0, s>>>(e, m, items, n);
}
void launch_gather_rows(const bf16* src, bf16* dst, const int* rows, int n, int d, cudaStream_t s) {
  k_gather_rows<<<n, 128, 0, s>>>(src, dst, rows, n, d);
}
void launch_logp_rows(const float* logits, int V, const int* target, int n, float inv_temp, double* out,
                      cudaStream_t s) {
  k_logp_rows<<<n, 256, 0, s>>>(logits, V, target, n, inv_temp, out);
}

void launch_release_handles(const EngineDev& e, const ModelDev& m, const int32_t* handles, int n, cudaStream_t s) {
  k_release<<<ceil_div(n, 128), 128, 0, s>>>(e, m, handles, n);
}

void launch_group_alloc(const EngineDev& e, const ModelDev& m, const int* groups, const int* lens, const int* last_tok,
                        int n, cudaStream_t s) {
  k_group_alloc<<<ceil_div(n, 128), 128, 0, s>>>(e, m, groups, lens, last_tok, n);
}

void launch_group_release(const EngineDev& e, const ModelDev& m, int group, cudaStream_t s) {
  k_group_release<<<1, 32, 0, s>>>(e, m, group);
}

}  // namespace ab
