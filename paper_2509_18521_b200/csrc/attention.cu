// K3: paged GQA decode attention, TMA-fed, warp-specialised flash-decoding.
//
// Work item = (live row, kv head, KV split of `chunk` tokens).  k_prep_decode
// writes the (row, split) list each iteration; a persistent grid (2 CTAs per
// SM) walks it.  Warp 4 is the producer: running up to kStages tiles ahead on
// empty/full mbarriers, it issues per 64-token tile cp.async.bulk.tensor
// loads of the kv head's K and V rows straight out of the paged pool (one 4-D
// box per tile with 64-token pages, else 2-D boxes; tensor map over
// kv[layer][page][k|v][head][slot][dim], 128-byte swizzle),
// plus on an item's first tile a 1-D bulk copy of the GQA group's q rows, and
// hands the item's metadata to the consumers through shared memory (all
// global-memory latency of the work list lives in the producer).  Warps 0-3
// consume: each owns 16 tokens of a tile, S = Q K^T and O += P V as mma.sync
// m16n8k16 bf16 tiles with the q heads as the 16-row M side
// (flash-attention-2 register layout, exp2 online softmax).  At an item's
// end the stage goes back to the producer and the 4 warps merge pairwise in
// a fixed order through a small buffer; rows with one split write the
// output directly, multi-split rows are merged in split order by the last
// CTA to finish (arrival counter, self-resetting): deterministic end to end.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <vector>

#include "model.cuh"

namespace ab {

namespace {

constexpr float kLog2e = 1.4426950408889634f;
__constant__ int c_pdl_mask = 6;  // see gemm.cu
constexpr int kTok = 64;        // tokens per tile
constexpr int kCons = 4;        // consumer warps (16 tokens each)
constexpr int kThreads = (kCons + 1) * 32;
constexpr int kStages = 3;
constexpr int kQSlots = 3;
constexpr int kMergeRows = 8;   // GQA group <= 8
constexpr int kMaxSplits = 64;  // KV splits per row (the model sizes the minimum split to respect it)

struct Meta {
  int row, kvh, sp, c0, c1, tile, ntiles, nsplit, qslot, done, pad0, pad1;
};

template <int HD>
struct AttCfg {
  static constexpr int kKV = kTok * HD * 2;  // K (or V) of one tile
  static constexpr int kQ = kMergeRows * HD * 2;
  static constexpr int oQ = kStages * 2 * kKV;
  static constexpr int oZero = oQ + kQSlots * kQ;
  // end-of-item merge buffer: [2][kMergeRows][HD] fp32 + [2][kMergeRows] (m, l); the split combine's
  // [kMergeRows][kMaxSplits] (m, l) aliases it (used only after the merge)
  static constexpr int kMB = 2 * kMergeRows * HD * 4 + 2 * kMergeRows * 8;
  static constexpr int oMB = oZero + HD * 2;
  static constexpr int oMLs = oMB;
  static constexpr int oMeta = oMB + (kMB > kMergeRows * kMaxSplits * 8 ? kMB : kMergeRows * kMaxSplits * 8);
  static constexpr int oBar = oMeta + kStages * (int)sizeof(Meta);
  static constexpr int kSmem = 1024 + oBar + 2 * kStages * 8;
  // two CTAs per SM: 228 KB of shared memory, 1 KB reserved per CTA
  static_assert(2 * (kSmem + 1024) <= 228 * 1024, "decode attention must fit two CTAs per SM");
};

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(su32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(su32(bar)), "r"(x), "r"(y)
      : "memory");
}
// 4-D view {64 dims, pool row, dim half, k|v}: one operation = a 64-token tile's K and V, both
// halves of the head dimension (32 KB at HD = 128), landing as [k|v][half][64 rows][128 B]
__device__ __forceinline__ void tma_4d(const CUtensorMap* map, uint64_t* bar, void* dst, int y) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %3, %3}], "
      "[%2];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(su32(bar)), "r"(0), "r"(y)
      : "memory");
}
__device__ __forceinline__ void bulk_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void cons_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr, bool trans) {
  if (trans)
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
  else
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

// byte offset of 16-byte chunk `ch` of row `r` in a TMA-swizzled [HD/64 halves][64 rows][128 B] tile
__device__ __forceinline__ uint32_t tile_off(int r, int ch) {
  return (uint32_t)((ch >> 3) * (kTok * 128) + r * 128 + (((ch & 7) ^ (r & 7)) << 4));
}

template <int HD>
__global__ void __launch_bounds__(kThreads, 2)
    k_decode_attn(const __grid_constant__ CUtensorMap kvmap, EngineDev e, ModelDev m, int layer,
                  const bf16* __restrict__ q, bf16* __restrict__ out, float* __restrict__ part_o,
                  float* __restrict__ part_ml, int max_splits) {
  using Cfg = AttCfg<HD>;
  pdl_wait();
  // the successor (the O GEMM) may start its pre-wait prologue on SMs this persistent grid leaves
  if (c_pdl_mask & 2) pdl_launch();
  const Ctl* c = e.ctl;
  if (c->stop) return;
  const int b = c->b;
  if (b <= 0) return;
  const int total = m.split_prefix[b] * m.hk;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float2* sMLs = reinterpret_cast<float2*>(base + Cfg::oMLs);  // [kMergeRows][kMaxSplits]
  Meta* meta = reinterpret_cast<Meta*>(base + Cfg::oMeta);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + Cfg::oBar);
  uint64_t* empty = full + kStages;
  __shared__ int s_last;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = m.gq;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCons);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < HD * 2 / 16; i += kThreads)
    reinterpret_cast<uint4*>(base + Cfg::oZero)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();

  if (warp == kCons) {
    // ------------------------------ producer ------------------------------
    // The whole warp walks the work list; lane 0 issues the barrier / TMA operations.  An item's
    // metadata is a chain of dependent loads (cursor claim -> (row, split) -> context / block-table
    // row -> page ids, ~2.5 us), resolved once the previous item's last tile is issued (kAhead = 1;
    // resolving it 3 tiles earlier was measured neutral at 768-3,072 items per launch, and it
    // commits the claimed item early).  With 64-token pages (one page per tile) the 32 lanes load 32
    // page ids at once and each tile is ONE 4-D TMA operation (K and V, both head-dim halves); other
    // page sizes keep per-box 2-D loads.
    if (lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&kvmap)) : "memory");
    constexpr int kAhead = 1;
    const int chunk = m.att_ctl[0];
    const uint32_t qbytes = (uint32_t)(gq * HD * 2);
    const int box_rows = m.P < kTok ? m.P : kTok;
    const bool tile_pages = m.P == kTok;
    struct Item {
      int valid, row, kvh, sp, c0, c1, ntiles, nsplit, pg;  // pg: page id of tile `lane` (tile_pages)
      const int32_t* bt;
    };
    auto resolve = [&](Item& it) {
      int idx = 0;
      if (lane == 0) idx = atomicAdd(&m.att_ctl[1 + layer], 1);
      idx = __shfl_sync(0xffffffffu, idx, 0);
      it.valid = idx < total;
      if (!it.valid) return;
      const int rs = idx / m.hk;
      it.kvh = idx % m.hk;
      const int packed = m.att_items[rs];
      it.row = packed & 0xffff;
      it.sp = packed >> 16;
      const int n = m.row_pos[it.row] + 1;
      // the row's nsplit = ceil(n / chunk) splits are balanced (64-token multiples)
      it.nsplit = (n + chunk - 1) / chunk;
      const int per = (((n + it.nsplit - 1) / it.nsplit) + kTok - 1) / kTok * kTok;
      it.c0 = it.sp * per;
      it.c1 = min(n, it.c0 + per);
      it.ntiles = (it.c1 - it.c0 + kTok - 1) / kTok;
      it.bt = m.bt + (size_t)m.row_btrow[it.row] * m.MP;
      it.pg = (tile_pages && lane < it.ntiles) ? it.bt[it.c0 / kTok + lane] : 0;
    };
    int g = 0;
    Item cur;
    resolve(cur);
    for (int k = 0; cur.valid; ++k) {
      Item nxt;
      nxt.valid = 0;
      const int t_next = max(0, cur.ntiles - kAhead);
      const int qslot = k % kQSlots;
      for (int t = 0; t < cur.ntiles; ++t, ++g) {
        if (tile_pages && t > 0 && (t & 31) == 0) {
          const int tt = t + lane;
          cur.pg = tt < cur.ntiles ? cur.bt[cur.c0 / kTok + tt] : 0;
        }
        const int page_t = tile_pages ? __shfl_sync(0xffffffffu, cur.pg, t & 31) : 0;
        if (lane == 0) {
          const int st = g % kStages;
          mbar_wait(&empty[st], ((g / kStages) & 1) ^ 1);
          Meta mt;
          mt.row = cur.row;
          mt.kvh = cur.kvh;
          mt.sp = cur.sp;
          mt.c0 = cur.c0;
          mt.c1 = cur.c1;
          mt.tile = t;
          mt.ntiles = cur.ntiles;
          mt.nsplit = cur.nsplit;
          mt.qslot = qslot;
          mt.done = 0;
          meta[st] = mt;
          uint8_t* sb = base + st * 2 * Cfg::kKV;
          mbar_expect_tx(&full[st], 2 * Cfg::kKV + (t == 0 ? qbytes : 0u));
          if (tile_pages) {
            const int64_t yk = (((int64_t)layer * m.NP + page_t) * 2 * m.hk + cur.kvh) * m.P;
            tma_4d(&kvmap, &full[st], sb, (int)yk);
          } else {
            const int tok0 = cur.c0 + t * kTok;
            for (int r0 = 0; r0 < kTok; r0 += box_rows) {
              const bool valid = tok0 + r0 < cur.c1;
              const int tok = valid ? tok0 + r0 : cur.c1 - 1;  // past the end: reload a valid page (masked)
              const int page = cur.bt[tok / m.P];
              const int slot = valid ? tok % m.P : 0;
              const int64_t yk = ((((int64_t)layer * m.NP + page) * 2) * m.hk + cur.kvh) * m.P + slot;
              const int64_t yv = yk + (int64_t)m.hk * m.P;
#pragma unroll
              for (int h = 0; h < HD / 64; ++h) {
                tma_2d(&kvmap, &full[st], sb + h * (kTok * 128) + r0 * 128, h * 64, (int)yk);
                tma_2d(&kvmap, &full[st], sb + Cfg::kKV + h * (kTok * 128) + r0 * 128, h * 64, (int)yv);
              }
            }
          }
          if (t == 0)
            bulk_1d(base + Cfg::oQ + qslot * Cfg::kQ, q + (size_t)cur.row * m.qd + cur.kvh * gq * HD, qbytes,
                    &full[st]);
        }
        __syncwarp();
        if (t == t_next) resolve(nxt);
      }
      cur = nxt;
    }
    if (lane == 0) {
      const int st = g % kStages;  // sentinel
      mbar_wait(&empty[st], ((g / kStages) & 1) ^ 1);
      meta[st].done = 1;
      mbar_arrive(&full[st]);
    }
    return;
  }

  // ------------------------------ consumers ------------------------------
  const int gr = lane >> 2, tq = lane & 3;
  const int tid = threadIdx.x;  // 0..127
  const float scale = rsqrtf((float)HD) * kLog2e;
  float o[HD / 8][4];
  float mrow[2] = {-FLT_MAX, -FLT_MAX}, lrow[2] = {0.f, 0.f};
  uint32_t qa[HD / 16][4];
  for (int g = 0;; ++g) {
    const int st = g % kStages;
    mbar_wait(&full[st], (g / kStages) & 1);
    const Meta mt = meta[st];
    if (mt.done) break;
    const uint32_t K = su32(base + st * 2 * Cfg::kKV), V = K + Cfg::kKV;
    if (mt.tile == 0) {
#pragma unroll
      for (int t = 0; t < HD / 8; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
      mrow[0] = mrow[1] = -FLT_MAX;
      lrow[0] = lrow[1] = 0.f;
      const int r = lane & 15;
      const uint32_t rowbase = r < gq ? su32(base + Cfg::oQ + mt.qslot * Cfg::kQ) + r * HD * 2
                                      : su32(base + Cfg::oZero);
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) ldsm_x4(qa[kk], rowbase + (kk * 2 + (lane >> 4)) * 16, false);
    }
    const int tb = mt.c0 + mt.tile * kTok, wt = warp * 16;
    float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      const int mi = lane >> 3;
      uint32_t bb[4];
      ldsm_x4(bb, K + tile_off(wt + (mi >> 1) * 8 + (lane & 7), kk * 2 + (mi & 1)), false);
      mma16816(s[0], qa[kk], bb[0], bb[1]);
      mma16816(s[1], qa[kk], bb[2], bb[3]);
    }
    float mx[2] = {-FLT_MAX, -FLT_MAX};
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const int tok = tb + wt + j * 8 + tq * 2 + (q4 & 1);
        const float v = tok < mt.c1 ? s[j][q4] * scale : -FLT_MAX;
        s[j][q4] = v;
        mx[q4 >> 1] = fmaxf(mx[q4 >> 1], v);
      }
    float alpha[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      const float mn = fmaxf(mrow[r], mx[r]);
      alpha[r] = (mrow[r] == -FLT_MAX) ? 0.f : exp2f(mrow[r] - mn);
      mrow[r] = mn;
    }
    float rsum[2] = {0.f, 0.f};
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const int r = q4 >> 1;
        const float p = (s[j][q4] == -FLT_MAX) ? 0.f : exp2f(s[j][q4] - mrow[r]);
        s[j][q4] = p;
        rsum[r] += p;
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) lrow[r] = lrow[r] * alpha[r] + rsum[r];
#pragma unroll
    for (int nt = 0; nt < HD / 8; ++nt) {
      o[nt][0] *= alpha[0];
      o[nt][1] *= alpha[0];
      o[nt][2] *= alpha[1];
      o[nt][3] *= alpha[1];
    }
    const uint32_t pa[4] = {pack_bf16(s[0][0], s[0][1]), pack_bf16(s[0][2], s[0][3]), pack_bf16(s[1][0], s[1][1]),
                            pack_bf16(s[1][2], s[1][3])};
#pragma unroll
    for (int nt2 = 0; nt2 < HD / 16; ++nt2) {
      const int mi = lane >> 3;
      uint32_t bb[4];
      ldsm_x4(bb, V + tile_off(wt + (mi & 1) * 8 + (lane & 7), nt2 * 2 + (mi >> 1)), true);
      mma16816(o[2 * nt2], pa, bb[0], bb[1]);
      mma16816(o[2 * nt2 + 1], pa, bb[2], bb[3]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done with the stage (the last one too)
    if (mt.tile != mt.ntiles - 1) continue;

    // ---- item complete: merge the 4 warps' unscaled outputs pairwise in fixed order (1 -> 0,
    // 3 -> 2, then 2 -> 0: deterministic) through a small dedicated buffer, so the item's last
    // stage has already gone back to the producer.  (Merging inside the held stage kept the ring at
    // two tiles in flight during every merge: ~1.2 us of CTA DRAM time per item, measured by
    // skipping the merge; a separate merge warp holding the stage longer was slower still.) ----
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 1);
      lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 2);
    }
    float* bO = reinterpret_cast<float*>(base + Cfg::oMB);                        // [2][kMergeRows][HD]
    float2* bML = reinterpret_cast<float2*>(base + Cfg::oMB + 2 * kMergeRows * HD * 4);  // [2][kMergeRows]
    auto put = [&](int slot) {
      if (gr < gq) {
        float* dst = bO + (slot * kMergeRows + gr) * HD;
#pragma unroll
        for (int nt = 0; nt < HD / 8; ++nt)
          *reinterpret_cast<float2*>(dst + nt * 8 + tq * 2) = make_float2(o[nt][0], o[nt][1]);
        if (tq == 0) bML[slot * kMergeRows + gr] = make_float2(mrow[0], lrow[0]);
      }
    };
    auto take = [&](int slot) {
      if (gr < gq) {
        const float2 ml = bML[slot * kMergeRows + gr];
        const float M = fmaxf(mrow[0], ml.x);
        const float a = mrow[0] == -FLT_MAX ? 0.f : exp2f(mrow[0] - M);
        const float bw = ml.x == -FLT_MAX ? 0.f : exp2f(ml.x - M);
        const float* src = bO + (slot * kMergeRows + gr) * HD;
#pragma unroll
        for (int nt = 0; nt < HD / 8; ++nt) {
          const float2 v = *reinterpret_cast<const float2*>(src + nt * 8 + tq * 2);
          o[nt][0] = o[nt][0] * a + v.x * bw;
          o[nt][1] = o[nt][1] * a + v.y * bw;
        }
        mrow[0] = M;
        lrow[0] = lrow[0] * a + ml.y * bw;
      }
    };
    cons_sync();  // the previous item's readers of the buffer are done
    if (warp & 1) put(warp >> 1);
    cons_sync();
    if (!(warp & 1)) take(warp >> 1);
    cons_sync();
    if (warp == 2) put(0);
    cons_sync();
    const int i = mt.row, kvh = mt.kvh, sp = mt.sp, nsplit = mt.nsplit;
    if (warp == 0) {
      take(0);
      if (gr < gq) {  // warp 0 holds the item's output rows
        const int head = kvh * gq + gr;
        if (nsplit == 1) {
          const float inv = 1.f / lrow[0];
          __nv_bfloat16* dst = out + (size_t)i * m.qd + head * HD + tq * 2;
#pragma unroll
          for (int nt = 0; nt < HD / 8; ++nt)
            *reinterpret_cast<uint32_t*>(dst + nt * 8) = pack_bf16(o[nt][0] * inv, o[nt][1] * inv);
        } else {
          const size_t pb = ((size_t)i * m.hq + head) * max_splits + sp;
#pragma unroll
          for (int nt = 0; nt < HD / 8; ++nt)
            *reinterpret_cast<float2*>(part_o + pb * HD + nt * 8 + tq * 2) = make_float2(o[nt][0], o[nt][1]);
          if (tq == 0) *reinterpret_cast<float2*>(part_ml + pb * 2) = make_float2(mrow[0], lrow[0]);
        }
      }
      __syncwarp();
    }
    if (nsplit > 1) {
      // split combine by the last CTA to finish a split of this (row, kv head): split order, deterministic
      if (tid == 0) {
        __threadfence();
        const int old = atomicAdd(&m.att_counter[i * m.hk + kvh], 1);
        const int last = old == nsplit - 1;
        if (last) {
          m.att_counter[i * m.hk + kvh] = 0;
          __threadfence();
        }
        s_last = last;
      }
      cons_sync();  // (also: warp 0 is done with the merge buffer, which sMLs aliases)
      if (s_last) {
        for (int idx = tid; idx < gq * nsplit; idx += kCons * 32) {
          const int row = idx / nsplit, s2 = idx % nsplit;
          const size_t pb = ((size_t)i * m.hq + kvh * gq + row) * max_splits + s2;
          sMLs[row * kMaxSplits + s2] = __ldcg(reinterpret_cast<const float2*>(part_ml + pb * 2));
        }
        cons_sync();
        for (int idx = tid; idx < gq * (HD / 4); idx += kCons * 32) {
          const int row = idx / (HD / 4), d4 = idx % (HD / 4);
          const int head = kvh * gq + row;
          const float2* ml = sMLs + row * kMaxSplits;
          float M = -FLT_MAX;
          for (int s2 = 0; s2 < nsplit; ++s2) M = fmaxf(M, ml[s2].x);
          const float4* src = reinterpret_cast<const float4*>(part_o + ((size_t)i * m.hq + head) * max_splits * HD) + d4;
          float L = 0.f;
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
          for (int s2 = 0; s2 < nsplit; ++s2) {
            const float wgt = exp2f(ml[s2].x - M);
            const float4 v = __ldcg(src + (size_t)s2 * (HD / 4));
            L += ml[s2].y * wgt;
            acc.x += v.x * wgt;
            acc.y += v.y * wgt;
            acc.z += v.z * wgt;
            acc.w += v.w * wgt;
          }
          const float inv = 1.f / L;
          uint2 w2;
          w2.x = pack_bf16(acc.x * inv, acc.y * inv);
          w2.y = pack_bf16(acc.z * inv, acc.w * inv);
          *reinterpret_cast<uint2*>(out + (size_t)i * m.qd + head * HD + d4 * 4) = w2;
        }
      }
      cons_sync();  // s_last / sMLs are reused by the next item
    }
  }
}

template <int HD>
int grid_t() {
  static int grid = 0;
  if (!grid) {
    AB_CUDA(cudaFuncSetAttribute(k_decode_attn<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, AttCfg<HD>::kSmem));
    int per_sm = 0, dev = 0, sms = 0;
    AB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_decode_attn<HD>, kThreads, AttCfg<HD>::kSmem));
    AB_CUDA(cudaGetDevice(&dev));
    AB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    grid = sms * (per_sm > 0 ? per_sm : 1);
  }
  return grid;
}

template <int HD>
void launch_t(const CUtensorMap& map, const EngineDev& e, const ModelDev& m, int layer, const bf16* q, bf16* out,
              float* part_o, float* part_ml, int max_splits, cudaStream_t s) {
  launch_pdl(k_decode_attn<HD>, dim3(grid_t<HD>()), dim3(kThreads), AttCfg<HD>::kSmem, s, map, e, m, layer, q, out,
             part_o, part_ml, max_splits);
}

// ---------------------------------------------------------------------------
// Causal prefill attention (prompt prefill and the re-prefill of resumed
// partials, §8 f1): flash-attention-2 over the paged pool.  Block = up to 128
// consecutive rows of one sequence (its block-table row and first position
// come from the host-built block list), one q head per CTA; 8 warps own 16
// rows each.  K / V tiles of 64 tokens are gathered page by page with
// cp.async into the same 128-byte-swizzled layout the decode kernel reads
// (double-buffered), S = Q K^T and O += P V run as mma.sync m16n8k16 with
// exp2 online softmax; tokens past a row's position are masked.
// ---------------------------------------------------------------------------

// Q block of kPfRows rows (8 warps x 16 rows): each K / V tile staged in shared memory serves 128 query
// rows (the first version used 64-row blocks and 4 warps: half the tile reuse, half the warps)
constexpr int kPfRows = 128;
constexpr int kPfThreads = kPfRows / 16 * 32;

template <int HD>
struct PfCfg {
  static constexpr int kTile = kTok * HD * 2;                  // 64 rows x HD bf16
  static constexpr int kTileQ = kPfRows * HD * 2;              // the Q block
  static constexpr int kSmem = 1024 + kTileQ + 4 * kTile;      // Q + 2 stages x (K, V)
};

// tile_off for a tile of R rows (the Q block): 16-byte chunk ch of row r, 128-byte swizzle
template <int R>
__device__ __forceinline__ uint32_t tile_off_r(int r, int ch) {
  return (uint32_t)((ch >> 3) * (R * 128) + r * 128 + (((ch & 7) ^ (r & 7)) << 4));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int HD>
__global__ void __launch_bounds__(kPfThreads, 1)
    k_prefill_flash(ModelDev m, int layer, const bf16* __restrict__ q, bf16* __restrict__ out,
                    const int4* __restrict__ blocks) {
  using Cfg = PfCfg<HD>;
  constexpr int CH = HD / 8;  // 16-byte chunks per row
  const int4 blk = blocks[blockIdx.x];  // {first row, rows, block-table row, first position}
  const int row0 = blk.x, nrows = blk.y, pos0 = blk.w;
  const int head = blockIdx.y, kvh = head / m.gq;
  const int32_t* bt = m.bt + (size_t)blk.z * m.MP;
  const int last_pos = pos0 + nrows - 1;
  const int n_kt = last_pos / kTok + 1;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sQ = su32(base), sKV = sQ + Cfg::kTileQ;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gr = lane >> 2, tq = lane & 3;

  for (int i = tid; i < kPfRows * CH; i += kPfThreads) {
    const int r = i / CH, ch = i % CH;
    const bool v = r < nrows;
    cp_async16(sQ + tile_off_r<kPfRows>(r, ch), q + (size_t)(row0 + (v ? r : 0)) * m.qd + head * HD + ch * 8, v);
  }
  auto load_kv = [&](int kt, int stage) {
    const uint32_t K = sKV + stage * 2 * Cfg::kTile, V = K + Cfg::kTile;
    for (int i = tid; i < kTok * CH; i += kPfThreads) {
      const int r = i / CH, ch = i % CH;
      const int tok = kt * kTok + r;
      const bool v = tok <= last_pos;
      const int t = v ? tok : 0;
      const int page = bt[t / m.P], slot = t % m.P;
      cp_async16(K + tile_off(r, ch), m.kv + m.kv_off(layer, page, 0, kvh, slot) + ch * 8, v);
      cp_async16(V + tile_off(r, ch), m.kv + m.kv_off(layer, page, 1, kvh, slot) + ch * 8, v);
    }
  };
  load_kv(0, 0);
  cp_async_commit();

  const float scale = rsqrtf((float)HD) * kLog2e;
  const int wq = warp * 16;
  const int qp[2] = {pos0 + wq + gr, pos0 + wq + gr + 8};
  const int warp_last = pos0 + wq + 15;
  float o[HD / 8][4];
#pragma unroll
  for (int t = 0; t < HD / 8; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
  float mrow[2] = {-FLT_MAX, -FLT_MAX}, lrow[2] = {0.f, 0.f};
  uint32_t qa[HD / 16][4];

  for (int kt = 0; kt < n_kt; ++kt) {
    if (kt + 1 < n_kt) load_kv(kt + 1, (kt + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (kt == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        ldsm_x4(qa[kk], sQ + tile_off_r<kPfRows>(wq + (lane & 15), kk * 2 + (lane >> 4)), false);
    }
    const int tb = kt * kTok;
    if (tb <= warp_last && wq < nrows) {
      const uint32_t K = sKV + (kt & 1) * 2 * Cfg::kTile, V = K + Cfg::kTile;
      float s[8][4];
#pragma unroll
      for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        const int mi = lane >> 3;
#pragma unroll
        for (int kg = 0; kg < 4; ++kg) {
          uint32_t bb[4];
          ldsm_x4(bb, K + tile_off(kg * 16 + (mi >> 1) * 8 + (lane & 7), kk * 2 + (mi & 1)), false);
          mma16816(s[2 * kg], qa[kk], bb[0], bb[1]);
          mma16816(s[2 * kg + 1], qa[kk], bb[2], bb[3]);
        }
      }
      float mx[2] = {-FLT_MAX, -FLT_MAX};
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const int tok = tb + j * 8 + tq * 2 + (q4 & 1);
          const float v = tok <= qp[q4 >> 1] ? s[j][q4] * scale : -FLT_MAX;
          s[j][q4] = v;
          mx[q4 >> 1] = fmaxf(mx[q4 >> 1], v);
        }
      float alpha[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
        mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
        const float mn = fmaxf(mrow[r], mx[r]);
        alpha[r] = (mrow[r] == -FLT_MAX) ? 0.f : exp2f(mrow[r] - mn);
        mrow[r] = mn;
      }
      float rsum[2] = {0.f, 0.f};
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const int r = q4 >> 1;
          const float p = (s[j][q4] == -FLT_MAX) ? 0.f : exp2f(s[j][q4] - mrow[r]);
          s[j][q4] = p;
          rsum[r] += p;
        }
#pragma unroll
      for (int r = 0; r < 2; ++r) lrow[r] = lrow[r] * alpha[r] + rsum[r];
#pragma unroll
      for (int nt = 0; nt < HD / 8; ++nt) {
        o[nt][0] *= alpha[0];
        o[nt][1] *= alpha[0];
        o[nt][2] *= alpha[1];
        o[nt][3] *= alpha[1];
      }
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint32_t pa[4] = {pack_bf16(s[2 * ks][0], s[2 * ks][1]), pack_bf16(s[2 * ks][2], s[2 * ks][3]),
                                pack_bf16(s[2 * ks + 1][0], s[2 * ks + 1][1]),
                                pack_bf16(s[2 * ks + 1][2], s[2 * ks + 1][3])};
#pragma unroll
        for (int nt2 = 0; nt2 < HD / 16; ++nt2) {
          const int mi = lane >> 3;
          uint32_t bb[4];
          ldsm_x4(bb, V + tile_off(ks * 16 + (mi & 1) * 8 + (lane & 7), nt2 * 2 + (mi >> 1)), true);
          mma16816(o[2 * nt2], pa, bb[0], bb[1]);
          mma16816(o[2 * nt2 + 1], pa, bb[2], bb[3]);
        }
      }
    }
    __syncthreads();  // the stage is reloaded two tiles later
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 1);
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 2);
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int rr = wq + gr + 8 * r;
    if (rr >= nrows) continue;
    const float inv = 1.f / lrow[r];
    bf16* dst = out + (size_t)(row0 + rr) * m.qd + head * HD + tq * 2;
#pragma unroll
    for (int nt = 0; nt < HD / 8; ++nt)
      *reinterpret_cast<uint32_t*>(dst + nt * 8) = pack_bf16(o[nt][2 * r] * inv, o[nt][2 * r + 1] * inv);
  }
}

template <int HD>
void launch_pf(const ModelDev& m, int layer, const bf16* q, bf16* out, const int4* blocks, int n_blocks,
               cudaStream_t s) {
  static bool init = false;
  if (!init) {
    AB_CUDA(cudaFuncSetAttribute(k_prefill_flash<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, PfCfg<HD>::kSmem));
    init = true;
  }
  k_prefill_flash<HD><<<dim3(n_blocks, m.hq), kPfThreads, PfCfg<HD>::kSmem, s>>>(m, layer, q, out, blocks);
}

}  // namespace

void launch_prefill_flash(const ModelDev& m, int layer, const bf16* q, bf16* out, const int4* blocks, int n_blocks,
                          cudaStream_t s) {
  if (n_blocks <= 0) return;
  if (m.hd == 128)
    launch_pf<128>(m, layer, q, out, blocks, n_blocks, s);
  else
    launch_pf<64>(m, layer, q, out, blocks, n_blocks, s);
}

void set_pdl_mask_attention(int mask) {
  AB_CUDA(cudaMemcpyToSymbol(c_pdl_mask, &mask, sizeof(int)));
}

void make_kv_tmap(CUtensorMap* map, const ModelDev& m) {
  AB_REQUIRE(m.gq <= kMergeRows, AB_ERR_CONFIG, "decode attention supports GQA groups of at most 8");
  AB_REQUIRE(m.P % 8 == 0 && (m.P <= kTok ? kTok % m.P == 0 : m.P % kTok == 0), AB_ERR_CONFIG,
             "page_size must divide 64 or be a multiple of 64");
  const int64_t rows = (int64_t)m.L * m.NP * 2 * m.hk * m.P;
  AB_REQUIRE(rows < (int64_t(1) << 31), AB_ERR_CONFIG, "KV pool too large for 32-bit TMA coordinates");
  if (m.P == kTok)  // one 4-D box per tile: K and V, every 64-wide half of the head dimension
    make_tmap_kv4(map, m.kv, rows, m.hd, (int64_t)m.hk * m.P, kTok);
  else
    make_tmap_bf16(map, m.kv, rows, m.hd, m.hd, 64, m.P < kTok ? m.P : kTok);
}

int decode_attention_ctas(const ModelDev& m) { return m.hd == 128 ? grid_t<128>() : grid_t<64>(); }

void launch_decode_attention(const CUtensorMap& map, const EngineDev& e, const ModelDev& m, int layer, const bf16* q,
                             bf16* out, float* part_o, float* part_ml, int max_splits, int chunk, cudaStream_t s) {
  (void)chunk;  // the split size of this iteration is on the device (ModelDev::att_ctl[0])
  AB_REQUIRE(max_splits <= kMaxSplits, AB_ERR_CONFIG, "too many KV splits per row for the decode attention");
  if (m.hd == 128)
    launch_t<128>(map, e, m, layer, q, out, part_o, part_ml, max_splits, s);
  else
    launch_t<64>(map, e, m, layer, q, out, part_o, part_ml, max_splits, s);
}

// The KV split size k_prep_decode picks for an iteration (host restatement for the test entry):
// about `items_per_cta` work items per persistent attention CTA, 64-token multiples, >= min_chunk.
static int default_chunk(const ModelDev& m, const int32_t* ctx, int rows, int min_chunk) {
  unsigned long long tot = 0;
  for (int i = 0; i < rows; ++i) tot += (unsigned long long)ctx[i];
  const unsigned long long ipc = (unsigned long long)attention_items_per_cta();
  const unsigned long long ctas = (unsigned long long)decode_attention_ctas(m);
  unsigned long long per = (tot * (unsigned long long)m.hk + ipc * ctas - 1) / (ipc * ctas);
  int ch = (int)std::min<unsigned long long>(per, 1ull << 30);
  ch = (ch + 63) & ~63;
  return std::max(ch, min_chunk);
}

}  // namespace ab

// Test entry (tests/test_attention_gpu.py): one launch of K3 over a caller-built single-layer paged
// pool.  Device pointers: q [rows, n_kv_heads * gq * head_dim] bf16; kv [n_pages][2][n_kv_heads]
// [page_size][head_dim] bf16 (the engine's per-layer page layout); block_table [rows, max_pages]
// int32 page ids; out [rows, n_kv_heads * gq * head_dim] bf16.  Host: ctx[rows] attended tokens per
// row (the row's own new token included).  chunk > 0 forces the KV split size (multiple of 64;
// ceil(ctx / chunk) <= 64 splits per row), chunk <= 0 uses the engine's per-iteration choice with
// min split -chunk (0: the engine's minimum).  *chunk_used receives the split size.
extern "C" int ab_debug_decode_attn(const void* q, const void* kv, int64_t n_pages, int page_size, int n_kv_heads,
                                    int head_dim, int gq, const int32_t* block_table, int max_pages,
                                    const int32_t* ctx, int rows, int chunk, void* out, int* chunk_used) {
  using namespace ab;
  try {
    AB_REQUIRE(rows >= 1 && rows <= 4096, AB_ERR_CONTRACT, "rows must lie in [1, 4096]");
    AB_REQUIRE(head_dim == 64 || head_dim == 128, AB_ERR_CONTRACT, "head_dim must be 64 or 128");
    AB_REQUIRE(gq >= 1 && gq <= kMergeRows, AB_ERR_CONTRACT, "GQA group must lie in [1, 8]");
    ModelDev m{};
    m.L = 1;
    m.hk = n_kv_heads;
    m.gq = gq;
    m.hq = gq * n_kv_heads;
    m.hd = head_dim;
    m.qd = m.hq * m.hd;
    m.kvd = m.hk * m.hd;
    m.P = page_size;
    m.MP = max_pages;
    m.NP = n_pages;
    m.kv = (bf16*)kv;
    int max_ctx = 1;
    for (int i = 0; i < rows; ++i) {
      AB_REQUIRE(ctx[i] >= 1 && ctx[i] <= max_pages * page_size, AB_ERR_CONTRACT, "context exceeds the block table");
      max_ctx = std::max(max_ctx, ctx[i]);
    }
    // the engine's minimum split: >= 256 tokens and <= 64 splits for the longest row (model_create)
    const int min_chunk = std::max(256, (ceil_div(max_ctx, kMaxSplits) + 63) / 64 * 64);
    const int ch = chunk > 0 ? chunk : default_chunk(m, ctx, rows, chunk < 0 ? -chunk : min_chunk);
    AB_REQUIRE(ch % 64 == 0, AB_ERR_CONTRACT, "chunk must be a multiple of 64");
    const int max_splits = ceil_div(max_ctx, ch);
    AB_REQUIRE(max_splits <= kMaxSplits, AB_ERR_CONTRACT, "more than 64 KV splits per row");
    if (chunk_used) *chunk_used = ch;
    // the work list k_prep_decode builds: (row, split) per row, exclusive prefix of split counts
    std::vector<int32_t> pos(rows), btrow(rows), prefix(rows + 1, 0), items;
    for (int i = 0; i < rows; ++i) {
      pos[i] = ctx[i] - 1;
      btrow[i] = i;
      const int ns = ceil_div(ctx[i], ch);
      prefix[i + 1] = prefix[i] + ns;
      for (int s2 = 0; s2 < ns; ++s2) items.push_back(i | (s2 << 16));
    }
    const int att_ctl[2] = {ch, 0};
    Ctl ctl{};
    ctl.b = rows;
    int32_t *d_pos, *d_btrow, *d_prefix, *d_items, *d_counter, *d_attctl;
    float *part_o, *part_ml;
    Ctl* d_ctl;
    AB_CUDA(cudaMalloc(&d_pos, sizeof(int32_t) * rows));
    AB_CUDA(cudaMalloc(&d_btrow, sizeof(int32_t) * rows));
    AB_CUDA(cudaMalloc(&d_prefix, sizeof(int32_t) * (rows + 1)));
    AB_CUDA(cudaMalloc(&d_items, sizeof(int32_t) * items.size()));
    AB_CUDA(cudaMalloc(&d_counter, sizeof(int32_t) * rows * m.hk));
    AB_CUDA(cudaMalloc(&d_attctl, sizeof(att_ctl)));
    AB_CUDA(cudaMalloc(&d_ctl, sizeof(Ctl)));
    AB_CUDA(cudaMalloc(&part_o, sizeof(float) * (size_t)rows * m.hq * max_splits * m.hd));
    AB_CUDA(cudaMalloc(&part_ml, sizeof(float) * (size_t)rows * m.hq * max_splits * 2));
    AB_CUDA(cudaMemcpy(d_pos, pos.data(), sizeof(int32_t) * rows, cudaMemcpyHostToDevice));
    AB_CUDA(cudaMemcpy(d_btrow, btrow.data(), sizeof(int32_t) * rows, cudaMemcpyHostToDevice));
    AB_CUDA(cudaMemcpy(d_prefix, prefix.data(), sizeof(int32_t) * (rows + 1), cudaMemcpyHostToDevice));
    AB_CUDA(cudaMemcpy(d_items, items.data(), sizeof(int32_t) * items.size(), cudaMemcpyHostToDevice));
    AB_CUDA(cudaMemset(d_counter, 0, sizeof(int32_t) * rows * m.hk));
    AB_CUDA(cudaMemcpy(d_attctl, att_ctl, sizeof(att_ctl), cudaMemcpyHostToDevice));
    AB_CUDA(cudaMemcpy(d_ctl, &ctl, sizeof(Ctl), cudaMemcpyHostToDevice));
    m.row_pos = d_pos;
    m.row_btrow = d_btrow;
    m.split_prefix = d_prefix;
    m.att_items = d_items;
    m.att_counter = d_counter;
    m.att_ctl = d_attctl;
    m.bt = const_cast<int32_t*>(block_table);
    EngineDev e{};
    e.ctl = d_ctl;
    CUtensorMap map;
    make_kv_tmap(&map, m);
    launch_decode_attention(map, e, m, 0, (const bf16*)q, (bf16*)out, part_o, part_ml, max_splits, ch, 0);
    AB_CUDA(cudaGetLastError());
    AB_CUDA(cudaDeviceSynchronize());
    // the split-combine arrival counters must have reset themselves
    std::vector<int32_t> cnt(rows * m.hk);
    AB_CUDA(cudaMemcpy(cnt.data(), d_counter, sizeof(int32_t) * cnt.size(), cudaMemcpyDeviceToHost));
    for (void* p : {(void*)d_pos, (void*)d_btrow, (void*)d_prefix, (void*)d_items, (void*)d_counter, (void*)d_attctl,
                    (void*)d_ctl, (void*)part_o, (void*)part_ml})
      cudaFree(p);
    for (int v : cnt) AB_REQUIRE(v == 0, AB_ERR_CUDA, "split-combine arrival counter did not reset");
    return AB_OK;
  } catch (const Error& err) {
    set_last_error(err.what());
    return err.code;
  } catch (const std::exception& err) {
    set_last_error(err.what());
    return AB_ERR_CUDA;
  }
}
