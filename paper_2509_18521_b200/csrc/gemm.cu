// K4: warp-specialised tcgen05 GEMM (sm_100a), TMA -> smem ring -> UMMA ->
// TMEM -> fused epilogue.
//
//   warp 0      TMA producer (one elected lane), STAGES-deep mbarrier ring
//   warp 1      TMEM allocator + MMA issuer (one lane, tcgen05.mma kind::f16)
//   warps 2-5   epilogue: tcgen05.ld 32x32b -> bias / residual / SwiGLU -> global
//
// D^T tile [128 weight rows x BN activation rows] accumulates in TMEM
// (lane = weight row, column = activation row), so the epilogue thread that
// owns TMEM lane t writes output feature n0+t for every activation row:
// a warp stores 32 consecutive features of one row per instruction.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "gemm.cuh"

namespace ab {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // one 128-byte swizzle atom of bf16
constexpr int kThreads = 192;
constexpr int kMaxBN = 256;
constexpr int kWBytes = kBM * kBK * 2;           // 16 KB weight tile per stage
constexpr int kRingBytes = 192 * 1024;           // TMA ring, carved into stages per launch
constexpr int kXchgBytes = 64 * 32 * 4;          // SwiGLU gate/up exchange
constexpr int kMaxStages = 12;
constexpr int kTmemCols = 2 * kMaxBN;            // double-buffered accumulator
constexpr int kSmem = 1024 + kRingBytes + kXchgBytes + 512;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int x, int y,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "l"(policy)
      : "memory");
}

// K-major operand, 128-byte swizzle, 8-row core groups 1024 bytes apart.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  return ((uint64_t)((saddr >> 4) & 0x3FFFu)) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float silu(float x) { return x / (1.f + __expf(-x)); }

// Per-launch schedule, chosen on the device from the live row count so one
// captured graph serves every batch size: activation tile width BN (the UMMA
// N), deterministic split-K factor, and the unit count of the persistent loop.
struct Sched {
  int bn, splits, m_tiles, n_tiles, units, nk, stages, stage_bytes;
};

// Cost model (SM clocks per CTA-wave): a 64-deep K block costs the larger of
// its MMA time (128 x BN x 64 MACs at ~4096 MAC/clk) and its operand fill
// (16 KB weights + BN x 128 B activations at ~64 B/clk from L2); split-K adds
// the partial-tile round trip; a CTA's last epilogue is exposed.
__device__ __forceinline__ Sched choose_sched(int rows, int N, int K, int max_bn, int max_splits, bool force,
                                              int grid, int64_t ws_cap) {
  Sched best{};
  best.units = 0;
  const int n_tiles = N / kBM, nk = K / kBK;
  int64_t best_cost = INT64_MAX;
  for (int bn = max_bn; bn >= 32; bn >>= 1) {
    const int m_tiles = (rows + bn - 1) / bn;
    const int tiles = n_tiles * m_tiles;
    for (int s = 1; s <= max_splits; ++s) {
      if (s > 1 && (tiles * s > 2 * grid || nk / s < 2 || (int64_t)s * rows * N > ws_cap)) break;
      const int units = tiles * s;
      const int64_t waves = (units + grid - 1) / grid;
      const int64_t kb = (nk + s - 1) / s;
      const int64_t per_kb = max(2 * bn, (kWBytes + 128 * bn) / 64);
      const int64_t split_cost = s > 1 ? (int64_t)bn * 40 : 0;
      const int64_t epi = (int64_t)min(bn, rows) * 12;
      const int64_t cost = waves * (kb * per_kb + 700 + split_cost) + epi;
      if (cost < best_cost) {
        best_cost = cost;
        best.bn = bn;
        best.splits = s;
        best.m_tiles = m_tiles;
        best.n_tiles = n_tiles;
        best.units = units;
        best.nk = nk;
      }
    }
    if (force) break;
  }
  best.stage_bytes = kWBytes + best.bn * kBK * 2;
  best.stages = min(kMaxStages, kRingBytes / best.stage_bytes);
  return best;
}

template <int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap ta, int N, int K,
              int M_cap, const int* __restrict__ rows_dev, const int* __restrict__ stop_dev, void* __restrict__ out,
              int64_t ldo, const __nv_bfloat16* __restrict__ bias, float* __restrict__ ws, int* __restrict__ cnt,
              int max_splits, int max_bn, int force_bn) {
  if (stop_dev && *stop_dev) return;
  const int rows = rows_dev ? min(*rows_dev, M_cap) : M_cap;
  if (rows <= 0) return;
  const Sched sc = choose_sched(rows, N, K, max_bn, (ws && cnt) ? max_splits : 1, force_bn != 0, gridDim.x,
                                kGemmWsElems);
  if ((int)blockIdx.x >= sc.units) return;

  extern __shared__ uint8_t smem_raw[];
  __shared__ int s_last_split;
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* xchg = reinterpret_cast<float*>(ring + kRingBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kRingBytes + kXchgBytes);
  uint64_t* empty = full + kMaxStages;
  uint64_t* tmem_full = empty + kMaxStages;  // [2]
  uint64_t* tmem_empty = tmem_full + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nst = sc.stages, bn = sc.bn, per_n = sc.m_tiles * sc.splits;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tw)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  auto unit_coords = [&](int u, int& n0, int& m0, int& z, int& kb0, int& kb1) {
    const int nt = u / per_n, r = u % per_n;
    n0 = nt * kBM;
    m0 = (r / sc.splits) * bn;
    z = r % sc.splits;
    kb0 = (int)(((int64_t)sc.nk * z) / sc.splits);
    kb1 = (int)(((int64_t)sc.nk * (z + 1)) / sc.splits);
  };

  if (warp == 0) {
    if (lane == 0) {
      // weights stream through once per launch unless several row tiles share them
      uint64_t pol_w, pol_a;
      if (sc.m_tiles > 1)
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_w));
      else
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_w));
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_a));
      int g = 0;
      for (int u = blockIdx.x; u < sc.units; u += gridDim.x) {
        int n0, m0, z, kb0, kb1;
        unit_coords(u, n0, m0, z, kb0, kb1);
        const int nbox = (min(bn, rows - m0) + 31) >> 5;  // skip activation boxes past the live rows
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % nst;
          const uint32_t ph = (g / nst) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = ring + s * sc.stage_bytes;
          mbar_expect_tx(&full[s], kWBytes + nbox * 32 * kBK * 2);
          tma_load_2d(&tw, &full[s], st, kb * kBK, n0, pol_w);
          for (int j = 0; j < nbox; ++j)
            tma_load_2d(&ta, &full[s], st + kWBytes + j * 32 * kBK * 2, kb * kBK, m0 + 32 * j, pol_a);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(bn >> 3) << 17) |
                             ((uint32_t)(kBM >> 4) << 24);
      const uint32_t ring_s = smem_u32(ring);
      int g = 0, t = 0;
      for (int u = blockIdx.x; u < sc.units; u += gridDim.x, ++t) {
        int n0, m0, z, kb0, kb1;
        unit_coords(u, n0, m0, z, kb0, kb1);
        const int acc = t & 1;
        mbar_wait(&tmem_empty[acc], ((t >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + (uint32_t)(acc * kMaxBN);
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % nst;
          mbar_wait(&full[s], (g / nst) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = ring_s + s * sc.stage_bytes;
          const uint64_t da = umma_desc(sa), db = umma_desc(sa + kWBytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)  // +32 bytes along K inside the swizzle atom
            umma_bf16(d, da + 2 * k, db + 2 * k, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        umma_commit(&tmem_full[acc]);
      }
    }
  } else {
    // epilogue warps 2..5 -> TMEM lane quadrants 2,3,0,1
    const int quad = warp & 3;
    const int lrow = quad * 32 + lane;  // TMEM lane = weight row within the tile
    const bool split = sc.splits > 1;
    int t = 0;
    for (int u = blockIdx.x; u < sc.units; u += gridDim.x, ++t) {
      int n0, m0, z, kb0, kb1;
      unit_coords(u, n0, m0, z, kb0, kb1);
      const int acc = t & 1;
      mbar_wait(&tmem_full[acc], (t >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * kMaxBN);
      const int live = min(bn, rows - m0);  // activation rows of this tile that exist
      auto release = [&]() {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&tmem_empty[acc]);
      };
      bool do_epi = true;
      if (split) {
        // deterministic split-K: partial tile -> workspace[split]; the last CTA of
        // the tile sums the partials in split order and runs the epilogue
        const int n = n0 + lrow;
        for (int c0 = 0; c0 < live; c0 += 32) {
          float v[32];
          tmem_ld32(taddr + c0, v);
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const int m = m0 + c0 + c;
            if (m < rows) ws[((int64_t)z * rows + m) * N + n] = v[c];
          }
        }
        release();
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 64) {
          const int tile = u / sc.splits;
          const int old = atomicAdd(&cnt[tile], 1);
          s_last_split = (old == sc.splits - 1);
          if (s_last_split) cnt[tile] = 0;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        do_epi = s_last_split != 0;
        asm volatile("bar.sync 1, 128;" ::: "memory");  // s_last_split is reused by the next unit
        if (!do_epi) continue;
        __threadfence();
      }
      auto fetch = [&](int c0, float (&v)[32]) {
        if (!split) {
          tmem_ld32(taddr + c0, v);
          return;
        }
        const int n = n0 + lrow;
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const int m = m0 + c0 + c;
          float a = 0.f;
          if (m < rows)
            for (int zz = 0; zz < sc.splits; ++zz) a += __ldcg(&ws[((int64_t)zz * rows + m) * N + n]);
          v[c] = a;
        }
      };
      if constexpr (EPI == kEpiSwiGLU) {
        // lanes 0-63: gate rows, lanes 64-127: up rows of the same 64 features
        const int j = (n0 >> 1) + (lrow & 63);
        for (int c0 = 0; c0 < live; c0 += 32) {
          float v[32];
          fetch(c0, v);
          if (lrow >= 64) {
#pragma unroll
            for (int c = 0; c < 32; ++c) xchg[c * 64 + (lrow - 64)] = v[c];
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (lrow < 64) {
            __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(out);
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              const int m = m0 + c0 + c;
              if (m < rows) o[(int64_t)m * ldo + j] = __float2bfloat16(silu(v[c]) * xchg[c * 64 + lrow]);
            }
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
        }
      } else {
        const int n = n0 + lrow;
        float bv = 0.f;
        if (EPI == kEpiBF16 && bias != nullptr) bv = __bfloat162float(bias[n]);
        for (int c0 = 0; c0 < live; c0 += 32) {
          float v[32];
          fetch(c0, v);
          if constexpr (EPI == kEpiAddF32) {
            // residual add: issue all 32 loads before any store (independent, in flight together)
            float* o = reinterpret_cast<float*>(out);
            float old[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              const int m = m0 + c0 + c;
              old[c] = m < rows ? __ldcg(o + (int64_t)m * ldo + n) : 0.f;
            }
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              const int m = m0 + c0 + c;
              if (m < rows) o[(int64_t)m * ldo + n] = old[c] + v[c];
            }
          } else {
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              const int m = m0 + c0 + c;
              if (m < rows) {
                if constexpr (EPI == kEpiBF16) {
                  reinterpret_cast<__nv_bfloat16*>(out)[(int64_t)m * ldo + n] = __float2bfloat16(v[c] + bv);
                } else {
                  reinterpret_cast<float*>(out)[(int64_t)m * ldo + n] = v[c];
                }
              }
            }
          }
        }
      }
      if (!split) release();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

// ---------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    AB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    AB_REQUIRE(p != nullptr && q == cudaDriverEntryPointSuccess, AB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

void make_map(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  AB_REQUIRE(r == CUDA_SUCCESS, AB_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
}

template <int EPI>
void launch_t(const GemmPlan& p, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    AB_CUDA(cudaFuncSetAttribute(k_gemm_tc<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    attr = true;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    AB_CUDA(cudaGetDevice(&dev));
    AB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const int zs = (p.ws && p.cnt) ? p.max_splits : 1;
  // persistent: one CTA per SM (never more CTAs than the largest possible unit count)
  const int64_t max_units = (int64_t)(p.N / kBM) * ceil_div(p.M_cap, 32) * zs;
  const int grid = (int)std::min<int64_t>(sms, max_units);
  k_gemm_tc<EPI><<<grid, kThreads, kSmem, s>>>(p.tw, p.ta, p.N, p.K, p.M_cap, p.rows_dev, p.stop_dev, p.out, p.ldo,
                                               p.bias, p.ws, p.cnt, zs, p.BN, p.force_bn ? 1 : 0);
}

}  // namespace

void gemm_plan(GemmPlan& p, const __nv_bfloat16* W, int N, int K, const __nv_bfloat16* A, int M_cap, int64_t lda,
               int BN, int epi, void* out, int64_t ldo, const __nv_bfloat16* bias, const int* rows_dev,
               const int* stop_dev, float* ws, int* cnt, int max_splits) {
  AB_REQUIRE(K % kBK == 0, AB_ERR_CONFIG, "GEMM K must be a multiple of 64");
  AB_REQUIRE(max_splits >= 1 && max_splits <= 16, AB_ERR_CONFIG, "GEMM max_splits must be in [1, 16]");
  AB_REQUIRE(max_splits == 1 || (ws && cnt), AB_ERR_CONFIG, "split-K needs a workspace");
  p.ws = ws;
  p.cnt = cnt;
  p.max_splits = max_splits;
  AB_REQUIRE(N % kBM == 0, AB_ERR_CONFIG, "GEMM N must be a multiple of 128");
  AB_REQUIRE(BN == 32 || BN == 64 || BN == 128 || BN == 256, AB_ERR_CONFIG, "GEMM BN must be 32/64/128/256");
  p.N = N;
  p.K = K;
  p.M_cap = M_cap;
  p.BN = BN;
  p.epi = epi;
  p.out = out;
  p.ldo = ldo;
  p.bias = bias;
  p.rows_dev = rows_dev;
  p.stop_dev = stop_dev;
  make_map(&p.tw, W, N, K, K, kBM);
  make_map(&p.ta, A, M_cap, K, lda, 32);  // activation tiles are loaded as 32-row boxes
}

void make_tmap_bf16(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_cols,
                    int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  AB_REQUIRE(r == CUDA_SUCCESS, AB_ERR_CUDA, "cuTensorMapEncodeTiled (KV) failed (" + std::to_string((int)r) + ")");
}

void gemm_launch(const GemmPlan& p, cudaStream_t s) {
  switch (p.epi) {
    case kEpiBF16: launch_t<kEpiBF16>(p, s); break;
    case kEpiF32: launch_t<kEpiF32>(p, s); break;
    case kEpiAddF32: launch_t<kEpiAddF32>(p, s); break;
    default: launch_t<kEpiSwiGLU>(p, s); break;
  }
}

}  // namespace ab

// Timing entry (tools/gemm_bench.py): median device time of `reps` launches,
// L2 flushed (256 MB memset) between launches, plan built outside the timing.
extern "C" int ab_debug_gemm_time(const void* W, const void* A, void* out, const void* bias, int N, int K, int M,
                                  int BN, int epi, int reps, float* ms_out) {
  try {
    static float* ws = nullptr;
    static int* cnt = nullptr;
    static void* flush = nullptr;
    // epi bit 4: split-K allowed (up to 8 splits); bit 5: automatic tile width (BN = max)
    const int max_splits = (epi & 16) ? 8 : 1;
    const bool force = (epi & 32) == 0;
    epi &= 15;
    if (!ws) {
      AB_CUDA(cudaMalloc(&ws, sizeof(float) * ab::kGemmWsElems));
      AB_CUDA(cudaMalloc(&cnt, sizeof(int) * ab::kGemmCounters));
      AB_CUDA(cudaMemset(cnt, 0, sizeof(int) * ab::kGemmCounters));
      AB_CUDA(cudaMalloc(&flush, size_t(256) << 20));
    }
    ab::GemmPlan p;
    ab::gemm_plan(p, (const __nv_bfloat16*)W, N, K, (const __nv_bfloat16*)A, M, K, BN, epi, out,
                  epi == ab::kEpiSwiGLU ? N / 2 : N, (const __nv_bfloat16*)bias, nullptr, nullptr,
                  max_splits > 1 ? ws : nullptr, max_splits > 1 ? cnt : nullptr, max_splits);
    p.force_bn = force;
    ab::gemm_launch(p, 0);  // warm: kernel attributes, TMA descriptors
    std::vector<float> t(reps);
    cudaEvent_t a, b;
    AB_CUDA(cudaEventCreate(&a));
    AB_CUDA(cudaEventCreate(&b));
    for (int r = 0; r < reps; ++r) {
      AB_CUDA(cudaMemsetAsync(flush, r & 0xff, size_t(256) << 20, 0));
      AB_CUDA(cudaEventRecord(a, 0));
      ab::gemm_launch(p, 0);
      AB_CUDA(cudaEventRecord(b, 0));
      AB_CUDA(cudaEventSynchronize(b));
      AB_CUDA(cudaEventElapsedTime(&t[r], a, b));
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    std::sort(t.begin(), t.end());
    *ms_out = t[reps / 2];
    return AB_OK;
  } catch (const ab::Error& e) {
    ab::set_last_error(e.what());
    return e.code;
  }
}

// Test entry: one GEMM on caller-provided device buffers (tests/test_kernels_gpu.py).
extern "C" int ab_debug_gemm(const void* W, const void* A, void* out, const void* bias, int N, int K, int M, int BN,
                             int epi) {
  // epi >= 16: the same epilogue (epi - 16) with split-K enabled (up to 8 splits)
  try {
    static float* ws = nullptr;
    static int* cnt = nullptr;
    // epi bit 4: split-K allowed (up to 8 splits); bit 5: automatic tile width (BN = max)
    const int max_splits = (epi & 16) ? 8 : 1;
    const bool force = (epi & 32) == 0;
    epi &= 15;
    if (max_splits > 1 && !ws) {
      AB_CUDA(cudaMalloc(&ws, sizeof(float) * ab::kGemmWsElems));
      AB_CUDA(cudaMalloc(&cnt, sizeof(int) * ab::kGemmCounters));
      AB_CUDA(cudaMemset(cnt, 0, sizeof(int) * ab::kGemmCounters));
    }
    ab::GemmPlan p;
    ab::gemm_plan(p, (const __nv_bfloat16*)W, N, K, (const __nv_bfloat16*)A, M, K, BN, epi, out,
                  epi == ab::kEpiSwiGLU ? N / 2 : N, (const __nv_bfloat16*)bias, nullptr, nullptr,
                  max_splits > 1 ? ws : nullptr, max_splits > 1 ? cnt : nullptr, max_splits);
    p.force_bn = force;
    ab::gemm_launch(p, 0);
    AB_CUDA(cudaGetLastError());
    AB_CUDA(cudaDeviceSynchronize());
    return AB_OK;
  } catch (const ab::Error& e) {
    ab::set_last_error(e.what());
    return e.code;
  }
}
