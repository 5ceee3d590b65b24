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
constexpr int kSmemBudget = 200 * 1024;

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

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

// K-major operand, 128-byte swizzle, 8-row core groups 1024 bytes apart.
__device__ __forceinline__ uint64_t umma_desc(const void* smem) {
  const uint64_t addr = smem_u32(smem);
  return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
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

template <int BN>
struct Cfg {
  static constexpr int kWBytes = kBM * kBK * 2;
  static constexpr int kABytes = BN * kBK * 2;
  static constexpr int kStageBytes = kWBytes + kABytes;
  // decode tiles (BN <= 128) fit two CTAs per SM; prefill tiles take the whole SM for a deep ring
  static constexpr int kBudget = kSmemBudget;
  static constexpr int kMinBlocks = 1;
  static constexpr int kStages = (kBudget - 2048) / kStageBytes > 8 ? 8 : (kBudget - 2048) / kStageBytes;
  static constexpr int kTmemCols = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  static constexpr int kSmem = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
  // kind::f16: D=f32 (bit 4), A=bf16 (bits 7-9 = 1), B=bf16 (bits 10-12 = 1), K-major both,
  // N>>3 at bits 17-22, M>>4 at bits 24-28.
  static constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                     ((uint32_t)(kBM >> 4) << 24);
};

__device__ __forceinline__ float silu(float x) { return x / (1.f + __expf(-x)); }

template <int BN, int EPI>
__global__ void __launch_bounds__(kThreads, Cfg<BN>::kMinBlocks)
    k_gemm_tc(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap ta, int N, int K,
              int M_cap, const int* __restrict__ rows_dev, const int* __restrict__ stop_dev, void* __restrict__ out,
              int64_t ldo, const __nv_bfloat16* __restrict__ bias, float* __restrict__ ws, int* __restrict__ cnt,
              int max_splits, int target_ctas) {
  using C = Cfg<BN>;
  if (stop_dev && *stop_dev) return;
  const int rows = rows_dev ? min(*rows_dev, M_cap) : M_cap;
  const int n0 = blockIdx.x * kBM, m0 = blockIdx.y * BN;
  if (m0 >= rows) return;
  // split-K sized from the live row count: enough CTAs to cover the SMs,
  // at least two 64-wide K blocks per split
  const int nk_all = K / kBK;
  const int tiles = gridDim.x * ((rows + BN - 1) / BN);
  // split only when the tiles leave most SMs idle (floor: never more CTAs than SMs)
  int splits = max(1, target_ctas / tiles);
  splits = min(splits, min(max_splits, max(1, nk_all / 2)));
  while (splits > 1 && (int64_t)splits * rows * N > kGemmWsElems) --splits;
  if ((int)blockIdx.z >= splits) return;
  const int kb0 = (int)(((int64_t)nk_all * blockIdx.z) / splits);
  const int kb1 = (int)(((int64_t)nk_all * (blockIdx.z + 1)) / splits);

  extern __shared__ uint8_t smem_raw[];
  __shared__ int s_last_split;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = base;
  uint8_t* sA = base + C::kStages * C::kWBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + C::kStages * C::kStageBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tmem_full = empty + C::kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tw)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const int nk = kb1 - kb0;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % C::kStages;
        const uint32_t ph = (kb / C::kStages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], C::kStageBytes);
        tma_load_2d(&tw, &full[s], sW + s * C::kWBytes, (kb0 + kb) * kBK, n0);
        tma_load_2d(&ta, &full[s], sA + s * C::kABytes, (kb0 + kb) * kBK, m0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % C::kStages;
        const uint32_t ph = (kb / C::kStages) & 1;
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t da = umma_desc(sW + s * C::kWBytes), db = umma_desc(sA + s * C::kABytes);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k)  // +32 bytes along K inside the swizzle atom
          umma_bf16(tmem, da + 2 * k, db + 2 * k, C::kIdesc, (kb | k) != 0);
        umma_commit(&empty[s]);
      }
      umma_commit(tmem_full);
    }
  } else {
    // epilogue warps 2..5 -> TMEM lane quadrants 2,3,0,1
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int quad = warp & 3;
    const int lrow = quad * 32 + lane;  // TMEM lane = weight row within the tile
    const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16);
    const bool split = splits > 1;
    bool do_epi = true;
    if (split) {
      // deterministic split-K: partial tile -> workspace[split]; the last CTA of
      // the tile sums the partials in split order and runs the epilogue
      const int n = n0 + lrow;
      for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        tmem_ld32(taddr + c0, v);
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const int m = m0 + c0 + c;
          if (m < rows) ws[((int64_t)blockIdx.z * rows + m) * N + n] = v[c];
        }
      }
      __threadfence();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 64) {
        const int tile = blockIdx.y * gridDim.x + blockIdx.x;
        const int old = atomicAdd(&cnt[tile], 1);
        s_last_split = (old == splits - 1);
        if (s_last_split) cnt[tile] = 0;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      do_epi = s_last_split != 0;
      if (do_epi) __threadfence();
    }
    auto fetch = [&](int c0, float (&v)[32]) {
      if (!split) {
        tmem_ld32(taddr + c0, v);
        return;
      }
      const int n = n0 + lrow;
#pragma unroll 4
      for (int c = 0; c < 32; ++c) {
        const int m = m0 + c0 + c;
        float acc = 0.f;
        if (m < rows)
          for (int z = 0; z < splits; ++z) acc += __ldcg(&ws[((int64_t)z * rows + m) * N + n]);
        v[c] = acc;
      }
    };
    if (!do_epi) {
    } else if constexpr (EPI == kEpiSwiGLU) {
      // lanes 0-63: gate rows, lanes 64-127: up rows of the same 64 features
      float* xchg = reinterpret_cast<float*>(sW);  // pipeline smem is idle now
      const int j = (n0 >> 1) + (lrow & 63);
      for (int c0 = 0; c0 < BN; c0 += 32) {
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
      if (EPI == kEpiBF16 && bias != nullptr && n < N) bv = __bfloat162float(bias[n]);
      for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        fetch(c0, v);
        if (n < N) {
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
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::kTmemCols));
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

template <int BN, int EPI>
void launch_t(const GemmPlan& p, cudaStream_t s) {
  using C = Cfg<BN>;
  static bool attr = false;
  if (!attr) {
    AB_CUDA(cudaFuncSetAttribute(k_gemm_tc<BN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    attr = true;
  }
  static int target = 0;
  if (!target) {
    int dev = 0, sms = 0;
    AB_CUDA(cudaGetDevice(&dev));
    AB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    target = sms * C::kMinBlocks;
  }
  const int zs = (p.ws && p.cnt) ? p.max_splits : 1;
  dim3 grid(ceil_div(p.N, kBM), ceil_div(p.M_cap, BN), zs);
  k_gemm_tc<BN, EPI><<<grid, kThreads, C::kSmem, s>>>(p.tw, p.ta, p.N, p.K, p.M_cap, p.rows_dev, p.stop_dev, p.out,
                                                      p.ldo, p.bias, p.ws, p.cnt, zs, target);
}

template <int BN>
void launch_bn(const GemmPlan& p, cudaStream_t s) {
  switch (p.epi) {
    case kEpiBF16: launch_t<BN, kEpiBF16>(p, s); break;
    case kEpiF32: launch_t<BN, kEpiF32>(p, s); break;
    case kEpiAddF32: launch_t<BN, kEpiAddF32>(p, s); break;
    default: launch_t<BN, kEpiSwiGLU>(p, s); break;
  }
}

}  // namespace

void gemm_plan(GemmPlan& p, const __nv_bfloat16* W, int N, int K, const __nv_bfloat16* A, int M_cap, int64_t lda,
               int BN, int epi, void* out, int64_t ldo, const __nv_bfloat16* bias, const int* rows_dev,
               const int* stop_dev, float* ws, int* cnt, int max_splits) {
  AB_REQUIRE(K % kBK == 0, AB_ERR_CONFIG, "GEMM K must be a multiple of 64");
  AB_REQUIRE(max_splits >= 1 && max_splits <= 16, AB_ERR_CONFIG, "GEMM max_splits must be in [1, 16]");
  AB_REQUIRE(max_splits == 1 || (ws && cnt), AB_ERR_CONFIG, "split-K needs a workspace");
  AB_REQUIRE((int64_t)ceil_div(N, kBM) * ceil_div(M_cap, BN) <= kGemmCounters, AB_ERR_CONFIG,
             "GEMM tile count exceeds the split-K counter array");
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
  make_map(&p.ta, A, M_cap, K, lda, BN);
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
  switch (p.BN) {
    case 32: launch_bn<32>(p, s); break;
    case 64: launch_bn<64>(p, s); break;
    case 128: launch_bn<128>(p, s); break;
    default: launch_bn<256>(p, s); break;
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
    const int max_splits = epi >= 16 ? 8 : 1;
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
    const int max_splits = epi >= 16 ? 8 : 1;
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
    ab::gemm_launch(p, 0);
    AB_CUDA(cudaGetLastError());
    AB_CUDA(cudaDeviceSynchronize());
    return AB_OK;
  } catch (const ab::Error& e) {
    ab::set_last_error(e.what());
    return e.code;
  }
}
