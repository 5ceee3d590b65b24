// tcgen05 GEMM for the decoder projections (K4).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <vector>

#include "common.cuh"

namespace ab {

enum GemmEpi : int {
  kEpiBF16 = 0,     // out bf16 = acc (+ bias)
  kEpiF32 = 1,      // out f32 = acc
  kEpiAddF32 = 2,   // out f32 += acc   (residual stream)
  kEpiSwiGLU = 3,   // weight rows interleaved in 64-row halves: out bf16[j] = silu(gate_j) * up_j
};

// D[M, N] = A[M, K] . W[N, K]^T, A = activations (rows dynamic), W = weights.
// Swap-AB on the tensor core: the 128-row UMMA M side walks W, the UMMA N
// side (BN) walks the activation rows, so small decode batches still issue
// full 128-wide MMAs.
struct GemmPlan {
  // 3-D TMA views [K/64][rows][64] (128-byte swizzle): one operation = two 64-deep k-blocks
  CUtensorMap tw3, tw3_256;                 // weights [N, K]: 128- / 256-row boxes
  CUtensorMap ta3_32, ta3_64, ta3, ta3_256;  // activations [M_cap, K]: 32- / 64- / 128- / 256-row boxes
  CUtensorMap tx_ns, tx_sw;                  // fp32 residual output: {32 x 128} swizzled / {128 x 32} boxes
  int N = 0, K = 0, M_cap = 0, BN = 0, epi = 0;  // BN: largest activation tile the kernel may pick
  void* out = nullptr;
  int64_t ldo = 0;
  const __nv_bfloat16* bias = nullptr;
  const int* rows_dev = nullptr;  // live row count on device (nullptr: M_cap)
  const int* stop_dev = nullptr;  // engine stop flag (nullptr: never stop)
  // deterministic split-K inside a thread-block cluster of `cluster` CTAs (1 = none):
  // the schedule table picks split = cluster (one tile per cluster) or none per row count
  int cluster = 1;
  bool pair = false;    // CTA-pair plan (cta_group::2, cluster of 2)
  bool nondet = false;  // fp32 residual plans may split K with TMA reduce-add (order not fixed)
  int grid = 0;  // persistent CTAs (a multiple of cluster)
  // tests: > 0 forces swap-AB with exactly `force` activation rows per tile, < 0 forces the
  // no-swap schedule with -force weight rows per tile, 0 = on-device choice
  int force = 0;
  const int* sched = nullptr;  // device table: packed schedule per live row count [0, M_cap]
  bool idle = false;           // the table is all zeros: gemm_launch skips the launch
  std::vector<int> host_tab;   // host copy of the schedule table (row counts known on the host)
  bool early_trigger = false;  // launch_dependents right after setup (successor = a small kernel)
  double extra_us = 0;         // autotuning: fixed cost added to this plan's measured time
  // autotuning: a follow-up kernel this plan needs (timed together with the GEMM), e.g. the SwiGLU
  // pass of the gate-up workspace plan; follow_arg is its extra operand
  void (*follow)(const GemmPlan&, cudaStream_t) = nullptr;
  void* follow_arg = nullptr;
};

void gemm_plan(GemmPlan& p, const __nv_bfloat16* W, int N, int K, const __nv_bfloat16* A, int M_cap, int64_t lda,
               int BN, int epi, void* out, int64_t ldo, const __nv_bfloat16* bias, const int* rows_dev,
               const int* stop_dev, int cluster = 1, bool pair = false);
// Split the row range between two plans of the same product (e.g. a cluster-8 split-K plan and a
// cluster-2 plan): each row count runs on the plan the cost model expects to be faster, the other
// launch exits at once.  Both plans are launched every time.
void gemm_partition(GemmPlan& a, GemmPlan& b);
void gemm_launch(const GemmPlan& p, cudaStream_t s);
// Launch only if the plan has work at `rows` (prefill: the row count is known on the host).
void gemm_launch_rows(const GemmPlan& p, int rows, cudaStream_t s);
void set_pdl_mask_gemm(int mask);  // early launch_dependents (programmatic dependent launch) per kernel class
// Autotuning (engine creation): the fixed schedule codes valid for the plan at `rows`; the
// median device time (us) of `reps` launches of one code at `rows` (L2 flushed before each by
// a memset of `flush`); install a per-row-count table built from measurements.
std::vector<int> gemm_candidates(const GemmPlan& p, int rows);
double gemm_time_code(const GemmPlan& p, int rows, int code, int reps, void* flush, size_t flush_bytes,
                      cudaStream_t s);
void gemm_set_table(GemmPlan& p, const std::vector<int>& tab);
// The cost model's schedule for the plan at `rows` (0: no valid schedule).
int gemm_default_code(const GemmPlan& p, int rows);
// Evict L2 for timing by reading `bytes` (> L2) of `buf` (reads leave no dirty lines behind).
void l2_flush(void* buf, size_t bytes, cudaStream_t s);
// Rebuild the plan's schedule table (force: see GemmPlan::force).
void gemm_set_schedule(GemmPlan& p, int force);

// 2-D bf16 TMA map: [rows, cols] with leading dimension `ld` elements, box {box_cols, box_rows},
// 128-byte swizzle (box_cols * 2 must be <= 128).
void make_tmap_bf16(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_cols,
                    int box_rows);
// 4-D bf16 KV-pool map {64, rows, hd / 64, k|v} (V `v_rows` rows after K), box {64, box_rows, hd / 64, 2},
// 128-byte swizzle: one operation loads a tile's K and V, both halves of each row.
void make_tmap_kv4(CUtensorMap* m, const void* ptr, int64_t rows, int hd, int64_t v_rows, int box_rows);

}  // namespace ab
