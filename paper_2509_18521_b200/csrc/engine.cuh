// Internal engine state shared by the engine, model and sampler translation units.
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"

namespace ab {

// NVTX range around a C-ABI call / engine phase (nsys / ncu --nvtx timelines; header-only NVTX3,
// a no-op unless a tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Device control block: one per engine, lives in device memory; copied to a
// pinned mirror at the host's polling points.
struct Ctl {
  int32_t b;                  // active slots (the live batch)
  int32_t stop;               // nonzero: every iteration kernel is a no-op
  int32_t stop_reason;        // AB_RUN_* or -1
  int32_t error;              // contract error code (see kErr*)
  int32_t error_handle;
  int32_t q_head, q_tail;     // FIFO ring indices (monotonic; slot = idx % Q)
  int32_t n_events, n_admits; // logged in the current run
  int32_t use_trigger, trigger_mode, stop_on_event, n_target, group_size;
  int32_t iters_to_next;      // trace mode: iterations until the next finish (-1 unknown)
  int32_t new_groups;         // scratch: groups completed in this iteration
  int64_t version;
  int64_t iteration_index, cumulative_tokens;
  int64_t run_iters, max_iters;
  int64_t completed_groups, completed_samples;
  int64_t kv_free_top;        // transformer: free-page stack top
  int64_t kv_fail;            // transformer: allocation failures
  uint64_t clock_ns;          // scratch for clock reads
  // data-parallel lockstep (dp_world > 1): this rank's share of the iteration, published to every
  // peer by k_dp_exchange, and the exchange epoch (same on every rank: one exchange per global
  // iteration)
  int32_t dp_done;            // the global stop of this run is decided: no more exchanges
  int32_t dp_pad;
  int64_t dp_epoch;
  int64_t dp_groups, dp_samples, dp_b, dp_next, dp_hint;
};

enum : int32_t {
  kErrNone = 0, kErrVersion = 1, kErrAtStop = 2, kErrNoTarget = 3, kErrOutOfKV = 4,
  kErrPeer = 5,      // data-parallel: another rank's iteration failed
  kErrDpTimeout = 6  // data-parallel: a peer's exchange record did not arrive in time
};

// internal stop reason: k_admit met a queued sample whose KV must be re-prefilled first (KV
// re-prefill mode, one engine): the host rebuilds the next admissions' KV and resumes the run
constexpr int32_t kRunNeedPrefill = 4;

struct Model;  // transformer (model.cu)

// POD view passed by value to kernels.
struct EngineDev {
  Ctl* ctl;
  int S, Q, H, L, G_cap;
  int stop_mode, model_kind, n_symbols, l_max, record;
  int n_eos;
  int eos[8];
  int32_t* slot_handle;
  int32_t* slot_tmp;
  int32_t* slot_finish;  // reason+1, 0 = continues
  int32_t* slot_token;   // token sampled this iteration
  int32_t* q_buf;
  int32_t* h_gen;
  int32_t* h_stop;
  int32_t* h_group;
  ulonglong2* h_key;
  int64_t* h_version;
  int32_t* h_tokens;  // [H * L]
  double* h_logp;     // [H * L]
  int32_t* g_done;
  int32_t* h_needs_pf;  // [H] or nullptr: 1 = queued resumed sample whose KV is not rebuilt yet
  // transformer: the KV page state k_finish needs to free a finished sample's private pages at once
  // (a fused run lasts thousands of iterations; pages must not wait for the host's release)
  int32_t* kv_bt;       // block tables [rows][kv_MP] (nullptr: no model)
  int32_t* kv_h_ctx;    // context length per handle
  int32_t* kv_h_shared; // leading pages shared with the prompt group
  int32_t* kv_free;     // free-page stack (top in Ctl::kv_free_top)
  int kv_P, kv_MP;
  ab_event* ev;
  ab_admit* adm;
  double* cf_logits;  // [n_symbols]
  double* cf_cdf;
  double* cf_logp;
  int32_t* it_b;       // per run iteration: live batch (profiling / roofline)
  int64_t* it_ctx;     // per run iteration: sum of context lengths
  int it_cap;
  uint64_t t0_ns;
  // data-parallel lockstep exchange: record slots [2][dp_world][8] int64 in every
  // rank's device memory; dp_peers[r] = rank r's slots (NVLink P2P / CUDA IPC mapped)
  int dp_world, dp_rank;
  int64_t* const* dp_peers;
  int64_t* dp_local;
  uint64_t dp_timeout_ns;
};

struct KernelTimer {
  std::string name;
  int64_t launches = 0;
  double ms = 0, bytes = 0, flops = 0;
};

struct Engine {
  ab_engine_config cfg{};
  ab_model_config mcfg{};
  int device = 0;
  cudaStream_t stream = nullptr;
  EngineDev d{};
  Ctl* ctl_host = nullptr;  // pinned mirror
  uint64_t* clock_host = nullptr;
  Model* model = nullptr;
  ab_sample_desc* stage_desc_host = nullptr;
  ab_sample_desc* stage_desc_dev = nullptr;
  int32_t* stage_i32_dev = nullptr;
  int32_t* stage_i32_host = nullptr;
  size_t stage_i32_cap = 0;
  int64_t prefill_tokens = 0;
  int64_t reprefill_tokens = 0;
  double reprefill_seconds = 0;  // host wall time of KV re-prefill (resumed partials + prompt recompute)
  int64_t launches = 0;  // kernels launched (gpu_launches claim)
  bool use_graphs = true;
  int64_t direct_launches = 0;
  // one captured iteration graph per decode plan variant (model_variant_for), plus a profiling
  // twin with event-record nodes
  std::vector<cudaGraphExec_t> iter_graphs, prof_graphs;
  std::vector<int64_t> graph_kernels;
  int variant = 0;  // variant of the chunk being launched
  bool capturing_prof = false;
  struct ProfSlot {
    int timer;
    cudaEvent_t a, b;
  };
  std::vector<std::vector<ProfSlot>> prof_slots;  // per variant's profiling graph
  int64_t prof_pending = -1;
  int prof_pending_variant = 0;
  int64_t prof_count = 0;
  // profiling
  bool profile = false;
  int sample_every = 8;
  std::vector<KernelTimer> timers;
  struct PendingTime {
    int timer;
    cudaEvent_t a, b;
    int64_t run_iter;  // -1: bytes known at launch
    double bytes, flops;
  };
  std::vector<PendingTime> pending;
  std::vector<cudaEvent_t> event_pool;

  // data-parallel exchange buffers
  int64_t* dp_buf = nullptr;            // this rank's record slots (exported to peers)
  int64_t** dp_peers_dev = nullptr;     // device array of the world's slot pointers
  std::vector<void*> dp_ipc_opened;     // peer buffers opened through CUDA IPC

  cudaEvent_t take_event();
  int timer_index(const char* name);
};

// model.cu
Model* model_create(Engine& e);
void model_destroy(Model* m);
int model_weight_count(Model* m);
void model_weight_info(Model* m, int idx, std::string* name, int64_t* rows, int64_t* cols, void** dev_ptr);
void model_open_group(Engine& e, int group_slot, const int32_t* prompt, int prompt_len);
void model_release_group(Engine& e, int group_slot);
void model_submit(Engine& e, const ab_sample_desc* descs_dev, int n);  // after per-handle state is set
// KV re-prefill mode: rebuild the KV of the next `count` deferred resumed samples (FIFO order)
int model_prefill_deferred(Engine& e, int count);  // returns how many were rebuilt
void model_drop_deferred(Engine& e);  // abort: queued resumed samples were never rebuilt
void model_forget_deferred(Engine& e, const int32_t* handles_host, int n);  // released handles
void model_release(Engine& e, const int32_t* handles_dev, int n);
void model_evict(Engine& e, const int32_t* handles_host, const int32_t* gen, int n);  // kv_resume: drop private KV
void model_begin_step(Engine& e, int64_t version);
void model_release_memory(Engine& e);
void model_resume_memory(Engine& e);
void model_score(Engine& e, const int32_t* tokens, const int64_t* offs, const int32_t* plen, int n, double* out);
int model_variants(Model* m);              // decode graph variants (plan selections)
int model_variant_for(Model* m, int rows);  // the variant for a chunk whose live batch is <= rows
int64_t model_iter_launches(Model* m, int variant);
void model_iteration(Engine& e, int64_t run_iter, bool timed, int variant);  // pages + forward + sampler
int64_t model_pages_total(Model* m);
std::string model_kv_report(Engine& e);  // for out-of-KV errors
void model_kernel_cost(Model* m, const std::string& name, double b, double sum_ctx, double* bytes, double* flops);

// profiling helper (engine.cu)
struct ScopedTimer {
  Engine& e;
  int idx;
  cudaEvent_t a = nullptr;
  double bytes, flops;
  int64_t run_iter;
  ScopedTimer(Engine& eng, bool on, const char* name, int64_t run_iter_, double bytes_ = 0, double flops_ = 0);
  ~ScopedTimer();
};

}  // namespace ab
