/*
 * april_b200.h — C-ABI of the B200-native APRIL rollout engine.
 *
 * The reference (`april_sim`, pure Python) has no FFI: its "plugin API" for
 * this path is the duck-typed `Engine` the `Scheduler` drives
 * (src/april_sim/scheduler.py:153-171, selected at src/april_sim/simulate.py:105-121).
 * Every entry point below replaces one member of that contract; the Python
 * shim `paper_2509_18521_b200/engine.py` binds them with ctypes and exposes
 * the reference names (see INTEGRATION.md for the binding a maintainer adds).
 *
 *   Engine.__init__ / EngineConfig        engine.py:38-66, 101-108   -> ab_engine_create
 *   Engine.begin_step(version, params)    engine.py:127-130, 253-260 -> ab_engine_begin_step
 *   Engine.submit(sample)                 engine.py:134-139          -> ab_engine_submit (+ ab_engine_open_group)
 *   Engine.decode_iteration()             engine.py:150-155          -> ab_engine_run(max_iters=1)
 *   Engine.decode_until_event()           engine.py:157-165          -> ab_engine_run(stop_on_event=1)
 *   Scheduler loop "while not check_trigger: decode_until_event()"
 *                                         scheduler.py:272-283       -> ab_engine_run(use_trigger=1)
 *   Engine.abort_active()                 engine.py:184-197          -> ab_engine_abort
 *   Segment.tokens / behavior_logprobs    rollouts.py:27-34          -> ab_engine_read_payload
 *   group_advantages(rewards, mode, eps)  policy.py:115-124          -> ab_group_advantages
 *   iteration_index / cumulative_tokens   engine.py:103-106          -> ab_engine_stats
 *
 * Errors follow src/april_sim/errors.py:4-9: AB_ERR_CONFIG maps to
 * ConfigError (raised only at construction), AB_ERR_CONTRACT to
 * ContractViolation.  ab_last_error() returns a thread-local message.
 * No torch types appear here: plain pointers, sizes and status codes.
 */
#ifndef APRIL_B200_H
#define APRIL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AB_OK 0
#define AB_ERR_CONFIG 1
#define AB_ERR_CONTRACT 2
#define AB_ERR_CUDA 3
#define AB_ERR_OUT_OF_KV 4
#define AB_ERR_NCCL 5

/* how sequences end (engine.py:214-289) */
#define AB_STOP_TRACE 0  /* stop at a pre-drawn target length (LengthDrivenEngine) */
#define AB_STOP_POLICY 1 /* stop on a drawn EOS/STOP symbol or l_max (PolicyDrivenEngine) */

/* what produces the next-token distribution */
#define AB_MODEL_NONE 0         /* no sampling at all (trace replay only)                 */
#define AB_MODEL_CONTEXT_FREE 1 /* one fp64 logits row per step (the reference's toy)     */
#define AB_MODEL_TRANSFORMER 2  /* Qwen-style decoder: paged KV, GQA attention, tcgen05  */

/* finish reasons (rollouts.py:107-110) */
#define AB_REASON_STOP_TOKEN 0
#define AB_REASON_TARGET_LENGTH 1
#define AB_REASON_MAX_LENGTH 2

/* why ab_engine_run returned */
#define AB_RUN_TRIGGER 0
#define AB_RUN_EVENT 1
#define AB_RUN_MAX_ITERS 2
#define AB_RUN_DRAINED 3

typedef struct ab_engine ab_engine;

typedef struct ab_model_config {
  int32_t n_layers, d_model, n_q_heads, n_kv_heads, head_dim, d_ff, vocab;
  int32_t qkv_bias;        /* Qwen2: bias on q/k/v projections            */
  int32_t qk_norm;         /* Qwen3: RMSNorm on q and k per head           */
  int32_t tied_embeddings; /* lm_head shares the embedding matrix         */
  float rope_theta, norm_eps;
} ab_model_config;

typedef struct ab_engine_config {
  int32_t max_slots;   /* S: concurrently decoding sequences (engine.py:45)  */
  int32_t l_max;       /* generation cap (engine.py:46)                       */
  int32_t max_handles; /* capacity of resident samples (active+queued+parked) */
  int32_t max_groups;  /* capacity of resident prompt groups                  */
  int32_t stop_mode;   /* AB_STOP_*                                           */
  int32_t model_kind;  /* AB_MODEL_*                                          */
  int32_t n_symbols;   /* context-free model: vocabulary incl. STOP (V+1)     */
  int32_t page_size;   /* transformer: KV page size in tokens                 */
  int64_t kv_pages;    /* transformer: KV pages to reserve (0 = auto)         */
  int32_t max_prompt;  /* transformer: longest prompt                         */
  float temperature;   /* 1.0 = plain softmax                                 */
  float top_p;         /* 1.0 = no nucleus truncation                         */
  int32_t greedy;      /* argmax decoding (lowest index on ties)              */
  int32_t n_eos;       /* transformer policy mode: EOS ids                    */
  int32_t eos_ids[8];
  int32_t record_payload; /* keep token ids + behaviour logprobs on device    */
  uint64_t weight_seed;   /* transformer: N(0, weight_std) init seed          */
  float weight_std;
  int32_t nondeterministic_gemm; /* 1: fp32 residual GEMMs may split K with TMA reduce-add
                                    (faster; split summation order not fixed run to run) */
  int32_t kv_resume; /* 0: a paused sample keeps its KV across steps; 1: the abort drops it and the
                        resubmit re-prefills prompt + carried tokens (prompt KV of resident groups is
                        recomputed when the step version changes) -- SURVEY §8 f1 */
  int32_t gemm_autotune; /* transformer: time the decode GEMM schedules on this GPU at engine creation
                            and run each live row count on the fastest (0: cost-model tables) */
  int32_t reserved[4];
} ab_engine_config;

typedef struct ab_sample_desc {
  int32_t handle;     /* 0..max_handles-1, owned by the caller            */
  int32_t group_slot; /* 0..max_groups-1                                  */
  int32_t gen_len;    /* tokens already generated (resumed samples)       */
  int32_t stop_at;    /* trace mode: min(target_length, l_max)            */
  uint64_t key0, key1; /* Philox4x64 key = blake2b(seed, lane 2, iid, sidx) */
} ab_sample_desc;

typedef struct ab_run_args {
  int64_t max_iters;     /* 0 = unbounded                                     */
  int32_t stop_on_event; /* return after the first iteration with a finish    */
  int32_t use_trigger;   /* return when check_trigger() fires                 */
  int32_t trigger_mode;  /* 0 groups, 1 samples (scheduler.py:59-64)          */
  int32_t n_target;      /* N                                                 */
  int32_t group_size;    /* G                                                 */
  int32_t reserved;
  int64_t completed_groups;  /* counters seeded by the caller at step start  */
  int64_t completed_samples;
} ab_run_args;

typedef struct ab_event {
  int32_t handle;
  int32_t tokens; /* sample total after this iteration                     */
  int64_t iteration;
  int32_t reason; /* AB_REASON_*                                           */
  int32_t group_complete; /* 1 if this finish completed its group          */
  double clock;   /* device wall seconds since engine creation             */
} ab_event;

typedef struct ab_admit {
  int32_t handle;
  int32_t slot;
  int64_t iteration; /* iteration_index before the admitting iteration    */
} ab_admit;

typedef struct ab_run_result {
  int64_t iterations; /* decode iterations executed by this call           */
  int32_t stop_reason; /* AB_RUN_*                                         */
  int32_t n_events, n_admits;
  int32_t reserved;
  int64_t completed_groups, completed_samples;
  int64_t iteration_index, cumulative_tokens; /* engine totals after the call */
} ab_run_result;

typedef struct ab_stats {
  int64_t iteration_index, cumulative_tokens;
  int32_t active, queued;
  double clock;        /* device wall seconds since engine creation         */
  int64_t kv_pages_total, kv_pages_free;
  int64_t prefill_tokens; /* prompt tokens prefilled (excluded from "generated") */
  int64_t kernel_launches; /* kernels this engine has launched */
  int64_t reprefill_tokens; /* carried tokens re-prefilled at resume (kv_resume = 1) */
  double reprefill_seconds; /* wall time spent re-prefilling (resumed partials + prompt recompute) */
} ab_stats;

typedef struct ab_kernel_stat {
  char name[32];
  int64_t launches;      /* timed launches                                   */
  double ms;             /* summed CUDA-event time of the timed launches     */
  double bytes;          /* summed algorithmic bytes of the timed launches   */
  double flops;          /* summed algorithmic flops                         */
} ab_kernel_stat;

const char* ab_last_error(void);
int ab_version(void);

int ab_engine_create(const ab_engine_config* cfg, const ab_model_config* model, int device, ab_engine** out);
int ab_engine_destroy(ab_engine* e);

/* weights (transformer): tensor i's name, shape and raw bf16 bytes */
int ab_engine_weight_count(ab_engine* e, int* n);
int ab_engine_weight_info(ab_engine* e, int idx, char* name, int name_cap, int64_t* rows, int64_t* cols);
int ab_engine_get_weight(ab_engine* e, int idx, void* host_dst, size_t bytes);
int ab_engine_set_weight(ab_engine* e, int idx, const void* src, size_t bytes);

/* context-free model: n_symbols fp64 logits (STOP last), or NULL */
int ab_engine_begin_step(ab_engine* e, int64_t version, const double* cf_logits);
/* transformer: prefill a prompt group's shared prefix into KV pages */
int ab_engine_open_group(ab_engine* e, int32_t group_slot, const int32_t* prompt, int32_t prompt_len);
int ab_engine_release_group(ab_engine* e, int32_t group_slot);
/* KV memory hand-off (kv_resume = 1 only): free the KV pool of an idle engine for a
 * co-located trainer, then re-acquire it (resident prompt KV is recomputed by the next submit). */
int ab_engine_release_memory(ab_engine* e);
int ab_engine_resume_memory(ab_engine* e);
int ab_engine_submit(ab_engine* e, const ab_sample_desc* descs, int n);
/* preset per-group completed-sample counts: n pairs (group_slot, count) */
int ab_engine_set_group_done(ab_engine* e, const int32_t* slot_count_pairs, int n);
int ab_engine_run(ab_engine* e, const ab_run_args* args, ab_run_result* res, ab_event* events, int event_cap,
                  ab_admit* admits, int admit_cap);
/* active handles (slot order) then queued handles (FIFO); gen counts of each */
int ab_engine_abort(ab_engine* e, int32_t* handles, int32_t* gen, int cap, int* n_active, int* n_queued);
int ab_engine_active(ab_engine* e, int32_t* handles, int32_t* gen, int cap, int* n_active);
int ab_engine_read_payload(ab_engine* e, const int32_t* handles, const int32_t* starts, const int32_t* counts, int n,
                           int32_t* tokens, double* logprobs);

// GSPO / sequence-level ratios: per-sample sum of the recorded behaviour log-probabilities over
// all generated tokens (device reduction of the partial-rollout payload) and the token count.
// Reference: the build's addition for SURVEY.md §8a row a17 (GSPO length-normalised log-prob);
// the reference computes sequence log-probs on the host (src/april_sim/policy.py:133-137).
int ab_engine_sequence_logprobs(ab_engine* e, const int32_t* handles, int n, double* sums, int32_t* lens);
/* Trainer-side recompute (the toy trainer's logp_now, policy.py:157-176): teacher-forced
 * log-probs of response tokens under the CURRENT weights, at the engine's temperature.  Host arrays:
 * sequence k = tokens[offs[k] .. offs[k+1]) (prompt + response), prompt_lens[k] >= 1 tokens of prompt;
 * logprobs receives sum_k (len_k - prompt_lens[k]) values, per sequence in token order. */
int ab_engine_score(ab_engine* e, const int32_t* tokens, const int64_t* offs, const int32_t* prompt_lens, int n,
                    double* logprobs);
int ab_engine_release(ab_engine* e, const int32_t* handles, int n);
int ab_engine_stats(ab_engine* e, ab_stats* out);
int ab_engine_profile(ab_engine* e, int enable, int sample_every);
int ab_engine_kernel_stats(ab_engine* e, ab_kernel_stat* out, int cap, int* n);
int ab_engine_synchronize(ab_engine* e);
/* data-parallel lockstep: align the device iteration counter with the global index */
int ab_engine_set_iteration(ab_engine* e, int64_t iteration_index);
int ab_engine_set_counters(ab_engine* e, int64_t iteration_index, int64_t cumulative_tokens);

/* Data-parallel lockstep on the device (the reference is one engine, and
 * its trigger loop scheduler.py:272-283 becomes global).  One engine per GPU, one process per GPU.
 * Each engine exports a small exchange buffer in its own HBM; after every rank attached the world's
 * buffers, every decode iteration ends with k_dp_exchange: each rank stores its (completed groups,
 * completed samples, live rows, next live rows, iterations-to-next-finish) into every peer's buffer
 * over NVLink and sums the world's records, so the APRIL trigger, drain, iteration_index and
 * cumulative_tokens are global on every rank with no host round trip per iteration.  ab_engine_run
 * then runs the lockstep loop (events / admissions in the logs are this rank's only).
 *   export: allocate + zero the buffer; *dev_ptr = its device address, ipc_handle (64 bytes, may be
 *           NULL) = its cudaIpcMemHandle_t for other processes.
 *   attach: peers[r] = rank r's buffer (kind 0: same-process device pointer; kind 1: IPC handle);
 *           every rank must have exported before any rank attaches; timeout_ms bounds each wait. */
typedef struct ab_dp_peer {
  uint64_t ptr;
  int32_t kind; /* 0 = device pointer in this process, 1 = CUDA IPC handle */
  int32_t reserved;
  uint8_t ipc[64];
} ab_dp_peer;
int ab_engine_dp_export(ab_engine* e, int world, uint64_t* dev_ptr, void* ipc_handle);
int ab_engine_dp_attach(ab_engine* e, int world, int rank, const ab_dp_peer* peers, int64_t timeout_ms);
int ab_engine_dp_detach(ab_engine* e);

/* K6: group-normalised advantages over contiguous groups of G rewards.
 * mode 0 = mean baseline, 1 = mean/std (GRPO), 2 = mean/std with a
 * zero-std flag (DAPO), 3 = mean/std for GSPO (whose sequence ratio uses
 * ab_engine_sequence_logprobs); pointers are device or host. */
int ab_group_advantages(const double* rewards, int n_groups, int group_size, int mode, double eps, double* adv,
                        int32_t* zero_std_flags, int device);

/* K7: clipped-ratio terms of a mixed-policy batch, host arrays.  Response k owns
 * tokens [offs[k], offs[k+1]) of logp_now / logp_beh; adv[k] its advantage.  Token level: ratios and
 * clipped get offs[n] entries (r = exp(now - beh); clipped iff A > 0 and r > 1 + eps_clip_high or
 * A < 0 and r < 1 - eps_clip, the clip rule of src/april_sim/policy.py:153-177); sequence_level
 * (GSPO): one ratio exp(mean_t(now - beh)) per response.  surrogate[k] = sum min(r A, clip(r) A). */
int ab_clipped_ratio_terms(const double* logp_now, const double* logp_beh, const int64_t* offs, int n,
                           const double* adv, double eps_clip, double eps_clip_high, int sequence_level,
                           double* ratios, int32_t* clipped, double* surrogate, int device);

/* Test entry points (device pointers; used by tests/test_kernels_gpu.py). */
int ab_debug_gemm(const void* W, const void* A, void* out, const void* bias, int N, int K, int M, int BN, int epi);
int ab_debug_gemm_time(const void* W, const void* A, void* out, const void* bias, int N, int K, int M, int BN, int epi,
                       int reps, float* ms_out);
/* packed GEMM schedule the cost model picks (host only, no GPU needed) */
int ab_debug_gemm_sched(int N, int K, int rows, int max_bn, int cluster, int n_clusters, int force, int epi);
/* co-resident persistent GEMM clusters of `cluster` CTAs */
int ab_debug_gemm_clusters(int cluster, int* out);
/* per-CTA %globaltimer timeline of the next GEMM launches (tools/gemm_trace.py) */
int ab_debug_gemm_trace(int on, unsigned long long* out);
int ab_debug_trace_mark(int slot);
/* K1's per-row routine on device logits [rows, V] and draws u [rows] (tests/test_sampler.py) */
/* K3 over a caller-built single-layer paged pool (tests/test_attention_gpu.py); device pointers:
 * q and out [rows, n_kv_heads*gq*head_dim] bf16, kv [n_pages][2][n_kv_heads][page_size][head_dim] bf16,
 * block_table [rows, max_pages] int32; host ctx[rows] = attended tokens per row.  chunk > 0 forces the
 * KV split size (multiple of 64), chunk <= 0 uses the engine's per-iteration choice (min split -chunk
 * or 256); *chunk_used receives it. */
int ab_debug_decode_attn(const void* q, const void* kv, int64_t n_pages, int page_size, int n_kv_heads, int head_dim,
                         int gq, const int32_t* block_table, int max_pages, const int32_t* ctx, int rows, int chunk,
                         void* out, int* chunk_used);
int ab_debug_sample_rows(const float* logits, int rows, int V, float temperature, int greedy, float top_p,
                         const double* u, int* tok, double* logp);

#ifdef __cplusplus
}
#endif
#endif
