// APRIL rollout engine: device-resident slots, FIFO admission, stable
// live-batch compaction, group done-counters and the early-termination
// trigger, driven by a host loop that polls a pinned control block only at
// iterations where something can finish.
//
// Semantics restate (reference paths relative to pkg/):
//   admission     src/april_sim/engine.py:141-146 (FIFO, up to S, at iteration start)
//   advance       src/april_sim/engine.py:167-180 (iteration_index += 1, cumulative += b,
//                 stable removal of finished slots, events in slot order)
//   trace stop    src/april_sim/engine.py:220-240
//   policy stop   src/april_sim/engine.py:274-289 (STOP before MAX_LENGTH)
//   trigger       src/april_sim/scheduler.py:59-64, checked after every iteration
//                 (counters only change at iterations with finishes, scheduler.py:272-283)
//   abort         src/april_sim/engine.py:184-197 (active in slot order, then queue FIFO)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "engine.cuh"

namespace ab {

static thread_local std::string g_last_error;
void set_last_error(const char* msg) { g_last_error = msg; }

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------

__global__ void k_run_begin(EngineDev d, ab_run_args a) {
  Ctl* c = d.ctl;
  c->stop = 0;
  c->stop_reason = -1;
  c->error = kErrNone;
  c->error_handle = -1;
  c->n_events = 0;
  c->n_admits = 0;
  c->run_iters = 0;
  c->max_iters = a.max_iters;
  c->use_trigger = a.use_trigger;
  c->trigger_mode = a.trigger_mode;
  c->stop_on_event = a.stop_on_event;
  c->n_target = a.n_target;
  c->group_size = a.group_size;
  c->completed_groups = a.completed_groups;
  c->completed_samples = a.completed_samples;
  c->iters_to_next = 1;
  c->dp_done = 0;
}

__device__ __forceinline__ bool trigger_fired(const Ctl* c) {
  // scheduler.py:59-64
  if (c->trigger_mode == 0) return c->completed_groups >= c->n_target;
  return c->completed_samples >= (int64_t)c->n_target * c->group_size && c->completed_groups >= c->n_target;
}

// Admission at the start of an iteration: pop the FIFO into free slots.
__global__ void k_admit(EngineDev d) {
  Ctl* c = d.ctl;
  if (c->stop) return;
  __shared__ int s_b, s_n, s_head;
  if (threadIdx.x == 0) {
    if (c->use_trigger && trigger_fired(c)) {  // trigger seeded as already fired: no decoding at all
      c->stop = 1;
      c->stop_reason = AB_RUN_TRIGGER;
      c->dp_done = 1;  // data-parallel: the seeded counters are global, every rank stops here
      s_n = -1;
    } else {
      s_b = c->b;
      s_head = c->q_head;
      s_n = min(d.S - s_b, c->q_tail - c->q_head);
    }
  }
  __syncthreads();
  const int n = s_n;
  if (n < 0) return;
  if (d.h_needs_pf) {
    // KV re-prefill mode: a resumed sample about to be admitted has no KV yet -- stop before
    // admitting anything (the iteration does not happen); the host rebuilds the next admissions'
    // KV and resumes the run, so admission order and iteration count are unchanged
    bool need = false;
    for (int i = threadIdx.x; i < n; i += blockDim.x) need |= d.h_needs_pf[d.q_buf[(s_head + i) % d.Q]] != 0;
    if (__syncthreads_or(need)) {
      if (threadIdx.x == 0) {
        c->stop = 1;
        c->stop_reason = kRunNeedPrefill;
      }
      return;
    }
  }
  const int b = s_b;
  const int64_t it = c->iteration_index;
  const int64_t ver = c->version;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int h = d.q_buf[(s_head + i) % d.Q];
    d.slot_handle[b + i] = h;
    if (d.h_version[h] >= ver) {  // rollouts.py:168-173: segment versions must strictly increase
      if (atomicCAS(&c->error, kErrNone, kErrVersion) == kErrNone) c->error_handle = h;
    }
    if (d.stop_mode == AB_STOP_TRACE) {
      if (d.h_stop[h] < 0) {  // engine.py:221-222
        if (atomicCAS(&c->error, kErrNone, kErrNoTarget) == kErrNone) c->error_handle = h;
      } else if (d.h_stop[h] - d.h_gen[h] <= 0) {  // engine.py:224-226
        if (atomicCAS(&c->error, kErrNone, kErrAtStop) == kErrNone) c->error_handle = h;
      }
    }
    d.h_version[h] = ver;
    ab_admit rec;
    rec.handle = h;
    rec.slot = b + i;
    rec.iteration = it;
    d.adm[c->n_admits + i] = rec;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    c->b = b + n;
    c->q_head = s_head + n;
    c->n_admits += n;
    if (d.dp_world > 1 && (c->error != kErrNone || c->b == 0)) {
      // data-parallel: this rank sits the iteration out (stop = 2 skips every kernel up to the
      // exchange); whether the job is drained or failed is decided globally by k_dp_exchange
      c->stop = 2;
      c->dp_groups = c->dp_samples = c->dp_b = c->dp_next = 0;
      c->dp_hint = 0x7fffffff;
    } else if (c->error != kErrNone) {
      c->stop = 1;
      c->stop_reason = -2;
    } else if (c->b == 0) {  // engine.py:153-154 / 161-162: nothing to decode
      c->stop = 1;
      c->stop_reason = AB_RUN_DRAINED;
    }
  }
}

__device__ __forceinline__ int searchsorted_right(const double* cdf, int n, double u) {
  int lo = 0, hi = n;  // number of cdf entries <= u
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (cdf[mid] <= u)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// Per-slot growth for the no-model / context-free engines: one Philox draw
// at position = generated tokens, inverse-CDF in index order, stop rules.
__global__ void k_grow_cf(EngineDev d) {
  const Ctl* c = d.ctl;
  if (c->stop) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= c->b) return;
  const int h = d.slot_handle[i];
  const int g = d.h_gen[h];
  int tok = -1;
  if (d.model_kind == AB_MODEL_CONTEXT_FREE) {
    const ulonglong2 k = d.h_key[h];
    const double u = philox_uniform(k.x, k.y, (uint64_t)g);           // engine.py:276 (unclamped)
    tok = min(searchsorted_right(d.cf_cdf, d.n_symbols, u), d.n_symbols - 1);  // engine.py:277-278
    if (d.record) {
      d.h_tokens[(int64_t)h * d.L + g] = tok;
      d.h_logp[(int64_t)h * d.L + g] = d.cf_logp[tok];
    }
  }
  const int g1 = g + 1;
  d.h_gen[h] = g1;
  int reason = -1;
  if (d.stop_mode == AB_STOP_TRACE) {
    const int stop_at = d.h_stop[h];
    if (g1 == stop_at) reason = stop_at >= d.l_max ? AB_REASON_MAX_LENGTH : AB_REASON_TARGET_LENGTH;
  } else {
    if (tok == d.n_symbols - 1)
      reason = AB_REASON_STOP_TOKEN;
    else if (g1 >= d.l_max)
      reason = AB_REASON_MAX_LENGTH;
  }
  d.slot_token[i] = tok;
  d.slot_finish[i] = reason + 1;
}

// Block-wide exclusive scan of two counters (1024 threads).
__device__ __forceinline__ void block_scan2(int a, int b, int* ea, int* eb, int* ta, int* tb) {
  __shared__ int sa[32], sb[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int xa = a, xb = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int ya = __shfl_up_sync(0xffffffffu, xa, o), yb = __shfl_up_sync(0xffffffffu, xb, o);
    if (lane >= o) {
      xa += ya;
      xb += yb;
    }
  }
  if (lane == 31) {
    sa[w] = xa;
    sb[w] = xb;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    int va = lane < nw ? sa[lane] : 0, vb = lane < nw ? sb[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int ya = __shfl_up_sync(0xffffffffu, va, o), yb = __shfl_up_sync(0xffffffffu, vb, o);
      if (lane >= o) {
        va += ya;
        vb += yb;
      }
    }
    if (lane < nw) {
      sa[lane] = va;
      sb[lane] = vb;
    }
  }
  __syncthreads();
  const int base_a = w ? sa[w - 1] : 0, base_b = w ? sb[w - 1] : 0;
  *ea = base_a + xa - a;
  *eb = base_b + xb - b;
  *ta = sa[(blockDim.x >> 5) - 1];
  *tb = sb[(blockDim.x >> 5) - 1];
  __syncthreads();
}

constexpr int kFinishThreads = 1024;
constexpr int kMaxIPT = 4;  // S <= 4096

// Stable compaction of the live batch + event log + group counters + trigger.
__global__ void __launch_bounds__(kFinishThreads) k_finish(EngineDev d) {
  Ctl* c = d.ctl;
  if (c->stop) return;
  const int b = c->b;
  const int ipt = (b + blockDim.x - 1) / blockDim.x;
  const int beg = min(b, (int)threadIdx.x * ipt), end = min(b, beg + ipt);
  int fin[kMaxIPT];
  int nk = 0, nd = 0;
  for (int j = 0; j < ipt; ++j) {
    const int i = beg + j;
    fin[j] = i < end ? d.slot_finish[i] : 0;
    if (i < end) {
      if (fin[j])
        ++nd;
      else
        ++nk;
    }
  }
  int ek, ed, tk, td;
  block_scan2(nk, nd, &ek, &ed, &tk, &td);
  __shared__ int s_new_groups;
  __shared__ int s_min_rem;
  if (threadIdx.x == 0) {
    s_new_groups = 0;
    s_min_rem = 0x7fffffff;
  }
  __syncthreads();
  const int64_t it1 = c->iteration_index + 1;  // engine.py:170: index advances before events
  const int ev_base = c->n_events;
  const int G = c->group_size;
  double clk = 0.0;
  if (nd) clk = (double)(globaltimer_ns() - d.t0_ns) * 1e-9;
  int min_rem = 0x7fffffff;
  for (int j = 0; j < ipt; ++j) {
    const int i = beg + j;
    if (i >= end) break;
    const int h = d.slot_handle[i];
    if (fin[j]) {
      if (d.kv_bt) {
        // free the finished sample's private KV pages now (k_release semantics; the host's later
        // release of the handle finds nothing left to free)
        const int have = (d.kv_h_ctx[h] + d.kv_P - 1) / d.kv_P, own0 = d.kv_h_shared[h];
        const int cnt = have - own0;
        if (cnt > 0) {
          const long long base =
              (long long)atomicAdd(reinterpret_cast<unsigned long long*>(&c->kv_free_top), (unsigned long long)cnt);
          for (int q = 0; q < cnt; ++q) d.kv_free[base + q] = d.kv_bt[(size_t)h * d.kv_MP + own0 + q];
        }
        d.kv_h_ctx[h] = 0;
        d.kv_h_shared[h] = 0;
      }
      int complete = 0;
      if (G > 0) {
        const int old = atomicAdd(&d.g_done[d.h_group[h]], 1);
        if (old + 1 == G) {
          complete = 1;
          atomicAdd(&s_new_groups, 1);
        }
      }
      ab_event e;
      e.handle = h;
      e.tokens = d.h_gen[h];
      e.iteration = it1;
      e.reason = fin[j] - 1;
      e.group_complete = complete;
      e.clock = clk;
      d.ev[ev_base + ed++] = e;
    } else {
      d.slot_tmp[ek++] = h;
      if (d.stop_mode == AB_STOP_TRACE) min_rem = min(min_rem, d.h_stop[h] - d.h_gen[h]);
    }
  }
  min_rem = warp_min_i(min_rem);
  if ((threadIdx.x & 31) == 0) atomicMin(&s_min_rem, min_rem);
  __syncthreads();
  for (int i = threadIdx.x; i < tk; i += blockDim.x) d.slot_handle[i] = d.slot_tmp[i];
  if (threadIdx.x == 0 && d.dp_world > 1) {
    // data-parallel: publish this rank's share; k_dp_exchange advances the global counters and
    // decides trigger / drain for every rank at once
    c->b = tk;
    c->n_events = ev_base + td;
    if (c->run_iters < d.it_cap) d.it_b[c->run_iters] = b;
    c->dp_groups = s_new_groups;
    c->dp_samples = td;
    c->dp_b = b;
    c->dp_next = tk + min(d.S - tk, c->q_tail - c->q_head);
    const bool queue_waiting = (c->q_tail - c->q_head) > 0 && tk < d.S;
    if (d.stop_mode == AB_STOP_TRACE)
      c->dp_hint = tk == 0 && !queue_waiting ? 0x7fffffff : (queue_waiting ? 1 : s_min_rem);
    else
      c->dp_hint = -1;
  } else if (threadIdx.x == 0) {
    c->b = tk;
    c->iteration_index = it1;
    c->cumulative_tokens += b;
    c->n_events = ev_base + td;
    c->completed_groups += s_new_groups;
    c->completed_samples += td;
    c->run_iters += 1;
    if (c->run_iters <= d.it_cap) {
      d.it_b[c->run_iters - 1] = b;
    }
    const bool queue_waiting = (c->q_tail - c->q_head) > 0 && tk < d.S;
    if (d.stop_mode == AB_STOP_TRACE && tk > 0 && !queue_waiting)
      c->iters_to_next = s_min_rem;
    else
      c->iters_to_next = (d.stop_mode == AB_STOP_TRACE) ? 1 : -1;
    if (c->use_trigger && td > 0 && trigger_fired(c)) {
      c->stop = 1;
      c->stop_reason = AB_RUN_TRIGGER;
    } else if (c->stop_on_event && td > 0) {
      c->stop = 1;
      c->stop_reason = AB_RUN_EVENT;
    } else if (c->max_iters > 0 && c->run_iters >= c->max_iters) {
      c->stop = 1;
      c->stop_reason = AB_RUN_MAX_ITERS;
    }
  }
}

__device__ __forceinline__ void st_release_sys(int64_t* p, int64_t v) {
  asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t* p) {
  int64_t v;
  asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(int64_t* p, int64_t v) {
  asm volatile("st.relaxed.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t ld_relaxed_sys(const int64_t* p) {
  int64_t v;
  asm volatile("ld.relaxed.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

constexpr int kDpRec = 8;  // int64 per record: epoch, groups, samples, b, next, hint, error, pad

// Data-parallel lockstep exchange, the last kernel of every iteration when the
// engine is one of dp_world ranks.  One warp: lane r stores this rank's record into slot
// [epoch & 1][rank] of rank r's buffer (peer memory over NVLink: payload relaxed, then the epoch
// with release semantics), then waits for slot [epoch & 1][r] of its own buffer to carry the same
// epoch (acquire).  The sums are integers, so every rank computes the same global decision:
// iteration_index / cumulative_tokens / completed counters advance by the global totals, the
// trigger (scheduler.py:59-64) fires on the global counters, and the job is drained when no rank
// has a live row.  Two parities: a rank can run at most one exchange ahead of the slowest, so
// it never overwrites a record that is still being read.  No host round trip per iteration.
__global__ void k_dp_exchange(EngineDev d) {
  Ctl* c = d.ctl;
  if (c->dp_done) return;
  const int lane = threadIdx.x, W = d.dp_world;
  const int64_t ep = c->dp_epoch + 1;
  const int par = (int)(ep & 1);
  const int64_t err = c->error != kErrNone ? 1 : 0;
  if (lane < W) {
    int64_t* dst = d.dp_peers[lane] + ((int64_t)par * W + d.dp_rank) * kDpRec;
    st_relaxed_sys(dst + 1, c->dp_groups);
    st_relaxed_sys(dst + 2, c->dp_samples);
    st_relaxed_sys(dst + 3, c->dp_b);
    st_relaxed_sys(dst + 4, c->dp_next);
    st_relaxed_sys(dst + 5, c->dp_hint);
    st_relaxed_sys(dst + 6, err);
    st_release_sys(dst, ep);
  }
  int64_t g = 0, smp = 0, b = 0, nx = 0, hint = 0x7fffffff, e = 0;
  int timed_out = 0;
  if (lane < W) {
    const int64_t* src = d.dp_local + ((int64_t)par * W + lane) * kDpRec;
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_sys(src) != ep) {
      if (globaltimer_ns() - t0 > d.dp_timeout_ns) {
        timed_out = 1;
        break;
      }
      __nanosleep(32);
    }
    if (!timed_out) {
      g = ld_relaxed_sys(src + 1);
      smp = ld_relaxed_sys(src + 2);
      b = ld_relaxed_sys(src + 3);
      nx = ld_relaxed_sys(src + 4);
      const int64_t h = ld_relaxed_sys(src + 5);
      hint = h < 0 ? 0x7fffffff : h;
      e = ld_relaxed_sys(src + 6);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    g += __shfl_xor_sync(0xffffffffu, g, o);
    smp += __shfl_xor_sync(0xffffffffu, smp, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    nx += __shfl_xor_sync(0xffffffffu, nx, o);
    e += __shfl_xor_sync(0xffffffffu, e, o);
    hint = min(hint, __shfl_xor_sync(0xffffffffu, hint, o));
    timed_out |= __shfl_xor_sync(0xffffffffu, timed_out, o);
  }
  if (lane != 0) return;
  c->dp_epoch = ep;
  if (timed_out || e) {
    if (c->error == kErrNone) c->error = timed_out ? kErrDpTimeout : kErrPeer;
    c->stop = 1;
    c->stop_reason = -2;
    c->dp_done = 1;
    return;
  }
  if (b == 0) {  // no rank had a live row: drained (the iteration did not happen)
    c->stop = 1;
    c->stop_reason = AB_RUN_DRAINED;
    c->dp_done = 1;
    return;
  }
  c->iteration_index += 1;
  c->cumulative_tokens += b;
  c->completed_groups += g;
  c->completed_samples += smp;
  c->run_iters += 1;
  // trace stop rules: no rank can finish a sample for `hint` iterations (policy rules: unknown)
  c->iters_to_next = d.stop_mode != AB_STOP_TRACE ? -1 : (int32_t)(hint < 1 ? 1 : (hint > (1 << 14) ? (1 << 14) : hint));
  c->stop = 0;
  if (c->use_trigger && smp > 0 && trigger_fired(c)) {
    c->stop = 1;
    c->stop_reason = AB_RUN_TRIGGER;
  } else if (c->stop_on_event && smp > 0) {
    c->stop = 1;
    c->stop_reason = AB_RUN_EVENT;
  } else if (c->max_iters > 0 && c->run_iters >= c->max_iters) {
    c->stop = 1;
    c->stop_reason = AB_RUN_MAX_ITERS;
  } else if (nx == 0) {
    c->stop = 1;
    c->stop_reason = AB_RUN_DRAINED;
  }
  if (c->stop) c->dp_done = 1;
}

// Queue submitted descriptors behind the FIFO tail.
__global__ void k_submit(EngineDev d, const ab_sample_desc* descs, int n) {
  Ctl* c = d.ctl;
  const int tail = c->q_tail;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const ab_sample_desc s = descs[i];
    const int h = s.handle;
    d.h_gen[h] = s.gen_len;
    d.h_stop[h] = s.stop_at;
    d.h_group[h] = s.group_slot;
    d.h_key[h] = make_ulonglong2(s.key0, s.key1);
    if (s.gen_len == 0) d.h_version[h] = INT64_MIN;
    d.q_buf[(tail + i) % d.Q] = h;
  }
}
__global__ void k_submit_tail(EngineDev d, int n) { d.ctl->q_tail += n; }

// Context-free model: numpy-exact softmax/cumsum/log of one fp64 logits row
// (policy.py:87-90 softmax; engine.py:257-259 cdf and logp).
__global__ void k_cf_prepare(EngineDev d) {
  if (threadIdx.x || blockIdx.x) return;
  const int n = d.n_symbols;
  double m = d.cf_logits[0];
  for (int i = 1; i < n; ++i) m = fmax(m, d.cf_logits[i]);
  double* e = d.cf_logp;  // scratch
  for (int i = 0; i < n; ++i) e[i] = exp(d.cf_logits[i] - m);
  const double s = np_pairwise_sum(e, n);
  double run = 0.0;
  for (int i = 0; i < n; ++i) {
    const double p = e[i] / s;
    run += p;
    d.cf_cdf[i] = run;
    e[i] = p;
  }
  for (int i = 0; i < n; ++i) e[i] = log(e[i]);
}

__global__ void k_read_clock(EngineDev d) {
  if (threadIdx.x == 0 && blockIdx.x == 0) d.ctl->clock_ns = globaltimer_ns();
}

__global__ void k_gather_payload(EngineDev d, const int32_t* handles, const int32_t* starts, const int64_t* offs,
                                 int n, int32_t* tok, double* logp) {
  const int r = blockIdx.x;
  if (r >= n) return;
  const int h = handles[r], s = starts[r];
  const int64_t o = offs[r], cnt = offs[r + 1] - offs[r];
  for (int64_t j = threadIdx.x; j < cnt; j += blockDim.x) {
    tok[o + j] = d.h_tokens[(int64_t)h * d.L + s + j];
    logp[o + j] = d.h_logp[(int64_t)h * d.L + s + j];
  }
}

__global__ void k_set_groups(EngineDev d, const int32_t* slots_and_counts, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    d.g_done[slots_and_counts[2 * i]] = slots_and_counts[2 * i + 1];
}

// ---------------------------------------------------------------------------
// profiling
// ---------------------------------------------------------------------------

cudaEvent_t Engine::take_event() {
  if (!event_pool.empty()) {
    cudaEvent_t e = event_pool.back();
    event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  AB_CUDA(cudaEventCreate(&e));
  return e;
}

int Engine::timer_index(const char* name) {
  for (size_t i = 0; i < timers.size(); ++i)
    if (timers[i].name == name) return (int)i;
  timers.push_back(KernelTimer{name});
  return (int)timers.size() - 1;
}

// Timed launches are only captured into the profiled iteration graph: the
// event-record nodes sit between the kernel nodes, so the measured interval
// is the kernel's device time with no host submission gap in it.
ScopedTimer::ScopedTimer(Engine& eng, bool on, const char* name, int64_t run_iter_, double bytes_, double flops_)
    : e(eng), idx(-1), bytes(bytes_), flops(flops_), run_iter(run_iter_) {
  if (!on || !e.capturing_prof) return;
  idx = e.timer_index(name);
  a = e.take_event();
  AB_CUDA(cudaEventRecordWithFlags(a, e.stream, cudaEventRecordExternal));
}
ScopedTimer::~ScopedTimer() {
  if (idx < 0) return;
  cudaEvent_t b = e.take_event();
  cudaEventRecordWithFlags(b, e.stream, cudaEventRecordExternal);
  if ((int)e.prof_slots.size() <= e.variant) e.prof_slots.resize(e.variant + 1);
  e.prof_slots[e.variant].push_back(Engine::ProfSlot{idx, a, b});
}

// Accumulate the profiled graph's event intervals for launch `run_iter`.
static void collect_prof(Engine& e) {
  if (e.prof_pending < 0) return;
  const int64_t it = e.prof_pending;
  e.prof_pending = -1;
  if (it >= e.d.it_cap) return;
  int32_t b = 0;
  int64_t ctx = 0;
  AB_CUDA(cudaMemcpy(&b, e.d.it_b + it, sizeof(int32_t), cudaMemcpyDeviceToHost));
  AB_CUDA(cudaMemcpy(&ctx, e.d.it_ctx + it, sizeof(int64_t), cudaMemcpyDeviceToHost));
  if (b <= 0) return;  // iteration queued past the stop point: all kernels were no-ops
  if (e.prof_pending_variant >= (int)e.prof_slots.size()) return;
  for (auto& s : e.prof_slots[e.prof_pending_variant]) {
    float ms = 0;
    AB_CUDA(cudaEventElapsedTime(&ms, s.a, s.b));
    auto& t = e.timers[s.timer];
    double bytes = 0, flops = 0;
    if (e.model) model_kernel_cost(e.model, t.name, (double)b, (double)ctx, &bytes, &flops);
    t.launches += 1;
    t.ms += ms;
    t.bytes += bytes;
    t.flops += flops;
  }
}

static void collect_timers(Engine& e) {
  if (e.pending.empty()) return;
  AB_CUDA(cudaStreamSynchronize(e.stream));
  int64_t max_it = -1;
  for (auto& p : e.pending) max_it = std::max(max_it, p.run_iter);
  std::vector<int32_t> it_b;
  std::vector<int64_t> it_ctx;
  if (max_it >= 0) {
    const int64_t n = std::min<int64_t>(max_it + 1, e.d.it_cap);
    it_b.resize(n);
    it_ctx.resize(n);
    AB_CUDA(cudaMemcpy(it_b.data(), e.d.it_b, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
    AB_CUDA(cudaMemcpy(it_ctx.data(), e.d.it_ctx, sizeof(int64_t) * n, cudaMemcpyDeviceToHost));
  }
  for (auto& p : e.pending) {
    float ms = 0;
    AB_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    auto& t = e.timers[p.timer];
    double bytes = p.bytes, flops = p.flops;
    bool live = true;
    if (p.run_iter >= 0 && p.run_iter < (int64_t)it_b.size()) {
      const double b = it_b[p.run_iter];
      live = b > 0;  // iterations queued past the stop point are no-ops
      if (e.model) model_kernel_cost(e.model, t.name, b, (double)it_ctx[p.run_iter], &bytes, &flops);
    }
    if (live) {
      t.launches += 1;
      t.ms += ms;
      t.bytes += bytes;
      t.flops += flops;
    }
    e.event_pool.push_back(p.a);
    e.event_pool.push_back(p.b);
  }
  e.pending.clear();
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

template <typename T>
static T* dalloc(size_t n) {
  T* p = nullptr;
  if (n == 0) n = 1;
  AB_CUDA(cudaMalloc(&p, n * sizeof(T)));
  AB_CUDA(cudaMemset(p, 0, n * sizeof(T)));
  return p;
}

static void sync_ctl(Engine& e) {
  AB_CUDA(cudaMemcpyAsync(e.ctl_host, e.d.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, e.stream));
  AB_CUDA(cudaStreamSynchronize(e.stream));
}

static void push_ctl_fields(Engine& e) {
  AB_CUDA(cudaMemcpyAsync(e.d.ctl, e.ctl_host, sizeof(Ctl), cudaMemcpyHostToDevice, e.stream));
  AB_CUDA(cudaStreamSynchronize(e.stream));
}

static void validate(const ab_engine_config& c, const ab_model_config* m) {
  AB_REQUIRE(c.max_slots >= 1, AB_ERR_CONFIG, "max_slots must be >= 1, got " + std::to_string(c.max_slots));
  AB_REQUIRE(c.max_slots <= kFinishThreads * kMaxIPT, AB_ERR_CONFIG, "max_slots must be <= 4096");
  AB_REQUIRE(c.l_max >= 1, AB_ERR_CONFIG, "l_max must be >= 1, got " + std::to_string(c.l_max));
  AB_REQUIRE(c.max_handles >= c.max_slots, AB_ERR_CONFIG, "max_handles must be >= max_slots");
  AB_REQUIRE(c.max_groups >= 1, AB_ERR_CONFIG, "max_groups must be >= 1");
  AB_REQUIRE(c.stop_mode == AB_STOP_TRACE || c.stop_mode == AB_STOP_POLICY, AB_ERR_CONFIG, "unknown stop_mode");
  AB_REQUIRE(c.model_kind >= AB_MODEL_NONE && c.model_kind <= AB_MODEL_TRANSFORMER, AB_ERR_CONFIG,
             "unknown model_kind");
  if (c.model_kind == AB_MODEL_CONTEXT_FREE)
    AB_REQUIRE(c.n_symbols >= 2, AB_ERR_CONFIG, "context-free model needs >= 1 token plus STOP");
  if (c.model_kind == AB_MODEL_NONE)
    AB_REQUIRE(c.stop_mode == AB_STOP_TRACE, AB_ERR_CONFIG, "policy stop mode needs a model");
  if (c.model_kind == AB_MODEL_TRANSFORMER) {
    AB_REQUIRE(m != nullptr, AB_ERR_CONFIG, "transformer engine needs a model config");
    AB_REQUIRE(c.temperature > 0.f || c.greedy, AB_ERR_CONFIG, "temperature must be > 0");
    AB_REQUIRE(c.top_p > 0.f && c.top_p <= 1.f, AB_ERR_CONFIG, "top_p must lie in (0, 1]");
    AB_REQUIRE(c.n_eos >= 0 && c.n_eos <= 8, AB_ERR_CONFIG, "at most 8 EOS ids");
    AB_REQUIRE(!c.kv_resume || c.record_payload, AB_ERR_CONFIG, "KV re-prefill needs the token payload on device");
  }
  AB_REQUIRE(c.kv_resume == 0 || c.kv_resume == 1, AB_ERR_CONFIG, "kv_resume must be 0 or 1");
}

static Engine* create(const ab_engine_config* cfgp, const ab_model_config* m, int device) {
  AB_REQUIRE(cfgp != nullptr, AB_ERR_CONFIG, "null config");
  validate(*cfgp, m);
  Engine* e = new Engine();
  e->cfg = *cfgp;
  if (m) e->mcfg = *m;
  e->device = device;
  AB_CUDA(cudaSetDevice(device));
  AB_CUDA(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
  const auto& c = e->cfg;
  EngineDev& d = e->d;
  d.S = c.max_slots;
  d.H = c.max_handles;
  d.Q = c.max_handles;
  d.L = c.l_max;
  d.G_cap = c.max_groups;
  d.stop_mode = c.stop_mode;
  d.model_kind = c.model_kind;
  d.n_symbols = c.n_symbols;
  d.l_max = c.l_max;
  d.record = c.record_payload && c.model_kind != AB_MODEL_NONE;
  d.n_eos = c.n_eos;
  for (int i = 0; i < 8; ++i) d.eos[i] = c.eos_ids[i];
  d.ctl = dalloc<Ctl>(1);
  d.slot_handle = dalloc<int32_t>(d.S);
  d.slot_tmp = dalloc<int32_t>(d.S);
  d.slot_finish = dalloc<int32_t>(d.S);
  d.slot_token = dalloc<int32_t>(d.S);
  d.q_buf = dalloc<int32_t>(d.Q);
  d.h_gen = dalloc<int32_t>(d.H);
  d.h_stop = dalloc<int32_t>(d.H);
  d.h_group = dalloc<int32_t>(d.H);
  d.h_key = dalloc<ulonglong2>(d.H);
  d.h_version = dalloc<int64_t>(d.H);
  if (d.record) {
    d.h_tokens = dalloc<int32_t>((size_t)d.H * d.L);
    d.h_logp = dalloc<double>((size_t)d.H * d.L);
  }
  d.g_done = dalloc<int32_t>(d.G_cap);
  if (c.model_kind == AB_MODEL_TRANSFORMER && c.kv_resume) d.h_needs_pf = dalloc<int32_t>(d.H);
  d.ev = dalloc<ab_event>(d.H + d.S);
  d.adm = dalloc<ab_admit>(d.H + d.S);
  if (c.model_kind == AB_MODEL_CONTEXT_FREE) {
    d.cf_logits = dalloc<double>(c.n_symbols);
    d.cf_cdf = dalloc<double>(c.n_symbols);
    d.cf_logp = dalloc<double>(c.n_symbols);
  }
  d.it_cap = 1 << 20;
  d.it_b = dalloc<int32_t>(d.it_cap);
  d.it_ctx = dalloc<int64_t>(d.it_cap);
  AB_CUDA(cudaMallocHost(&e->ctl_host, sizeof(Ctl)));
  memset(e->ctl_host, 0, sizeof(Ctl));
  e->ctl_host->version = INT64_MIN;
  e->ctl_host->stop = 1;
  push_ctl_fields(*e);
  {
    std::vector<int64_t> v(d.H, INT64_MIN);
    AB_CUDA(cudaMemcpy(d.h_version, v.data(), d.H * sizeof(int64_t), cudaMemcpyHostToDevice));
  }
  AB_CUDA(cudaMallocHost(&e->stage_desc_host, sizeof(ab_sample_desc) * (d.H + 1)));
  e->stage_desc_dev = dalloc<ab_sample_desc>(d.H + 1);
  e->stage_i32_cap = (size_t)4 * d.H + 16;
  AB_CUDA(cudaMallocHost(&e->stage_i32_host, sizeof(int32_t) * e->stage_i32_cap));
  e->stage_i32_dev = dalloc<int32_t>(e->stage_i32_cap);
  k_read_clock<<<1, 1, 0, e->stream>>>(d);
  sync_ctl(*e);
  d.t0_ns = e->ctl_host->clock_ns;
  if (c.model_kind == AB_MODEL_TRANSFORMER) e->model = model_create(*e);
  AB_CUDA(cudaStreamSynchronize(e->stream));
  return e;
}

static void destroy(Engine* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  cudaStreamSynchronize(e->stream);
  for (auto g : e->iter_graphs)
    if (g) cudaGraphExecDestroy(g);
  for (auto g : e->prof_graphs)
    if (g) cudaGraphExecDestroy(g);
  for (auto& v : e->prof_slots)
    for (auto& s : v) {
      cudaEventDestroy(s.a);
      cudaEventDestroy(s.b);
    }
  if (e->model) model_destroy(e->model);
  EngineDev& d = e->d;
  void* ptrs[] = {d.ctl,     d.slot_handle, d.slot_tmp, d.slot_finish, d.slot_token, d.q_buf,  d.h_gen,
                  d.h_stop,  d.h_group,     d.h_key,    d.h_version,   d.h_tokens,   d.h_logp, d.g_done,
                  d.ev,      d.adm,         d.cf_logits, d.cf_cdf,     d.cf_logp,    d.it_b,   d.it_ctx,
                  d.h_needs_pf,
                  e->stage_desc_dev, e->stage_i32_dev};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (e->ctl_host) cudaFreeHost(e->ctl_host);
  if (e->stage_desc_host) cudaFreeHost(e->stage_desc_host);
  if (e->stage_i32_host) cudaFreeHost(e->stage_i32_host);
  for (void* p : e->dp_ipc_opened) cudaIpcCloseMemHandle(p);
  if (e->dp_peers_dev) cudaFree(e->dp_peers_dev);
  if (e->dp_buf) cudaFree(e->dp_buf);
  for (auto ev : e->event_pool) cudaEventDestroy(ev);
  for (auto& p : e->pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  cudaStreamDestroy(e->stream);
  delete e;
}

static void begin_step(Engine& e, int64_t version, const double* logits) {
  sync_ctl(e);
  AB_REQUIRE(e.ctl_host->b == 0 && e.ctl_host->q_tail == e.ctl_host->q_head, AB_ERR_CONTRACT,
             "begin_step requires an idle engine");
  e.ctl_host->version = version;
  AB_CUDA(cudaMemcpyAsync(&e.d.ctl->version, &version, sizeof(int64_t), cudaMemcpyHostToDevice, e.stream));
  if (e.cfg.model_kind == AB_MODEL_CONTEXT_FREE) {
    AB_REQUIRE(logits != nullptr, AB_ERR_CONTRACT, "policy-driven decode needs policy parameters");
    for (int i = 0; i < e.cfg.n_symbols; ++i)
      AB_REQUIRE(std::isfinite(logits[i]), AB_ERR_CONTRACT, "logits must be finite");
    AB_CUDA(cudaMemcpyAsync(e.d.cf_logits, logits, sizeof(double) * e.cfg.n_symbols, cudaMemcpyHostToDevice,
                            e.stream));
    k_cf_prepare<<<1, 1, 0, e.stream>>>(e.d);
  }
  if (e.model) model_begin_step(e, version);
  AB_CUDA(cudaStreamSynchronize(e.stream));
}

static void submit(Engine& e, const ab_sample_desc* descs, int n) {
  if (n <= 0) return;
  sync_ctl(e);
  const int queued = e.ctl_host->q_tail - e.ctl_host->q_head;
  AB_REQUIRE(queued + n <= e.d.Q, AB_ERR_CONTRACT, "submission queue full");
  for (int i = 0; i < n; ++i) {
    const auto& s = descs[i];
    AB_REQUIRE(s.handle >= 0 && s.handle < e.d.H, AB_ERR_CONTRACT, "sample handle out of range");
    AB_REQUIRE(s.group_slot >= 0 && s.group_slot < e.d.G_cap, AB_ERR_CONTRACT, "group slot out of range");
    AB_REQUIRE(s.gen_len >= 0 && s.gen_len <= e.cfg.l_max, AB_ERR_CONTRACT, "gen_len out of range");
  }
  memcpy(e.stage_desc_host, descs, sizeof(ab_sample_desc) * n);
  AB_CUDA(cudaMemcpyAsync(e.stage_desc_dev, e.stage_desc_host, sizeof(ab_sample_desc) * n, cudaMemcpyHostToDevice,
                          e.stream));
  k_submit<<<ceil_div(n, 256), 256, 0, e.stream>>>(e.d, e.stage_desc_dev, n);
  if (e.model) model_submit(e, e.stage_desc_dev, n);
  k_submit_tail<<<1, 1, 0, e.stream>>>(e.d, n);
  AB_CUDA(cudaStreamSynchronize(e.stream));
}

static void launch_iteration(Engine& e, int64_t run_iter, bool timed = false) {
  e.launches += 2 + (e.model ? model_iter_launches(e.model, e.variant) : 1);
  {
    ScopedTimer t(e, timed, "admit", run_iter);
    k_admit<<<1, 256, 0, e.stream>>>(e.d);
  }
  if (e.model) {
    model_iteration(e, run_iter, timed, e.variant);
  } else {
    ScopedTimer t(e, timed, "grow", run_iter);
    k_grow_cf<<<ceil_div(e.d.S, 128), 128, 0, e.stream>>>(e.d);
  }
  {
    ScopedTimer t(e, timed, "finish", run_iter);
    k_finish<<<1, kFinishThreads, 0, e.stream>>>(e.d);
  }
  if (e.d.dp_world > 1) {
    ScopedTimer t(e, timed, "dp_exchange", run_iter);
    k_dp_exchange<<<1, 32, 0, e.stream>>>(e.d);
    e.launches += 1;
  }
}

// Iterations are replayed from one captured CUDA graph: every kernel reads the
// live batch size and the stop flag from the device control block, so the
// same graph serves every batch size.  When profiling, the first iteration of
// every `sample_every`-th host chunk replays a second graph that also holds
// event-record nodes around each kernel class.
static cudaGraphExec_t capture_iteration(Engine& e, bool timed) {
  const int64_t before = e.launches;
  cudaGraph_t g;
  cudaGraphExec_t x;
  e.capturing_prof = timed;
  AB_CUDA(cudaStreamBeginCapture(e.stream, cudaStreamCaptureModeThreadLocal));
  launch_iteration(e, -1, timed);
  AB_CUDA(cudaStreamEndCapture(e.stream, &g));
  e.capturing_prof = false;
  AB_CUDA(cudaGraphInstantiate(&x, g, 0));
  AB_CUDA(cudaGraphDestroy(g));
  if ((int)e.graph_kernels.size() <= e.variant) e.graph_kernels.resize(e.variant + 1, 0);
  e.graph_kernels[e.variant] = e.launches - before;
  e.launches = before;
  return x;
}

static void launch_iteration_fast(Engine& e, int64_t run_iter, bool first_in_chunk) {
  if (!e.use_graphs || e.direct_launches < 1) {  // first call: plain launches set up kernel attributes
    launch_iteration(e, run_iter);
    ++e.direct_launches;
    return;
  }
  const int v = e.variant;
  if ((int)e.iter_graphs.size() <= v) {
    e.iter_graphs.resize(v + 1, nullptr);
    e.prof_graphs.resize(v + 1, nullptr);
  }
  if (!e.iter_graphs[v]) e.iter_graphs[v] = capture_iteration(e, false);
  bool prof = false;
  if (e.profile && first_in_chunk && e.prof_pending < 0) prof = (e.prof_count++ % e.sample_every) == 0;
  if (prof) {
    if (!e.prof_graphs[v]) e.prof_graphs[v] = capture_iteration(e, true);
    AB_CUDA(cudaGraphLaunch(e.prof_graphs[v], e.stream));
    e.prof_pending = run_iter;
    e.prof_pending_variant = v;
  } else {
    AB_CUDA(cudaGraphLaunch(e.iter_graphs[v], e.stream));
  }
  e.launches += e.graph_kernels[v];
}

static void run(Engine& e, const ab_run_args* a, ab_run_result* r, ab_event* ev, int ev_cap, ab_admit* adm,
                int adm_cap) {
  AB_REQUIRE(a && r, AB_ERR_CONTRACT, "null run arguments");
  AB_REQUIRE(a->group_size >= 0, AB_ERR_CONTRACT, "group_size must be >= 0");
  k_run_begin<<<1, 1, 0, e.stream>>>(e.d, *a);
  if (e.profile) {
    AB_CUDA(cudaMemsetAsync(e.d.it_b, 0, sizeof(int32_t) * e.d.it_cap, e.stream));
    AB_CUDA(cudaMemsetAsync(e.d.it_ctx, 0, sizeof(int64_t) * e.d.it_cap, e.stream));
  }
  if (e.model) sync_ctl(e);  // live batch + queue: the first chunk's graph variant
  int64_t launched = 0;
  int chunk = 1;
  const int policy_chunk = 4;
  while (true) {
    int n = chunk;
    if (a->max_iters > 0) n = (int)std::min<int64_t>(n, std::max<int64_t>(1, a->max_iters - launched));
    if (e.model) {
      // admission only happens at iteration starts from the FIFO: no iteration of this chunk can
      // have more live rows than the current batch plus the queue (capped at S)
      const Ctl& c0 = *e.ctl_host;
      const int bmax = (int)std::min<int64_t>(e.d.S, (int64_t)c0.b + (c0.q_tail - c0.q_head));
      e.variant = model_variant_for(e.model, bmax);
    }
    {
      NvtxRange r("april.chunk");
      for (int i = 0; i < n; ++i) launch_iteration_fast(e, launched + i, i == 0);
      launched += n;
      sync_ctl(e);
    }
    collect_prof(e);
    const Ctl& c = *e.ctl_host;
    if (c.stop && c.stop_reason == kRunNeedPrefill && c.error == kErrNone) {
      // rebuild the KV of the samples the next admission takes (plus a few beyond it), then go on
      const int want = std::min(e.d.S - c.b, c.q_tail - c.q_head);
      AB_REQUIRE(model_prefill_deferred(e, std::max(1, want) + 8) > 0, AB_ERR_CONTRACT,
                 "a queued sample waits for a KV rebuild that is not pending");
      e.ctl_host->stop = 0;
      e.ctl_host->stop_reason = -1;
      static_assert(offsetof(Ctl, stop_reason) == offsetof(Ctl, stop) + 4, "layout");
      AB_CUDA(cudaMemcpyAsync(&e.d.ctl->stop, &e.ctl_host->stop, 2 * sizeof(int32_t), cudaMemcpyHostToDevice,
                              e.stream));
      chunk = 1;
      continue;
    }
    if (c.stop) break;
    if (c.iters_to_next > 0)
      chunk = c.iters_to_next;
    else
      chunk = policy_chunk;
    chunk = std::min(chunk, 1 << 14);
  }
  collect_timers(e);
  const Ctl& c = *e.ctl_host;
  if (c.error != kErrNone) {
    // roll back nothing: the reference raises mid-admission as well (engine.py:141-146)
    std::string msg;
    if (c.error == kErrVersion)
      msg = "segment versions must strictly increase (handle " + std::to_string(c.error_handle) + ")";
    else if (c.error == kErrAtStop)
      msg = "sample handle " + std::to_string(c.error_handle) + " already at its stop point";
    else if (c.error == kErrNoTarget)
      msg = "sample handle " + std::to_string(c.error_handle) + " has no target length";
    else if (c.error == kErrOutOfKV)
      throw Error(AB_ERR_OUT_OF_KV, "KV page pool exhausted during decode (" + model_kv_report(e) + ")");
    else if (c.error == kErrPeer)
      throw Error(AB_ERR_NCCL, "data-parallel: a peer rank's iteration failed");
    else if (c.error == kErrDpTimeout)
      throw Error(AB_ERR_NCCL, "data-parallel: a peer rank's exchange record did not arrive in time");
    throw Error(AB_ERR_CONTRACT, msg);
  }
  AB_REQUIRE(c.n_events <= ev_cap || ev == nullptr, AB_ERR_CONTRACT, "event buffer too small");
  AB_REQUIRE(c.n_admits <= adm_cap || adm == nullptr, AB_ERR_CONTRACT, "admit buffer too small");
  if (ev && c.n_events)
    AB_CUDA(cudaMemcpyAsync(ev, e.d.ev, sizeof(ab_event) * c.n_events, cudaMemcpyDeviceToHost, e.stream));
  if (adm && c.n_admits)
    AB_CUDA(cudaMemcpyAsync(adm, e.d.adm, sizeof(ab_admit) * c.n_admits, cudaMemcpyDeviceToHost, e.stream));
  AB_CUDA(cudaStreamSynchronize(e.stream));
  r->iterations = c.run_iters;
  r->stop_reason = c.stop_reason;
  r->n_events = c.n_events;
  r->n_admits = c.n_admits;
  r->completed_groups = c.completed_groups;
  r->completed_samples = c.completed_samples;
  r->iteration_index = c.iteration_index;
  r->cumulative_tokens = c.cumulative_tokens;
}

static void abort_active(Engine& e, int32_t* handles, int32_t* gen, int cap, int* n_active, int* n_queued) {
  sync_ctl(e);
  Ctl& c = *e.ctl_host;
  const int b = c.b, q = c.q_tail - c.q_head;
  AB_REQUIRE(b + q <= cap, AB_ERR_CONTRACT, "abort buffer too small");
  std::vector<int32_t> qh(e.d.Q);
  if (b) AB_CUDA(cudaMemcpy(handles, e.d.slot_handle, sizeof(int32_t) * b, cudaMemcpyDeviceToHost));
  if (q) {
    AB_CUDA(cudaMemcpy(qh.data(), e.d.q_buf, sizeof(int32_t) * e.d.Q, cudaMemcpyDeviceToHost));
    for (int i = 0; i < q; ++i) handles[b + i] = qh[(c.q_head + i) % e.d.Q];
  }
  if (gen && b + q) {
    std::vector<int32_t> all(e.d.H);
    AB_CUDA(cudaMemcpy(all.data(), e.d.h_gen, sizeof(int32_t) * e.d.H, cudaMemcpyDeviceToHost));
    for (int i = 0; i < b + q; ++i) gen[i] = all[handles[i]];
  }
  c.b = 0;
  c.q_head = c.q_tail;
  if (e.model) model_drop_deferred(e);
  AB_CUDA(cudaMemcpy(&e.d.ctl->b, &c.b, sizeof(int32_t), cudaMemcpyHostToDevice));
  AB_CUDA(cudaMemcpy(&e.d.ctl->q_head, &c.q_head, sizeof(int32_t), cudaMemcpyHostToDevice));
  if (e.model && e.cfg.kv_resume && b + q) {
    std::vector<int32_t> g2(b + q);
    if (!gen) {
      std::vector<int32_t> all(e.d.H);
      AB_CUDA(cudaMemcpy(all.data(), e.d.h_gen, sizeof(int32_t) * e.d.H, cudaMemcpyDeviceToHost));
      for (int i = 0; i < b + q; ++i) g2[i] = all[handles[i]];
    }
    model_evict(e, handles, gen ? gen : g2.data(), b + q);
  }
  *n_active = b;
  *n_queued = q;
}

static void active(Engine& e, int32_t* handles, int32_t* gen, int cap, int* n_active) {
  sync_ctl(e);
  const int b = e.ctl_host->b;
  AB_REQUIRE(b <= cap, AB_ERR_CONTRACT, "buffer too small");
  if (b) AB_CUDA(cudaMemcpy(handles, e.d.slot_handle, sizeof(int32_t) * b, cudaMemcpyDeviceToHost));
  if (gen && b) {
    std::vector<int32_t> all(e.d.H);
    AB_CUDA(cudaMemcpy(all.data(), e.d.h_gen, sizeof(int32_t) * e.d.H, cudaMemcpyDeviceToHost));
    for (int i = 0; i < b; ++i) gen[i] = all[handles[i]];
  }
  *n_active = b;
}

static void read_payload(Engine& e, const int32_t* handles, const int32_t* starts, const int32_t* counts, int n,
                         int32_t* tok, double* logp) {
  AB_REQUIRE(e.d.record, AB_ERR_CONTRACT, "engine does not record token payloads");
  if (n <= 0) return;
  std::vector<int64_t> offs(n + 1, 0);
  for (int i = 0; i < n; ++i) {
    AB_REQUIRE(handles[i] >= 0 && handles[i] < e.d.H, AB_ERR_CONTRACT, "handle out of range");
    AB_REQUIRE(starts[i] >= 0 && counts[i] >= 0 && starts[i] + counts[i] <= e.d.L, AB_ERR_CONTRACT,
               "payload range out of bounds");
    offs[i + 1] = offs[i] + counts[i];
  }
  const int64_t total = offs[n];
  int32_t *dh, *ds, *dt;
  int64_t* doff;
  double* dl;
  // stream-ordered scratch: no device-wide synchronisation (other engines of this process may be
  // decoding on the same device)
  AB_CUDA(cudaMallocAsync(&dh, sizeof(int32_t) * n, e.stream));
  AB_CUDA(cudaMallocAsync(&ds, sizeof(int32_t) * n, e.stream));
  AB_CUDA(cudaMallocAsync(&doff, sizeof(int64_t) * (n + 1), e.stream));
  AB_CUDA(cudaMallocAsync(&dt, sizeof(int32_t) * std::max<int64_t>(1, total), e.stream));
  AB_CUDA(cudaMallocAsync(&dl, sizeof(double) * std::max<int64_t>(1, total), e.stream));
  AB_CUDA(cudaMemcpyAsync(dh, handles, sizeof(int32_t) * n, cudaMemcpyHostToDevice, e.stream));
  AB_CUDA(cudaMemcpyAsync(ds, starts, sizeof(int32_t) * n, cudaMemcpyHostToDevice, e.stream));
  AB_CUDA(cudaMemcpyAsync(doff, offs.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, e.stream));
  k_gather_payload<<<n, 128, 0, e.stream>>>(e.d, dh, ds, doff, n, dt, dl);
  if (total) {
    if (tok) AB_CUDA(cudaMemcpyAsync(tok, dt, sizeof(int32_t) * total, cudaMemcpyDeviceToHost, e.stream));
    if (logp) AB_CUDA(cudaMemcpyAsync(logp, dl, sizeof(double) * total, cudaMemcpyDeviceToHost, e.stream));
  }
  cudaFreeAsync(dh, e.stream);
  cudaFreeAsync(ds, e.stream);
  cudaFreeAsync(doff, e.stream);
  cudaFreeAsync(dt, e.stream);
  cudaFreeAsync(dl, e.stream);
  AB_CUDA(cudaStreamSynchronize(e.stream));
}

// Per-sample sum of the recorded behaviour log-probabilities over all generated tokens (one
// warp per handle, lane-strided partial sums combined by a fixed xor tree: deterministic).
// GSPO's length-normalised sequence log-ratio uses sum / length.
__global__ void k_seq_logprob(EngineDev e, const int32_t* __restrict__ handles, int n, double* __restrict__ sums,
                              int32_t* __restrict__ lens) {
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= n) return;
  const int h = handles[i];
  const int len = e.h_gen[h];
  const double* lp = e.h_logp + (size_t)h * e.L;
  double acc = 0.0;
  for (int j = lane; j < len; j += 32) acc += lp[j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) {
    sums[i] = acc;
    lens[i] = len;
  }
}

static void seq_logprob(Engine& e, const int32_t* handles, int n, double* sums, int32_t* lens) {
  AB_REQUIRE(e.d.record, AB_ERR_CONTRACT, "engine does not record token payloads");
  if (n <= 0) return;
  for (int i = 0; i < n; ++i) AB_REQUIRE(handles[i] >= 0 && handles[i] < e.d.H, AB_ERR_CONTRACT, "handle out of range");
  int32_t *dh, *dn;
  double* ds;
  AB_CUDA(cudaMallocAsync(&dh, sizeof(int32_t) * n, e.stream));
  AB_CUDA(cudaMallocAsync(&dn, sizeof(int32_t) * n, e.stream));
  AB_CUDA(cudaMallocAsync(&ds, sizeof(double) * n, e.stream));
  AB_CUDA(cudaMemcpyAsync(dh, handles, sizeof(int32_t) * n, cudaMemcpyHostToDevice, e.stream));
  k_seq_logprob<<<ceil_div(n, 8), 256, 0, e.stream>>>(e.d, dh, n, ds, dn);
  AB_CUDA(cudaGetLastError());
  AB_CUDA(cudaMemcpyAsync(sums, ds, sizeof(double) * n, cudaMemcpyDeviceToHost, e.stream));
  AB_CUDA(cudaMemcpyAsync(lens, dn, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, e.stream));
  cudaFreeAsync(dh, e.stream);
  cudaFreeAsync(dn, e.stream);
  cudaFreeAsync(ds, e.stream);
  AB_CUDA(cudaStreamSynchronize(e.stream));
}

static void set_groups(Engine& e, const int32_t* pairs, int n) {
  if (n <= 0) return;
  AB_REQUIRE((size_t)2 * n <= e.stage_i32_cap, AB_ERR_CONTRACT, "too many groups");
  for (int i = 0; i < n; ++i) AB_REQUIRE(pairs[2 * i] >= 0 && pairs[2 * i] < e.d.G_cap, AB_ERR_CONTRACT,
                                         "group slot out of range");
  memcpy(e.stage_i32_host, pairs, sizeof(int32_t) * 2 * n);
  AB_CUDA(cudaMemcpyAsync(e.stage_i32_dev, e.stage_i32_host, sizeof(int32_t) * 2 * n, cudaMemcpyHostToDevice,
                          e.stream));
  k_set_groups<<<ceil_div(n, 256), 256, 0, e.stream>>>(e.d, e.stage_i32_dev, n);
  AB_CUDA(cudaStreamSynchronize(e.stream));
}

static double read_clock(Engine& e) {
  k_read_clock<<<1, 1, 0, e.stream>>>(e.d);
  sync_ctl(e);
  return (double)(e.ctl_host->clock_ns - e.d.t0_ns) * 1e-9;
}

static void drop_graphs(Engine& e) {
  for (auto& x : e.iter_graphs)
    if (x) cudaGraphExecDestroy(x), x = nullptr;
  for (auto& x : e.prof_graphs)
    if (x) cudaGraphExecDestroy(x), x = nullptr;
}

static void dp_detach(Engine& e) {
  AB_CUDA(cudaStreamSynchronize(e.stream));
  for (void* p : e.dp_ipc_opened) cudaIpcCloseMemHandle(p);
  e.dp_ipc_opened.clear();
  if (e.dp_peers_dev) cudaFree(e.dp_peers_dev);
  e.dp_peers_dev = nullptr;
  e.d.dp_world = 0;
  e.d.dp_rank = 0;
  e.d.dp_peers = nullptr;
  drop_graphs(e);
}

static void dp_export(Engine& e, int world, uint64_t* dev_ptr, void* ipc) {
  AB_REQUIRE(world >= 2 && world <= 32, AB_ERR_CONFIG, "data-parallel world size must lie in [2, 32]");
  if (e.dp_buf) {
    dp_detach(e);
    cudaFree(e.dp_buf);
    e.dp_buf = nullptr;
  }
  const size_t bytes = sizeof(int64_t) * 2 * world * kDpRec;
  AB_CUDA(cudaMalloc(&e.dp_buf, bytes));
  AB_CUDA(cudaMemset(e.dp_buf, 0, bytes));
  AB_CUDA(cudaDeviceSynchronize());
  *dev_ptr = (uint64_t)(uintptr_t)e.dp_buf;
  if (ipc) {
    cudaIpcMemHandle_t h;
    AB_CUDA(cudaIpcGetMemHandle(&h, e.dp_buf));
    static_assert(sizeof(h) == 64, "CUDA IPC handle is 64 bytes");
    memcpy(ipc, &h, sizeof(h));
  }
}

static void dp_attach(Engine& e, int world, int rank, const ab_dp_peer* peers, int64_t timeout_ms) {
  AB_REQUIRE(e.dp_buf != nullptr, AB_ERR_CONTRACT, "ab_engine_dp_export must precede ab_engine_dp_attach");
  AB_REQUIRE(world >= 2 && world <= 32 && rank >= 0 && rank < world, AB_ERR_CONFIG, "bad data-parallel rank");
  sync_ctl(e);
  AB_REQUIRE(e.ctl_host->b == 0 && e.ctl_host->q_tail == e.ctl_host->q_head, AB_ERR_CONTRACT,
             "dp_attach requires an idle engine");
  std::vector<int64_t*> ptrs(world, nullptr);
  for (int r = 0; r < world; ++r) {
    if (r == rank) {
      ptrs[r] = e.dp_buf;
    } else if (peers[r].kind == 0) {  // same process (tests: several engines on one device)
      ptrs[r] = (int64_t*)(uintptr_t)peers[r].ptr;
    } else {
      cudaIpcMemHandle_t h;
      memcpy(&h, peers[r].ipc, sizeof(h));
      void* p = nullptr;
      AB_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      e.dp_ipc_opened.push_back(p);
      ptrs[r] = (int64_t*)p;
    }
    AB_REQUIRE(ptrs[r] != nullptr, AB_ERR_CONTRACT, "null peer exchange buffer");
  }
  if (e.dp_peers_dev) cudaFree(e.dp_peers_dev);
  AB_CUDA(cudaMalloc(&e.dp_peers_dev, sizeof(int64_t*) * world));
  AB_CUDA(cudaMemcpy(e.dp_peers_dev, ptrs.data(), sizeof(int64_t*) * world, cudaMemcpyHostToDevice));
  e.d.dp_world = world;
  e.d.dp_rank = rank;
  e.d.dp_peers = e.dp_peers_dev;
  e.d.dp_local = e.dp_buf;
  e.d.dp_timeout_ns = (uint64_t)(timeout_ms > 0 ? timeout_ms : 60000) * 1000000ull;
  e.ctl_host->dp_epoch = 0;
  e.ctl_host->dp_done = 0;
  AB_CUDA(cudaMemcpy(&e.d.ctl->dp_epoch, &e.ctl_host->dp_epoch, sizeof(int64_t), cudaMemcpyHostToDevice));
  drop_graphs(e);  // the iteration graphs now end with the exchange
}

template <typename F>
static int guard(F&& f) {
  try {
    f();
    return AB_OK;
  } catch (const Error& err) {
    g_last_error = err.what();
    return err.code;
  } catch (const std::exception& err) {
    g_last_error = err.what();
    return AB_ERR_CUDA;
  }
}

}  // namespace ab

using ab::Engine;

struct ab_engine {
  Engine* impl;
};

extern "C" {

const char* ab_last_error(void) { return ab::g_last_error.c_str(); }
int ab_version(void) { return 1; }

int ab_engine_create(const ab_engine_config* cfg, const ab_model_config* model, int device, ab_engine** out) {
  return ab::guard([&] {
    AB_REQUIRE(out != nullptr, AB_ERR_CONFIG, "null output pointer");
    *out = nullptr;
    Engine* e = ab::create(cfg, model, device);
    *out = new ab_engine{e};
  });
}

int ab_engine_destroy(ab_engine* e) {
  return ab::guard([&] {
    if (!e) return;
    ab::destroy(e->impl);
    delete e;
  });
}

int ab_engine_begin_step(ab_engine* e, int64_t version, const double* cf_logits) {
  ab::NvtxRange nvtx("april.begin_step");
  return ab::guard([&] { ab::begin_step(*e->impl, version, cf_logits); });
}

int ab_engine_submit(ab_engine* e, const ab_sample_desc* descs, int n) {
  ab::NvtxRange nvtx("april.submit");
  return ab::guard([&] { ab::submit(*e->impl, descs, n); });
}

int ab_engine_set_group_done(ab_engine* e, const int32_t* slot_count_pairs, int n) {
  return ab::guard([&] { ab::set_groups(*e->impl, slot_count_pairs, n); });
}

int ab_engine_run(ab_engine* e, const ab_run_args* args, ab_run_result* res, ab_event* events, int event_cap,
                  ab_admit* admits, int admit_cap) {
  ab::NvtxRange nvtx("april.run");
  return ab::guard([&] { ab::run(*e->impl, args, res, events, event_cap, admits, admit_cap); });
}

int ab_engine_abort(ab_engine* e, int32_t* handles, int32_t* gen, int cap, int* n_active, int* n_queued) {
  ab::NvtxRange nvtx("april.abort");
  return ab::guard([&] { ab::abort_active(*e->impl, handles, gen, cap, n_active, n_queued); });
}

int ab_engine_active(ab_engine* e, int32_t* handles, int32_t* gen, int cap, int* n_active) {
  return ab::guard([&] { ab::active(*e->impl, handles, gen, cap, n_active); });
}

int ab_engine_read_payload(ab_engine* e, const int32_t* handles, const int32_t* starts, const int32_t* counts, int n,
                           int32_t* tokens, double* logprobs) {
  ab::NvtxRange nvtx("april.read_payload");
  return ab::guard([&] { ab::read_payload(*e->impl, handles, starts, counts, n, tokens, logprobs); });
}

int ab_engine_sequence_logprobs(ab_engine* e, const int32_t* handles, int n, double* sums, int32_t* lens) {
  ab::NvtxRange nvtx("april.sequence_logprobs");
  return ab::guard([&] { ab::seq_logprob(*e->impl, handles, n, sums, lens); });
}

int ab_engine_score(ab_engine* e, const int32_t* tokens, const int64_t* offs, const int32_t* prompt_lens, int n,
                    double* logprobs) {
  ab::NvtxRange nvtx("april.score");
  return ab::guard([&] {
    Engine& g = *e->impl;
    AB_REQUIRE(g.model != nullptr, AB_ERR_CONTRACT, "scoring needs the transformer model");
    AB_REQUIRE(n >= 0 && tokens && offs && prompt_lens && logprobs, AB_ERR_CONTRACT, "score: null argument");
    if (n) ab::model_score(g, tokens, offs, prompt_lens, n, logprobs);
  });
}

int ab_engine_release(ab_engine* e, const int32_t* handles, int n) {
  return ab::guard([&] {
    Engine& g = *e->impl;
    if (!g.model || n <= 0) return;
    AB_REQUIRE((size_t)n <= g.stage_i32_cap, AB_ERR_CONTRACT, "too many handles");
    ab::model_forget_deferred(g, handles, n);
    memcpy(g.stage_i32_host, handles, sizeof(int32_t) * n);
    AB_CUDA(cudaMemcpyAsync(g.stage_i32_dev, g.stage_i32_host, sizeof(int32_t) * n, cudaMemcpyHostToDevice,
                            g.stream));
    if (g.d.h_needs_pf) {  // a released handle is never waiting for a rebuild
      const int32_t zero = 0;
      for (int i = 0; i < n; ++i)
        AB_CUDA(cudaMemcpyAsync(g.d.h_needs_pf + handles[i], &zero, sizeof(int32_t), cudaMemcpyHostToDevice, g.stream));
    }
    ab::model_release(g, g.stage_i32_dev, n);
    AB_CUDA(cudaStreamSynchronize(g.stream));
  });
}

int ab_engine_open_group(ab_engine* e, int32_t group_slot, const int32_t* prompt, int32_t prompt_len) {
  ab::NvtxRange nvtx("april.open_group");
  return ab::guard([&] {
    Engine& g = *e->impl;
    AB_REQUIRE(group_slot >= 0 && group_slot < g.d.G_cap, AB_ERR_CONTRACT, "group slot out of range");
    if (!g.model) return;
    ab::model_open_group(g, group_slot, prompt, prompt_len);
  });
}

// KV memory hand-off: free the KV pool while a co-located trainer runs, then
// re-acquire it.  Re-prefill mode only (paused partials hold no KV there); the resident prompt KV
// is recomputed by the next submit.  The captured iteration graphs embed the pool address and are
// re-captured.
int ab_engine_release_memory(ab_engine* e) {
  ab::NvtxRange nvtx("april.release_memory");
  return ab::guard([&] {
    Engine& g = *e->impl;
    AB_REQUIRE(g.model != nullptr, AB_ERR_CONTRACT, "engine has no transformer model");
    AB_REQUIRE(g.cfg.kv_resume == 1, AB_ERR_CONTRACT, "releasing the KV pool needs kv_resume = reprefill");
    sync_ctl(g);
    AB_REQUIRE(g.ctl_host->b == 0 && g.ctl_host->q_tail == g.ctl_host->q_head, AB_ERR_CONTRACT,
               "release_memory requires an idle engine");
    ab::model_release_memory(g);
  });
}

int ab_engine_resume_memory(ab_engine* e) {
  ab::NvtxRange nvtx("april.resume_memory");
  return ab::guard([&] {
    Engine& g = *e->impl;
    AB_REQUIRE(g.model != nullptr, AB_ERR_CONTRACT, "engine has no transformer model");
    ab::model_resume_memory(g);
    ab::drop_graphs(g);
  });
}

int ab_engine_dp_export(ab_engine* e, int world, uint64_t* dev_ptr, void* ipc_handle) {
  return ab::guard([&] { ab::dp_export(*e->impl, world, dev_ptr, ipc_handle); });
}

int ab_engine_dp_attach(ab_engine* e, int world, int rank, const ab_dp_peer* peers, int64_t timeout_ms) {
  ab::NvtxRange nvtx("april.dp_attach");
  return ab::guard([&] { ab::dp_attach(*e->impl, world, rank, peers, timeout_ms); });
}

int ab_engine_dp_detach(ab_engine* e) {
  return ab::guard([&] { ab::dp_detach(*e->impl); });
}

int ab_engine_set_counters(ab_engine* e, int64_t iteration_index, int64_t cumulative_tokens) {
  return ab::guard([&] {
    Engine& g = *e->impl;
    AB_CUDA(cudaStreamSynchronize(g.stream));
    int64_t v[2] = {iteration_index, cumulative_tokens};
    static_assert(offsetof(ab::Ctl, cumulative_tokens) == offsetof(ab::Ctl, iteration_index) + 8, "layout");
    AB_CUDA(cudaMemcpy(&g.d.ctl->iteration_index, v, sizeof(v), cudaMemcpyHostToDevice));
    g.ctl_host->iteration_index = iteration_index;
    g.ctl_host->cumulative_tokens = cumulative_tokens;
  });
}

int ab_engine_release_group(ab_engine* e, int32_t group_slot) {
  return ab::guard([&] {
    Engine& g = *e->impl;
    AB_REQUIRE(group_slot >= 0 && group_slot < g.d.G_cap, AB_ERR_CONTRACT, "group slot out of range");
    if (g.model) ab::model_release_group(g, group_slot);
  });
}

int ab_engine_stats(ab_engine* e, ab_stats* out) {
  return ab::guard([&] {
    Engine& g = *e->impl;
    out->clock = ab::read_clock(g);
    const ab::Ctl& c = *g.ctl_host;
    out->iteration_index = c.iteration_index;
    out->cumulative_tokens = c.cumulative_tokens;
    out->active = c.b;
    out->queued = c.q_tail - c.q_head;
    out->kv_pages_total = g.model ? ab::model_pages_total(g.model) : 0;
    out->kv_pages_free = c.kv_free_top;
    out->prefill_tokens = g.prefill_tokens;
    out->reprefill_tokens = g.reprefill_tokens;
    out->reprefill_seconds = g.reprefill_seconds;
    out->kernel_launches = g.launches;
  });
}

int ab_engine_profile(ab_engine* e, int enable, int sample_every) {
  return ab::guard([&] {
    Engine& g = *e->impl;
    g.profile = enable != 0;
    g.sample_every = sample_every > 0 ? sample_every : 1;
    if (!enable)  // keep the names: captured profiling slots refer to timer indices
      for (auto& t : g.timers) {
        t.launches = 0;
        t.ms = t.bytes = t.flops = 0;
      }
  });
}

int ab_engine_kernel_stats(ab_engine* e, ab_kernel_stat* out, int cap, int* n) {
  return ab::guard([&] {
    Engine& g = *e->impl;
    *n = (int)g.timers.size();
    for (int i = 0; i < *n && i < cap; ++i) {
      memset(&out[i], 0, sizeof(ab_kernel_stat));
      strncpy(out[i].name, g.timers[i].name.c_str(), sizeof(out[i].name) - 1);
      out[i].launches = g.timers[i].launches;
      out[i].ms = g.timers[i].ms;
      out[i].bytes = g.timers[i].bytes;
      out[i].flops = g.timers[i].flops;
    }
  });
}

int ab_engine_set_iteration(ab_engine* e, int64_t iteration_index) {
  return ab::guard([&] {
    Engine& g = *e->impl;
    AB_CUDA(cudaStreamSynchronize(g.stream));
    AB_CUDA(cudaMemcpy(&g.d.ctl->iteration_index, &iteration_index, sizeof(int64_t), cudaMemcpyHostToDevice));
    g.ctl_host->iteration_index = iteration_index;
  });
}

int ab_engine_synchronize(ab_engine* e) {
  return ab::guard([&] { AB_CUDA(cudaStreamSynchronize(e->impl->stream)); });
}

int ab_engine_weight_count(ab_engine* e, int* n) {
  return ab::guard([&] { *n = e->impl->model ? ab::model_weight_count(e->impl->model) : 0; });
}

int ab_engine_weight_info(ab_engine* e, int idx, char* name, int name_cap, int64_t* rows, int64_t* cols) {
  return ab::guard([&] {
    AB_REQUIRE(e->impl->model, AB_ERR_CONTRACT, "engine has no transformer model");
    AB_REQUIRE(idx >= 0 && idx < ab::model_weight_count(e->impl->model), AB_ERR_CONTRACT, "weight index");
    std::string nm;
    void* p;
    ab::model_weight_info(e->impl->model, idx, &nm, rows, cols, &p);
    if (name && name_cap > 0) {
      strncpy(name, nm.c_str(), name_cap - 1);
      name[name_cap - 1] = 0;
    }
  });
}

static int weight_copy(ab_engine* e, int idx, void* host, const void* src, size_t bytes) {
  return ab::guard([&] {
    AB_REQUIRE(e->impl->model, AB_ERR_CONTRACT, "engine has no transformer model");
    AB_REQUIRE(idx >= 0 && idx < ab::model_weight_count(e->impl->model), AB_ERR_CONTRACT, "weight index");
    std::string nm;
    int64_t r, c;
    void* p;
    ab::model_weight_info(e->impl->model, idx, &nm, &r, &c, &p);
    AB_REQUIRE(bytes == (size_t)(r * c * 2), AB_ERR_CONTRACT, "weight byte count mismatch");
    if (host)
      AB_CUDA(cudaMemcpy(host, p, bytes, cudaMemcpyDeviceToHost));
    else
      AB_CUDA(cudaMemcpy(p, src, bytes, cudaMemcpyDefault));
  });
}

int ab_engine_get_weight(ab_engine* e, int idx, void* host_dst, size_t bytes) {
  return weight_copy(e, idx, host_dst, nullptr, bytes);
}
int ab_engine_set_weight(ab_engine* e, int idx, const void* src, size_t bytes) {
  return weight_copy(e, idx, nullptr, src, bytes);
}

}  // extern "C"
