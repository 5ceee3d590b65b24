// Transformer decode path of the engine: weights, paged KV pool, batched
// prompt prefill with prefix sharing, and one decode iteration over the
// device-resident live batch (prep -> embed -> L x [norm, QKV GEMM, RoPE+KV,
// paged attention, O GEMM(+res), norm, gate-up GEMM(SwiGLU), down GEMM(+res)]
// -> norm -> lm_head GEMM -> fused sampler).  Every kernel reads the live
// batch size and the stop flag from the device control block, so a chunk of
// iterations can be queued without host round-trips.
#include <cuda_bf16.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <string>
#include <vector>

#include "model.cuh"

namespace ab {

struct WeightInfo {
  std::string name;
  int64_t rows, cols;
  bf16* ptr;
};

struct Model {
  ModelDev md{};
  ab_model_config cfg{};
  std::vector<LayerW> layers;
  bf16 *embed = nullptr, *lm_head = nullptr, *final_norm = nullptr;
  std::vector<WeightInfo> winfo;
  bf16* wbuf = nullptr;
  size_t wbytes = 0;
  int S = 0, M_pf = 0, rows_cap = 0;
  float *x = nullptr, *logits = nullptr, *part_o = nullptr, *part_ml = nullptr;
  float* gu_ws = nullptr;      // gate-up reduce-add workspace [S, 2f] fp32 (nondeterministic_gemm only)
  uint8_t* samp_part = nullptr;  // split sampler: per-piece (max, argmax, sum) partials
  bool samp_split = false;       // the sampler runs as two kernels (pieces + finish)
  bf16 *xn = nullptr, *qkv = nullptr, *qrot = nullptr, *attn = nullptr, *hbuf = nullptr;
  float* qkv32 = nullptr;
  int max_splits = 1, chunk = 256;
  struct Plans {
    GemmPlan qkv, o, gu, down;
    // decode only: the same QKV / O / down products on clusters of 2 (148 CTAs, split-K <= 2);
    // gemm_partition gives each row count to the faster of the pair of plans
    GemmPlan qkv2, o2, down2;
    GemmPlan gu2;  // decode gate-up on a cluster-of-8 (non-pair) plan: small row counts (autotuned)
    // prefill only: CTA-pair alternatives of the four projections (autotuned against the 1-SM plans)
    GemmPlan qkv_p, o_p, gu_p, down_p;
  };
  std::vector<Plans> dec, pf;
  GemmPlan lm_dec, lm_dec2;  // lm_head: CTA pair / 1-SM alternative (autotuned)
  // Decode plan selection without idle launches.  Every decode projection has two plans whose
  // cluster shapes differ (a launch attribute), so one captured graph cannot switch between them on
  // the device.  After autotuning both plans hold FULL schedule tables (valid at every row count)
  // and each row count has a preferred plan; the distinct preference vectors are the graph
  // variants (bit j set: projection j = qkv, o, gate-up, down, lm_head runs its second plan).  The
  // host picks the variant of a chunk of iterations from the chunk's largest possible live batch;
  // inside the chunk the live batch only shrinks, and the chosen plans are valid at any row count.
  // Empty: cost-model tables (gemm_autotune = 0), both plans launched with complementary tables.
  std::vector<int> variant_sel;
  std::vector<int> variant_of;  // [S + 1]
  // log-prob scoring (model_score): gathered final-norm rows -> lm_head -> log-softmax at the targets
  GemmPlan lm_score;
  bf16* score_a = nullptr;
  int *score_rows = nullptr, *score_idx = nullptr, *score_tgt = nullptr;
  double* score_out = nullptr;
  int2* score_items = nullptr;
  int* pf_rows = nullptr;  // device row count for prefill GEMMs
  CUtensorMap kvmap;         // TMA view of the KV pool for the decode attention
  int32_t *ga_g = nullptr, *ga_len = nullptr, *ga_last = nullptr;
  int32_t* host_stage = nullptr;
  size_t host_stage_cap = 0;
  struct PendingGroup {
    int g;
    std::vector<int32_t> prompt;
    bool in_place;  // re-prefill of a resident group's prompt (pages already allocated)
  };
  std::vector<PendingGroup> pending;
  // KV re-prefill mode, one engine: resumed samples whose KV is rebuilt only when their admission is
  // next (bounded KV: a long partial-rollout buffer is never rebuilt all at once), FIFO order
  std::deque<ab_sample_desc> deferred;
  // causal attention blocks of a prefill chunk ({first row, rows, block-table row, first position})
  int4 *pf_blocks = nullptr, *pf_blocks_host = nullptr;
  int pf_blocks_cap = 0;
  // KV re-prefill mode (§8 f1): prompts of resident groups, their prefilled context, evicted handles
  std::map<int, std::vector<int32_t>> prompts;
  std::vector<int32_t> g_ctx_host;
  std::vector<char> evicted;
  int4 *rs_items = nullptr, *rs_pieces = nullptr;
  int64_t last_version = -1;
  size_t kv_bytes = 0;
  bool kv_released = false;
  float inv_temp = 1.f;
};

namespace {

constexpr int kScoreRows = 64;  // scratch block-table rows: sequences scored per batch

template <typename T>
T* dalloc(size_t n) {
  T* p = nullptr;
  AB_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
  AB_CUDA(cudaMemset(p, 0, std::max<size_t>(n, 1) * sizeof(T)));
  return p;
}

// Largest activation tile the decode GEMMs may use; the kernel picks the
// actual width (and split-K) on the device from the live row count.
int pick_bn(int rows) {
  if (rows <= 32) return 32;
  if (rows <= 64) return 64;
  if (rows <= 128) return 128;
  return 256;
}

}  // namespace

// the gate-up workspace plan's follow-up pass (timed with it by the autotuner)
static void follow_swiglu(const GemmPlan& p, cudaStream_t s) {
  launch_swiglu_ws(reinterpret_cast<float*>(p.out), reinterpret_cast<bf16*>(p.follow_arg), p.N / 2, p.sched,
                   p.rows_dev, p.M_cap, p.stop_dev, s);
}

// Decode GEMM autotuning: for every projection, each of its alternative plans (cluster-8 split-K,
// cluster-1 reduce-add / cluster-2, CTA pair) and every valid fixed schedule is timed on this GPU
// at a ladder of live row counts (L2 flushed before each launch); each row count then runs the
// fastest (plan, schedule) and the other plan's table entry is 0.  Layers share shapes, so layer 0
// is tuned and its tables are installed on every layer; results are cached per process.
static void autotune_decode(Engine& e, Model* M) {
  const char* lv = getenv("AB_AUTOTUNE_LOG");
  const bool log = lv != nullptr, log_all = lv && lv[0] == '2';
  cudaStream_t s = e.stream;
  const int S = M->S;
  std::vector<int> ladder;
  for (int r : {1, 2, 4, 8, 12, 16, 24, 32, 40, 48, 56, 64, 80, 96, 112, 128, 160, 192, 224, 256, 320, 384, 448, 512,
                640, 768, 896, 1024, 1280, 1536, 1792, 2048})
    if (r < S) ladder.push_back(r);
  ladder.push_back(S);
  void* flush = nullptr;
  const size_t flush_bytes = (size_t)192 << 20;  // > L2 (126 MB)
  int cur_cap = S;  // table size - 1 of the plans being tuned
  auto key_of = [&](const std::vector<GemmPlan*>& g) {
    std::string k;
    for (auto* p : g)
      k += std::to_string(p->N) + "," + std::to_string(p->K) + "," + std::to_string(p->epi) + "," +
           std::to_string(p->M_cap) + "," + std::to_string(p->BN) + "," + std::to_string(p->cluster) + "," +
           std::to_string(p->pair) + "," + std::to_string(p->nondet) + "," + std::to_string(p->grid) + ";";
    return k;
  };
  // tables: per plan, its best measured schedule at every row count (the cost model's where it has
  // no valid candidate); choice: per row count, the fastest plan
  struct Tuned {
    std::vector<std::vector<int>> tabs;
    std::vector<int> choice;
  };
  static std::map<std::string, Tuned> cache2;
  auto tune = [&](std::vector<GemmPlan*> g) -> Tuned {
    const std::string key = key_of(g);
    auto it = cache2.find(key);
    if (it != cache2.end()) return it->second;
    if (!flush) {
      AB_CUDA(cudaMalloc(&flush, flush_bytes));
      AB_CUDA(cudaMemsetAsync(flush, 0, flush_bytes, s));
      l2_flush(flush, flush_bytes, s);  // (the memset's dirty lines are written back before any timing)
    }
    Tuned out;
    out.tabs.assign(g.size(), std::vector<int>(cur_cap + 1, 0));
    out.choice.assign(cur_cap + 1, 0);
    std::vector<std::vector<std::pair<double, int>>> best(ladder.size(),
                                                          std::vector<std::pair<double, int>>(g.size(), {1e30, 0}));
    for (size_t li = 0; li < ladder.size(); ++li) {
      const int r = ladder[li];
      for (size_t i = 0; i < g.size(); ++i)
        for (int c : gemm_candidates(*g[i], r)) {
          if (log_all) {
            fprintf(stderr, "[autotune]   try N=%d K=%d rows=%d plan=%zu code=0x%x\n", g[i]->N, g[i]->K, r, i, c);
            fflush(stderr);
          }
          const double us = gemm_time_code(*g[i], r, c, 3, flush, flush_bytes, s) + g[i]->extra_us;
          if (us < best[li][i].first) best[li][i] = {us, c};
        }
    }
    int lo = 1;
    for (size_t li = 0; li < ladder.size(); ++li) {
      const int r = ladder[li];
      int bp = 0;
      for (size_t i = 1; i < g.size(); ++i)
        if (best[li][i].first < best[li][bp].first) bp = (int)i;
      for (int x = lo; x <= r; ++x) {
        out.choice[x] = bp;
        for (size_t i = 0; i < g.size(); ++i)
          out.tabs[i][x] = best[li][i].first < 1e29 ? best[li][i].second : gemm_default_code(*g[i], x);
      }
      if (log)
        fprintf(stderr, "[autotune] N=%d K=%d epi=%d rows=%d plan=%d (cluster %d%s) code=0x%x %.1f us (other %.1f us)\n",
                g[0]->N, g[0]->K, g[0]->epi, r, bp, g[bp]->cluster, g[bp]->pair ? " pair" : "",
                best[li][bp].second, best[li][bp].first, best[li][1 - bp].first);
      lo = r + 1;
    }
    out.tabs[0][0] = out.tabs[1][0] = 0;
    // a plan with no schedule at some row count is never chosen (it could not cover a shrinking batch)
    for (size_t i = 0; i < g.size(); ++i)
      for (int x = 1; x <= cur_cap; ++x)
        if (out.tabs[i][x] == 0) {
          for (int y = 1; y <= cur_cap; ++y)
            if (out.choice[y] == (int)i) out.choice[y] = 1 - (int)i;
          break;
        }
    cache2[key] = out;
    return out;
  };
  const int L = (int)M->dec.size();
  std::vector<std::vector<int>> choices;  // per projection (qkv, o, gate-up, down, lm_head)
  auto apply = [&](std::vector<Model::Plans>& v, GemmPlan Model::Plans::*a, GemmPlan Model::Plans::*b,
                   bool decode) {
    std::vector<GemmPlan*> g = {&(v[0].*a), &(v[0].*b)};
    Tuned t = tune(g);
    if (!decode) {  // prefill: the host knows the row count, launch only the chosen plan's entry
      for (int x = 0; x <= cur_cap; ++x) t.tabs[1 - t.choice[x]][x] = 0;
    }
    for (int l = 0; l < L; ++l) {
      gemm_set_table(v[l].*a, t.tabs[0]);
      gemm_set_table(v[l].*b, t.tabs[1]);
    }
    if (decode) choices.push_back(t.choice);
  };
  apply(M->dec, &Model::Plans::qkv, &Model::Plans::qkv2, true);
  apply(M->dec, &Model::Plans::o, &Model::Plans::o2, true);
  apply(M->dec, &Model::Plans::gu, &Model::Plans::gu2, true);
  apply(M->dec, &Model::Plans::down, &Model::Plans::down2, true);
  {
    Tuned t = tune({&M->lm_dec, &M->lm_dec2});
    gemm_set_table(M->lm_dec, t.tabs[0]);
    gemm_set_table(M->lm_dec2, t.tabs[1]);
    choices.push_back(t.choice);
  }
  // graph variants: the distinct per-row-count plan choices
  M->variant_sel.clear();
  M->variant_of.assign(S + 1, 0);
  for (int r = 1; r <= S; ++r) {
    int sel = 0;
    for (size_t j = 0; j < choices.size(); ++j) sel |= choices[j][r] << j;
    int v = -1;
    for (size_t k = 0; k < M->variant_sel.size(); ++k)
      if (M->variant_sel[k] == sel) v = (int)k;
    if (v < 0) {
      v = (int)M->variant_sel.size();
      M->variant_sel.push_back(sel);
    }
    M->variant_of[r] = v;
  }
  M->variant_of[0] = M->variant_of[1];
  if (log)
    for (size_t k = 0; k < M->variant_sel.size(); ++k) {
      int lo = -1, hi = -1;
      for (int r = 1; r <= S; ++r)
        if (M->variant_of[r] == (int)k) {
          if (lo < 0) lo = r;
          hi = r;
        }
      fprintf(stderr, "[autotune] graph variant %zu: plan bits 0x%x (qkv,o,gu,down,lm), rows %d..%d\n", k,
              M->variant_sel[k], lo, hi);
    }
  // prefill chunks (up to M_pf rows): 1-SM plans against CTA-pair plans on a coarse ladder
  ladder.clear();
  for (int r = 64; r < M->M_pf; r *= 4) ladder.push_back(r);
  ladder.push_back(M->M_pf);
  cur_cap = M->M_pf;
  apply(M->pf, &Model::Plans::qkv, &Model::Plans::qkv_p, false);
  apply(M->pf, &Model::Plans::o, &Model::Plans::o_p, false);
  apply(M->pf, &Model::Plans::gu, &Model::Plans::gu_p, false);
  apply(M->pf, &Model::Plans::down, &Model::Plans::down_p, false);
  if (flush) AB_CUDA(cudaFree(flush));
  // the timing runs accumulated into the decode workspaces: the QKV accumulator must start at zero
  AB_CUDA(cudaMemsetAsync(M->qkv32, 0, sizeof(float) * (size_t)S * M->md.qkv_dim, s));
  AB_CUDA(cudaStreamSynchronize(s));
}

Model* model_create(Engine& e) {
  const ab_model_config& c = e.mcfg;
  const ab_engine_config& ec = e.cfg;
  AB_REQUIRE(c.n_layers >= 1 && c.d_model % 128 == 0, AB_ERR_CONFIG, "d_model must be a multiple of 128");
  AB_REQUIRE(c.head_dim == 64 || c.head_dim == 128, AB_ERR_CONFIG, "head_dim must be 64 or 128");
  AB_REQUIRE(c.n_kv_heads >= 1 && c.n_q_heads % c.n_kv_heads == 0, AB_ERR_CONFIG, "GQA group must divide heads");
  AB_REQUIRE(c.n_q_heads / c.n_kv_heads <= 16, AB_ERR_CONFIG, "GQA group > 16 unsupported");
  AB_REQUIRE(c.d_ff % 64 == 0 && c.vocab % 128 == 0, AB_ERR_CONFIG, "d_ff % 64 and vocab % 128 required");
  AB_REQUIRE(ec.page_size >= 16 && ec.page_size % 16 == 0, AB_ERR_CONFIG, "page_size must be a multiple of 16");
  AB_REQUIRE(ec.max_prompt >= 2, AB_ERR_CONFIG, "max_prompt must be >= 2");
  {
    // which kernels trigger their dependents early (bit 1 GEMM at start, 2 attention, 4 RMSNorm,
    // 8 GEMM after its last MMA)
    const char* pm = getenv("AB_PDL_MASK");
    const int mask = pm ? atoi(pm) : 6;  // measured: the GEMM's own early trigger costs 4-6 %
    set_pdl_mask_gemm(mask);
    set_pdl_mask_attention(mask);
    set_pdl_mask_layers(mask);
  }
  Model* M = new Model();
  M->cfg = c;
  ModelDev& m = M->md;
  m.L = c.n_layers;
  m.d = c.d_model;
  m.hq = c.n_q_heads;
  m.hk = c.n_kv_heads;
  m.hd = c.head_dim;
  m.f = c.d_ff;
  m.V = c.vocab;
  m.qd = m.hq * m.hd;
  m.kvd = m.hk * m.hd;
  m.qkv_dim = m.qd + 2 * m.kvd;
  m.gq = m.hq / m.hk;
  m.qk_norm = c.qk_norm;
  m.eps = c.norm_eps;
  m.P = ec.page_size;
  m.H = e.d.H;
  m.G_cap = e.d.G_cap;
  m.max_pos = ec.max_prompt + ec.l_max + 1;
  m.MP = ceil_div(m.max_pos, m.P) + 1;
  AB_REQUIRE(m.qkv_dim % 128 == 0, AB_ERR_CONFIG, "q+k+v projection width must be a multiple of 128");
  cudaStream_t s = e.stream;

  // ---- weights (one allocation, N(0, std) matrices, unit norms) ----
  auto add = [&](const std::string& n, int64_t r, int64_t cc) {
    M->winfo.push_back({n, r, cc, nullptr});
  };
  add("embed", m.V, m.d);
  if (!c.tied_embeddings) add("lm_head", m.V, m.d);
  add("final_norm", 1, m.d);
  for (int l = 0; l < m.L; ++l) {
    const std::string p = "layers." + std::to_string(l) + ".";
    add(p + "attn_norm", 1, m.d);
    add(p + "wqkv", m.qkv_dim, m.d);
    if (c.qkv_bias) add(p + "bqkv", 1, m.qkv_dim);
    if (c.qk_norm) {
      add(p + "q_norm", 1, m.hd);
      add(p + "k_norm", 1, m.hd);
    }
    add(p + "wo", m.d, m.qd);
    add(p + "mlp_norm", 1, m.d);
    add(p + "wgu", 2 * m.f, m.d);  // rows per 128-row tile: 64 gate rows then the matching 64 up rows
    add(p + "wd", m.d, m.f);
  }
  size_t total = 0;
  for (auto& w : M->winfo) total += (size_t)((w.rows * w.cols + 63) / 64 * 64);
  M->wbuf = dalloc<bf16>(total);
  M->wbytes = total * 2;
  size_t off = 0;
  for (size_t i = 0; i < M->winfo.size(); ++i) {
    auto& w = M->winfo[i];
    w.ptr = M->wbuf + off;
    off += (size_t)((w.rows * w.cols + 63) / 64 * 64);
    const bool is_norm = w.name.find("norm") != std::string::npos;
    launch_init_weights(w.ptr, (size_t)(w.rows * w.cols), ec.weight_seed, i, is_norm ? 0.f : ec.weight_std, 1.f, s);
  }
  auto find = [&](const std::string& n) -> bf16* {
    for (auto& w : M->winfo)
      if (w.name == n) return w.ptr;
    return nullptr;
  };
  M->embed = find("embed");
  M->lm_head = c.tied_embeddings ? M->embed : find("lm_head");
  M->final_norm = find("final_norm");
  for (int l = 0; l < m.L; ++l) {
    const std::string p = "layers." + std::to_string(l) + ".";
    LayerW lw{find(p + "attn_norm"), find(p + "wqkv"), find(p + "bqkv"), find(p + "q_norm"), find(p + "k_norm"),
              find(p + "wo"),        find(p + "mlp_norm"), find(p + "wgu"), find(p + "wd")};
    M->layers.push_back(lw);
  }

  // ---- buffers ----
  M->S = e.d.S;
  M->M_pf = std::max(ec.max_prompt, 16384);
  M->rows_cap = std::max(M->S, M->M_pf);
  const size_t R = M->rows_cap;
  M->x = dalloc<float>(R * m.d);
  M->xn = dalloc<bf16>(R * std::max(m.d, m.f));
  M->qkv = dalloc<bf16>(R * m.qkv_dim);
  M->qkv32 = dalloc<float>((size_t)M->S * m.qkv_dim);  // decode QKV accumulator (kept zeroed between uses)
  M->qrot = dalloc<bf16>(R * m.qd);
  M->attn = dalloc<bf16>(R * m.qd);
  M->hbuf = dalloc<bf16>(R * m.f);
  M->logits = dalloc<float>((size_t)M->S * m.V);
  // gate-up stream-K workspace plan (experimental, AB_GU_WORKSPACE=1): measured slower than the
  // cluster-8 SwiGLU plan at decode batches once its SwiGLU pass is included, so off by default
  {
    const char* gw = getenv("AB_GU_WORKSPACE");
    if (ec.nondeterministic_gemm && gw && atoi(gw) != 0)
      M->gu_ws = dalloc<float>((size_t)M->S * 2 * m.f);  // kept zeroed between uses
  }
  M->samp_part = dalloc<uint8_t>(sampler_scratch_bytes(M->S, m.V));
  M->samp_split = sampler_uses_split(ec.greedy, ec.top_p);
  // smallest KV split of an attention work item (the prep kernel picks the split per iteration);
  // at most 64 splits per row
  M->chunk = std::max(256, (ceil_div(m.max_pos, 64) + 63) / 64 * 64);
  M->max_splits = ceil_div(m.max_pos, M->chunk);
  M->part_o = dalloc<float>((size_t)M->S * m.hq * M->max_splits * m.hd);
  M->part_ml = dalloc<float>((size_t)M->S * m.hq * M->max_splits * 2);
  m.row_tok = dalloc<int32_t>(R);
  m.row_pos = dalloc<int32_t>(R);
  m.row_btrow = dalloc<int32_t>(R);
  m.row_pslot = dalloc<int32_t>(R);
  m.split_prefix = dalloc<int32_t>(M->S + 1);
  m.att_counter = dalloc<int32_t>((size_t)M->S * m.hk);
  m.att_items = dalloc<int32_t>((size_t)M->S * M->max_splits + 1);
  m.att_ctl = dalloc<int32_t>(1 + m.L);
  m.h_ctx = dalloc<int32_t>(m.H);
  m.h_last_tok = dalloc<int32_t>(m.H);
  m.h_shared = dalloc<int32_t>(m.H);
  m.g_ctx = dalloc<int32_t>(m.G_cap);
  m.g_last_tok = dalloc<int32_t>(m.G_cap);
  m.g_npages = dalloc<int32_t>(m.G_cap);
  m.bt = dalloc<int32_t>((size_t)(m.H + m.G_cap + kScoreRows) * m.MP);  // + scratch rows for scoring
  m.rope = dalloc<float2>((size_t)m.max_pos * (m.hd / 2));
  launch_rope_table(m.rope, m.max_pos, m.hd, c.rope_theta, s);
  M->pf_rows = dalloc<int>(1);
  M->ga_g = dalloc<int32_t>(M->M_pf + 1);
  M->ga_len = dalloc<int32_t>(M->M_pf + 1);
  M->ga_last = dalloc<int32_t>(M->M_pf + 1);
  M->pf_blocks_cap = M->M_pf / 64 + M->M_pf + 16;  // a chunk holds <= M_pf rows, each piece adds one block
  M->pf_blocks = dalloc<int4>(M->pf_blocks_cap);
  AB_CUDA(cudaMallocHost(&M->pf_blocks_host, sizeof(int4) * M->pf_blocks_cap));
  M->rs_items = dalloc<int4>(m.H + 1);
  M->rs_pieces = dalloc<int4>(M->M_pf + 2);
  M->g_ctx_host.assign(m.G_cap, 0);
  M->evicted.assign(m.H, 0);
  M->host_stage_cap = (size_t)8 * (M->M_pf + 16);
  AB_CUDA(cudaMallocHost(&M->host_stage, sizeof(int32_t) * M->host_stage_cap));

  // ---- KV pool: everything left after a safety margin, unless requested ----
  const size_t page_bytes = (size_t)m.L * 2 * m.hk * m.P * m.hd * 2;
  AB_CUDA(cudaStreamSynchronize(s));
  size_t free_b = 0, total_b = 0;
  AB_CUDA(cudaMemGetInfo(&free_b, &total_b));
  int64_t np = ec.kv_pages;
  if (np <= 0) {
    const size_t margin = (size_t)4 << 30;
    np = free_b > margin ? (int64_t)((free_b - margin) / page_bytes) : 0;
  }
  AB_REQUIRE(np >= 1, AB_ERR_CONFIG, "no HBM left for the KV pool");
  AB_REQUIRE((size_t)np * page_bytes + ((size_t)1 << 30) <= free_b, AB_ERR_CONFIG, "KV pool does not fit in HBM");
  AB_REQUIRE(np * m.P < (int64_t(1) << 31), AB_ERR_CONFIG, "KV pool too large for 32-bit token slots");
  m.NP = np;
  m.kv = dalloc<bf16>((size_t)np * page_bytes / 2);
  M->kv_bytes = (size_t)np * page_bytes;
  m.free_pages = dalloc<int32_t>(np);
  {
    std::vector<int32_t> fp(np);
    for (int64_t i = 0; i < np; ++i) fp[i] = (int32_t)(np - 1 - i);
    AB_CUDA(cudaMemcpy(m.free_pages, fp.data(), sizeof(int32_t) * np, cudaMemcpyHostToDevice));
  }
  AB_CUDA(cudaMemcpy(&e.d.ctl->kv_free_top, &np, sizeof(int64_t), cudaMemcpyHostToDevice));
  make_kv_tmap(&M->kvmap, m);
  e.ctl_host->kv_free_top = np;
  e.d.kv_bt = m.bt;
  e.d.kv_h_ctx = m.h_ctx;
  e.d.kv_h_shared = m.h_shared;
  e.d.kv_free = m.free_pages;
  e.d.kv_P = m.P;
  e.d.kv_MP = m.MP;

  // ---- GEMM plans ----
  const int* b = &e.d.ctl->b;
  const int* stop = &e.d.ctl->stop;
  const int bn_dec = pick_bn(M->S);
  for (int l = 0; l < m.L; ++l) {
    const LayerW& w = M->layers[l];
    Model::Plans d, p;
    const bool nd = ec.nondeterministic_gemm != 0;
    // decode QKV: fp32 accumulator reduce-added into a zeroed workspace (it may then split K like the
    // residual GEMMs); bias, bf16 rounding and RoPE / KV write happen in k_rope_kv_f32
    gemm_plan(d.qkv, w.wqkv, m.qkv_dim, m.d, M->xn, M->S, m.d, bn_dec, kEpiAddF32, M->qkv32, m.qkv_dim, nullptr, b,
              stop, 8);
    gemm_plan(d.o, w.wo, m.d, m.qd, M->attn, M->S, m.qd, bn_dec, kEpiAddF32, M->x, m.d, nullptr, b, stop, 8);
    gemm_plan(d.gu, w.wgu, 2 * m.f, m.d, M->xn, M->S, m.d, bn_dec, kEpiSwiGLU, M->hbuf, m.f, nullptr, b, stop,
              2, true);
    gemm_plan(d.down, w.wd, m.d, m.f, M->hbuf, M->S, m.f, bn_dec, kEpiAddF32, M->x, m.d, nullptr, b, stop, 8);
    gemm_plan(d.qkv2, w.wqkv, m.qkv_dim, m.d, M->xn, M->S, m.d, bn_dec, kEpiAddF32, M->qkv32, m.qkv_dim, nullptr, b,
              stop, nd ? 1 : 2);
    // fp32 residual GEMMs: the second plan is either a cluster-of-2 plan (deterministic) or, when
    // the engine allows it, a cluster-of-1 plan whose split-K partials are reduce-added by TMA
    gemm_plan(d.o2, w.wo, m.d, m.qd, M->attn, M->S, m.qd, bn_dec, kEpiAddF32, M->x, m.d, nullptr, b, stop, nd ? 1 : 2);
    gemm_plan(d.down2, w.wd, m.d, m.f, M->hbuf, M->S, m.f, bn_dec, kEpiAddF32, M->x, m.d, nullptr, b, stop,
              nd ? 1 : 2);
    if (nd) {
      d.qkv2.nondet = d.o2.nondet = d.down2.nondet = true;
      gemm_set_schedule(d.qkv2, 0);
      gemm_set_schedule(d.o2, 0);
      gemm_set_schedule(d.down2, 0);
    }
    gemm_partition(d.qkv, d.qkv2);
    gemm_partition(d.o, d.o2);
    gemm_partition(d.down, d.down2);
    {
      // the residual GEMMs are followed by an RMSNorm: AB_GEMM_TRIGGER=1 lets it launch and wait while
      // they run (measured neutral at b = 64-1024, so off by default)
      const char* gt = getenv("AB_GEMM_TRIGGER");
      const bool et = gt ? atoi(gt) != 0 : false;
      d.o.early_trigger = d.o2.early_trigger = d.down.early_trigger = d.down2.early_trigger = et;
    }
    if (nd && M->gu_ws) {
      // gate-up alternative: raw gate / up accumulators reduce-added into a zeroed fp32 workspace by
      // stream-K ranges (every SM streams the same weight bytes whatever the tile count), then
      // k_swiglu_ws forms h = silu(gate) * up and re-zeroes the workspace
      gemm_plan(d.gu2, w.wgu, 2 * m.f, m.d, M->xn, M->S, m.d, bn_dec, kEpiAddF32, M->gu_ws, 2 * m.f, nullptr, b,
                stop, 1);
      d.gu2.nondet = true;
      d.gu2.follow = follow_swiglu;  // the autotuner times the plan together with its SwiGLU pass
      d.gu2.follow_arg = M->hbuf;
    } else {
      gemm_plan(d.gu2, w.wgu, 2 * m.f, m.d, M->xn, M->S, m.d, bn_dec, kEpiSwiGLU, M->hbuf, m.f, nullptr, b, stop, 8);
    }
    gemm_set_table(d.gu2, std::vector<int>(M->S + 1, 0));  // idle unless the autotuner picks it
    gemm_plan(p.qkv, w.wqkv, m.qkv_dim, m.d, M->xn, M->M_pf, m.d, 256, kEpiBF16, M->qkv, m.qkv_dim, w.bqkv,
              M->pf_rows, nullptr);
    gemm_plan(p.o, w.wo, m.d, m.qd, M->attn, M->M_pf, m.qd, 256, kEpiAddF32, M->x, m.d, nullptr, M->pf_rows,
              nullptr);
    gemm_plan(p.gu, w.wgu, 2 * m.f, m.d, M->xn, M->M_pf, m.d, 256, kEpiSwiGLU, M->hbuf, m.f, nullptr, M->pf_rows,
              nullptr);
    gemm_plan(p.down, w.wd, m.d, m.f, M->hbuf, M->M_pf, m.f, 256, kEpiAddF32, M->x, m.d, nullptr, M->pf_rows,
              nullptr);
    gemm_plan(p.qkv_p, w.wqkv, m.qkv_dim, m.d, M->xn, M->M_pf, m.d, 256, kEpiBF16, M->qkv, m.qkv_dim, w.bqkv,
              M->pf_rows, nullptr, 2, true);
    gemm_plan(p.o_p, w.wo, m.d, m.qd, M->attn, M->M_pf, m.qd, 256, kEpiAddF32, M->x, m.d, nullptr, M->pf_rows,
              nullptr, 2, true);
    gemm_plan(p.gu_p, w.wgu, 2 * m.f, m.d, M->xn, M->M_pf, m.d, 256, kEpiSwiGLU, M->hbuf, m.f, nullptr,
              M->pf_rows, nullptr, 2, true);
    gemm_plan(p.down_p, w.wd, m.d, m.f, M->hbuf, M->M_pf, m.f, 256, kEpiAddF32, M->x, m.d, nullptr, M->pf_rows,
              nullptr, 2, true);
    for (GemmPlan* pp : {&p.qkv_p, &p.o_p, &p.gu_p, &p.down_p})  // idle unless the autotuner picks them
      gemm_set_table(*pp, std::vector<int>(M->M_pf + 1, 0));
    M->dec.push_back(d);
    M->pf.push_back(p);
  }
  gemm_plan(M->lm_dec, M->lm_head, m.V, m.d, M->xn, M->S, m.d, bn_dec, kEpiF32, M->logits, m.V, nullptr, b, stop, 2, true);
  M->score_a = dalloc<bf16>((size_t)M->S * m.d);
  M->score_rows = dalloc<int>(1);
  M->score_idx = dalloc<int>(M->S);
  M->score_tgt = dalloc<int>(M->S);
  M->score_out = dalloc<double>(M->S);
  M->score_items = dalloc<int2>(kScoreRows);
  gemm_plan(M->lm_score, M->lm_head, m.V, m.d, M->score_a, M->S, m.d, bn_dec, kEpiF32, M->logits, m.V, nullptr,
            M->score_rows, nullptr, 2, true);
  gemm_plan(M->lm_dec2, M->lm_head, m.V, m.d, M->xn, M->S, m.d, bn_dec, kEpiF32, M->logits, m.V, nullptr, b, stop, 1);
  gemm_set_table(M->lm_dec2, std::vector<int>(M->S + 1, 0));  // idle unless the autotuner picks it
  if (ec.gemm_autotune) autotune_decode(e, M);
  M->inv_temp = ec.greedy ? 1.f / std::max(ec.temperature, 1e-6f) : 1.f / ec.temperature;
  if (ec.temperature <= 0.f) M->inv_temp = 1.f;
  AB_CUDA(cudaStreamSynchronize(s));
  return M;
}

void model_destroy(Model* M) {
  if (!M) return;
  ModelDev& m = M->md;
  void* ptrs[] = {M->wbuf,     M->x,        M->xn,        M->qkv,       M->qkv32,     M->qrot,     M->attn,     M->hbuf,
                  M->logits,   M->part_o,   M->part_ml,   m.row_tok,    m.row_pos,    m.row_btrow, m.row_pslot, m.h_ctx,
                  m.h_last_tok, m.h_shared, m.g_ctx,      m.g_last_tok, m.g_npages,   m.bt,        m.rope,
                  M->pf_rows,  M->ga_g,     M->ga_len,    M->ga_last,  m.kv,
                  m.free_pages, m.split_prefix, m.att_counter, m.att_ctl, M->pf_blocks, M->rs_items,
                  M->rs_pieces, M->score_a, M->score_rows, M->score_idx, M->score_tgt, M->score_out,
                  M->score_items, M->samp_part, M->gu_ws};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (M->host_stage) cudaFreeHost(M->host_stage);
  if (M->pf_blocks_host) cudaFreeHost(M->pf_blocks_host);
  delete M;
}

int model_weight_count(Model* M) { return (int)M->winfo.size(); }

void model_weight_info(Model* M, int idx, std::string* name, int64_t* rows, int64_t* cols, void** dev_ptr) {
  const auto& w = M->winfo[idx];
  *name = w.name;
  *rows = w.rows;
  *cols = w.cols;
  *dev_ptr = w.ptr;
}

int64_t model_pages_total(Model* M) { return M->md.NP; }

// pool / batch / resident-state summary for out-of-KV errors
std::string model_kv_report(Engine& e) {
  Model* M = e.model;
  if (!M) return "no model";
  AB_CUDA(cudaMemcpyAsync(e.ctl_host, e.d.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, e.stream));
  AB_CUDA(cudaStreamSynchronize(e.stream));
  const Ctl& c = *e.ctl_host;
  return "pages " + std::to_string(M->md.NP) + ", free top " + std::to_string(c.kv_free_top) + ", live rows " +
         std::to_string(c.b) + ", queued " + std::to_string(c.q_tail - c.q_head) + ", resident prompt groups " +
         std::to_string(M->prompts.size()) + ", deferred rebuilds " + std::to_string(M->deferred.size()) +
         ", page " + std::to_string(M->md.P) + " tokens";
}

void model_open_group(Engine& e, int group_slot, const int32_t* prompt, int prompt_len) {
  Model* M = e.model;
  AB_REQUIRE(prompt != nullptr && prompt_len >= 2, AB_ERR_CONTRACT, "prompt needs >= 2 tokens");
  AB_REQUIRE(prompt_len <= e.cfg.max_prompt, AB_ERR_CONTRACT, "prompt longer than max_prompt");
  for (int i = 0; i < prompt_len; ++i)
    AB_REQUIRE(prompt[i] >= 0 && prompt[i] < M->md.V, AB_ERR_CONTRACT, "prompt token out of vocabulary");
  M->pending.push_back({group_slot, std::vector<int32_t>(prompt, prompt + prompt_len), false});
  if (e.cfg.kv_resume) M->prompts[group_slot] = M->pending.back().prompt;
}

static void check_kv(Engine& e) {
  AB_CUDA(cudaMemcpyAsync(&e.ctl_host->error, &e.d.ctl->error, sizeof(int32_t), cudaMemcpyDeviceToHost, e.stream));
  AB_CUDA(cudaStreamSynchronize(e.stream));
  if (e.ctl_host->error == kErrOutOfKV)
    throw Error(AB_ERR_OUT_OF_KV, "KV page pool exhausted (" + model_kv_report(e) + ")");
}

// Append the causal-attention blocks (<= kPfBlockRows rows, attention.cu kPfRows) of one run of rows of a
// sequence.
constexpr int kPfBlockRows = 128;
static int add_blocks(Model* M, int nb, int row0, int n, int btrow, int pos0) {
  for (int i = 0; i < n; i += kPfBlockRows) {
    AB_REQUIRE(nb < M->pf_blocks_cap, AB_ERR_CONFIG, "prefill block list overflow");
    M->pf_blocks_host[nb++] = make_int4(row0 + i, std::min(kPfBlockRows, n - i), btrow, pos0 + i);
  }
  return nb;
}

// Prefill forward over R rows already described on the device (row_tok / row_pos / row_btrow):
// writes every row's K / V into its pages.  Attention blocks go longest-context first.
static void prefill_rows(Engine& e, int R, int nb) {
  Model* M = e.model;
  ModelDev& m = M->md;
  cudaStream_t s = e.stream;
  std::sort(M->pf_blocks_host, M->pf_blocks_host + nb,
            [](const int4& x, const int4& y) { return x.w + x.y > y.w + y.y; });
  AB_CUDA(cudaMemcpyAsync(M->pf_blocks, M->pf_blocks_host, sizeof(int4) * nb, cudaMemcpyHostToDevice, s));
  AB_CUDA(cudaMemcpyAsync(M->pf_rows, &R, sizeof(int), cudaMemcpyHostToDevice, s));
  launch_embed(m, M->embed, M->x, nullptr, R, nullptr, s);
  for (int l = 0; l < m.L; ++l) {
    const LayerW& w = M->layers[l];
    const Model::Plans& p = M->pf[l];
    launch_rmsnorm(M->x, w.attn_norm, M->xn, m.d, m.eps, nullptr, R, nullptr, s);
    gemm_launch_rows(p.qkv, R, s);
    gemm_launch_rows(p.qkv_p, R, s);
    launch_rope_kv(m, l, M->qkv, w.q_norm, w.k_norm, M->qrot, nullptr, R, nullptr, s);
    launch_prefill_flash(m, l, M->qrot, M->attn, M->pf_blocks, nb, s);
    gemm_launch_rows(p.o, R, s);
    gemm_launch_rows(p.o_p, R, s);
    launch_rmsnorm(M->x, w.mlp_norm, M->xn, m.d, m.eps, nullptr, R, nullptr, s);
    gemm_launch_rows(p.gu, R, s);
    gemm_launch_rows(p.gu_p, R, s);
    gemm_launch_rows(p.down, R, s);
    gemm_launch_rows(p.down_p, R, s);
  }
  AB_CUDA(cudaGetLastError());
  AB_CUDA(cudaStreamSynchronize(s));  // host staging is reused by the next chunk
  int64_t g = 0;
  for (const GemmPlan* pp : {&M->pf[0].qkv, &M->pf[0].qkv_p, &M->pf[0].o, &M->pf[0].o_p, &M->pf[0].gu,
                             &M->pf[0].gu_p, &M->pf[0].down, &M->pf[0].down_p})
    g += (pp->idle || (!pp->host_tab.empty() && pp->host_tab[R] == 0)) ? 0 : 1;
  e.launches += 1 + (4 + g) * (int64_t)m.L;
}

// Prefill every pending prompt group (positions 0..len-2) in packed chunks.
static void flush_prefill(Engine& e) {
  Model* M = e.model;
  if (M->pending.empty()) return;
  ModelDev& m = M->md;
  cudaStream_t s = e.stream;
  size_t k = 0;
  while (k < M->pending.size()) {
    int R = 0;
    size_t k1 = k;
    while (k1 < M->pending.size() && R + (int)M->pending[k1].prompt.size() - 1 <= M->M_pf) {
      R += (int)M->pending[k1].prompt.size() - 1;
      ++k1;
    }
    const int ng = (int)(k1 - k);
    int32_t* hs = M->host_stage;
    int32_t* tok = hs;
    int32_t* pos = tok + R;
    int32_t* btr = pos + R;
    int32_t* gg = btr + R;
    int32_t* gl = gg + ng;
    int32_t* glast = gl + ng;
    int r = 0, na = 0, nb = 0;
    for (int j = 0; j < ng; ++j) {
      const auto& pg = M->pending[k + j];
      const int len = (int)pg.prompt.size() - 1;
      if (!pg.in_place) {
        gg[na] = pg.g;
        gl[na] = len;
        glast[na] = pg.prompt[len];
        ++na;
      }
      M->g_ctx_host[pg.g] = len;
      nb = add_blocks(M, nb, r, len, m.H + pg.g, 0);
      for (int t = 0; t < len; ++t, ++r) {
        tok[r] = pg.prompt[t];
        pos[r] = t;
        btr[r] = m.H + pg.g;
      }
    }
    AB_CUDA(cudaMemcpyAsync(m.row_tok, tok, sizeof(int32_t) * R, cudaMemcpyHostToDevice, s));
    AB_CUDA(cudaMemcpyAsync(m.row_pos, pos, sizeof(int32_t) * R, cudaMemcpyHostToDevice, s));
    AB_CUDA(cudaMemcpyAsync(m.row_btrow, btr, sizeof(int32_t) * R, cudaMemcpyHostToDevice, s));
    if (na) {
      AB_CUDA(cudaMemcpyAsync(M->ga_g, gg, sizeof(int32_t) * na, cudaMemcpyHostToDevice, s));
      AB_CUDA(cudaMemcpyAsync(M->ga_len, gl, sizeof(int32_t) * na, cudaMemcpyHostToDevice, s));
      AB_CUDA(cudaMemcpyAsync(M->ga_last, glast, sizeof(int32_t) * na, cudaMemcpyHostToDevice, s));
      launch_group_alloc(e.d, m, M->ga_g, M->ga_len, M->ga_last, na, s);
      e.launches += 1;
      AB_CUDA(cudaMemcpyAsync(&e.ctl_host->error, &e.d.ctl->error, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      AB_CUDA(cudaStreamSynchronize(s));
      if (e.ctl_host->error == kErrOutOfKV) {
        // the pool cannot hold this chunk's prompts: return what the chunk's groups got, drop them
        // and every later pending group (not prefilled), clear the error, and report it
        for (int j = 0; j < na; ++j) launch_group_release(e.d, m, gg[j], s);
        AB_CUDA(cudaMemsetAsync(&e.d.ctl->error, 0, sizeof(int32_t), s));
        AB_CUDA(cudaStreamSynchronize(s));
        for (size_t j = k; j < M->pending.size(); ++j) M->prompts.erase(M->pending[j].g);
        M->pending.erase(M->pending.begin() + k, M->pending.end());
        throw Error(AB_ERR_OUT_OF_KV, "KV page pool exhausted (prompt prefill)");
      }
    }
    prefill_rows(e, R, nb);
    e.prefill_tokens += R;
    k = k1;
  }
  M->pending.clear();
  check_kv(e);
}

// KV re-prefill mode: drop the private KV pages of samples leaving the live batch with generated
// tokens (the abort of an APRIL step); they are rebuilt by prefill when the sample is resubmitted.
void model_evict(Engine& e, const int32_t* handles, const int32_t* gen, int n) {
  Model* M = e.model;
  int k = 0;
  for (int i = 0; i < n; ++i)
    if (gen[i] > 0 && !M->evicted[handles[i]]) {
      e.stage_i32_host[k++] = handles[i];
      M->evicted[handles[i]] = 1;
    }
  if (!k) return;
  AB_CUDA(cudaMemcpyAsync(e.stage_i32_dev, e.stage_i32_host, sizeof(int32_t) * k, cudaMemcpyHostToDevice, e.stream));
  launch_release_handles(e.d, M->md, e.stage_i32_dev, k, e.stream);
  e.launches += 1;
  AB_CUDA(cudaStreamSynchronize(e.stream));
}

// Rebuild the KV of resubmitted evicted samples: re-fork the group prompt pages, then prefill
// the prompt's last token and every generated token but the newest (which the next decode
// iteration feeds), in chunks of <= M_pf rows; a sample may span chunks (in position order).
static void resume_reprefill(Engine& e, const ab_sample_desc* descs, int n) {
  Model* M = e.model;
  ModelDev& m = M->md;
  cudaStream_t s = e.stream;
  std::vector<int4> items;
  for (int i = 0; i < n; ++i)
    if (descs[i].gen_len > 0 && M->evicted[descs[i].handle]) {
      items.push_back(make_int4(descs[i].handle, descs[i].group_slot, descs[i].gen_len, 0));
      M->evicted[descs[i].handle] = 0;
    }
  if (items.empty()) return;
  AB_CUDA(cudaMemcpyAsync(M->rs_items, items.data(), sizeof(int4) * items.size(), cudaMemcpyHostToDevice, s));
  launch_resume_fork(e.d, m, M->rs_items, (int)items.size(), s);
  e.launches += 2;
  check_kv(e);
  std::vector<int4> pieces;
  int R = 0, nb = 0;
  auto run_chunk = [&]() {
    if (!R) return;
    pieces.push_back(make_int4(0, 0, 0, R));  // sentinel: end row of the last piece
    AB_CUDA(cudaMemcpyAsync(M->rs_pieces, pieces.data(), sizeof(int4) * pieces.size(), cudaMemcpyHostToDevice, s));
    launch_extend_rows(e.d, m, M->rs_pieces, (int)pieces.size() - 1, s);
    e.launches += 1;
    prefill_rows(e, R, nb);  // synchronises: the piece list may be rebuilt
    e.reprefill_tokens += R;
    pieces.clear();
    R = nb = 0;
  };
  for (const int4& it : items) {
    const int h = it.x, g = it.y, gen = it.z;
    for (int j0 = 0; j0 < gen;) {
      if (R == M->M_pf) run_chunk();
      const int cnt = std::min(gen - j0, M->M_pf - R);
      pieces.push_back(make_int4(h, g, j0, R));
      nb = add_blocks(M, nb, R, cnt, h, M->g_ctx_host[g] + j0);
      R += cnt;
      j0 += cnt;
    }
  }
  run_chunk();
}

// Teacher-forced log-probs of response tokens under the current weights (the trainer's
// recompute of pi_theta on a mixed-policy batch).  Sequence k = tokens[offs[k], offs[k+1]), its first
// plen[k] tokens the prompt; out receives, per sequence in order, log pi(token_p | tokens_<p) / T for
// p = plen .. len-1.  Runs the prefill pass over positions 0..len-2 into scratch block-table rows
// (pages borrowed from the pool and returned), then the final norm, lm_head and a log-softmax at the
// target token for the rows that predict a response token.
void model_score(Engine& e, const int32_t* tokens, const int64_t* offs, const int32_t* plen, int n, double* out) {
  Model* M = e.model;
  ModelDev& m = M->md;
  cudaStream_t s = e.stream;
  flush_prefill(e);
  std::vector<int64_t> ob(n + 1, 0);
  for (int k = 0; k < n; ++k) {
    const int64_t len = offs[k + 1] - offs[k];
    AB_REQUIRE(plen[k] >= 1 && len > plen[k], AB_ERR_CONTRACT, "score: every sequence needs a prompt and a response");
    AB_REQUIRE(len <= (int64_t)m.max_pos, AB_ERR_CONTRACT, "score: sequence longer than the engine's positions");
    for (int64_t p = offs[k]; p < offs[k + 1]; ++p)
      AB_REQUIRE(tokens[p] >= 0 && tokens[p] < m.V, AB_ERR_CONTRACT, "score: token out of vocabulary");
    ob[k + 1] = ob[k] + (len - plen[k]);
  }
  const int row0 = m.H + m.G_cap;
  std::vector<int32_t> tok, pos, btr;
  std::vector<int> tgt_row, tgt_tok;
  std::vector<int64_t> tgt_out;
  auto run_targets = [&]() {
    for (size_t c0 = 0; c0 < tgt_row.size(); c0 += M->S) {
      const int cnt = (int)std::min<size_t>(M->S, tgt_row.size() - c0);
      AB_CUDA(cudaMemcpyAsync(M->score_idx, tgt_row.data() + c0, sizeof(int) * cnt, cudaMemcpyHostToDevice, s));
      AB_CUDA(cudaMemcpyAsync(M->score_tgt, tgt_tok.data() + c0, sizeof(int) * cnt, cudaMemcpyHostToDevice, s));
      AB_CUDA(cudaMemcpyAsync(M->score_rows, &cnt, sizeof(int), cudaMemcpyHostToDevice, s));
      launch_gather_rows(M->xn, M->score_a, M->score_idx, cnt, m.d, s);
      gemm_launch(M->lm_score, s);
      launch_logp_rows(M->logits, m.V, M->score_tgt, cnt, M->inv_temp, M->score_out, s);
      std::vector<double> h(cnt);
      AB_CUDA(cudaMemcpyAsync(h.data(), M->score_out, sizeof(double) * cnt, cudaMemcpyDeviceToHost, s));
      AB_CUDA(cudaStreamSynchronize(s));
      for (int i = 0; i < cnt; ++i) out[tgt_out[c0 + i]] = h[i];
      e.launches += 3;
    }
  };
  for (int k0 = 0; k0 < n; k0 += kScoreRows) {
    const int nb_items = std::min(kScoreRows, n - k0);
    std::vector<int2> items(nb_items);
    for (int i = 0; i < nb_items; ++i) items[i] = make_int2(row0 + i, (int)(offs[k0 + i + 1] - offs[k0 + i] - 1));
    AB_CUDA(cudaMemcpyAsync(M->score_items, items.data(), sizeof(int2) * nb_items, cudaMemcpyHostToDevice, s));
    launch_score_alloc(e.d, m, M->score_items, nb_items, s);
    e.launches += 1;
    check_kv(e);
    int R = 0, nb = 0;
    tok.clear(), pos.clear(), btr.clear(), tgt_row.clear(), tgt_tok.clear(), tgt_out.clear();
    auto run_chunk = [&]() {
      if (!R) return;
      AB_CUDA(cudaMemcpyAsync(m.row_tok, tok.data(), sizeof(int32_t) * R, cudaMemcpyHostToDevice, s));
      AB_CUDA(cudaMemcpyAsync(m.row_pos, pos.data(), sizeof(int32_t) * R, cudaMemcpyHostToDevice, s));
      AB_CUDA(cudaMemcpyAsync(m.row_btrow, btr.data(), sizeof(int32_t) * R, cudaMemcpyHostToDevice, s));
      prefill_rows(e, R, nb);
      launch_rmsnorm(M->x, M->final_norm, M->xn, m.d, m.eps, nullptr, R, nullptr, s);
      e.launches += 1;
      run_targets();
      tok.clear(), pos.clear(), btr.clear(), tgt_row.clear(), tgt_tok.clear(), tgt_out.clear();
      R = nb = 0;
    };
    for (int i = 0; i < nb_items; ++i) {
      const int k = k0 + i;
      const int32_t* seq = tokens + offs[k];
      const int len = (int)(offs[k + 1] - offs[k]);
      for (int p0 = 0; p0 < len - 1;) {
        if (R == M->M_pf) run_chunk();
        const int cnt = std::min(len - 1 - p0, M->M_pf - R);
        nb = add_blocks(M, nb, R, cnt, row0 + i, p0);
        for (int p = p0; p < p0 + cnt; ++p, ++R) {
          tok.push_back(seq[p]);
          pos.push_back(p);
          btr.push_back(row0 + i);
          if (p >= plen[k] - 1) {
            tgt_row.push_back(R);
            tgt_tok.push_back(seq[p + 1]);
            tgt_out.push_back(ob[k] + (p - (plen[k] - 1)));
          }
        }
        p0 += cnt;
      }
    }
    run_chunk();
    launch_score_release(e.d, m, M->score_items, nb_items, s);
    e.launches += 1;
    AB_CUDA(cudaStreamSynchronize(s));
  }
}

void model_release_memory(Engine& e) {
  Model* M = e.model;
  AB_REQUIRE(!M->kv_released, AB_ERR_CONTRACT, "KV pool already released");
  AB_CUDA(cudaStreamSynchronize(e.stream));
  AB_CUDA(cudaFree(M->md.kv));
  M->md.kv = nullptr;
  M->kv_released = true;
}

void model_resume_memory(Engine& e) {
  Model* M = e.model;
  AB_REQUIRE(M->kv_released, AB_ERR_CONTRACT, "KV pool is not released");
  void* p = nullptr;
  AB_CUDA(cudaMalloc(&p, M->kv_bytes));
  M->md.kv = reinterpret_cast<bf16*>(p);
  make_kv_tmap(&M->kvmap, M->md);
  M->kv_released = false;
  // the pool's contents are gone: every resident prompt group is prefilled again in place
  for (auto& kv : M->prompts) {
    bool queued = false;
    for (auto& pg : M->pending) queued |= pg.g == kv.first;
    if (!queued) M->pending.push_back({kv.first, kv.second, true});
  }
}

void model_begin_step(Engine& e, int64_t version) {
  Model* M = e.model;
  if (!e.cfg.kv_resume) return;
  // new policy weights: every resident prompt group's KV is recomputed in place (the paused
  // samples' KV was already dropped at the abort).  Queued here and run by the step's first
  // submit, so that its cost lands inside the step's rollout wall time (scheduler clock0 is
  // read after begin_step).
  if (M->last_version >= 0 && version != M->last_version) {
    for (auto& kv : M->prompts) {
      bool queued = false;
      for (auto& pg : M->pending) queued |= pg.g == kv.first;
      if (!queued) M->pending.push_back({kv.first, kv.second, true});
    }
  }
  M->last_version = version;
}

__global__ void k_set_flags(int32_t* flags, const int32_t* idx, int n, int32_t v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flags[idx[i]] = v;
}

// flags[stage_i32_host[0..n)] = v on the device (stage_i32 holds the handles)
static void set_handle_flags(Engine& e, int n, int32_t v) {
  if (n <= 0 || !e.d.h_needs_pf) return;
  AB_CUDA(cudaMemcpyAsync(e.stage_i32_dev, e.stage_i32_host, sizeof(int32_t) * n, cudaMemcpyHostToDevice, e.stream));
  k_set_flags<<<ceil_div(n, 256), 256, 0, e.stream>>>(e.d.h_needs_pf, e.stage_i32_dev, n, v);
  AB_CUDA(cudaGetLastError());
  AB_CUDA(cudaStreamSynchronize(e.stream));  // stage_i32 is reused by the caller
  e.launches += 1;
}

void model_submit(Engine& e, const ab_sample_desc* descs_dev, int n) {
  AB_REQUIRE(!e.model->kv_released, AB_ERR_CONTRACT, "KV pool released: call resume_memory first");
  const auto t0 = std::chrono::steady_clock::now();
  bool recompute = false;
  for (auto& pg : e.model->pending) recompute |= pg.in_place;
  {
    NvtxRange r("april.prompt_prefill");
    flush_prefill(e);
  }
  if (recompute) e.reprefill_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  launch_fork_groups(e.d, e.model->md, descs_dev, n, e.stream);
  AB_CUDA(cudaGetLastError());
  check_kv(e);
  if (e.cfg.kv_resume) {
    if (e.d.h_needs_pf && e.d.dp_world <= 1) {
      // defer: flag the resumed samples; k_admit stops the run when one of them is next and
      // model_prefill_deferred rebuilds the KV of that admission
      Model* M = e.model;
      int k = 0;
      for (int i = 0; i < n; ++i) {
        const ab_sample_desc& d = e.stage_desc_host[i];
        if (d.gen_len > 0 && M->evicted[d.handle]) {
          M->deferred.push_back(d);
          e.stage_i32_host[k++] = d.handle;
        }
      }
      set_handle_flags(e, k, 1);
    } else {
      const auto t1 = std::chrono::steady_clock::now();
      NvtxRange r("april.reprefill");
      resume_reprefill(e, e.stage_desc_host, n);  // synchronous
      e.reprefill_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
    }
  }
}

int model_prefill_deferred(Engine& e, int count) {
  Model* M = e.model;
  const int n = std::min<int>(count, (int)M->deferred.size());
  if (n <= 0) return 0;
  const auto t1 = std::chrono::steady_clock::now();
  NvtxRange r("april.reprefill");
  std::vector<ab_sample_desc> descs(M->deferred.begin(), M->deferred.begin() + n);
  M->deferred.erase(M->deferred.begin(), M->deferred.begin() + n);
  resume_reprefill(e, descs.data(), n);  // synchronous
  for (int i = 0; i < n; ++i) e.stage_i32_host[i] = descs[i].handle;
  set_handle_flags(e, n, 0);
  e.reprefill_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
  return n;
}

void model_forget_deferred(Engine& e, const int32_t* handles, int n) {
  Model* M = e.model;
  if (M->deferred.empty()) return;
  for (int i = 0; i < n; ++i)
    for (auto it = M->deferred.begin(); it != M->deferred.end(); ++it)
      if (it->handle == handles[i]) {
        M->deferred.erase(it);
        break;
      }
}

void model_drop_deferred(Engine& e) {
  Model* M = e.model;
  int k = 0;
  for (const auto& d : M->deferred) e.stage_i32_host[k++] = d.handle;
  M->deferred.clear();
  set_handle_flags(e, k, 0);
}

void model_release(Engine& e, const int32_t* handles_dev, int n) {
  launch_release_handles(e.d, e.model->md, handles_dev, n, e.stream);
  AB_CUDA(cudaGetLastError());
}

void model_release_group(Engine& e, int group_slot) {
  Model* M = e.model;
  // a group still waiting for prefill is simply dropped
  M->prompts.erase(group_slot);
  bool resident = true;
  for (size_t i = 0; i < M->pending.size(); ++i)
    if (M->pending[i].g == group_slot) {
      resident = M->pending[i].in_place;
      M->pending.erase(M->pending.begin() + i);
      break;
    }
  if (!resident) return;
  launch_group_release(e.d, M->md, group_slot, e.stream);
  AB_CUDA(cudaGetLastError());
}

int model_variants(Model* M) { return std::max<int>(1, (int)M->variant_sel.size()); }

int model_variant_for(Model* M, int rows) {
  if (M->variant_sel.empty()) return 0;
  return M->variant_of[std::max(0, std::min(rows, M->S))];
}

// Launch the plan of projection j the variant selects (legacy tables: both, idle ones are skipped).
static void launch_pair(Model* M, int variant, int j, const GemmPlan& a, const GemmPlan& b, cudaStream_t s) {
  if (M->variant_sel.empty()) {
    gemm_launch(a, s);
    gemm_launch(b, s);
  } else {
    gemm_launch(((M->variant_sel[variant] >> j) & 1) ? b : a, s);
  }
}

static int pair_launches(Model* M, int variant, int j, const GemmPlan& a, const GemmPlan& b) {
  if (M->variant_sel.empty()) return (a.idle ? 0 : 1) + (b.idle ? 0 : 1);
  return (((M->variant_sel[variant] >> j) & 1) ? b : a).idle ? 0 : 1;
}

// the gate-up workspace plan (gu2 with an fp32 output) runs in this variant: its SwiGLU pass follows
static bool gu_ws_runs(Model* M, int variant, const Model::Plans& p) {
  if (!M->gu_ws || p.gu2.epi != kEpiAddF32 || p.gu2.idle) return false;
  return M->variant_sel.empty() || ((M->variant_sel[variant] >> 2) & 1);
}

// kernels one decode iteration of graph variant `variant` launches
int64_t model_iter_launches(Model* M, int variant) {
  // prep, embed, final norm, sampler (+ its finish pass)
  int64_t n = 4 + (M->samp_split ? 1 : 0) + pair_launches(M, variant, 4, M->lm_dec, M->lm_dec2);
  for (const auto& p : M->dec)
    n += 4 + pair_launches(M, variant, 0, p.qkv, p.qkv2) + pair_launches(M, variant, 1, p.o, p.o2) +
         pair_launches(M, variant, 2, p.gu, p.gu2) + pair_launches(M, variant, 3, p.down, p.down2) +
         (gu_ws_runs(M, variant, p) ? 1 : 0);
  return n;
}

void model_iteration(Engine& e, int64_t run_iter, bool timed, int variant) {
  Model* M = e.model;
  ModelDev& m = M->md;
  cudaStream_t s = e.stream;
  const int* b = &e.d.ctl->b;
  const int* stop = &e.d.ctl->stop;
  const int S = M->S;
  {
    ScopedTimer t(e, timed, "prep", run_iter);
    launch_prep_decode(e.d, m, M->chunk, s);
  }
  {
    ScopedTimer t(e, timed, "embed", run_iter);
    launch_embed(m, M->embed, M->x, b, S, stop, s);
  }
  for (int l = 0; l < m.L; ++l) {
    const LayerW& w = M->layers[l];
    const Model::Plans& p = M->dec[l];
    {
      ScopedTimer t(e, timed, "rmsnorm", run_iter);
      launch_rmsnorm(M->x, w.attn_norm, M->xn, m.d, m.eps, b, S, stop, s);
    }
    {
      ScopedTimer t(e, timed, "gemm_qkv", run_iter);
      launch_pair(M, variant, 0, p.qkv, p.qkv2, s);
    }
    {
      ScopedTimer t(e, timed, "rope_kv", run_iter);
      launch_rope_kv_f32(m, l, M->qkv32, w.bqkv, w.q_norm, w.k_norm, M->qrot, b, S, stop, s);
    }
    {
      ScopedTimer t(e, timed, "attention", run_iter);
      launch_decode_attention(M->kvmap, e.d, m, l, M->qrot, M->attn, M->part_o, M->part_ml, M->max_splits, M->chunk,
                              s);
    }
    {
      ScopedTimer t(e, timed, "gemm_o", run_iter);
      launch_pair(M, variant, 1, p.o, p.o2, s);
    }
    {
      ScopedTimer t(e, timed, "rmsnorm", run_iter);
      launch_rmsnorm(M->x, w.mlp_norm, M->xn, m.d, m.eps, b, S, stop, s);
    }
    {
      ScopedTimer t(e, timed, "gemm_gate_up", run_iter);
      launch_pair(M, variant, 2, p.gu, p.gu2, s);
    }
    if (gu_ws_runs(M, variant, p)) {
      ScopedTimer t(e, timed, "swiglu", run_iter);
      launch_swiglu_ws(M->gu_ws, M->hbuf, m.f, p.gu2.sched, b, S, stop, s);
    }
    {
      ScopedTimer t(e, timed, "gemm_down", run_iter);
      launch_pair(M, variant, 3, p.down, p.down2, s);
    }
  }
  {
    ScopedTimer t(e, timed, "rmsnorm", run_iter);
    launch_rmsnorm(M->x, M->final_norm, M->xn, m.d, m.eps, b, S, stop, s);
  }
  {
    ScopedTimer t(e, timed, "gemm_lm_head", run_iter);
    launch_pair(M, variant, 4, M->lm_dec, M->lm_dec2, s);
  }
  {
    ScopedTimer t(e, timed, "sampler", run_iter);
    launch_sampler(e.d, m, M->logits, M->inv_temp, e.cfg.greedy, e.cfg.top_p, M->samp_part, s);
  }
}

// Algorithmic bytes / flops of one launch of kernel class `name` at live
// batch b with sum_ctx = sum over live rows of the attended context length.
void model_kernel_cost(Model* M, const std::string& name, double b, double sum_ctx, double* bytes, double* flops) {
  const ModelDev& m = M->md;
  const double d = m.d, f = m.f, V = m.V, qkv = m.qkv_dim, qd = m.qd, kvd = m.kvd;
  *bytes = 0;
  *flops = 0;
  auto gemm = [&](double N, double K, double out_bytes) {
    *bytes = N * K * 2 + b * K * 2 + b * N * out_bytes;
    *flops = 2 * b * N * K;
  };
  if (name == "gemm_qkv") gemm(qkv, d, 2);
  else if (name == "gemm_o") gemm(d, qd, 8);
  else if (name == "gemm_gate_up") {
    gemm(2 * f, d, 0);
    *bytes += b * f * 2;
  } else if (name == "gemm_down") gemm(d, f, 8);
  else if (name == "gemm_lm_head") gemm(V, d, 4);
  else if (name == "attention") {
    *bytes = sum_ctx * kvd * 2 * 2 + b * qd * 2 * 2;
    *flops = 4 * sum_ctx * qd;
  } else if (name == "sampler") *bytes = b * V * 4;
  else if (name == "rmsnorm") *bytes = b * d * 6;
  else if (name == "rope_kv") *bytes = b * qkv * 2 + b * (qd + 2 * kvd) * 2;
  else if (name == "swiglu") *bytes = b * 2 * f * 4 * 2 + b * f * 2;
  else if (name == "embed") *bytes = b * d * 6;
}

}  // namespace ab
