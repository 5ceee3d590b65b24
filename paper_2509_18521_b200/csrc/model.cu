// Transformer decode path of the engine: weights, paged KV pool, batched
// prompt prefill with prefix sharing, and one decode iteration over the
// device-resident live batch (prep -> embed -> L x [norm, QKV GEMM, RoPE+KV,
// paged attention, O GEMM(+res), norm, gate-up GEMM(SwiGLU), down GEMM(+res)]
// -> norm -> lm_head GEMM -> fused sampler).  Every kernel reads the live
// batch size and the stop flag from the device control block, so a chunk of
// iterations can be queued without host round-trips.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstring>
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
  bf16 *xn = nullptr, *qkv = nullptr, *qrot = nullptr, *attn = nullptr, *hbuf = nullptr;
  int max_splits = 1, chunk = 256;
  struct Plans {
    GemmPlan qkv, o, gu, down;
    // decode only: the same QKV / O / down products on clusters of 2 (148 CTAs, split-K <= 2);
    // gemm_partition gives each row count to the faster of the pair of plans
    GemmPlan qkv2, o2, down2;
  };
  std::vector<Plans> dec, pf;
  GemmPlan lm_dec;
  int* pf_rows = nullptr;  // device row count for prefill GEMMs
  CUtensorMap kvmap;         // TMA view of the KV pool for the decode attention
  int32_t *seg_start = nullptr, *seg_group = nullptr, *ga_g = nullptr, *ga_len = nullptr, *ga_last = nullptr;
  int32_t* host_stage = nullptr;
  size_t host_stage_cap = 0;
  struct PendingGroup {
    int g;
    std::vector<int32_t> prompt;
  };
  std::vector<PendingGroup> pending;
  float inv_temp = 1.f;
};

namespace {

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
  AB_REQUIRE(ec.top_p >= 1.f, AB_ERR_CONFIG, "top_p < 1 is not supported by this build");
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
  M->qrot = dalloc<bf16>(R * m.qd);
  M->attn = dalloc<bf16>(R * m.qd);
  M->hbuf = dalloc<bf16>(R * m.f);
  M->logits = dalloc<float>((size_t)M->S * m.V);
  // smallest KV split of an attention work item (the prep kernel picks the split per iteration);
  // at most 64 splits per row
  M->chunk = std::max(256, (ceil_div(m.max_pos, 64) + 63) / 64 * 64);
  M->max_splits = ceil_div(m.max_pos, M->chunk);
  M->part_o = dalloc<float>((size_t)M->S * m.hq * M->max_splits * m.hd);
  M->part_ml = dalloc<float>((size_t)M->S * m.hq * M->max_splits * 2);
  m.row_tok = dalloc<int32_t>(R);
  m.row_pos = dalloc<int32_t>(R);
  m.row_btrow = dalloc<int32_t>(R);
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
  m.bt = dalloc<int32_t>((size_t)(m.H + m.G_cap) * m.MP);
  m.rope = dalloc<float2>((size_t)m.max_pos * (m.hd / 2));
  launch_rope_table(m.rope, m.max_pos, m.hd, c.rope_theta, s);
  M->pf_rows = dalloc<int>(1);
  M->seg_start = dalloc<int32_t>(M->M_pf + 1);
  M->seg_group = dalloc<int32_t>(M->M_pf + 1);
  M->ga_g = dalloc<int32_t>(M->M_pf + 1);
  M->ga_len = dalloc<int32_t>(M->M_pf + 1);
  M->ga_last = dalloc<int32_t>(M->M_pf + 1);
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
  m.NP = np;
  m.kv = dalloc<bf16>((size_t)np * page_bytes / 2);
  m.free_pages = dalloc<int32_t>(np);
  {
    std::vector<int32_t> fp(np);
    for (int64_t i = 0; i < np; ++i) fp[i] = (int32_t)(np - 1 - i);
    AB_CUDA(cudaMemcpy(m.free_pages, fp.data(), sizeof(int32_t) * np, cudaMemcpyHostToDevice));
  }
  AB_CUDA(cudaMemcpy(&e.d.ctl->kv_free_top, &np, sizeof(int64_t), cudaMemcpyHostToDevice));
  make_kv_tmap(&M->kvmap, m);
  e.ctl_host->kv_free_top = np;

  // ---- GEMM plans ----
  const int* b = &e.d.ctl->b;
  const int* stop = &e.d.ctl->stop;
  const int bn_dec = pick_bn(M->S);
  for (int l = 0; l < m.L; ++l) {
    const LayerW& w = M->layers[l];
    Model::Plans d, p;
    gemm_plan(d.qkv, w.wqkv, m.qkv_dim, m.d, M->xn, M->S, m.d, bn_dec, kEpiBF16, M->qkv, m.qkv_dim, w.bqkv, b, stop,
              8);
    gemm_plan(d.o, w.wo, m.d, m.qd, M->attn, M->S, m.qd, bn_dec, kEpiAddF32, M->x, m.d, nullptr, b, stop, 8);
    gemm_plan(d.gu, w.wgu, 2 * m.f, m.d, M->xn, M->S, m.d, bn_dec, kEpiSwiGLU, M->hbuf, m.f, nullptr, b, stop,
              2, true);
    gemm_plan(d.down, w.wd, m.d, m.f, M->hbuf, M->S, m.f, bn_dec, kEpiAddF32, M->x, m.d, nullptr, b, stop, 8);
    gemm_plan(d.qkv2, w.wqkv, m.qkv_dim, m.d, M->xn, M->S, m.d, bn_dec, kEpiBF16, M->qkv, m.qkv_dim, w.bqkv, b,
              stop, 2);
    // fp32 residual GEMMs: the second plan is either a cluster-of-2 plan (deterministic) or, when
    // the engine allows it, a cluster-of-1 plan whose split-K partials are reduce-added by TMA
    const bool nd = ec.nondeterministic_gemm != 0;
    gemm_plan(d.o2, w.wo, m.d, m.qd, M->attn, M->S, m.qd, bn_dec, kEpiAddF32, M->x, m.d, nullptr, b, stop, nd ? 1 : 2);
    gemm_plan(d.down2, w.wd, m.d, m.f, M->hbuf, M->S, m.f, bn_dec, kEpiAddF32, M->x, m.d, nullptr, b, stop,
              nd ? 1 : 2);
    if (nd) {
      d.o2.nondet = d.down2.nondet = true;
      gemm_set_schedule(d.o2, 0);
      gemm_set_schedule(d.down2, 0);
    }
    gemm_partition(d.qkv, d.qkv2);
    gemm_partition(d.o, d.o2);
    gemm_partition(d.down, d.down2);
    gemm_plan(p.qkv, w.wqkv, m.qkv_dim, m.d, M->xn, M->M_pf, m.d, 256, kEpiBF16, M->qkv, m.qkv_dim, w.bqkv,
              M->pf_rows, nullptr);
    gemm_plan(p.o, w.wo, m.d, m.qd, M->attn, M->M_pf, m.qd, 256, kEpiAddF32, M->x, m.d, nullptr, M->pf_rows,
              nullptr);
    gemm_plan(p.gu, w.wgu, 2 * m.f, m.d, M->xn, M->M_pf, m.d, 256, kEpiSwiGLU, M->hbuf, m.f, nullptr, M->pf_rows,
              nullptr);
    gemm_plan(p.down, w.wd, m.d, m.f, M->hbuf, M->M_pf, m.f, 256, kEpiAddF32, M->x, m.d, nullptr, M->pf_rows,
              nullptr);
    M->dec.push_back(d);
    M->pf.push_back(p);
  }
  gemm_plan(M->lm_dec, M->lm_head, m.V, m.d, M->xn, M->S, m.d, bn_dec, kEpiF32, M->logits, m.V, nullptr, b, stop, 2, true);
  M->inv_temp = ec.greedy ? 1.f / std::max(ec.temperature, 1e-6f) : 1.f / ec.temperature;
  if (ec.temperature <= 0.f) M->inv_temp = 1.f;
  AB_CUDA(cudaStreamSynchronize(s));
  return M;
}

void model_destroy(Model* M) {
  if (!M) return;
  ModelDev& m = M->md;
  void* ptrs[] = {M->wbuf,     M->x,        M->xn,        M->qkv,       M->qrot,      M->attn,     M->hbuf,
                  M->logits,   M->part_o,   M->part_ml,   m.row_tok,    m.row_pos,    m.row_btrow, m.h_ctx,
                  m.h_last_tok, m.h_shared, m.g_ctx,      m.g_last_tok, m.g_npages,   m.bt,        m.rope,
                  M->pf_rows,  M->seg_start, M->seg_group, M->ga_g,     M->ga_len,    M->ga_last,  m.kv,
                  m.free_pages, m.split_prefix, m.att_counter, m.att_ctl};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (M->host_stage) cudaFreeHost(M->host_stage);
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

void model_open_group(Engine& e, int group_slot, const int32_t* prompt, int prompt_len) {
  Model* M = e.model;
  AB_REQUIRE(prompt != nullptr && prompt_len >= 2, AB_ERR_CONTRACT, "prompt needs >= 2 tokens");
  AB_REQUIRE(prompt_len <= e.cfg.max_prompt, AB_ERR_CONTRACT, "prompt longer than max_prompt");
  for (int i = 0; i < prompt_len; ++i)
    AB_REQUIRE(prompt[i] >= 0 && prompt[i] < M->md.V, AB_ERR_CONTRACT, "prompt token out of vocabulary");
  M->pending.push_back({group_slot, std::vector<int32_t>(prompt, prompt + prompt_len)});
}

static void check_kv(Engine& e) {
  AB_CUDA(cudaMemcpyAsync(&e.ctl_host->error, &e.d.ctl->error, sizeof(int32_t), cudaMemcpyDeviceToHost, e.stream));
  AB_CUDA(cudaStreamSynchronize(e.stream));
  if (e.ctl_host->error == kErrOutOfKV) throw Error(AB_ERR_OUT_OF_KV, "KV page pool exhausted");
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
    int32_t* segs = btr + R;
    int32_t* segg = segs + ng + 1;
    int32_t* gg = segg + ng;
    int32_t* gl = gg + ng;
    int32_t* glast = gl + ng;
    int r = 0;
    for (int j = 0; j < ng; ++j) {
      const auto& pg = M->pending[k + j];
      const int len = (int)pg.prompt.size() - 1;
      segs[j] = r;
      segg[j] = pg.g;
      gg[j] = pg.g;
      gl[j] = len;
      glast[j] = pg.prompt[len];
      for (int t = 0; t < len; ++t, ++r) {
        tok[r] = pg.prompt[t];
        pos[r] = t;
        btr[r] = m.H + pg.g;
      }
    }
    segs[ng] = R;
    AB_CUDA(cudaMemcpyAsync(m.row_tok, tok, sizeof(int32_t) * R, cudaMemcpyHostToDevice, s));
    AB_CUDA(cudaMemcpyAsync(m.row_pos, pos, sizeof(int32_t) * R, cudaMemcpyHostToDevice, s));
    AB_CUDA(cudaMemcpyAsync(m.row_btrow, btr, sizeof(int32_t) * R, cudaMemcpyHostToDevice, s));
    AB_CUDA(cudaMemcpyAsync(M->seg_start, segs, sizeof(int32_t) * (ng + 1), cudaMemcpyHostToDevice, s));
    AB_CUDA(cudaMemcpyAsync(M->seg_group, segg, sizeof(int32_t) * ng, cudaMemcpyHostToDevice, s));
    AB_CUDA(cudaMemcpyAsync(M->ga_g, gg, sizeof(int32_t) * ng, cudaMemcpyHostToDevice, s));
    AB_CUDA(cudaMemcpyAsync(M->ga_len, gl, sizeof(int32_t) * ng, cudaMemcpyHostToDevice, s));
    AB_CUDA(cudaMemcpyAsync(M->ga_last, glast, sizeof(int32_t) * ng, cudaMemcpyHostToDevice, s));
    AB_CUDA(cudaMemcpyAsync(M->pf_rows, &R, sizeof(int), cudaMemcpyHostToDevice, s));
    launch_group_alloc(e.d, m, M->ga_g, M->ga_len, M->ga_last, ng, s);
    int max_len = 0;
    for (int j = 0; j < ng; ++j) max_len = std::max(max_len, gl[j]);
    launch_embed(m, M->embed, M->x, nullptr, R, nullptr, s);
    for (int l = 0; l < m.L; ++l) {
      const LayerW& w = M->layers[l];
      const Model::Plans& p = M->pf[l];
      launch_rmsnorm(M->x, w.attn_norm, M->xn, m.d, m.eps, nullptr, R, nullptr, s);
      gemm_launch(p.qkv, s);
      launch_rope_kv(m, l, M->qkv, w.q_norm, w.k_norm, M->qrot, nullptr, R, nullptr, s);
      launch_prefill_attention(m, l, M->qrot, M->attn, M->seg_start, M->seg_group, ng, R, max_len, s);
      gemm_launch(p.o, s);
      launch_rmsnorm(M->x, w.mlp_norm, M->xn, m.d, m.eps, nullptr, R, nullptr, s);
      gemm_launch(p.gu, s);
      gemm_launch(p.down, s);
    }
    AB_CUDA(cudaGetLastError());
    AB_CUDA(cudaStreamSynchronize(s));  // host staging is reused by the next chunk
    e.prefill_tokens += R;
    e.launches += 2 + 8 * (int64_t)m.L;
    k = k1;
  }
  M->pending.clear();
  check_kv(e);
}

void model_submit(Engine& e, const ab_sample_desc* descs_dev, int n) {
  flush_prefill(e);
  launch_fork_groups(e.d, e.model->md, descs_dev, n, e.stream);
  AB_CUDA(cudaGetLastError());
  check_kv(e);
}

void model_release(Engine& e, const int32_t* handles_dev, int n) {
  launch_release_handles(e.d, e.model->md, handles_dev, n, e.stream);
  AB_CUDA(cudaGetLastError());
}

void model_release_group(Engine& e, int group_slot) {
  Model* M = e.model;
  // a group still waiting for prefill is simply dropped
  for (size_t i = 0; i < M->pending.size(); ++i)
    if (M->pending[i].g == group_slot) {
      M->pending.erase(M->pending.begin() + i);
      return;
    }
  launch_group_release(e.d, M->md, group_slot, e.stream);
  AB_CUDA(cudaGetLastError());
}

void model_iteration(Engine& e, int64_t run_iter, bool timed) {
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
      gemm_launch(p.qkv, s);
      gemm_launch(p.qkv2, s);
    }
    {
      ScopedTimer t(e, timed, "rope_kv", run_iter);
      launch_rope_kv(m, l, M->qkv, w.q_norm, w.k_norm, M->qrot, b, S, stop, s);
    }
    {
      ScopedTimer t(e, timed, "attention", run_iter);
      launch_decode_attention(M->kvmap, e.d, m, l, M->qrot, M->attn, M->part_o, M->part_ml, M->max_splits, M->chunk,
                              s);
    }
    {
      ScopedTimer t(e, timed, "gemm_o", run_iter);
      gemm_launch(p.o, s);
      gemm_launch(p.o2, s);
    }
    {
      ScopedTimer t(e, timed, "rmsnorm", run_iter);
      launch_rmsnorm(M->x, w.mlp_norm, M->xn, m.d, m.eps, b, S, stop, s);
    }
    {
      ScopedTimer t(e, timed, "gemm_gate_up", run_iter);
      gemm_launch(p.gu, s);
    }
    {
      ScopedTimer t(e, timed, "gemm_down", run_iter);
      gemm_launch(p.down, s);
      gemm_launch(p.down2, s);
    }
  }
  {
    ScopedTimer t(e, timed, "rmsnorm", run_iter);
    launch_rmsnorm(M->x, M->final_norm, M->xn, m.d, m.eps, b, S, stop, s);
  }
  {
    ScopedTimer t(e, timed, "gemm_lm_head", run_iter);
    gemm_launch(M->lm_dec, s);
  }
  {
    ScopedTimer t(e, timed, "sampler", run_iter);
    launch_sampler(e.d, m, M->logits, M->inv_temp, e.cfg.greedy, e.cfg.top_p, s);
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
  else if (name == "embed") *bytes = b * d * 6;
}

}  // namespace ab
