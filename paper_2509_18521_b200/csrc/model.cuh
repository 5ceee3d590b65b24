// Transformer decode path: device layout shared by model.cu, decoder_kernels.cu, sampler.cu.
#pragma once

#include <cuda_bf16.h>

#include "engine.cuh"
#include "gemm.cuh"

namespace ab {

using bf16 = __nv_bfloat16;

// KV pool layout (HBM): kv[layer][page][k|v][kv_head][page_slot][head_dim] bf16.
// One page id addresses the same token range in every layer; a page's K (or V)
// for one kv head is a contiguous page_size*head_dim*2-byte block.
struct ModelDev {
  int L, d, hq, hk, hd, f, V, qkv_dim, qd, kvd, gq;
  int P, MP, H, G_cap;
  int qk_norm;
  float eps;
  bf16* kv;
  int64_t NP;
  int32_t* free_pages;  // stack, top in Ctl::kv_free_top
  int32_t* bt;          // [(H + G_cap) * MP]: rows [0,H) samples, [H, H+G_cap) prompt groups
  int32_t* h_ctx;       // tokens with KV in cache
  int32_t* h_last_tok;  // next input token
  int32_t* h_shared;    // leading pages shared with the prompt group
  int32_t* g_ctx;
  int32_t* g_last_tok;
  int32_t* g_npages;
  float2* rope;         // [max_pos][hd/2] (cos, sin)
  int max_pos;
  int32_t* row_tok;
  int32_t* row_pos;
  int32_t* row_btrow;
  int32_t* row_pslot;     // [S] decode: page * P + slot of the row's new token (k_prep_decode)
  int32_t* split_prefix;  // [S+1] attention work list: exclusive prefix of KV splits per live row
  int32_t* att_counter;   // [S * hk] split-combine arrival counters (self-resetting)
  int32_t* att_items;     // [S * max_splits] work list: row | split << 16
  int32_t* att_ctl;       // [1 + L]: KV split size of this iteration, per-layer work-list cursors

  __device__ __forceinline__ size_t kv_off(int l, int page, int which, int head, int slot) const {
    return ((((size_t)l * NP + page) * 2 + which) * hk + head) * (size_t)P * hd + (size_t)slot * hd;
  }
};

struct LayerW {
  bf16 *attn_norm, *wqkv, *bqkv, *q_norm, *k_norm, *wo, *mlp_norm, *wgu, *wd;
};

// decoder_kernels.cu
void launch_init_weights(bf16* w, size_t n, uint64_t seed, uint64_t tensor_id, float std, float constant,
                         cudaStream_t s);
void launch_rope_table(float2* rope, int max_pos, int hd, float theta, cudaStream_t s);
void launch_prep_decode(const EngineDev& e, const ModelDev& m, int chunk, cudaStream_t s);
void launch_embed(const ModelDev& m, const bf16* emb, float* x, const int* rows_dev, int rows_cap,
                  const int* stop, cudaStream_t s);
void launch_rmsnorm(const float* x, const bf16* w, bf16* out, int d, float eps, const int* rows_dev, int rows_cap,
                    const int* stop, cudaStream_t s);
void launch_rope_kv(const ModelDev& m, int layer, const bf16* qkv, const bf16* q_norm, const bf16* k_norm, bf16* q_out,
                    const int* rows_dev, int rows_cap, const int* stop, cudaStream_t s);
void launch_rope_kv_f32(const ModelDev& m, int layer, float* qkv, const bf16* bias, const bf16* q_norm,
                        const bf16* k_norm, bf16* q_out, const int* rows_dev, int rows_cap, const int* stop,
                        cudaStream_t s);
// attention.cu
void make_kv_tmap(CUtensorMap* map, const ModelDev& m);
int decode_attention_ctas(const ModelDev& m);  // persistent grid of the decode attention kernel
void launch_decode_attention(const CUtensorMap& map, const EngineDev& e, const ModelDev& m, int layer, const bf16* q,
                             bf16* out, float* part_o, float* part_ml, int max_splits, int chunk, cudaStream_t s);
// causal flash prefill over the paged pool; blocks[i] = {first row, rows (<= 64), block-table row, first position}
void set_pdl_mask_attention(int mask);
void set_pdl_mask_layers(int mask);
int attention_items_per_cta();  // decode attention work items per persistent CTA (AB_ATT_ITEMS, default 1)
void launch_prefill_flash(const ModelDev& m, int layer, const bf16* q, bf16* out, const int4* blocks, int n_blocks,
                          cudaStream_t s);
void launch_fork_groups(const EngineDev& e, const ModelDev& m, const ab_sample_desc* descs, int n, cudaStream_t s);
void launch_resume_fork(const EngineDev& e, const ModelDev& m, const int4* items, int n, cudaStream_t s);
void launch_extend_rows(const EngineDev& e, const ModelDev& m, const int4* pieces, int n_pieces, cudaStream_t s);
void launch_score_alloc(const EngineDev& e, const ModelDev& m, const int2* items, int n, cudaStream_t s);
void launch_score_release(const EngineDev& e, const ModelDev& m, const int2* items, int n, cudaStream_t s);
void launch_gather_rows(const bf16* src, bf16* dst, const int* rows, int n, int d, cudaStream_t s);
void launch_logp_rows(const float* logits, int V, const int* target, int n, float inv_temp, double* out,
                      cudaStream_t s);
void launch_release_handles(const EngineDev& e, const ModelDev& m, const int32_t* handles, int n, cudaStream_t s);
void launch_group_alloc(const EngineDev& e, const ModelDev& m, const int* groups, const int* lens,
                        const int* last_tok, int n, cudaStream_t s);
void launch_group_release(const EngineDev& e, const ModelDev& m, int group, cudaStream_t s);
// h[r][j] = bf16(silu(g) * u) from the gate-up fp32 workspace (interleaved 64-row halves per 128
// rows), re-zeroing it; a no-op when the plan's schedule entry for the live row count is 0
void launch_swiglu_ws(float* ws, bf16* h, int f, const int* sched, const int* rows_dev, int rows_cap, const int* stop,
                      cudaStream_t s);
// sampler.cu
// top_p = 1 or greedy: split kernels over fixed logit pieces (part: sampler_scratch_bytes);
// nucleus: one CTA per row
void launch_sampler(const EngineDev& e, const ModelDev& m, const float* logits, float inv_temp, int greedy,
                    float top_p, void* part, cudaStream_t s);
size_t sampler_scratch_bytes(int rows, int V);
bool sampler_uses_split(int greedy, float top_p);  // two kernels (pieces + finish) per iteration

}  // namespace ab
