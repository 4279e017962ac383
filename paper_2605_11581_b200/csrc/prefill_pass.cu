// One C entry for the whole Prefill pass (`adamk_prefill`; PAPER.md:244-249 runs Prefill on the
// serving engine's operators -- here on this library's tcgen05 GEMM, flash attention and row kernels, in the order
// paper_2605_11581_b200/prefill.py documents).  Host code only: it carves the caller's workspace and enqueues the
// operators of include/adamk_prefill.h on one stream, so a host without Python can fill the decode kernel's KV cache.
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "../../include/adamk_prefill.h"

namespace {

thread_local char g_pass_err[256] = "";

int pass_fail(const char* what, int layer, const char* detail) {
  snprintf(g_pass_err, sizeof(g_pass_err), "adamk_prefill: %s (layer %d)%s%s", what, layer, detail && detail[0] ? ": " : "",
           detail ? detail : "");
  return -1;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct PassBuffers {
  size_t xp, qkv, q, ap, act, vt, total;
};

PassBuffers carve(const AdamkPrefillModel& m, int T, int pos0, int planes) {
  PassBuffers b{};
  const size_t P = (size_t)planes, Tn = (size_t)T;
  const size_t ctx_pad = (size_t)((pos0 + T + 63) / 64) * 64;
  size_t off = 0;
  auto take = [&](size_t bytes) { const size_t o = off; off += align256(bytes); return o; };
  b.xp = take(P * Tn * m.hidden * 2);
  b.qkv = take(Tn * (size_t)(m.n_q_heads + 2 * m.n_kv_heads) * m.head_dim * 4);
  b.q = take((size_t)m.n_q_heads * Tn * m.head_dim * 2);
  b.ap = take(P * Tn * (size_t)m.n_q_heads * m.head_dim * 2);
  b.act = take(P * Tn * (size_t)m.intermediate_padded * 2);
  b.vt = take((size_t)m.n_kv_heads * m.head_dim * ctx_pad * 2);
  b.total = off;
  return b;
}

bool model_ok(const AdamkPrefillModel* m) {
  return m && m->n_layers > 0 && m->hidden > 0 && m->hidden % 8 == 0 && m->n_q_heads > 0 && m->n_kv_heads > 0 &&
         m->n_q_heads % m->n_kv_heads == 0 && (m->head_dim == 64 || m->head_dim == 128) && m->intermediate_padded > 0 &&
         m->intermediate_padded % 128 == 0 && m->max_ctx > 0 && m->kv_layer_stride > 0;
}

}  // namespace

extern "C" {

const char* adamk_prefill_pass_last_error(void) { return g_pass_err; }

size_t adamk_prefill_workspace_bytes(const AdamkPrefillModel* model, int T, int pos0, int planes) {
  if (!model_ok(model) || T <= 0 || pos0 < 0 || (planes != 1 && planes != 2)) return 0;
  return carve(*model, T, pos0, planes).total;
}

int adamk_prefill(const AdamkPrefillModel* model, const AdamkPrefillLayer* layers, const void* embed, const float* rope_cos,
                  const float* rope_sin, const int32_t* tokens, int T, int pos0, int planes, void* k_cache, void* v_cache,
                  void* workspace, float* hidden, adamk_pf_stream stream) {
  if (!model_ok(model)) return pass_fail("invalid model description", -1, "");
  if (!layers || !embed || !rope_cos || !rope_sin || !tokens || !k_cache || !v_cache || !workspace || !hidden)
    return pass_fail("NULL argument", -1, "");
  if (T <= 0 || pos0 < 0 || (planes != 1 && planes != 2)) return pass_fail("T, pos0 or planes out of range", -1, "");
  if ((long long)pos0 + T > model->max_ctx) return pass_fail("prompt does not fit the KV cache", -1, "");
  const AdamkPrefillModel& m = *model;
  const PassBuffers b = carve(m, T, pos0, planes);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  void* xp = ws + b.xp;
  float* qkv = reinterpret_cast<float*>(ws + b.qkv);
  void* q = ws + b.q;
  void* ap = ws + b.ap;
  void* act = ws + b.act;
  void* vt = ws + b.vt;
  const int H = m.hidden, D = m.head_dim, nq = m.n_q_heads, nkv = m.n_kv_heads, I = m.intermediate_padded;
  const int n_qkv = (nq + 2 * nkv) * D, ctx = pos0 + T, ctx_pad = (ctx + 63) / 64 * 64;
  auto gemm_err = [&](const char* what, int l) { return pass_fail(what, l, adamk_prefill_last_error()); };
  if (adamk_prefill_embed(tokens, T, embed, H, hidden, stream)) return gemm_err("embedding gather", -1);
  for (int l = 0; l < m.n_layers; ++l) {
    const AdamkPrefillLayer& w = layers[l];
    if (!w.ln1 || !w.ln2 || !w.wqkv || !w.wo || !w.wgu || !w.wdown) return pass_fail("NULL weight", l, "");
    uint8_t* kc = static_cast<uint8_t*>(k_cache) + (size_t)l * m.kv_layer_stride;
    uint8_t* vc = static_cast<uint8_t*>(v_cache) + (size_t)l * m.kv_layer_stride;
    if (adamk_prefill_rmsnorm_split(hidden, w.ln1, m.rms_eps, T, H, xp, planes, stream)) return gemm_err("input norm", l);
    if (adamk_prefill_gemm(xp, planes, T, H, w.wqkv, n_qkv, w.bqkv, qkv, n_qkv, ADAMK_PF_EPI_STORE, 1, 0, ADAMK_PF_TILE_AUTO, stream))
      return gemm_err("QKV projection", l);
    if (adamk_prefill_rope_store(qkv, T, nq, nkv, D, w.q_norm, w.k_norm, m.rms_eps, rope_cos, rope_sin, pos0, m.max_ctx, q, 1, kc, vc,
                                 stream))
      return gemm_err("rotary embedding / cache write", l);
    if (adamk_prefill_vt(vc, nkv, D, m.max_ctx, ctx, ctx_pad, vt, stream))
      return pass_fail("V transpose", l, adamk_prefill_attention_last_error());
    if (adamk_prefill_attention(q, kc, vt, T, pos0, nq, nkv, D, m.max_ctx, ctx_pad, ap, planes, stream))
      return pass_fail("flash attention", l, adamk_prefill_attention_last_error());
    if (adamk_prefill_gemm(ap, planes, T, nq * D, w.wo, H, nullptr, hidden, H, ADAMK_PF_EPI_RESID, 1, 0, ADAMK_PF_TILE_AUTO, stream))
      return gemm_err("O projection", l);
    if (adamk_prefill_rmsnorm_split(hidden, w.ln2, m.rms_eps, T, H, xp, planes, stream)) return gemm_err("post-attention norm", l);
    if (adamk_prefill_gemm(xp, planes, T, H, w.wgu, 2 * I, nullptr, act, I, ADAMK_PF_EPI_SWIGLU, planes, (long long)T * I,
                           ADAMK_PF_TILE_AUTO, stream))
      return gemm_err("gate / up projection", l);
    if (adamk_prefill_gemm(act, planes, T, I, w.wdown, H, nullptr, hidden, H, ADAMK_PF_EPI_RESID, 1, 0, ADAMK_PF_TILE_AUTO, stream))
      return gemm_err("down projection", l);
  }
  return 0;
}

}  // extern "C"
