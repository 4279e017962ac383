/*
 * adamk_prefill.h -- C ABI of the Prefill-phase operators in libadamk.so.
 *
 * The paper's online half runs Prefill on the serving engine's own operators and Decode on the MegaKernel
 * (/root/reference/PAPER.md:244-249); the reference ships neither.  These entry
 * points are the hand-written sm_100a Prefill operators a TensorRT-LLM style engine would call in place of
 * its library GEMMs: a tcgen05 / tensor-memory GEMM with the fused epilogues a decoder layer needs, and the
 * element-wise kernels around it.  Same conventions as adamk.h: 0 on success, negative ADAMK_PF_E_* code
 * otherwise, adamk_prefill_last_error() for the message, asynchronous on the given stream, no C++ or torch
 * types in the signatures, the caller owns every buffer.
 */
#ifndef ADAMK_PREFILL_H_
#define ADAMK_PREFILL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADAMK_PF_OK 0
#define ADAMK_PF_E_INVALID (-1)
#define ADAMK_PF_E_CUDA (-2)

/* GEMM epilogues */
#define ADAMK_PF_EPI_STORE 0  /* out fp32 [T, ldo]  = acc (+ bias)                                          */
#define ADAMK_PF_EPI_RESID 1  /* out fp32 [T, ldo] += acc          (residual stream update)                 */
#define ADAMK_PF_EPI_SWIGLU 2 /* out bf16 planes [parts_out][T, ldo] = split(silu(gate) * up); the weight   */
                              /* interleaves gate and up rows in blocks of tile_n / 2 features              */

/* GEMM tile shapes (tokens x output features) */
#define ADAMK_PF_TILE_AUTO 0
#define ADAMK_PF_TILE_128 128  /* 128 x 128, one CTA                                                         */
#define ADAMK_PF_TILE_256 256  /* 128 x 256, one CTA                                                         */
#define ADAMK_PF_TILE_PAIR 512 /* 256 x 256 on a CTA pair (cluster of 2, tcgen05.mma.cta_group::2)           */

#define ADAMK_PF_EPI_ATOMIC 3 /* out fp32 [T, ldo] += acc (+ bias once) with fp32 atomics: decode-sized T, where the  */
                              /* library splits K across SMs to stream the weight at full width (one-CTA tiles)     */

typedef void* adamk_pf_stream; /* cudaStream_t */

const char* adamk_prefill_last_error(void);

/* Launch the operators below with programmatic dependent launch (stream serialization attribute): each kernel's
 * prologue overlaps the previous kernel's tail and `griddepcontrol.wait` orders the data.  Process-wide, off by
 * default; the batched decode step (dozens of ~10 us kernels per layer) turns it on.
 *   0 = off; 1 = on; 2 = on, and every GEMM issues the WEIGHT boxes of its first pass over the shared-memory ring
 *   ahead of the wait (the weight is constant data: only token rows, bias and outputs are ordered behind the previous
 *   kernel) -- the batched decode default; 3 = 2 + the next k blocks of the CTA's weight share requested into L2
 *   (measured slower than 2; kept for A/B, tools/batch_pdl_ab.py).  Modes 2 / 3 require that no kernel in the stream
 *   writes a GEMM's weight operand. */
void adamk_prefill_set_pdl(int on);

/* Decode-sized ATOMIC calls whose stacked planes hold at most 32 tokens each (batch <= 32): plane p is placed in rows
 * [32 p, 32 p + T) of the 128-row token tile (a 3-D tensor map of the token operand), so that every plane's accumulator
 * rows sit in their own tensor-memory lane quarter and one epilogue warp per plane sends the atomics instead of one
 * warp for all planes.  Process-wide, on by default; 0 restores consecutive rows (A/B). */
void adamk_prefill_set_plane_quarters(int on);

/* Tile walk order of adamk_prefill_gemm, process-wide: -1 (default) = chosen per call -- tile column fastest when the
 * activation operand is larger than the weight and the weight fits L2 (the down projection of a long prompt), token
 * block fastest otherwise; 0 / 1 force one of them (A/B measurements, tools/ncu_prefill.py). */
void adamk_prefill_set_walk(int mode);

/* One-shot hint for the NEXT adamk_prefill_gemm call on this thread (one-CTA tiles): while that GEMM waits for its own
 * operands, its idle warps pull `bytes` at `ptr` -- the weight the kernel AFTER it will stream -- into L2
 * (cp.async.bulk.prefetch.L2).  The batched decode step chains its GEMMs this way; 16-byte aligned, < L2 size. */
void adamk_prefill_prefetch_next(const void* ptr, long long bytes);

/* Debug: when non-null, CTA 0 of every one-CTA-tile GEMM launch writes six %globaltimer stamps (ns) to `stamps`
 * (device memory, 8 x uint64): start, prologue done, first operands landed, last MMA issued, epilogue done, exit,
 * accumulator visible to the epilogue. */
void adamk_prefill_set_trace(void* stamps);

/* D[T, N] = X[T, K] . W[N, K]^T on the tensor cores, fp32 accumulation in tensor memory.
 *   x_planes  bf16 [parts][T, K] row-major: the activation as `parts` bf16 planes whose sum is the fp32 value
 *             (parts 1 = plain bf16; 2 = hi + lo, ~2^-17 relative; 3 = hi + mid + lo, below fp32 resolution --
 *             free for decode-sized T, where all planes ride in one token tile).
 *   w         bf16 [N, K] row-major (Hugging Face layout).
 *   tile_n    one of ADAMK_PF_TILE_*; the SwiGLU weight interleaves gate / up in blocks of 128 features for the
 *             256-wide tiles (ADAMK_PF_TILE_256 / _PAIR) and 64 for ADAMK_PF_TILE_128.
 * K, N and ldo must be multiples of 8 and the pointers 16-byte aligned. */
int adamk_prefill_gemm(const void* x_planes, int parts, int T, int K, const void* w, int N, const float* bias, void* out, int ldo,
                       int epilogue, int parts_out, long long part_stride, int tile_n, adamk_pf_stream stream);

/* How adamk_prefill_gemm would cut this problem on a GPU with n_sms SMs -- host arithmetic only, no device needed:
 * plan_out = {tile (ADAMK_PF_TILE_*), tiles, whole-tile items, column slices per last-wave tile, work items, K splits,
 * k blocks (of 64) per split, planes stacked in one token tile (0/1), grid size}. */
int adamk_prefill_gemm_plan(int parts, int T, int K, int N, int epilogue, int tile_n, int n_sms, int32_t plan_out[9]);

/* Causal flash attention of a Prefill pass on the tensor cores (csrc/prefill_attn.cu; replaces the serving engine's
 * attention operator of PAPER.md:248).  q bf16 [n_q][T][D] (rotary applied, unscaled); k_cache bf16 [n_kv][max_ctx][D]
 * (one layer of the decode kernel's cache, rows pos0 .. pos0 + T - 1 already written); vt bf16 [n_kv][D][ctx_pad] =
 * adamk_prefill_vt of the same layer's V cache.  Row t attends to positions 0 .. pos0 + t.  out: bf16 planes
 * [parts][T][n_q * D] (parts 1: the bf16 value; 2: value + residual), the activation operand of the O projection. */
int adamk_prefill_attention(const void* q, const void* k_cache, const void* vt, int T, int pos0, int n_q, int n_kv, int D, int max_ctx,
                            int ctx_pad, void* out_planes, int parts, adamk_pf_stream stream);

/* vt bf16 [n_kv][D][ctx_pad] = transpose of v_cache bf16 [n_kv][max_ctx][D] rows 0 .. ctx - 1, zero padded to ctx_pad (a multiple of 64). */
int adamk_prefill_vt(const void* v_cache, int n_kv, int D, int max_ctx, int ctx, int ctx_pad, void* vt, adamk_pf_stream stream);

const char* adamk_prefill_attention_last_error(void);

/* Which flash kernel adamk_prefill_attention launches, process-wide: 0 (default) = a pair of 128-row q tiles per CTA
 * (one tile when the pass has at most 128 rows), 1 = always one tile per CTA with its rows split between two softmax
 * warpgroups.  Same results up to summation order; for A/B measurements and tests. */
void adamk_prefill_attention_set_kernel(int one_tile);

/* h fp32 [T, H] = embed[tokens[t]] (bf16 table). */
int adamk_prefill_embed(const int32_t* tokens, int T, const void* embed, int H, float* h, adamk_pf_stream stream);

/* The same for a device-resident decode loop, whose token ids the host never sees: ids outside [0, vocab) read row 0. */
int adamk_batch_embed(const int32_t* tokens, int T, const void* embed, int H, int vocab, float* h, adamk_pf_stream stream);

/* planes bf16 [parts][T, H] = split(RMSNorm(h) * gain): the GEMM's activation operand. */
int adamk_prefill_rmsnorm_split(const float* h, const void* gain, float eps, int T, int H, void* planes, int parts,
                                adamk_pf_stream stream);

/* planes bf16 [parts][n] = split(x fp32 [n]). */
int adamk_prefill_split(const float* x, long long n, void* planes, int parts, adamk_pf_stream stream);

/* qkv fp32 [T, (n_q + 2 n_kv) D] (bias already added) -> optional per-head RMSNorm of q and k (Qwen3), rotate-half
 * rotary embedding with the decode kernel's fp32 cos/sin tables [max_ctx, D/2], then
 *   q_out   [n_q][T][D]  fp32 or bf16 (q_is_bf16)
 *   k_cache / v_cache  bf16 [n_kv][max_ctx][D] of one layer, rows pos0 .. pos0 + T - 1. */
int adamk_prefill_rope_store(const float* qkv, int T, int n_q, int n_kv, int D, const void* q_gain, const void* k_gain, float eps,
                             const float* cos, const float* sin, int pos0, int max_ctx, void* q_out, int q_is_bf16, void* k_cache,
                             void* v_cache, adamk_pf_stream stream);

/* ---- the whole Prefill pass behind one call (csrc/prefill_pass.cu) ------------------------
 * What the serving engine's Prefill phase hands to this library: T prompt tokens in, rows
 * pos0 .. pos0 + T - 1 of every layer of the decode kernel's KV cache filled, final hidden states out.  Host-side
 * orchestration of the operators above on one stream (embedding, then per layer: RMSNorm + plane split, QKV GEMM + bias,
 * rotary embedding + cache write, V transpose, causal flash attention, O GEMM += residual, RMSNorm + split, gate/up GEMM
 * with SwiGLU, down GEMM += residual): 1 + 9 launches per layer, asynchronous, no allocation. */
typedef struct {
  int n_layers, hidden, n_q_heads, n_kv_heads, head_dim;
  int intermediate_padded;      /* I rounded up to a multiple of 128: rows / 2 of wgu, columns of wdown (zero padded) */
  int max_ctx;                  /* rows per head of the KV cache and of the rope tables */
  float rms_eps;
  long long kv_layer_stride;    /* BYTES between consecutive layers of k_cache / v_cache (the plugin's cache:
                                   max_batch * n_kv_heads * max_ctx * head_dim * 2) */
} AdamkPrefillModel;

typedef struct {
  const void* ln1;      /* bf16 [hidden] */
  const void* ln2;      /* bf16 [hidden] */
  const void* wqkv;     /* bf16 [(n_q + 2 n_kv) * head_dim, hidden]: q, k, v rows concatenated */
  const float* bqkv;    /* fp32 [(n_q + 2 n_kv) * head_dim] or NULL */
  const void* wo;       /* bf16 [hidden, n_q * head_dim] */
  const void* wgu;      /* bf16 [2 * intermediate_padded, hidden]: gate / up interleaved in blocks of 128 features */
  const void* wdown;    /* bf16 [hidden, intermediate_padded] */
  const void* q_norm;   /* bf16 [head_dim] or NULL (Qwen3) */
  const void* k_norm;   /* bf16 [head_dim] or NULL */
} AdamkPrefillLayer;

/* Scratch the pass needs for T tokens at offset pos0 with `planes` (1 | 2) bf16 planes per activation; 0 = bad arguments. */
size_t adamk_prefill_workspace_bytes(const AdamkPrefillModel* model, int T, int pos0, int planes);

/* tokens: DEVICE int32 [T]; embed bf16 [vocab, hidden]; rope_cos / rope_sin fp32 [max_ctx, head_dim / 2] (the decode
 * kernel's tables); k_cache / v_cache: sequence 0 of layer 0 of the decode kernel's cache; workspace: DEVICE,
 * adamk_prefill_workspace_bytes, 256-byte aligned; hidden: DEVICE fp32 [T, hidden], the final hidden states (before
 * the final norm).  pos0 > 0 = chunked Prefill: rows 0 .. pos0 - 1 must already be cached. */
int adamk_prefill(const AdamkPrefillModel* model, const AdamkPrefillLayer* layers, const void* embed, const float* rope_cos,
                  const float* rope_sin, const int32_t* tokens, int T, int pos0, int planes, void* k_cache, void* v_cache,
                  void* workspace, float* hidden, adamk_pf_stream stream);

const char* adamk_prefill_pass_last_error(void);

/* ---- batched decode: one new token per sequence, B sequences per step -------------
 * The projections are adamk_prefill_gemm with T = B and the ATOMIC / SWIGLU / STORE epilogues; these are the operators
 * between them.  Caches: bf16 [B][n_kv][max_ctx][D] per layer (seq_stride = elements between sequences). */

/* rmsnorm_split that also clears `zero_n` floats at `zero` (the fp32 targets of the ATOMIC GEMMs that follow). */
int adamk_batch_rmsnorm_split(const float* h, const void* gain, float eps, int B, int H, void* planes, int parts, float* zero, long long zero_n,
                              adamk_pf_stream stream);

/* rope_store for a batch: token b sits at positions[b] of sequence b; q_out fp32 [n_q][B][D]. */
int adamk_batch_rope_store(const float* qkv, int B, int n_q, int n_kv, int D, const void* q_gain, const void* k_gain, float eps,
                           const float* cos, const float* sin, const int32_t* positions, long long seq_stride, int max_ctx, float* q_out,
                           void* k_cache, void* v_cache, adamk_pf_stream stream);

/* Attention of every sequence's new token over cache rows 0 .. positions[b] (split over 64-row chunks, merged),
 * output as bf16 planes [parts][B][n_q * D].  workspace: adamk_batch_attention_workspace() bytes. */
size_t adamk_batch_attention_workspace(int B, int n_q, int D, int max_ctx);
int adamk_batch_attention(const float* q, const void* k_cache, const void* v_cache, const int32_t* positions, int B, int n_q, int n_kv, int D,
                          int max_ctx, long long seq_stride, float* workspace, void* out_planes, int parts, adamk_pf_stream stream);

/* planes bf16 [parts][B, I] = split(silu(gate) * up) from gu fp32 [B, 2 I] (gate / up interleaved in blocks of `block`
 * features, the column order the interleaved gate/up weight produces). */
int adamk_batch_swiglu_split(const float* gu, int B, int I, int block, void* planes, int parts, adamk_pf_stream stream);

/* next[b] = argmax(logits[b]) (lowest index on ties); when non-null, tokens[b] = next[b] and positions[b] += 1. */
int adamk_batch_argmax(const float* logits, int B, int V, int32_t* next, int32_t* tokens, int32_t* positions, adamk_pf_stream stream);

/* The same pick with every row scanned by 64 CTAs instead of one (73 -> a few microseconds for a 150 K vocabulary).
 * scratch: DEVICE, adamk_batch_argmax_workspace(B) bytes, ZERO before the first call (the kernel leaves it ready for the
 * next one); one scratch per stream of steps. */
size_t adamk_batch_argmax_workspace(int B);
int adamk_batch_argmax_sliced(const float* logits, int B, int V, void* scratch, int32_t* next, int32_t* tokens, int32_t* positions,
                              adamk_pf_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* ADAMK_PREFILL_H_ */
