/*
 * adamk.h -- C ABI of the B200 decode MegaKernel plugin (libadamk.so).
 *
 * Drop-in boundary.  The reference describes this call
 * only in prose: "embed MegaKernel ... into TensorRT-LLM's execution topology
 * via a Plugin mechanism", "replace only the core Transformer Block with a
 * custom MegaKernel plugin", Prefill on native ops / Decode on the MegaKernel
 * (/root/reference/PAPER.md:244-249), and its SPEC puts the plugin itself out
 * of scope.  There is therefore no reference
 * signature to copy; these entry points have the shape of a TensorRT
 * IPluginV2::enqueue(inputs, outputs, workspace, stream) call and are what a
 * maintainer of the reference's online half would bind (see INTEGRATION.md for
 * the ctypes stub).  What the plugin consumes is the reference's own artifact:
 * the SolidifiedTrace written by `mkplan search`
 * (/root/reference/pkg/src/mkplan/search.py:79-107,138-171), lowered by
 * paper_2605_11581_b200/task_table.py to the flat device task table passed to
 * adamk_create().
 *
 * Conventions: every function returns 0 on success or a negative ADAMK_E_*
 * code; adamk_last_error() returns a thread-local message.  No exceptions and
 * no C++/torch types cross the boundary.  The caller owns every device buffer
 * (weights, packed weights, KV cache, workspace, outputs); the library owns
 * only its handle and the device copy of the task table.  decode_step is
 * asynchronous on the given stream and not re-entrant per handle.
 */
#ifndef ADAMK_H_
#define ADAMK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADAMK_ABI_VERSION 2

#define ADAMK_OK 0
#define ADAMK_E_INVALID (-1)     /* bad argument / malformed task table        */
#define ADAMK_E_CUDA (-2)        /* a CUDA runtime call failed                 */
#define ADAMK_E_UNSUPPORTED (-3) /* valid request this build cannot execute    */
#define ADAMK_E_STATE (-4)       /* call order violated (e.g. step before bind) */
#define ADAMK_E_DEVICE (-5)      /* the kernel reported an error (watchdog...) */

typedef struct AdamkHandle_* adamk_handle;
typedef void* adamk_stream; /* cudaStream_t */

/* Decoder dimensions.  Mirrors paper_2605_11581_b200.model_config.ModelConfig. */
typedef struct AdamkModelDesc {
  int32_t hidden, n_layers, n_q_heads, n_kv_heads, head_dim, intermediate, vocab;
  int32_t max_ctx;   /* KV-cache capacity in positions                          */
  int32_t max_batch; /* sequences per step the task table was built for         */
  int32_t qkv_bias;  /* Qwen2/Qwen2.5: 1                                        */
  int32_t qk_norm;   /* Qwen3: 1                                                */
  int32_t tied_embed;
  float rms_eps;
  float rope_theta;  /* informational; the kernel reads the cos/sin tables      */
} AdamkModelDesc;

/* Per-layer bf16 weights in Hugging Face layout ([out_features, in_features],
 * row-major).  Optional pointers are NULL when the model has no such tensor. */
typedef struct AdamkLayerWeights {
  const void* ln1;    /* [hidden]                      */
  const void* wq;     /* [q_dim, hidden]               */
  const void* wk;     /* [kv_dim, hidden]              */
  const void* wv;     /* [kv_dim, hidden]              */
  const void* bq;     /* [q_dim]      or NULL          */
  const void* bk;     /* [kv_dim]     or NULL          */
  const void* bv;     /* [kv_dim]     or NULL          */
  const void* q_norm; /* [head_dim]   or NULL (Qwen3)  */
  const void* k_norm; /* [head_dim]   or NULL (Qwen3)  */
  const void* wo;     /* [hidden, q_dim]               */
  const void* ln2;    /* [hidden]                      */
  const void* wgate;  /* [intermediate, hidden]        */
  const void* wup;    /* [intermediate, hidden]        */
  const void* wdown;  /* [hidden, intermediate]        */
} AdamkLayerWeights;

typedef struct AdamkWeightPtrs {
  const void* embed;      /* bf16 [vocab, hidden]; must stay alive (row gather)  */
  const void* final_norm; /* bf16 [hidden]                                       */
  const void* lm_head;    /* bf16 [vocab, hidden]; NULL = tied to embed          */
  const AdamkLayerWeights* layers; /* HOST array of n_layers entries             */
  const float* rope_cos;  /* fp32 [max_ctx, head_dim/2] device                   */
  const float* rope_sin;  /* fp32 [max_ctx, head_dim/2] device                   */
} AdamkWeightPtrs;

/* ABI / device queries (no handle needed). */
int adamk_abi_version(void);
int adamk_device_sm_count(int device, int* out_sms);
const char* adamk_last_error(void);

/* Create a plugin instance from the model description and the device task
 * table blob (task_table.py: header, per-SM ranges, 64-byte task records).
 * The table is validated against the description and the device, then copied
 * to the GPU.  tp_rank/tp_size select the tensor-parallel shard (1 GPU: 0/1;
 * tp_size 2, 4 or 8 otherwise).  The handle belongs to the CUDA device that is
 * current at this call: every buffer and stream later passed with it must live
 * on that device, and a step may be issued from a thread whose current device
 * differs (the library switches for the launch and switches back). */
int adamk_create(const AdamkModelDesc* desc, const void* task_table, size_t task_table_bytes,
                 int tp_rank, int tp_size, adamk_handle* out);
void adamk_destroy(adamk_handle h);

/* Bytes of the caller-allocated packed-weight buffer (tile-major per-SM weight
 * streams + fp32 copies of the norm/bias vectors). */
size_t adamk_packed_bytes(adamk_handle h);
/* Repack the HF-layout weights into `packed` (device, 256-byte aligned) on
 * `stream` and remember the pointers.  The source matrices may be freed after
 * the stream has drained, except `embed`. */
int adamk_bind_weights(adamk_handle h, const AdamkWeightPtrs* w, void* packed, adamk_stream stream);

/* W4A16 (GPTQ-format) weights of one layer: for every projection matrix W [N, K] the 4-bit codes q uint8 [N, K / 2]
 * (element k of a row in byte k / 2, even k in the low nibble) and the fp16 scales s [N, ceil(K / 128)];
 * W[n][k] = (q[n][k] - 8) * s[n][k / 128]  (reference byte model: pkg/src/mkplan/graph_ir.py:296-318, group 128,
 * two bytes per scale).  K must be a multiple of 8. */
typedef struct AdamkW4A16Layer {
  const void *q_wq, *s_wq, *q_wk, *s_wk, *q_wv, *s_wv, *q_wo, *s_wo, *q_wgate, *s_wgate, *q_wup, *s_wup, *q_wdown, *s_wdown;
} AdamkW4A16Layer;

/* adamk_bind_weights for a task table built with the W4A16 schedule flag: the layer matrices come from `qlayers` (HOST
 * array of n_layers entries, device pointers inside); `w->layers` still supplies norms / biases (its matrix pointers
 * are ignored); embedding and LM head stay bf16. */
int adamk_bind_weights_w4a16(adamk_handle h, const AdamkWeightPtrs* w, const AdamkW4A16Layer* qlayers, void* packed, adamk_stream stream);

/* Let `h` stream the packed weights another handle already bound (no repacking, no second copy in HBM).
 * Both handles must have been created from identical task tables.  Used by the batch lanes of
 * plugin.BatchLanes: B instances of the kernel on disjoint SM subsets, one sequence each, reading ONE
 * packed stream (the second reader of a stage hits L2).  `w` supplies embed / rope pointers as in
 * adamk_bind_weights (`layers` is not read). */
int adamk_share_weights(adamk_handle h, adamk_handle owner, const AdamkWeightPtrs* w);

/* Tensor parallelism only (tp_size > 1 at adamk_create; `desc` then holds the
 * rank's shard: n_q_heads, n_kv_heads, intermediate and vocab divided by
 * tp_size): base pointers of EVERY rank's workspace as seen from this GPU
 * (peer-mapped memory; own rank included, rank order).  The kernel stores its
 * partial O-proj / down-proj rows and its LM-head argmax into slot tp_rank of
 * each of them and sums its own slots in rank order; no collective library is
 * involved.  decode_step fails with ADAMK_E_STATE until this has been called. */
int adamk_bind_peers(adamk_handle h, void* const* peer_workspaces, int n_peers);

/* Workspace: the tagged activation vectors ({fp32 value, tag} words), split-KV
 * partial records, per-SM argmax partials and the step epoch.  Must be
 * initialised once with workspace_init (zeroes it and opens epoch 1). */
size_t adamk_workspace_bytes(adamk_handle h);
int adamk_workspace_init(adamk_handle h, void* workspace, adamk_stream stream);

/* KV cache geometry: each of k_cache / v_cache is bf16
 * [n_layers, max_batch, n_kv_heads, max_ctx, head_dim]. */
size_t adamk_kv_cache_bytes(adamk_handle h);

/* One decode step for `batch` sequences: ONE launch of the persistent kernel.
 * token_ids / positions / next_token_out are DEVICE int32[batch]; logits_out is
 * DEVICE fp32 [batch, vocab] or NULL.  Writes K/V of the new token at
 * positions[b] and the greedy next token.  With auto_advance != 0 the kernel
 * also stores next_token into token_ids and increments positions, so steps can
 * be enqueued back to back with no host round trip. */
int adamk_decode_step(adamk_handle h, int32_t* token_ids, int32_t* positions, int batch,
                      void* k_cache, void* v_cache, void* workspace,
                      float* logits_out, int32_t* next_token_out, int auto_advance,
                      adamk_stream stream);

/* The same step with HOST buffers, for a caller that feeds one token at a time (the serving engine's
 * decode hook): copies token_ids / positions (HOST int32[batch], pinned memory for the copies
 * to be asynchronous) into the device state, launches the step (auto_advance = 0), copies the greedy next token
 * into next_token_host (HOST int32[batch]) and waits for the stream.  One library call per token instead of
 * three copies, a launch and a synchronise issued from the host language.  A position outside [0, max_ctx) or a
 * token id outside the vocabulary is refused with ADAMK_E_INVALID before anything is copied or launched (on the
 * device the same input ends in a trap and a lost context: the device-resident loop must be bounded by its driver). */
int adamk_decode_step_host(adamk_handle h, const int32_t* token_ids_host, const int32_t* positions_host, int batch,
                           int32_t* token_ids, int32_t* positions,
                           void* k_cache, void* v_cache, void* workspace,
                           float* logits_out, int32_t* next_token_out, int32_t* next_token_host,
                           adamk_stream stream);

/* Poll the device-written status block (host-mapped); 0 = no error recorded.
 * Fills `info` (8 ints: code, sm, task, tag seen, tag expected, detail, thread, -) if not NULL. */
int adamk_device_status(adamk_handle h, int32_t* info);

/* Optional per-task timeline (the device analogue of the reference's
 * chrome_trace_events, /root/reference/pkg/src/mkplan/simulator.py:381-411):
 * when a device buffer of adamk_trace_bytes() is set, consumer thread 0 of every
 * CTA stores four %globaltimer stamps per task (start, dependency met, prologue
 * done, end).  NULL disables tracing. */
size_t adamk_trace_bytes(adamk_handle h);
int adamk_set_trace(adamk_handle h, void* trace_buf);

/* Standalone weight-streaming probe used by the measurement harness: runs only
 * the Loader/Consumer ring over the packed stream (no dependencies), to
 * separate HBM streaming efficiency from dependency stalls.  mode 1: Loader +
 * Consumer math; mode 2: Loader only (consumers release slots untouched);
 * mode 3: like 1 with the Loader re-reading an L2-resident window; mode 4:
 * Consumer math only (no Loader, no barriers).  `sink` is n_sms * 64 floats. */
int adamk_stream_probe(adamk_handle h, float* sink, int mode, adamk_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* ADAMK_H_ */
