// adamk.cu -- persistent, warp-specialised decode MegaKernel for sm_100a + its C ABI.
//
// One launch = one decode step of the whole model (every layer + LM head + argmax).
// grid = one CTA per SM; each CTA walks its static, program-ordered task list
// (paper_2605_11581_b200/task_table.py).  Roles follow the reference's role split
// (/root/reference/pkg/src/mkplan/planner.py:60-77):
//   Loader   : warp 0, one elected lane.  Streams the CTA's weight sub-tiles with
//              cp.async.bulk (TMA, SASS UBLKCP) into an n_stage-deep shared-memory
//              ring; never looks at activations, so it runs ahead across operator
//              and layer boundaries (the paper's "asynchronous prefetching and
//              logical decoupling") limited only by free ring slots.
//   Consumer : warps 1..C.  Wait on the operator's dependency counter, stage the
//              fp32 activation vector in shared memory (fusing RMSNorm), then GEMV
//              out of the ring with LDS.128 + FFMA and warp-shuffle reductions.
//   Storer   : the consumers' epilogue (bias / residual / SiLU*up / argmax) and the
//              release of the operator's global counter.
// Page states Empty -> Locked -> Ready (planner.py:84-94) = ring slot `empty`
// mbarrier phase -> TMA in flight -> `full` mbarrier phase.
// Inter-SM dependencies are monotonically increasing global counters whose target
// values are fixed in the task table ("path solidification").
//
// Numerical contract (shared with oracle/decode_ref.py): bf16 weights used exactly,
// fp32 activations and accumulation, bf16 KV cache, fp32 RoPE tables from the host.

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/adamk.h"

// ----------------------------------------------------------------------------------
// task table format (keep in sync with task_table.py)
// ----------------------------------------------------------------------------------
namespace {

constexpr int kMagic = 0x4B4D4441;
constexpr int kVersion = 1;
constexpr int kHeaderInts = 16;
constexpr int kTaskInts = 16;
constexpr int kChunk = 256;          // K elements per chunk
constexpr int kSmemMax = 232448;
constexpr int kSmemReserved = 1024;  // barriers + reduction scratch
constexpr int kMaxStages = 16;
constexpr int kAttnPBMax = 128;      // positions per attention block (8 per consumer warp)
constexpr int kAttnChunksMax = 128;  // split-KV units per (sequence, kv head)
constexpr int kGMax = 8;             // max q heads per kv head

enum TaskType { T_END = 0, T_QKV = 1, T_ATTN = 2, T_OPROJ = 3, T_GATEUP = 4, T_DOWN = 5, T_LMHEAD = 6 };
enum Ctr { CTR_A = 0, CTR_B = 1, CTR_C = 2, CTR_D = 3, CTR_E = 4, CTR_F = 5, CTR_HEAD0 = 6 };

struct Task {  // 64 bytes
  int type, layer, a, b, k, kchunks, rt, ktc, n_tiles, n_ktiles, w_off, n_stages, wait_ctr, wait_val, sig_ctr, aux;
};
static_assert(sizeof(Task) == kTaskInts * 4, "task record is 64 bytes");

// device error codes written to the host-mapped status block
enum DevErr { DE_NONE = 0, DE_WATCHDOG_CTR = 1, DE_WATCHDOG_FULL = 2, DE_WATCHDOG_EMPTY = 3, DE_BAD_POS = 4 };

struct KParams {
  // model
  int H, L, nq, nkv, D, I, V, G, q_dim, kv_dim, qkv_rows, max_ctx, batch;
  int has_bias, qk_norm;
  float eps;
  // schedule
  int C, n_stage, stage_bytes, attn_chunks, attn_min_chunk, scratch_bytes, n_lm_tasks, n_counters;
  int xs_floats;  // floats reserved for the staged activation vector; the merge weights follow it
  // task table
  const Task* tasks;
  const int* sm_begin;
  const unsigned* sm_stream;  // [n_sms + 1] packed-stream range of every SM (16-byte units)
  int pf_min_bytes, pf_max_bytes;  // L2 prefetch distance ahead of the ring: steady state / while stalled
  // weights
  const uint8_t* wpacked;   // tile-major bf16 weight streams
  const float* fparams;     // fp32 norm gains / biases
  int fp_layer_stride, fp_ln1, fp_ln2, fp_bias, fp_qn, fp_kn, fp_final;
  const __nv_bfloat16* embed;
  const float* rope_cos;
  const float* rope_sin;
  // per-step buffers
  __nv_bfloat16* kcache;
  __nv_bfloat16* vcache;
  float* h_a;
  float* h_b;
  float* qkv;
  float* attn;
  float* act;
  float* part;
  float* lm_val;
  int* lm_idx;
  unsigned* counters;
  float* logits;
  int* tokens;
  int* positions;
  int* next_tokens;
  int* status;  // host-mapped, 8 ints
  int auto_advance;
  int probe;    // 1 = stream probe: consumers skip dependencies and epilogues; 2 = also skip the math
  float* probe_sink;
  unsigned long long* trace;  // optional [n_tasks][8] globaltimer stamps (0 start, 1 dependency met, 2 prologue done, 7 end, 3-6 op specific)
};

// ----------------------------------------------------------------------------------
// PTX helpers
// ----------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint32_t mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok;
}
// TMA bulk copy global -> shared, completion on an mbarrier (SASS: UBLKCP)
__device__ __forceinline__ void tma_bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_bulk_g2s_hint(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void l2_prefetch_bulk(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_acqrel_add(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
// named barrier over the consumer warps only (barrier 0 is __syncthreads)
__device__ __forceinline__ void consumer_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}
__device__ __forceinline__ float4 lds128f(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint4 lds128u(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

constexpr long long kWatchdogCycles = 6000000000LL;  // ~3 s at 2 GHz; a step takes < 1 ms

__device__ __noinline__ void dev_fail(const KParams& p, int code, int task, int a, int b, int c) {
  volatile int* s = p.status;
  if (s) {
    s[1] = blockIdx.x; s[2] = task; s[3] = a; s[4] = b; s[5] = c; s[6] = threadIdx.x;
    __threadfence_system();
    s[0] = code;
    __threadfence_system();
  }
  __trap();
}

__device__ __forceinline__ uint32_t mbar_try_wait_hint(uint32_t bar, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity), "r"(ns)
      : "memory");
  return ok;
}
__device__ __noinline__ void mbar_wait_slow(const KParams& p, uint32_t bar, uint32_t parity, int code, int task) {
  const long long t0 = clock64();
  while (!mbar_try_wait_hint(bar, parity, 2000u)) {
    if (clock64() - t0 > kWatchdogCycles) dev_fail(p, code, task, (int)bar, (int)parity, 0);
  }
}
__device__ __forceinline__ void mbar_wait(const KParams& p, uint32_t bar, uint32_t parity, int code, int task) {
  if (!mbar_try_wait(bar, parity)) mbar_wait_slow(p, bar, parity, code, task);
}

// ----------------------------------------------------------------------------------
// shared-memory layout
// ----------------------------------------------------------------------------------
struct SmemHdr {
  unsigned long long full[kMaxStages];
  unsigned long long empty[kMaxStages];
  float red[64];
  int misc[32];
};
static_assert(sizeof(SmemHdr) <= kSmemReserved, "smem header too large");

struct ConsumerCtx {
  uint32_t slot;      // ring slot of the next stage to drain
  uint32_t ph;        // its mbarrier phase parity
  int cw;             // consumer warp index 0..C-1
  int lane;
  int ctid;           // thread index among consumers
  int nct;            // number of consumer threads
  float rs;           // RMSNorm scale of the current GEMV's input (applied in the epilogue), else 1
  float best_val;     // LM-head running argmax (lane 0 of each warp)
  int best_idx;
};

__device__ __forceinline__ void stamp(const KParams& p, const ConsumerCtx& c, int task, int k) {
  if (p.trace && c.ctid == 0) p.trace[(size_t)task * 8 + k] = globaltimer_ns();
}

// ----------------------------------------------------------------------------------
// dependency wait / signal
// ----------------------------------------------------------------------------------
__device__ __noinline__ void poll_counter_slow(const KParams& p, const unsigned* addr, int val, int ctr, int task) {
  const long long t0 = clock64();
  unsigned seen;
  while ((seen = ld_relaxed_u32(addr)) < (unsigned)val) {
    if (clock64() - t0 > kWatchdogCycles) dev_fail(p, DE_WATCHDOG_CTR, task, ctr, (int)seen, val);
  }
}
__device__ __forceinline__ void wait_counter(const KParams& p, const ConsumerCtx& c, int ctr, int val, int task) {
  if (ctr >= 0 && !p.probe) {
    if (c.ctid == 0) {
      const unsigned* addr = p.counters + ctr;
      if (ld_relaxed_u32(addr) < (unsigned)val) poll_counter_slow(p, addr, val, ctr, task);
      fence_acq_rel_gpu();  // one acquire for the whole poll loop (no per-poll L1 invalidate)
    }
  }
  consumer_sync(c.nct);
}

// all consumer threads have finished their global writes for this task
__device__ __forceinline__ void signal_counter(const KParams& p, const ConsumerCtx& c, int ctr) {
  consumer_sync(c.nct);
  if (c.ctid == 0 && ctr >= 0 && !p.probe) red_release_add(p.counters + ctr, 1u);
}

// Split-KV geometry of one decode step, shared by the Loader (which streams the K/V
// blocks of a unit through the ring) and the Consumers (which drain them).
struct AttnGeom {
  int CL, n_active, t0, n, PB, nblk;
};
__device__ __forceinline__ AttnGeom attn_geometry(const KParams& p, int pos, int slot) {
  AttnGeom g;
  const int ctx = pos + 1;
  g.CL = max(p.attn_min_chunk, (ctx + p.attn_chunks - 1) / p.attn_chunks);
  g.CL = (g.CL + 7) & ~7;
  g.n_active = (ctx + g.CL - 1) / g.CL;
  g.t0 = slot * g.CL;
  g.n = min(ctx, g.t0 + g.CL) - g.t0;           // <= 0 for inactive slots
  g.PB = min(64, (p.stage_bytes / (p.D * 2)) & ~7);  // positions per ring stage
  g.nblk = g.n > 0 ? (g.n + g.PB - 1) / g.PB : 0;
  return g;
}

// Flash-decoding merge of the split-KV partial records, done by every consumer of the
// attention output (O-projection prologue): xs[h*D + d] = sum_s w[h][s] * o_s[h][d] with
// w = exp(m_s - M) / sum_s l_s exp(m_s - M).  `wts` holds n_q_heads * n_active floats.
// All global loads of a phase are independent and issued back to back (one L2 round trip).
__device__ __forceinline__ void attn_merge_into(const KParams& p, const ConsumerCtx& c, int pos, float* xs, int kpad,
                                                float* wts) {
  const AttnGeom ge = attn_geometry(p, pos, 0);
  const int na = ge.n_active, D = p.D, G = p.G, PS = D + 4;
  const float* part = p.part;  // [nkv][attn_chunks][G][PS]   (batch 1)
  // phase 1: (m, l) of every (head, chunk) -> shared memory
  for (int i = c.ctid; i < p.nq * na; i += c.nct) {
    const int h = i / na, s2 = i - h * na;
    const int kvh = h / G, g = h - kvh * G;
    const float2 ml = __ldcg(reinterpret_cast<const float2*>(part + (((size_t)kvh * p.attn_chunks + s2) * G + g) * PS + D));
    wts[i] = ml.x;
    wts[p.nq * na + i] = ml.y;
  }
  consumer_sync(c.nct);
  // phase 2: normalised weights, one warp per head, lanes over chunks
  for (int h = c.cw; h < p.nq; h += p.C) {
    float M = -INFINITY;
    for (int s2 = c.lane; s2 < na; s2 += 32) M = fmaxf(M, wts[h * na + s2]);
    M = warp_max(M);
    float L = 0.f;
    for (int s2 = c.lane; s2 < na; s2 += 32) {
      const float wgt = expf(wts[h * na + s2] - M);
      L = fmaf(wts[p.nq * na + h * na + s2], wgt, L);
      wts[h * na + s2] = wgt;
    }
    L = warp_sum(L);
    const float inv = 1.0f / L;
    for (int s2 = c.lane; s2 < na; s2 += 32) wts[h * na + s2] *= inv;
  }
  consumer_sync(c.nct);
  // phase 3: weighted sum, four output dims per thread, chunks batched by four
  const int q4 = p.q_dim >> 2;
  for (int i = c.ctid; i < (kpad >> 2); i += c.nct) {
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < q4) {
      const int h = (i * 4) / D, d = i * 4 - h * D;
      const int kvh = h / G, g = h - kvh * G;
      const float* rec = part + ((size_t)kvh * p.attn_chunks * G + g) * PS + d;
      const size_t cs = (size_t)G * PS;
      const float* w = wts + h * na;
      for (int s0 = 0; s0 < na; s0 += 8) {  // eight independent 16-byte loads in flight per thread
        float4 a[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          a[u] = (s0 + u < na) ? __ldcg(reinterpret_cast<const float4*>(rec + (s0 + u) * cs)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const float wu = (s0 + u < na) ? w[s0 + u] : 0.f;
          x.x = fmaf(a[u].x, wu, x.x); x.y = fmaf(a[u].y, wu, x.y); x.z = fmaf(a[u].z, wu, x.z); x.w = fmaf(a[u].w, wu, x.w);
        }
      }
    }
    reinterpret_cast<float4*>(xs)[i] = x;
  }
  consumer_sync(c.nct);
}

// ----------------------------------------------------------------------------------
// GEMV task
// ----------------------------------------------------------------------------------
__device__ __forceinline__ float silu(float g) { return g / (1.0f + expf(-g)); }

// fp32 hidden-state element of the layer input: layer 0 reads the embedding row
__device__ __forceinline__ float4 load_h4(const KParams& p, int layer, bool mid, int tok, int i4) {
  if (mid) return __ldcg(reinterpret_cast<const float4*>(p.h_b) + i4);
  if (layer == 0) {
    const uint2 raw = __ldg(reinterpret_cast<const uint2*>(p.embed + (size_t)tok * p.H) + i4);
    return make_float4(bf_lo(raw.x), bf_hi(raw.x), bf_lo(raw.y), bf_hi(raw.y));
  }
  return __ldcg(reinterpret_cast<const float4*>(p.h_a) + i4);
}
__device__ __forceinline__ float load_h1(const KParams& p, int layer, int tok, int i) {
  if (layer == 0) return __bfloat162float(p.embed[(size_t)tok * p.H + i]);
  return __ldcg(p.h_a + i);
}

constexpr int kPreG = 4;  // float4 gain vectors per thread preloaded before the dependency wait

__device__ __forceinline__ const float* gemv_gain(const KParams& p, const Task& t) {
  if (t.type == T_LMHEAD) return p.fparams + p.fp_final;
  return p.fparams + (size_t)t.layer * p.fp_layer_stride + (t.type == T_GATEUP ? p.fp_ln2 : p.fp_ln1);
}

// Stage the activation vector of a GEMV in shared memory (fp32, zero padded to kpad).
__device__ __forceinline__ void gemv_prologue(const KParams& p, ConsumerCtx& c, const Task& t, float* xs,
                                              SmemHdr* hdr, int tok, int pos, const float4 (&g4)[kPreG]) {
  const int kpad = t.kchunks * kChunk;
  const int type = t.type;
  c.rs = 1.0f;
  if (type == T_OPROJ) {  // input = merged split-KV attention output
    attn_merge_into(p, c, pos, xs, kpad, xs + p.xs_floats);
    return;
  }
  if (type == T_DOWN) {
    const int k4 = t.k >> 2, kp4 = kpad >> 2;
    for (int i0 = c.ctid; i0 < kp4; i0 += 4 * c.nct) {  // four independent loads in flight per thread
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * c.nct;
        v[u] = (i < k4) ? __ldcg(reinterpret_cast<const float4*>(p.act) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * c.nct;
        if (i < kp4) reinterpret_cast<float4*>(xs)[i] = v[u];
      }
    }
    consumer_sync(c.nct);
    return;
  }
  // RMSNorm-fused prologues: QKV (ln1 over layer input), GATEUP (ln2 over h_mid), LMHEAD (final norm).
  // Single pass: stage h * gain, accumulate sum(h^2); the scalar rsqrt(mean + eps) commutes with
  // the dot products and is applied to each output row in the epilogue.
  const bool mid = (type == T_GATEUP);
  const int layer = (type == T_LMHEAD) ? p.L : t.layer;  // LM head reads h_a (layer index L > 0)
  const float4* gain4 = reinterpret_cast<const float4*>(gemv_gain(p, t));
  const int h4 = p.H >> 2, kp4 = kpad >> 2;
  float ss = 0.f;
  auto stage = [&](int i, const float4& g) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < h4) {
      v = load_h4(p, layer, mid, tok, i);
      ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
      v.x *= g.x; v.y *= g.y; v.z *= g.z; v.w *= g.w;
    }
    reinterpret_cast<float4*>(xs)[i] = v;
  };
#pragma unroll
  for (int k = 0; k < kPreG; ++k) {
    const int i = c.ctid + k * c.nct;
    if (i < kp4) stage(i, g4[k]);
  }
  for (int i = c.ctid + kPreG * c.nct; i < kp4; i += c.nct)
    stage(i, i < h4 ? __ldg(gain4 + i) : make_float4(0.f, 0.f, 0.f, 0.f));
  ss = warp_sum(ss);
  if (c.lane == 0) hdr->red[c.cw] = ss;
  consumer_sync(c.nct);
  float tot = 0.f;
  for (int w = 0; w < p.C; ++w) tot += hdr->red[w];
  c.rs = rsqrtf(tot / (float)p.H + p.eps);
}

// Epilogue operand of one output row that is known before the dot product finishes (bias,
// residual input): loaded ahead of the K loop so its latency hides behind the stream.
__device__ __forceinline__ float load_eop(const KParams& p, const Task& t, int vrow, int tok) {
  switch (t.type) {
    case T_QKV: return p.has_bias ? __ldg(p.fparams + (size_t)t.layer * p.fp_layer_stride + p.fp_bias + vrow) : 0.f;
    case T_OPROJ: return load_h1(p, t.layer, tok, vrow);
    case T_DOWN: return __ldcg(p.h_b + vrow);
    default: return 0.f;
  }
}

__device__ __forceinline__ void gemv_epilogue(const KParams& p, ConsumerCtx& c, const Task& t, int vrow, float v,
                                              float v_pair, float eop) {
  switch (t.type) {
    case T_QKV: p.qkv[vrow] = v + eop; break;
    case T_OPROJ: p.h_b[vrow] = eop + v; break;
    case T_GATEUP: p.act[vrow >> 1] = silu(v) * v_pair; break;  // vrow even = gate, pair = up
    case T_DOWN: p.h_a[vrow] = eop + v; break;
    case T_LMHEAD: {
      if (p.logits) p.logits[vrow] = v;
      if (v > c.best_val) { c.best_val = v; c.best_idx = vrow; }  // rows ascend: first max wins ties
    } break;
    default: break;
  }
}

// One 256-element K chunk of RW rows: acc[i] += w[i][chunk] . x[chunk].  bf16 -> fp32 is a
// shift / mask per element; the products go through the packed FFMA2 pipe (sm_100).
template <int RW, bool ALL>
__device__ __forceinline__ void gemv_chunk(uint32_t waddr, uint32_t row_stride, uint32_t xaddr, int nrows,
                                           float2 (&accA)[RW], float2 (&accB)[RW]) {
  const float4 xa = lds128f(xaddr);
  const float4 xb = lds128f(xaddr + 512);
#pragma unroll
  for (int i = 0; i < RW; ++i) {
    if (ALL || i < nrows) {
      const uint4 w = lds128u(waddr + i * row_stride);
      accA[i] = __ffma2_rn(make_float2(bf_lo(w.x), bf_hi(w.x)), make_float2(xa.x, xa.y), accA[i]);
      accB[i] = __ffma2_rn(make_float2(bf_lo(w.y), bf_hi(w.y)), make_float2(xa.z, xa.w), accB[i]);
      accA[i] = __ffma2_rn(make_float2(bf_lo(w.z), bf_hi(w.z)), make_float2(xb.x, xb.y), accA[i]);
      accB[i] = __ffma2_rn(make_float2(bf_lo(w.w), bf_hi(w.w)), make_float2(xb.z, xb.w), accB[i]);
    }
  }
}

template <int RW>
__device__ __forceinline__ void gemv_tiles(const KParams& p, ConsumerCtx& c, const Task& t, int task_idx,
                                           const float* xs, SmemHdr* hdr, uint8_t* ring, int tok,
                                           const float (&eop0)[4]) {
  const uint32_t xs_addr = smem_u32(xs) + c.lane * 16;
  const uint32_t ring_addr = smem_u32(ring) + c.lane * 16;
  const uint32_t full0 = smem_u32(&hdr->full[0]);
  const uint32_t empty0 = smem_u32(&hdr->empty[0]);
  const int r0 = c.cw * RW;
  const uint32_t n_stage = (uint32_t)p.n_stage;
  for (int tile = 0; tile < t.n_tiles; ++tile) {
    const int rows = min(t.rt, t.b - tile * t.rt);
    const int nrows = min(RW, rows - r0);  // rows of this tile owned by this warp (<= 0: none)
    float2 accA[RW], accB[RW];
    float eop[RW];
#pragma unroll
    for (int i = 0; i < RW; ++i) {
      accA[i] = make_float2(0.f, 0.f);
      accB[i] = make_float2(0.f, 0.f);
      eop[i] = eop0[i];
      if (tile > 0 && c.lane == 0 && i < nrows && !p.probe) eop[i] = load_eop(p, t, t.a + tile * t.rt + r0 + i, tok);
    }
    int kc0 = 0;
    for (int kt = 0; kt < t.n_ktiles; ++kt, kc0 += t.ktc) {
      const int chunks = min(t.ktc, t.kchunks - kc0);
      mbar_wait(p, full0 + c.slot * 8, c.ph, DE_WATCHDOG_FULL, task_idx);
      if (nrows > 0 && p.probe != 2) {
        const uint32_t row_stride = (uint32_t)chunks * 512u;
        uint32_t wa = ring_addr + c.slot * (uint32_t)p.stage_bytes + (uint32_t)r0 * row_stride;
        uint32_t xa = xs_addr + (uint32_t)kc0 * (kChunk * 4);
        if (nrows == RW) {
#pragma unroll 2
          for (int ch = 0; ch < chunks; ++ch, wa += 512, xa += kChunk * 4)
            gemv_chunk<RW, true>(wa, row_stride, xa, RW, accA, accB);
        } else {
          for (int ch = 0; ch < chunks; ++ch, wa += 512, xa += kChunk * 4)
            gemv_chunk<RW, false>(wa, row_stride, xa, nrows, accA, accB);
        }
      }
      __syncwarp();
      if (c.lane == 0) mbar_arrive(empty0 + c.slot * 8);
      if (++c.slot == n_stage) { c.slot = 0; c.ph ^= 1u; }
    }
    if (p.probe) {
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < RW; ++i) s += accA[i].x + accA[i].y + accB[i].x + accB[i].y;
      if (s == 1.2345678e-30f) p.probe_sink[blockIdx.x] = s;  // keep the math alive
      continue;
    }
    if (nrows > 0) {
      float v[RW];
#pragma unroll
      for (int i = 0; i < RW; ++i) v[i] = c.rs * warp_sum((accA[i].x + accB[i].x) + (accA[i].y + accB[i].y));
      if (c.lane == 0) {
        const int vrow0 = t.a + tile * t.rt + r0;
        if (t.type == T_GATEUP) {
#pragma unroll
          for (int i = 0; i < RW; i += 2)
            if (i < nrows) gemv_epilogue(p, c, t, vrow0 + i, v[i], v[(i + 1) % RW], 0.f);
        } else {
#pragma unroll
          for (int i = 0; i < RW; ++i)
            if (i < nrows) gemv_epilogue(p, c, t, vrow0 + i, v[i], 0.f, eop[i]);
        }
      }
    }
  }
}

__device__ __forceinline__ void lm_finish(const KParams& p, ConsumerCtx& c, SmemHdr* hdr) {
  // per-warp best -> CTA best -> global partial -> last CTA reduces, publishes, resets counters
  float bv = __shfl_sync(0xffffffffu, c.best_val, 0);
  int bi = __shfl_sync(0xffffffffu, c.best_idx, 0);
  if (c.lane == 0) { hdr->red[c.cw] = bv; hdr->misc[c.cw] = bi; }
  consumer_sync(c.nct);
  if (c.ctid == 0) {
    float best = hdr->red[0];
    int idx = hdr->misc[0];
    for (int w = 1; w < p.C; ++w) {
      const float v = hdr->red[w];
      const int i = hdr->misc[w];
      if (v > best || (v == best && i < idx)) { best = v; idx = i; }
    }
    p.lm_val[blockIdx.x] = best;
    p.lm_idx[blockIdx.x] = idx;
    __threadfence();
    const unsigned old = atom_acqrel_add(p.counters + CTR_F, 1u);
    hdr->misc[31] = (old == (unsigned)(p.n_lm_tasks - 1)) ? 1 : 0;
  }
  consumer_sync(c.nct);
  if (hdr->misc[31] && c.cw == 0) {
    __threadfence();
    float best = -INFINITY;
    int idx = 0x7fffffff;
    for (int s = c.lane; s < (int)gridDim.x; s += 32) {
      const int i = __ldcg(p.lm_idx + s);
      const float v = __ldcg(p.lm_val + s);
      if (i >= 0 && (v > best || (v == best && i < idx))) { best = v; idx = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      if (ov > best || (ov == best && oi < idx)) { best = ov; idx = oi; }
    }
    if (c.lane == 0) {
      p.next_tokens[0] = idx;
      if (p.auto_advance) { p.tokens[0] = idx; p.positions[0] = p.positions[0] + 1; }
    }
    // every CTA has passed its last wait: reset the dependency counters for the next launch
    for (int i = c.lane; i < p.n_counters; i += 32) p.counters[i] = 0u;
  }
}

__device__ __forceinline__ void run_gemv(const KParams& p, ConsumerCtx& c, const Task& t, int task_idx, float* xs,
                                         SmemHdr* hdr, uint8_t* ring, int tok, int pos) {
  stamp(p, c, task_idx, 0);
  const int rw = t.rt / p.C;
  // ---- before the dependency wait: everything that does not depend on the awaited data ----
  // (per-layer vectors are always DRAM misses under the weight stream: ~1 us each if loaded late)
  float4 g4[kPreG];
  float eop0[4] = {0.f, 0.f, 0.f, 0.f};
  if (!p.probe) {
    if (t.type == T_QKV || t.type == T_GATEUP || t.type == T_LMHEAD) {
      const float4* gain4 = reinterpret_cast<const float4*>(gemv_gain(p, t));
#pragma unroll
      for (int k = 0; k < kPreG; ++k) {
        const int i = c.ctid + k * c.nct;
        g4[k] = (i < (p.H >> 2)) ? __ldg(gain4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    if (c.lane == 0 && t.type != T_DOWN) {  // DOWN's residual (h_mid) is preloaded after its own dependency
      const int r0 = c.cw * rw, rows0 = min(t.rt, t.b);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i < rw && r0 + i < rows0) eop0[i] = load_eop(p, t, t.a + r0 + i, tok);
    }
  }
  wait_counter(p, c, t.wait_ctr, t.wait_val, task_idx);
  stamp(p, c, task_idx, 1);
  if (!p.probe) {
    if (c.lane == 0 && t.type == T_DOWN) {
      const int r0 = c.cw * rw, rows0 = min(t.rt, t.b);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i < rw && r0 + i < rows0) eop0[i] = load_eop(p, t, t.a + r0 + i, tok);
    }
    gemv_prologue(p, c, t, xs, hdr, tok, pos, g4);
  }
  stamp(p, c, task_idx, 2);
  if (rw == 2) gemv_tiles<2>(p, c, t, task_idx, xs, hdr, ring, tok, eop0);
  else gemv_tiles<4>(p, c, t, task_idx, xs, hdr, ring, tok, eop0);
  if (p.probe) return;
  stamp(p, c, task_idx, 3);
  if (t.type == T_LMHEAD) lm_finish(p, c, hdr);
  else signal_counter(p, c, t.sig_ctr);
  stamp(p, c, task_idx, 7);
}

// Per-lane operands of rope_norm_head that do not depend on this step's projections:
// loaded BEFORE the dependency wait so their DRAM latency is off the critical path
// (small per-layer vectors never survive in L2 under the weight stream).
template <int D>
struct HeadParams {
  float gq[D / 32], gk[D / 32], cs[D / 64], sn[D / 64];
};
template <int D>
__device__ __forceinline__ HeadParams<D> load_head_params(const KParams& p, const float* lay_fp, int pos, int lane) {
  HeadParams<D> hp;
#pragma unroll
  for (int j = 0; j < D / 32; ++j) {
    hp.gq[j] = p.qk_norm ? __ldg(lay_fp + p.fp_qn + lane + 32 * j) : 1.0f;
    hp.gk[j] = p.qk_norm ? __ldg(lay_fp + p.fp_kn + lane + 32 * j) : 1.0f;
  }
#pragma unroll
  for (int j = 0; j < D / 64; ++j) {
    hp.cs[j] = __ldg(p.rope_cos + (size_t)pos * (D / 2) + lane + 32 * j);
    hp.sn[j] = __ldg(p.rope_sin + (size_t)pos * (D / 2) + lane + 32 * j);
  }
  return hp;
}

// one warp, one head: optional RMSNorm over D, rotate-half RoPE, scale
// PADL > 0: the output is laid out in segments of PADL floats separated by 4 floats of padding
// (bank-conflict-free reads by the score step); PADL = 0: dense.
template <int D, int PADL>
__device__ __forceinline__ void rope_norm_head(const KParams& p, const float* raw, const float (&gain)[D / 32],
                                               const HeadParams<D>& hp, float scale, int lane, float* out) {
  auto at = [](int d) { return PADL > 0 ? d + (d / (PADL > 0 ? PADL : 1)) * 4 : d; };
  constexpr int PER = D / 32;  // 4 (D=128) or 2 (D=64): elements lane, lane+32, ...
  constexpr int HALF = D / 2;
  float v[PER];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < PER; ++j) { v[j] = __ldcg(raw + lane + 32 * j); ss += v[j] * v[j]; }
  if (p.qk_norm) {
    ss = warp_sum(ss);
    const float rs = rsqrtf(ss / (float)D + p.eps);
#pragma unroll
    for (int j = 0; j < PER; ++j) v[j] = v[j] * rs * gain[j];
  }
#pragma unroll
  for (int j = 0; j < PER / 2; ++j) {
    const int d1 = lane + 32 * j;  // < HALF
    const float x1 = v[j], x2 = v[j + PER / 2];
    out[at(d1)] = (x1 * hp.cs[j] - x2 * hp.sn[j]) * scale;
    out[at(d1 + HALF)] = (x2 * hp.cs[j] + x1 * hp.sn[j]) * scale;
  }
}

// Layout of the attention scratch (floats); must match task_table.scratch_bytes / adamk_create.
//   qs[G][D] | sc[8][kAttnPBMax] | rsc[C][8] | prob[8][kAttnPBMax] | red[C][G][D] | lw[C][8] | mw[C][8] | knew[D] | vnew[D]
//
// The K and V rows of a unit's context chunk arrive through the weight ring (the paper's
// "KV-cache loads advanced into the pipeline window"): per block of PB positions
// one K stage and one V stage, issued by the Loader long before the QKV projections of this
// layer are done.  The row of the new token is patched into the staged copy.  Every unit
// publishes a partial record (o[D], m, l) per q head; the flash-decoding merge of the records
// is done by the consumers of the attention output (the O-projection prologue), so no unit
// waits for another.
template <int D, int PPW>
__device__ __forceinline__ void run_attn(const KParams& p, ConsumerCtx& c, const Task& t, int task_idx, float* scratch,
                                         SmemHdr* hdr, uint8_t* ring, int pos) {
  constexpr int DPL = D / 32;  // V / output elements per lane (lanes split the head dim)
  const int G = p.G;
  const int kvh = t.a, slot = t.b, bidx = t.aux;
  if (p.probe) return;
  const AttnGeom ge = attn_geometry(p, pos, slot);
  if (slot >= ge.n_active) {  // no context for this slot at this length: only keep the counter target static
    signal_counter(p, c, CTR_C);
    return;
  }
  stamp(p, c, task_idx, 0);
  const int n = ge.n, t0 = ge.t0, PB = ge.PB, nblk = ge.nblk;
  const bool owns_new = (slot == ge.n_active - 1);  // this chunk contains position `pos`

  // compile-time lane mapping of the score step (see below) -- needed here for the padded q layout
  constexpr int GS = PPW < 8 ? PPW : 8, LPP = 32 / GS, DL = D / LPP;
  constexpr int QP = D + LPP * 4;           // padded q row: LPP segments of DL floats, 4 floats apart
  constexpr int SR = kAttnPBMax + 4;        // padded score / probability row
  float* qs = scratch;                      // [G][QP]
  float* sc = qs + kGMax * (128 + 8 * 4);   // [kGMax][SR]   (q region sized for the largest QP)
  float* rsc = sc + kGMax * SR;             // per-warp rescale factors [C][kGMax]
  float* prob = rsc + p.C * kGMax;          // probabilities [kGMax][SR] (scores stay intact: other warps still read them)
  float* red = prob + kGMax * SR;
  float* lw = red + p.C * G * D;
  float* mw = lw + p.C * kGMax;
  float* knew = mw + p.C * kGMax;
  float* vnew = knew + D;

  const float* qkv = p.qkv + (size_t)bidx * p.qkv_rows;
  const float* lay_fp = p.fparams + (size_t)t.layer * p.fp_layer_stride;
  const float scale = rsqrtf((float)D);
  const size_t head_base = ((size_t)(t.layer * p.batch + bidx) * p.nkv + kvh) * (size_t)p.max_ctx * D;
  __nv_bfloat16* Kc = p.kcache + head_base;
  __nv_bfloat16* Vc = p.vcache + head_base;
  const uint32_t ring_addr = smem_u32(ring);
  const uint32_t full0 = smem_u32(&hdr->full[0]);
  const uint32_t empty0 = smem_u32(&hdr->empty[0]);
  const uint32_t n_stage = (uint32_t)p.n_stage;

  const HeadParams<D> hp = load_head_params<D>(p, lay_fp, pos, c.lane);  // before the wait
  wait_counter(p, c, t.wait_ctr, t.wait_val, task_idx);
  stamp(p, c, task_idx, 1);

  // q heads of this group: (norm) + RoPE + 1/sqrt(D); the owner of `pos` also appends K/V
  for (int g = c.cw; g < G; g += p.C)
    rope_norm_head<D, DL>(p, qkv + (size_t)(kvh * G + g) * D, hp.gq, hp, scale, c.lane, qs + g * QP);
  if (owns_new) {
    const int wk = G % p.C, wv = (G + 1) % p.C;  // warps with the least q work
    if (c.cw == wk) {
      rope_norm_head<D, 0>(p, qkv + p.q_dim + (size_t)kvh * D, hp.gk, hp, 1.0f, c.lane, knew);
      __syncwarp();
      for (int d = c.lane; d < D; d += 32) Kc[(size_t)pos * D + d] = __float2bfloat16_rn(knew[d]);
    }
    if (c.cw == wv) {
      const float* vraw = qkv + p.q_dim + p.kv_dim + (size_t)kvh * D;
      for (int d = c.lane; d < D; d += 32) {
        const float v = __ldcg(vraw + d);
        vnew[d] = v;
        Vc[(size_t)pos * D + d] = __float2bfloat16_rn(v);
      }
    }
  }
  consumer_sync(c.nct);
  stamp(p, c, task_idx, 2);

  // Per-warp running softmax state lives in shared memory (red = unnormalised output, mw = running
  // max, lw = running sum) and every loop over heads is a plain runtime loop: this path runs once
  // per layer on a few SMs, so its instruction footprint -- not its FLOPs -- is what costs time.
  for (int g = 0; g < G; ++g) {
#pragma unroll
    for (int e = 0; e < DPL; ++e) red[(c.cw * G + g) * D + c.lane * DPL + e] = 0.f;
    if (c.lane == 0) { mw[c.cw * kGMax + g] = -INFINITY; lw[c.cw * kGMax + g] = 0.f; }
  }
  __syncwarp();

  auto lds_row = [&](uint32_t base, int tl, float (&out)[DPL]) {  // one bf16 row, DPL elements per lane
    if constexpr (DPL == 4) {
      uint2 raw;
      asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(raw.x), "=r"(raw.y) : "r"(base + (uint32_t)(tl * D + c.lane * 4) * 2u));
      out[0] = bf_lo(raw.x); out[1] = bf_hi(raw.x); out[2] = bf_lo(raw.y); out[3] = bf_hi(raw.y);
    } else {
      uint32_t raw;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(raw) : "r"(base + (uint32_t)(tl * D + c.lane * 2) * 2u));
      out[0] = bf_lo(raw); out[1] = bf_hi(raw);
    }
  };

  // Lane mapping of the score step: the warp's PPW positions are handled GS = min(PPW, 8) at a
  // time by LPP = 32 / GS lanes each; a lane owns DL = D / LPP contiguous dims, so one dot product
  // needs log2(LPP) shuffle steps and all GS positions reduce in parallel.  All compile-time.
  const int lsub = c.lane % LPP, lpos = c.lane / LPP;
  // Lane mapping of the softmax bookkeeping: lane -> (head hg = lane % 8, part hpart = lane / 8)
  const int hg = c.lane & 7, hpart = c.lane >> 3;

  for (int blk = 0; blk < nblk; ++blk) {
    const bool patch = owns_new && blk == nblk - 1;
    const int new_row = (pos - t0) - blk * PB;  // row of the new token inside this block (if patch)
    const int nvalid = min(PPW, n - blk * PB - c.cw * PPW);  // valid positions of this warp in this block (may be <= 0)
    // ---------------- K stage: scores of this warp's PPW positions ----------------
    mbar_wait(p, full0 + c.slot * 8, c.ph, DE_WATCHDOG_FULL, task_idx);
    if (blk == 0) stamp(p, c, task_idx, 5);
    const uint32_t kb = ring_addr + c.slot * (uint32_t)p.stage_bytes;
    if (patch) {  // the staged copy predates this step's K row: overwrite it (bf16, as the cache holds it)
      for (int d = c.ctid; d < D; d += c.nct) {
        const unsigned short bits = __bfloat16_as_ushort(__float2bfloat16_rn(knew[d]));
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(kb + (uint32_t)(new_row * D + d) * 2u), "h"(bits) : "memory");
      }
      consumer_sync(c.nct);
    }
#pragma unroll
    for (int j0 = 0; j0 < PPW; j0 += GS) {
      const int j = j0 + lpos;
      const int tl = c.cw * PPW + j;
      const uint32_t krow = kb + (uint32_t)(tl * D + lsub * DL) * 2u;
      float kf[DL];  // this lane's slice of the K row, converted once and reused for every head
#pragma unroll
      for (int e = 0; e < DL; e += 8) {
        const uint4 raw = lds128u(krow + e * 2);
        kf[e + 0] = bf_lo(raw.x); kf[e + 1] = bf_hi(raw.x); kf[e + 2] = bf_lo(raw.y); kf[e + 3] = bf_hi(raw.y);
        kf[e + 4] = bf_lo(raw.z); kf[e + 5] = bf_hi(raw.z); kf[e + 6] = bf_lo(raw.w); kf[e + 7] = bf_hi(raw.w);
      }
#pragma unroll 2
      for (int g = 0; g < G; ++g) {
        const float4* qp = reinterpret_cast<const float4*>(qs + g * QP + lsub * (DL + 4));
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
        for (int e = 0; e < DL / 4; ++e) {
          const float4 q4 = qp[e];
          s0 = fmaf(q4.x, kf[e * 4 + 0], s0); s1 = fmaf(q4.y, kf[e * 4 + 1], s1);
          s2 = fmaf(q4.z, kf[e * 4 + 2], s2); s3 = fmaf(q4.w, kf[e * 4 + 3], s3);
        }
        float sdot = (s0 + s1) + (s2 + s3);
#pragma unroll
        for (int o = LPP >> 1; o > 0; o >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, o);
        if (lsub == 0) sc[g * SR + tl] = (j < nvalid) ? sdot : -INFINITY;
      }
    }
    __syncwarp();
    if (c.lane == 0) mbar_arrive(empty0 + c.slot * 8);
    if (++c.slot == n_stage) { c.slot = 0; c.ph ^= 1u; }
    consumer_sync(c.nct);
    if (blk == 0) stamp(p, c, task_idx, 3);
    // ---------------- online softmax bookkeeping for all heads at once ----------------
    // block max of head hg over the quarter hpart of the block, then across the 4 parts
    float resc_l = 0.f;
    {
      float mb = -INFINITY;
      if (hg < G)
        for (int i = hpart; i < PB; i += 4) mb = fmaxf(mb, sc[hg * SR + i]);  // conflict-free: bank = 4 hg + hpart + 4k
      mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 8));
      mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 16));
      const float m_old = (hg < G) ? mw[c.cw * kGMax + hg] : 0.f;
      const float m_new = fmaxf(m_old, mb);
      resc_l = expf(m_old - m_new);  // exp(-inf) = 0 on the first block
      // probabilities of this warp's own positions (entries written by this warp only): part hpart
      // covers positions hpart, hpart + 4, ... of the warp
      float lsum = 0.f;
      if (hg < G) {
        for (int j = hpart; j < PPW; j += 4) {
          const int idx = hg * SR + c.cw * PPW + j;
          const float pj = (j < nvalid) ? expf(sc[idx] - m_new) : 0.f;
          prob[idx] = pj;
          lsum += pj;
        }
      }
      lsum += __shfl_xor_sync(0xffffffffu, lsum, 8);
      lsum += __shfl_xor_sync(0xffffffffu, lsum, 16);
      __syncwarp();
      if (hpart == 0 && hg < G) {
        mw[c.cw * kGMax + hg] = m_new;
        lw[c.cw * kGMax + hg] = lw[c.cw * kGMax + hg] * resc_l + lsum;
        rsc[c.cw * kGMax + hg] = resc_l;  // per-warp rescale factors for the P.V step
      }
      __syncwarp();
    }
    // ---------------- V stage: P.V over this warp's positions, one head at a time ----------------
    mbar_wait(p, full0 + c.slot * 8, c.ph, DE_WATCHDOG_FULL, task_idx);
    if (blk == 0) stamp(p, c, task_idx, 6);
    const uint32_t vb = ring_addr + c.slot * (uint32_t)p.stage_bytes;
    if (patch) {
      for (int d = c.ctid; d < D; d += c.nct) {
        const unsigned short bits = __bfloat16_as_ushort(__float2bfloat16_rn(vnew[d]));
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(vb + (uint32_t)(new_row * D + d) * 2u), "h"(bits) : "memory");
      }
      consumer_sync(c.nct);
    }
#pragma unroll 1
    for (int g = 0; g < G; ++g) {
      const float resc = rsc[c.cw * kGMax + g];
      float acc[DPL];
      float* ra = red + (c.cw * G + g) * D + c.lane * DPL;
#pragma unroll
      for (int e = 0; e < DPL; ++e) acc[e] = ra[e] * resc;
      const float* pr = prob + g * SR + c.cw * PPW;
#pragma unroll 4
      for (int j = 0; j < nvalid; ++j) {
        float vf[DPL];
        lds_row(vb, c.cw * PPW + j, vf);
        const float pg = pr[j];
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc[e] = fmaf(pg, vf[e], acc[e]);
      }
#pragma unroll
      for (int e = 0; e < DPL; ++e) ra[e] = acc[e];
    }
    __syncwarp();
    if (c.lane == 0) mbar_arrive(empty0 + c.slot * 8);
    if (++c.slot == n_stage) { c.slot = 0; c.ph ^= 1u; }
    if (blk + 1 < nblk) consumer_sync(c.nct);  // sc is rewritten by the next block
  }
  stamp(p, c, task_idx, 4);
  consumer_sync(c.nct);

  // cross-warp reduction -> partial record (o[D], m, l) of every q head of the group
  const int PS = D + 4;  // o[D], m, l, pad (records stay 16-byte aligned)
  float* part = p.part + ((size_t)(bidx * p.nkv + kvh) * p.attn_chunks + slot) * (size_t)G * PS;
  for (int i = c.ctid; i < G * D; i += c.nct) {
    const int g = i / D, d = i - g * D;
    float o = 0.f;
    for (int w = 0; w < p.C; ++w) o += red[(w * G + g) * D + d];
    part[(size_t)g * PS + d] = o;
    if (d == 0) {
      float l = 0.f;
      for (int w = 0; w < p.C; ++w) l += lw[w * kGMax + g];
      part[(size_t)g * PS + D] = mw[g];  // warp 0's copy; identical in every warp
      part[(size_t)g * PS + D + 1] = l;
    }
  }
  signal_counter(p, c, CTR_C);
  stamp(p, c, task_idx, 7);
}

// ----------------------------------------------------------------------------------
// the persistent kernel
// ----------------------------------------------------------------------------------
template <int CW>
__global__ void __launch_bounds__((CW + 1) * 32, 1) adamk_decode_kernel(const __grid_constant__ KParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  SmemHdr* hdr = reinterpret_cast<SmemHdr*>(smem);
  float* scratch = reinterpret_cast<float*>(smem + kSmemReserved);
  uint8_t* ring = smem + kSmemReserved + p.scratch_bytes;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.n_stage; ++s) {
      mbar_init(smem_u32(&hdr->full[s]), 1);
      mbar_init(smem_u32(&hdr->empty[s]), (uint32_t)p.C);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  const int tb = p.sm_begin[blockIdx.x], te = p.sm_begin[blockIdx.x + 1];

  if (warp == 0) {
    // ------------------------------ Loader ------------------------------
    if (lane == 0) {
      uint32_t slot = 0, ph = 0;
      const uint32_t ring_addr = smem_u32(ring);
      const uint32_t n_stage = (uint32_t)p.n_stage;
      const uint64_t pol = l2_evict_first_policy();  // weights are read once per step
      int lpos = 0;
      if (!p.probe) {
        lpos = __ldcg(p.positions);
        if (lpos < 0 || lpos >= p.max_ctx) return;  // the consumers report the error
      }
      // L2 prefetch cursor: runs pf_min bytes ahead of the ring in steady state and up to
      // pf_max bytes ahead while the ring is full (consumers stalled on a dependency), so
      // HBM keeps streaming through dependency stalls.
      const uint8_t* pf = p.wpacked + (size_t)p.sm_stream[blockIdx.x] * 16u;
      const uint8_t* const pf_end = p.wpacked + (size_t)p.sm_stream[blockIdx.x + 1] * 16u;
      constexpr uint32_t kPfGranule = 16384;
      auto prefetch_to = [&](const uint8_t* upto) {
        if (upto > pf_end) upto = pf_end;
        while (pf < upto) {
          const uint32_t nb = (uint32_t)min((size_t)kPfGranule, (size_t)(pf_end - pf));
          l2_prefetch_bulk(pf, nb);
          pf += nb;
        }
      };
      if (p.pf_min_bytes > 0) prefetch_to(pf + p.pf_min_bytes);
      for (int ti = tb; ti < te; ++ti) {
        const int4* tp = reinterpret_cast<const int4*>(p.tasks + ti);
        const int4 q0 = __ldg(tp), q1 = __ldg(tp + 1), q2 = __ldg(tp + 2);
        const int type = q0.x, nrows = q0.w, kchunks = q1.y, rt = q1.z, ktc = q1.w;
        const int n_tiles = q2.x, n_ktiles = q2.y;
        if (type == T_END) continue;
        if (type == T_ATTN) {
          // K / V blocks of this unit's context chunk, one ring stage each (skipped in probe mode)
          if (p.probe) continue;
          const AttnGeom ge = attn_geometry(p, lpos, q0.w);
          if (q0.w >= ge.n_active) continue;
          const int4 q3 = __ldg(tp + 3);
          const size_t head_base = ((size_t)(q0.y * p.batch + q3.w) * p.nkv + q0.z) * (size_t)p.max_ctx * p.D;
          for (int blk = 0; blk < ge.nblk; ++blk) {
            const int nb = min(ge.PB, ge.n - blk * ge.PB);
            const uint32_t bytes = (uint32_t)nb * (uint32_t)p.D * 2u;
            const size_t off = head_base + (size_t)(ge.t0 + blk * ge.PB) * p.D;
            for (int kv = 0; kv < 2; ++kv) {
              const uint32_t eb = smem_u32(&hdr->empty[slot]);
              if (!mbar_try_wait(eb, ph ^ 1u)) mbar_wait_slow(p, eb, ph ^ 1u, DE_WATCHDOG_EMPTY, ti);
              const uint32_t fb = smem_u32(&hdr->full[slot]);
              mbar_arrive_expect_tx(fb, bytes);
              tma_bulk_g2s(ring_addr + slot * (uint32_t)p.stage_bytes, (kv ? p.vcache : p.kcache) + off, bytes, fb);
              if (++slot == n_stage) { slot = 0; ph ^= 1u; }
            }
          }
          continue;
        }
        const uint8_t* src = p.wpacked + (size_t)(uint32_t)q2.z * 16u;
        for (int tile = 0; tile < n_tiles; ++tile) {
          const int rows = min(rt, nrows - tile * rt);
          for (int kt = 0; kt < n_ktiles; ++kt) {
            const int chunks = min(ktc, kchunks - kt * ktc);
            const uint32_t bytes = (uint32_t)rows * (uint32_t)chunks * 512u;
            const uint32_t eb = smem_u32(&hdr->empty[slot]);
            if (!mbar_try_wait(eb, ph ^ 1u)) {
              const long long t0 = clock64();
              while (!mbar_try_wait_hint(eb, ph ^ 1u, 300u)) {
                if (p.pf_max_bytes > 0 && pf < src + p.pf_max_bytes) prefetch_to(pf + 2 * kPfGranule);
                if (clock64() - t0 > kWatchdogCycles) dev_fail(p, DE_WATCHDOG_EMPTY, ti, (int)slot, (int)ph, 0);
              }
            }
            const uint32_t fb = smem_u32(&hdr->full[slot]);
            mbar_arrive_expect_tx(fb, bytes);
            const uint8_t* lsrc = src;
            if (p.probe == 3) lsrc = p.wpacked + (size_t)p.sm_stream[blockIdx.x] * 16u + ((size_t)(src - p.wpacked) & 0x3ffffu & ~(size_t)0xffff);
            tma_bulk_g2s_hint(ring_addr + slot * (uint32_t)p.stage_bytes, lsrc, bytes, fb, pol);
            src += bytes;
            if (p.pf_min_bytes > 0) prefetch_to(src + p.pf_min_bytes);
            if (++slot == n_stage) { slot = 0; ph ^= 1u; }
          }
        }
      }
    }
    return;
  }

  // ------------------------------ Consumers ------------------------------
  ConsumerCtx c;
  c.slot = 0; c.ph = 0; c.cw = warp - 1; c.lane = lane; c.ctid = threadIdx.x - 32; c.nct = p.C * 32;
  c.rs = 1.0f; c.best_val = -INFINITY; c.best_idx = -1;
  int tok = 0, pos = 0;
  if (!p.probe) {
    tok = __ldcg(p.tokens);
    pos = __ldcg(p.positions);
    if (pos < 0 || pos >= p.max_ctx || tok < 0 || tok >= p.V) {
      if (c.ctid == 0) dev_fail(p, DE_BAD_POS, -1, pos, tok, p.max_ctx);
      return;
    }
  }
  auto fetch_task = [&](int ti) {
    const int4* tp = reinterpret_cast<const int4*>(p.tasks + ti);
    const int4 a = __ldg(tp), b = __ldg(tp + 1), cc = __ldg(tp + 2), d = __ldg(tp + 3);
    Task t;
    t.type = a.x; t.layer = a.y; t.a = a.z; t.b = a.w;
    t.k = b.x; t.kchunks = b.y; t.rt = b.z; t.ktc = b.w;
    t.n_tiles = cc.x; t.n_ktiles = cc.y; t.w_off = cc.z; t.n_stages = cc.w;
    t.wait_ctr = d.x; t.wait_val = d.y; t.sig_ctr = d.z; t.aux = d.w;
    return t;
  };
  Task next = fetch_task(tb < te ? tb : 0);
  for (int ti = tb; ti < te; ++ti) {
    const Task t = next;
    if (ti + 1 < te) next = fetch_task(ti + 1);  // the record is a DRAM miss: fetch one task ahead
    if (t.type == T_ATTN) {
      if (p.D == 128) run_attn<128, 64 / CW>(p, c, t, ti, scratch, hdr, ring, pos);
      else run_attn<64, 64 / CW>(p, c, t, ti, scratch, hdr, ring, pos);
    } else if (t.type != T_END) {
      run_gemv(p, c, t, ti, scratch, hdr, ring, tok, pos);
    }
  }
}

// ----------------------------------------------------------------------------------
// weight packer: HF row-major bf16 -> per-SM tile-major streams (+ fp32 parameter tail)
// ----------------------------------------------------------------------------------
struct PackParams {
  const Task* tasks;
  int n_tasks;
  const AdamkLayerWeights* layers;  // device copy
  const void* lm_head;
  uint8_t* wpacked;
  int H, I, q_dim, kv_dim;
};

__device__ __forceinline__ const __nv_bfloat16* resolve_row(const PackParams& pp, const Task& t, int vrow, int* K) {
  const AdamkLayerWeights* lw = (t.type == T_LMHEAD) ? nullptr : pp.layers + t.layer;
  switch (t.type) {
    case T_QKV:
      *K = pp.H;
      if (vrow < pp.q_dim) return (const __nv_bfloat16*)lw->wq + (size_t)vrow * pp.H;
      if (vrow < pp.q_dim + pp.kv_dim) return (const __nv_bfloat16*)lw->wk + (size_t)(vrow - pp.q_dim) * pp.H;
      return (const __nv_bfloat16*)lw->wv + (size_t)(vrow - pp.q_dim - pp.kv_dim) * pp.H;
    case T_OPROJ: *K = pp.q_dim; return (const __nv_bfloat16*)lw->wo + (size_t)vrow * pp.q_dim;
    case T_GATEUP:
      *K = pp.H;
      return ((vrow & 1) ? (const __nv_bfloat16*)lw->wup : (const __nv_bfloat16*)lw->wgate) + (size_t)(vrow >> 1) * pp.H;
    case T_DOWN: *K = pp.I; return (const __nv_bfloat16*)lw->wdown + (size_t)vrow * pp.I;
    default: *K = pp.H; return (const __nv_bfloat16*)pp.lm_head + (size_t)vrow * pp.H;
  }
}

__global__ void adamk_pack_kernel(const PackParams pp) {
  const int ti = blockIdx.x;
  if (ti >= pp.n_tasks) return;
  const Task t = pp.tasks[ti];
  if (t.type == T_ATTN || t.type == T_END) return;
  uint4* dst = reinterpret_cast<uint4*>(pp.wpacked + (size_t)(uint32_t)t.w_off * 16u);
  size_t done = 0;  // 16-byte elements written so far
  for (int tile = 0; tile < t.n_tiles; ++tile) {
    const int rows = min(t.rt, t.b - tile * t.rt);
    for (int kt = 0; kt < t.n_ktiles; ++kt) {
      const int chunks = min(t.ktc, t.kchunks - kt * t.ktc);
      const int n = rows * chunks * 32;
      for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const int ln = e & 31;
        const int ch = (e >> 5) % chunks;
        const int r = (e >> 5) / chunks;
        int K;
        const __nv_bfloat16* row = resolve_row(pp, t, t.a + tile * t.rt + r, &K);
        const int k0 = (kt * t.ktc + ch) * kChunk + ln * 4;
        uint2 lo = make_uint2(0u, 0u), hi = make_uint2(0u, 0u);
        if (k0 + 3 < K) lo = *reinterpret_cast<const uint2*>(row + k0);
        else {
          unsigned short v[4] = {0, 0, 0, 0};
          for (int j = 0; j < 4; ++j) if (k0 + j < K) v[j] = reinterpret_cast<const unsigned short*>(row)[k0 + j];
          lo = make_uint2(v[0] | ((unsigned)v[1] << 16), v[2] | ((unsigned)v[3] << 16));
        }
        const int k1 = k0 + 128;
        if (k1 + 3 < K) hi = *reinterpret_cast<const uint2*>(row + k1);
        else {
          unsigned short v[4] = {0, 0, 0, 0};
          for (int j = 0; j < 4; ++j) if (k1 + j < K) v[j] = reinterpret_cast<const unsigned short*>(row)[k1 + j];
          hi = make_uint2(v[0] | ((unsigned)v[1] << 16), v[2] | ((unsigned)v[3] << 16));
        }
        dst[done + e] = make_uint4(lo.x, lo.y, hi.x, hi.y);
      }
      done += (size_t)n;
    }
  }
}

__global__ void adamk_cvt_kernel(const __nv_bfloat16* src, float* dst, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = __bfloat162float(src[i]);
}

// ----------------------------------------------------------------------------------
// host side
// ----------------------------------------------------------------------------------
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
#define CUDA_TRY(expr)                                                                                   \
  do {                                                                                                   \
    cudaError_t _e = (expr);                                                                             \
    if (_e != cudaSuccess)                                                                               \
      return fail(ADAMK_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));                     \
  } while (0)

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace

struct AdamkHandle_ {
  AdamkModelDesc desc{};
  int n_sms = 0, C = 0, n_stage = 0, stage_bytes = 0, n_tasks = 0, batch = 0, n_counters = 0;
  int attn_chunks = 0, attn_min_chunk = 0, scratch_bytes = 0, n_lm_tasks = 0, pf_min_bytes = 0, pf_max_bytes = 0;
  int xs_floats = 0;
  const unsigned* d_sm_stream = nullptr;
  size_t packed_weight_bytes = 0;  // matrix streams only
  size_t fparam_floats = 0;
  int fp_layer_stride = 0, fp_ln1 = 0, fp_ln2 = 0, fp_bias = 0, fp_qn = 0, fp_kn = 0, fp_final = 0;
  std::vector<int> host_table;
  int* d_table = nullptr;  // sm_begin + tasks
  const int* d_sm_begin = nullptr;
  const Task* d_tasks = nullptr;
  bool bound = false;
  const uint8_t* wpacked = nullptr;
  const float* fparams = nullptr;
  AdamkWeightPtrs w{};
  int* status_host = nullptr;
  int* status_dev = nullptr;
  unsigned long long* trace = nullptr;
  int smem_bytes = 0;
  // workspace layout (byte offsets)
  size_t ws_h_a = 0, ws_h_b = 0, ws_qkv = 0, ws_attn = 0, ws_act = 0, ws_part = 0, ws_lm_val = 0, ws_lm_idx = 0,
         ws_counters = 0, ws_total = 0;
};

extern "C" {

int adamk_abi_version(void) { return ADAMK_ABI_VERSION; }

const char* adamk_last_error(void) { return g_err.c_str(); }

int adamk_device_sm_count(int device, int* out_sms) {
  if (!out_sms) return fail(ADAMK_E_INVALID, "out_sms is NULL");
  int n = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device));
  *out_sms = n;
  return ADAMK_OK;
}

int adamk_create(const AdamkModelDesc* desc, const void* task_table, size_t task_table_bytes, int tp_rank, int tp_size,
                 adamk_handle* out) {
  if (!desc || !task_table || !out) return fail(ADAMK_E_INVALID, "NULL argument");
  if (tp_size != 1 || tp_rank != 0) return fail(ADAMK_E_UNSUPPORTED, "tensor parallel shards are not built yet (tp_size must be 1)");
  if (task_table_bytes < (size_t)kHeaderInts * 4 || task_table_bytes % 4) return fail(ADAMK_E_INVALID, "task table too small");
  const int* tt = static_cast<const int*>(task_table);
  if (tt[0] != kMagic || tt[1] != kVersion) return fail(ADAMK_E_INVALID, "task table magic/version mismatch");
  auto h = new AdamkHandle_();
  h->desc = *desc;
  h->n_sms = tt[2]; h->C = tt[3]; h->n_stage = tt[4]; h->stage_bytes = tt[5]; h->n_tasks = tt[6]; h->batch = tt[7];
  h->n_counters = tt[8]; h->attn_chunks = tt[9]; h->attn_min_chunk = tt[10]; h->scratch_bytes = tt[11];
  h->n_lm_tasks = tt[12];
  h->pf_min_bytes = tt[14] * 1024; h->pf_max_bytes = tt[15] * 1024;
  auto bad = [&](const std::string& m) { delete h; return fail(ADAMK_E_INVALID, m); };
  const AdamkModelDesc& d = *desc;
  if (d.head_dim != 64 && d.head_dim != 128) return bad("head_dim must be 64 or 128");
  if (d.n_kv_heads < 1 || d.n_q_heads % d.n_kv_heads) return bad("n_q_heads must be a multiple of n_kv_heads");
  if (d.n_q_heads / d.n_kv_heads > kGMax) return bad("more than 8 q heads per kv head");
  if (d.hidden % 8 || d.intermediate % 8) return bad("hidden/intermediate must be multiples of 8");
  if (h->batch != 1 || d.max_batch != 1) { delete h; return fail(ADAMK_E_UNSUPPORTED, "batch > 1 is not built yet"); }
  if (h->C != 4 && h->C != 8 && h->C != 16) return bad("consumer_warps must be 4, 8 or 16");
  if (h->n_stage < 1 || h->n_stage > kMaxStages) return bad("n_stage out of range");
  if (h->stage_bytes <= 0 || h->stage_bytes % 1024) return bad("stage_bytes must be a positive multiple of 1024");
  if (h->n_sms < 1 || h->n_tasks < 1) return bad("empty task table");
  if (h->attn_chunks < 1 || h->attn_chunks > kAttnChunksMax || h->attn_min_chunk < 8)
    return bad("attention chunking out of range");
  {
    const int pb = std::min(64, (h->stage_bytes / (d.head_dim * 2)) & ~7);
    if (pb != 64) return bad("stage_bytes too small: a K/V block is 64 positions (64 * head_dim * 2 bytes)");
  }
  const size_t need = ((size_t)kHeaderInts + (size_t)h->n_sms + 1 + (size_t)h->n_tasks * kTaskInts) * 4;
  if (task_table_bytes != need) return bad("task table size does not match its header");
  if (h->n_counters != CTR_HEAD0 + h->batch * d.n_kv_heads) return bad("counter count mismatch");
  h->smem_bytes = kSmemReserved + h->scratch_bytes + h->n_stage * h->stage_bytes;
  if (h->smem_bytes > kSmemMax) return bad("ring + scratch exceed 227 KB shared memory");
  {  // the scratch region must hold the widest activation vector + merge weights, and the attention buffers
    const int G = d.n_q_heads / d.n_kv_heads;
    const int kmax = std::max(std::max(d.hidden, d.n_q_heads * d.head_dim), d.intermediate);
    h->xs_floats = (int)align_up((size_t)kmax, kChunk);
    const size_t xb = ((size_t)h->xs_floats + 2 * (size_t)d.n_q_heads * h->attn_chunks) * 4;
    const size_t ab = ((size_t)kGMax * (128 + 32) + 2 * (size_t)kGMax * (kAttnPBMax + 4) + (size_t)h->C * G * d.head_dim +
                       3 * (size_t)h->C * kGMax + 2 * (size_t)d.head_dim) * 4;
    if ((size_t)h->scratch_bytes < std::max(xb, ab)) return bad("scratch_bytes too small for this model");
  }
  const int* sm_begin = tt + kHeaderInts;
  const Task* tasks = reinterpret_cast<const Task*>(tt + kHeaderInts + h->n_sms + 1);
  if (sm_begin[0] != 0 || sm_begin[h->n_sms] != h->n_tasks) return bad("sm_begin does not cover the task list");
  size_t wbytes = 0;
  for (int s = 0; s < h->n_sms; ++s)
    if (sm_begin[s] > sm_begin[s + 1]) return bad("sm_begin not monotone");
  const int qkv_rows = (d.n_q_heads + 2 * d.n_kv_heads) * d.head_dim;
  for (int i = 0; i < h->n_tasks; ++i) {
    const Task& t = tasks[i];
    if (t.type == T_ATTN) {
      if (t.a < 0 || t.a >= d.n_kv_heads || t.b < 0 || t.b >= h->attn_chunks || t.layer < 0 || t.layer >= d.n_layers)
        return bad("attention task out of range");
      continue;
    }
    if (t.type < T_QKV || t.type > T_LMHEAD) return bad("unknown task type");
    int n_rows = 0, K = 0;
    switch (t.type) {
      case T_QKV: n_rows = qkv_rows; K = d.hidden; break;
      case T_OPROJ: n_rows = d.hidden; K = d.n_q_heads * d.head_dim; break;
      case T_GATEUP: n_rows = 2 * d.intermediate; K = d.hidden; break;
      case T_DOWN: n_rows = d.hidden; K = d.intermediate; break;
      default: n_rows = d.vocab; K = d.hidden; break;
    }
    if (t.k != K || t.kchunks != (K + kChunk - 1) / kChunk) return bad("task K mismatch");
    if (t.a < 0 || t.b < 1 || t.a + t.b > n_rows) return bad("task rows out of range");
    if (t.rt % h->C || (t.rt / h->C != 2 && t.rt / h->C != 4)) return bad("rows_per_tile / consumer_warps must be 2 or 4");
    if (t.type == T_GATEUP && ((t.a | t.b) & 1)) return bad("gate/up rows must come in pairs");
    if (t.ktc < 1 || t.n_ktiles != (t.kchunks + t.ktc - 1) / t.ktc || t.n_tiles != (t.b + t.rt - 1) / t.rt)
      return bad("task tiling inconsistent");
    if ((size_t)t.rt * t.ktc * 512 > (size_t)h->stage_bytes) return bad("stage larger than stage_bytes");
    if (t.type != T_LMHEAD && (t.layer < 0 || t.layer >= d.n_layers)) return bad("task layer out of range");
    if (t.wait_ctr >= h->n_counters || t.sig_ctr >= h->n_counters) return bad("counter index out of range");
    const size_t bytes = (size_t)t.b * t.kchunks * 512;
    const size_t off = (size_t)(uint32_t)t.w_off * 16;
    wbytes = std::max(wbytes, off + bytes);
  }
  h->packed_weight_bytes = align_up(wbytes, 256);
  // fp32 parameter tail
  h->fp_ln1 = 0; h->fp_ln2 = d.hidden; h->fp_bias = 2 * d.hidden; h->fp_qn = h->fp_bias + qkv_rows;
  h->fp_kn = h->fp_qn + d.head_dim; h->fp_layer_stride = (int)align_up((size_t)h->fp_kn + d.head_dim, 4);
  h->fp_final = h->fp_layer_stride * d.n_layers;
  h->fparam_floats = (size_t)h->fp_final + d.hidden;
  // workspace layout
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes, 256); return r; };
  const int G = d.n_q_heads / d.n_kv_heads;
  h->ws_counters = take((size_t)h->n_counters * 4);
  h->ws_h_a = take((size_t)d.hidden * 4);
  h->ws_h_b = take((size_t)d.hidden * 4);
  h->ws_qkv = take((size_t)qkv_rows * 4);
  h->ws_attn = take((size_t)d.n_q_heads * d.head_dim * 4);
  h->ws_act = take(align_up((size_t)d.intermediate, kChunk) * 4);
  h->ws_part = take((size_t)d.n_kv_heads * h->attn_chunks * G * (d.head_dim + 4) * 4);
  h->ws_lm_val = take((size_t)h->n_sms * 4);
  h->ws_lm_idx = take((size_t)h->n_sms * 4);
  h->ws_total = o;

  // device copy: task records first (64-byte aligned for the int4 loads), then sm_begin
  h->host_table.assign(reinterpret_cast<const int*>(tasks), reinterpret_cast<const int*>(tasks) + (size_t)h->n_tasks * kTaskInts);
  h->host_table.insert(h->host_table.end(), sm_begin, sm_begin + h->n_sms + 1);
  {  // per-SM packed-stream ranges (streams are SM-major and contiguous)
    std::vector<unsigned> sm_stream(h->n_sms + 1, 0u);
    unsigned cursor = 0;
    for (int sm = 0; sm < h->n_sms; ++sm) {
      sm_stream[sm] = cursor;
      for (int i = sm_begin[sm]; i < sm_begin[sm + 1]; ++i) {
        const Task& t = tasks[i];
        if (t.type == T_ATTN) continue;
        if ((unsigned)t.w_off != cursor) return bad("packed streams must be contiguous per SM, SM-major");
        cursor += (unsigned)((size_t)t.b * t.kchunks * 512 / 16);
      }
    }
    sm_stream[h->n_sms] = cursor;
    for (unsigned v : sm_stream) h->host_table.push_back((int)v);
  }
  cudaError_t e = cudaMalloc(&h->d_table, h->host_table.size() * 4);
  if (e == cudaSuccess) e = cudaMemcpy(h->d_table, h->host_table.data(), h->host_table.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaHostAlloc(&h->status_host, 64, cudaHostAllocMapped);
  if (e == cudaSuccess) {
    memset(h->status_host, 0, 64);
    e = cudaHostGetDevicePointer(&h->status_dev, h->status_host, 0);
  }
  if (e == cudaSuccess) e = cudaFuncSetAttribute(adamk_decode_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(adamk_decode_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(adamk_decode_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
  if (e != cudaSuccess) {
    std::string m = std::string("adamk_create: ") + cudaGetErrorString(e);
    adamk_destroy(h);
    return fail(ADAMK_E_CUDA, m);
  }
  h->d_tasks = reinterpret_cast<const Task*>(h->d_table);
  h->d_sm_begin = h->d_table + (size_t)h->n_tasks * kTaskInts;
  h->d_sm_stream = reinterpret_cast<const unsigned*>(h->d_sm_begin + h->n_sms + 1);
  *out = h;
  return ADAMK_OK;
}

void adamk_destroy(adamk_handle h) {
  if (!h) return;
  if (h->d_table) cudaFree(h->d_table);
  if (h->status_host) cudaFreeHost(h->status_host);
  delete h;
}

size_t adamk_packed_bytes(adamk_handle h) { return h ? h->packed_weight_bytes + align_up(h->fparam_floats * 4, 256) : 0; }

size_t adamk_workspace_bytes(adamk_handle h) { return h ? h->ws_total : 0; }

size_t adamk_kv_cache_bytes(adamk_handle h) {
  if (!h) return 0;
  const AdamkModelDesc& d = h->desc;
  return (size_t)d.n_layers * d.max_batch * d.n_kv_heads * d.max_ctx * d.head_dim * 2;
}

int adamk_workspace_init(adamk_handle h, void* workspace, adamk_stream stream) {
  if (!h || !workspace) return fail(ADAMK_E_INVALID, "NULL argument");
  CUDA_TRY(cudaMemsetAsync(workspace, 0, h->ws_total, (cudaStream_t)stream));
  return ADAMK_OK;
}

int adamk_bind_weights(adamk_handle h, const AdamkWeightPtrs* w, void* packed, adamk_stream stream_) {
  if (!h || !w || !packed) return fail(ADAMK_E_INVALID, "NULL argument");
  if (!w->embed || !w->final_norm || !w->layers || !w->rope_cos || !w->rope_sin) return fail(ADAMK_E_INVALID, "missing weight pointer");
  if ((uintptr_t)packed % 256) return fail(ADAMK_E_INVALID, "packed buffer must be 256-byte aligned");
  const AdamkModelDesc& d = h->desc;
  cudaStream_t stream = (cudaStream_t)stream_;
  for (int l = 0; l < d.n_layers; ++l) {
    const AdamkLayerWeights& lw = w->layers[l];
    if (!lw.ln1 || !lw.wq || !lw.wk || !lw.wv || !lw.wo || !lw.ln2 || !lw.wgate || !lw.wup || !lw.wdown)
      return fail(ADAMK_E_INVALID, "layer " + std::to_string(l) + ": missing matrix pointer");
    if (d.qkv_bias && (!lw.bq || !lw.bk || !lw.bv)) return fail(ADAMK_E_INVALID, "qkv_bias set but bias pointer missing");
    if (d.qk_norm && (!lw.q_norm || !lw.k_norm)) return fail(ADAMK_E_INVALID, "qk_norm set but norm pointer missing");
  }
  AdamkLayerWeights* d_layers = nullptr;
  CUDA_TRY(cudaMalloc(&d_layers, sizeof(AdamkLayerWeights) * d.n_layers));
  cudaError_t e = cudaMemcpyAsync(d_layers, w->layers, sizeof(AdamkLayerWeights) * d.n_layers, cudaMemcpyHostToDevice, stream);
  if (e != cudaSuccess) { cudaFree(d_layers); return fail(ADAMK_E_CUDA, cudaGetErrorString(e)); }
  PackParams pp{};
  pp.tasks = h->d_tasks; pp.n_tasks = h->n_tasks; pp.layers = d_layers;
  pp.lm_head = w->lm_head ? w->lm_head : w->embed;
  pp.wpacked = static_cast<uint8_t*>(packed);
  pp.H = d.hidden; pp.I = d.intermediate; pp.q_dim = d.n_q_heads * d.head_dim; pp.kv_dim = d.n_kv_heads * d.head_dim;
  adamk_pack_kernel<<<h->n_tasks, 256, 0, stream>>>(pp);
  // fp32 parameter tail
  float* fp = reinterpret_cast<float*>(static_cast<uint8_t*>(packed) + h->packed_weight_bytes);
  auto cvt = [&](const void* src, size_t off, int n) {
    if (src && n > 0) adamk_cvt_kernel<<<(n + 255) / 256, 256, 0, stream>>>((const __nv_bfloat16*)src, fp + off, n);
  };
  e = cudaMemsetAsync(fp, 0, h->fparam_floats * 4, stream);
  for (int l = 0; l < d.n_layers && e == cudaSuccess; ++l) {
    const AdamkLayerWeights& lw = w->layers[l];
    const size_t base = (size_t)l * h->fp_layer_stride;
    cvt(lw.ln1, base + h->fp_ln1, d.hidden);
    cvt(lw.ln2, base + h->fp_ln2, d.hidden);
    if (d.qkv_bias) {
      cvt(lw.bq, base + h->fp_bias, pp.q_dim);
      cvt(lw.bk, base + h->fp_bias + pp.q_dim, pp.kv_dim);
      cvt(lw.bv, base + h->fp_bias + pp.q_dim + pp.kv_dim, pp.kv_dim);
    }
    if (d.qk_norm) {
      cvt(lw.q_norm, base + h->fp_qn, d.head_dim);
      cvt(lw.k_norm, base + h->fp_kn, d.head_dim);
    }
  }
  cvt(w->final_norm, h->fp_final, d.hidden);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  cudaFree(d_layers);
  if (e != cudaSuccess) return fail(ADAMK_E_CUDA, std::string("adamk_bind_weights: ") + cudaGetErrorString(e));
  h->w = *w;
  h->w.layers = nullptr;
  h->wpacked = static_cast<const uint8_t*>(packed);
  h->fparams = fp;
  h->bound = true;
  return ADAMK_OK;
}

int adamk_bind_peers(adamk_handle h, void* const* peer_workspaces, int n_peers) {
  (void)peer_workspaces;
  if (!h) return fail(ADAMK_E_INVALID, "NULL handle");
  if (n_peers == 1) return ADAMK_OK;
  return fail(ADAMK_E_UNSUPPORTED, "tensor parallel shards are not built yet");
}

static int fill_params(adamk_handle h, KParams& p, void* workspace) {
  const AdamkModelDesc& d = h->desc;
  memset(&p, 0, sizeof(p));
  p.H = d.hidden; p.L = d.n_layers; p.nq = d.n_q_heads; p.nkv = d.n_kv_heads; p.D = d.head_dim; p.I = d.intermediate;
  p.V = d.vocab; p.G = d.n_q_heads / d.n_kv_heads; p.q_dim = d.n_q_heads * d.head_dim; p.kv_dim = d.n_kv_heads * d.head_dim;
  p.qkv_rows = p.q_dim + 2 * p.kv_dim; p.max_ctx = d.max_ctx; p.batch = h->batch;
  p.has_bias = d.qkv_bias; p.qk_norm = d.qk_norm; p.eps = d.rms_eps;
  p.C = h->C; p.n_stage = h->n_stage; p.stage_bytes = h->stage_bytes; p.attn_chunks = h->attn_chunks;
  p.attn_min_chunk = h->attn_min_chunk; p.scratch_bytes = h->scratch_bytes; p.n_lm_tasks = h->n_lm_tasks;
  p.n_counters = h->n_counters;
  p.xs_floats = h->xs_floats;
  p.tasks = h->d_tasks; p.sm_begin = h->d_sm_begin; p.sm_stream = h->d_sm_stream;
  p.pf_min_bytes = h->pf_min_bytes; p.pf_max_bytes = h->pf_max_bytes;
  p.wpacked = h->wpacked; p.fparams = h->fparams;
  p.fp_layer_stride = h->fp_layer_stride; p.fp_ln1 = h->fp_ln1; p.fp_ln2 = h->fp_ln2; p.fp_bias = h->fp_bias;
  p.fp_qn = h->fp_qn; p.fp_kn = h->fp_kn; p.fp_final = h->fp_final;
  p.embed = (const __nv_bfloat16*)h->w.embed; p.rope_cos = h->w.rope_cos; p.rope_sin = h->w.rope_sin;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  if (ws) {
    p.counters = (unsigned*)(ws + h->ws_counters);
    p.h_a = (float*)(ws + h->ws_h_a); p.h_b = (float*)(ws + h->ws_h_b); p.qkv = (float*)(ws + h->ws_qkv);
    p.attn = (float*)(ws + h->ws_attn); p.act = (float*)(ws + h->ws_act); p.part = (float*)(ws + h->ws_part);
    p.lm_val = (float*)(ws + h->ws_lm_val); p.lm_idx = (int*)(ws + h->ws_lm_idx);
  }
  p.status = h->status_dev;
  p.trace = h->trace;
  return ADAMK_OK;
}

static int launch(adamk_handle h, const KParams& p, cudaStream_t stream) {
  int dev = 0, sms = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (sms < h->n_sms) return fail(ADAMK_E_INVALID, "task table was built for more SMs than this device has");
  void* args[] = {(void*)&p};
  // cooperative launch: all CTAs must be co-resident (they wait on each other's counters)
  const void* fn = h->C == 4 ? (const void*)adamk_decode_kernel<4>
                   : h->C == 8 ? (const void*)adamk_decode_kernel<8> : (const void*)adamk_decode_kernel<16>;
  CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(h->n_sms), dim3((h->C + 1) * 32), args, (size_t)h->smem_bytes, stream));
  return ADAMK_OK;
}

int adamk_decode_step(adamk_handle h, int32_t* token_ids, int32_t* positions, int batch, void* k_cache, void* v_cache,
                      void* workspace, float* logits_out, int32_t* next_token_out, int auto_advance,
                      adamk_stream stream) {
  if (!h || !token_ids || !positions || !k_cache || !v_cache || !workspace || !next_token_out)
    return fail(ADAMK_E_INVALID, "NULL argument");
  if (!h->bound) return fail(ADAMK_E_STATE, "adamk_bind_weights has not been called");
  if (batch != h->batch) return fail(ADAMK_E_INVALID, "batch does not match the task table");
  if (h->status_host[0] != 0) return fail(ADAMK_E_DEVICE, "a previous step reported a device error; see adamk_device_status");
  KParams p;
  fill_params(h, p, workspace);
  p.kcache = (__nv_bfloat16*)k_cache; p.vcache = (__nv_bfloat16*)v_cache;
  p.logits = logits_out; p.tokens = token_ids; p.positions = positions; p.next_tokens = next_token_out;
  p.auto_advance = auto_advance;
  return launch(h, p, (cudaStream_t)stream);
}

int adamk_stream_probe(adamk_handle h, float* sink, int mode, adamk_stream stream) {
  if (!h || !sink) return fail(ADAMK_E_INVALID, "NULL argument");
  if (!h->bound) return fail(ADAMK_E_STATE, "adamk_bind_weights has not been called");
  KParams p;
  fill_params(h, p, nullptr);
  p.probe = (mode == 2 || mode == 3) ? mode : 1; p.probe_sink = sink;
  if (mode == 3) { p.pf_min_bytes = 0; p.pf_max_bytes = 0; }
  return launch(h, p, (cudaStream_t)stream);
}

int adamk_set_trace(adamk_handle h, void* trace_buf) {
  if (!h) return fail(ADAMK_E_INVALID, "NULL handle");
  h->trace = static_cast<unsigned long long*>(trace_buf);
  return ADAMK_OK;
}

size_t adamk_trace_bytes(adamk_handle h) { return h ? (size_t)h->n_tasks * 8 * sizeof(unsigned long long) : 0; }

int adamk_device_status(adamk_handle h, int32_t* info) {
  if (!h) return fail(ADAMK_E_INVALID, "NULL handle");
  if (info) memcpy(info, h->status_host, 32);
  return h->status_host[0];
}

}  // extern "C"
