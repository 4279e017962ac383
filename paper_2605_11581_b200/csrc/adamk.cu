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
//              logical decoupling") limited by free ring slots and by
//              a cap on the stages in flight (keeps the loaded memory latency low).
//   Consumer : warps 1..C.  Gather the operator's input vector, stage it in shared
//              memory (fusing RMSNorm), then GEMV out of the ring with LDS.128 +
//              packed FFMA2.  The warps of a CTA form a WR x WK grid per operator:
//              WR row groups of up to 8 rows, WK interleaved K groups.
//   Storer   : the consumers' epilogue (bias / residual / SiLU*up / argmax).
// Page states Empty -> Locked -> Ready (planner.py:84-94) = ring slot `empty`
// mbarrier phase -> TMA in flight -> `full` mbarrier phase.
//
// Inter-SM dependencies carry no counters and no fences: every activation element is
// published as one 64-bit word {fp32 value, 32-bit tag} with a single relaxed store, and
// the consumers of the vector poll the words themselves until every tag equals the
// (step, layer) tag they expect -- the data is its own flag.  Which words an operator
// reads and the tag it expects are fixed by the task table ("path solidification",
// PAPER.md:197); nothing is scheduled at run time.
//
// Numerical contract (shared with oracle/decode_ref.py): bf16 weights used exactly,
// fp32 activations and accumulation, bf16 KV cache, fp32 RoPE tables from the host.

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
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

typedef unsigned long long u64;

constexpr int kMagic = 0x4B4D4441;
constexpr int kVersion = 2;
constexpr int kHeaderInts = 16;
constexpr int kTaskInts = 16;
constexpr int kChunk = 256;          // K elements per chunk
constexpr int kSmemMax = 232448;
constexpr int kSmemReserved = 3584;  // barriers + reduction scratch + the shared-memory copy of the kernel parameters
constexpr int kMaxStages = 16;
constexpr int kAttnWarps = 8;        // consumer warps that take part in an attention unit
constexpr int kAttnChunksMax = 128;  // split-KV units per (sequence, kv head)
constexpr int kGMax = 8;             // max q heads per kv head
constexpr int kRW = 8;               // max rows per warp per tile
constexpr int kGatherBatch = 4;      // 16-byte tagged-word loads a thread keeps in flight while gathering a vector
constexpr int kMaxTP = 8;
constexpr int kRep = 2;              // copies of the vectors every SM gathers whole (single-GPU kernel; measured 1 / 2 / 4 / 8 copies: 804 / 796 / 800 / 805 us per token)
constexpr int kTagStride = 256;      // tag = epoch * kTagStride + layer + 1

enum TaskType { T_END = 0, T_QKV = 1, T_ATTN = 2, T_OPROJ = 3, T_GATEUP = 4, T_DOWN = 5, T_LMHEAD = 6, T_MERGE = 7, T_DOWNK = 8, T_HRED = 9 };

struct Task {  // 64 bytes
  int type, layer, a, b, k, kchunks, rt, ktc, n_tiles, n_ktiles, w_off, geom, r12, r13, r14, aux;
};
static_assert(sizeof(Task) == kTaskInts * 4, "task record is 64 bytes");

// device error codes written to the host-mapped status block
enum DevErr { DE_NONE = 0, DE_WATCHDOG_TAG = 1, DE_WATCHDOG_FULL = 2, DE_WATCHDOG_EMPTY = 3, DE_BAD_POS = 4, DE_WATCHDOG_INFLIGHT = 5 };

struct KParams {
  // model
  int H, L, nq, nkv, D, I, V, G, q_dim, kv_dim, qkv_rows, max_ctx, batch;
  int has_bias, qk_norm;
  float eps;
  // schedule
  int C, n_stage, stage_bytes, attn_chunks, attn_min_chunk, scratch_bytes, n_lm_tasks, inflight;
  int stream_down;         // 1: the down projection streams its input vector in k-tile by k-tile (down_streamed)
  int attn_block;          // positions per K / V block = 8 x attention warps: one pass of the unit's warps per block
  int pf_window_bytes;     // how far past the ring the Loader prefetches into L2 while it is blocked (0 = off)
  int poll_inflight;       // ring stages the Loader keeps in flight (and no L2 prefetch) while its consumers poll for inputs (0 = no change)
  int pace_clk_per_64k;    // Loader pacing: SM clocks per 64 KB of NEW bytes this SM asks HBM for (0 = unpaced)
  int task_cache_bytes;    // shared-memory copy of this SM's task list (32-byte packed records)
  unsigned poll_sleep_ns;  // back-off between polls of a not-yet-complete vector (0 = none)
  // task table
  const Task* tasks;
  const int* sm_begin;
  const unsigned* sm_stream;  // [n_sms + 1] packed-stream range of every SM (16-byte units)
  // weights
  const uint8_t* wpacked;   // tile-major bf16 weight streams
  const float* fparams;     // fp32 norm gains / biases
  int fp_layer_stride, fp_ln1, fp_ln2, fp_bias, fp_qn, fp_kn, fp_final;
  unsigned fp_bytes;        // size of the fp32 parameter tail
  const __nv_bfloat16* embed;
  const float* rope_cos;
  const float* rope_sin;
  // per-step buffers
  __nv_bfloat16* kcache;
  __nv_bfloat16* vcache;
  // tagged activation vectors ({fp32, tag} words)
  // The vectors every SM gathers whole (hx, hm, attn) are published in `rep` copies; SM s reads copy s % rep.  A
  // 12 KB vector sits in ~48 of the ~184 L2 slices (256-byte hash granules): with one copy, 148 SMs polling it
  // queue 100 K requests on those slices and every hop pays that queue twice (the producers' stores wait in it too).
  int rep;
  u64* ll_hx;    // [rep][2][tp][H]  layer input, ping-pong by layer parity; one slot of partial rows per TP rank
  u64* ll_hm;    // [rep][tp][H]     hidden state after attention, likewise
  u64* ll_lmx;   // [tp][2]     (value, index) of every rank's LM-head argmax
  u64* ll_qkv;   // [qkv_rows]
  u64* ll_attn;  // [rep][q_dim]  merged attention output
  u64* ll_act;   // [I]
  u64* ll_part;  // [nq][attn_chunks][D + 2]  split-KV partial records (o[D], m, l)
  u64* ll_part2; // [H / 4][n_sms][4]  fused down projection: every SM's partial rows (T_DOWNK -> T_HRED), row-quad major
  float* lm_val;
  int* lm_idx;
  unsigned* sync;  // [0] = epoch, [1] = CTAs that finished the LM head
  float* logits;
  int* tokens;
  int* positions;
  int* next_tokens;
  int* status;  // host-mapped, 8 ints
  int auto_advance;
  // tensor parallelism: this rank publishes its partial O-proj / down-proj rows (and its LM-head argmax) into
  // slot tp_rank of EVERY rank's workspace with the same 64-bit tagged stores (NVLink peer memory)
  int tp_rank, tp_size, vocab_off;
  u64* peer_hx[kMaxTP];
  u64* peer_hm[kMaxTP];
  u64* peer_lmx[kMaxTP];
  int probe;    // 1 = stream probe: consumers skip dependencies and epilogues; 2 = also skip the math;
                // 3 = like 1 but the Loader re-reads an L2-resident window; 4 = consumers only (no Loader, no waits)
  float* probe_sink;
  u64* trace;  // optional [n_tasks][8] globaltimer stamps (0 start, 1 inputs gathered, 2 body done, 7 end, 3-6 op specific)
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
__device__ __forceinline__ uint32_t mbar_test_wait(uint32_t bar, uint32_t parity) {  // non-blocking probe
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok;
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
__device__ __forceinline__ void l2_prefetch_bulk(const void* src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(src), "r"(bytes), "l"(pol) : "memory");
}
// The small per-layer fp32 vectors (norm gains, biases) sit on the critical path of every hop; the
// weight stream flushes them out of L2 between two uses unless they are loaded evict-last.
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ float2 ldg_keep_f2(const float2* p) {
  float2 v;
  const uint64_t pol = l2_evict_last_policy();
  asm volatile("ld.global.nc.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(v.x), "=f"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float4 ldg_keep_f4(const float4* p) {
  float4 v;
  const uint64_t pol = l2_evict_last_policy();
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ldg_keep_f1(const float* p) {
  float v;
  const uint64_t pol = l2_evict_last_policy();
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u64 globaltimer_ns() {
  u64 t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
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

// ---- tagged words: {fp32 value (low half), tag (high half)} ----
// A 64-bit aligned scalar store / load is single-copy atomic, so a reader that sees the
// expected tag also sees the value written with it: no fence, no separate flag.
__device__ __forceinline__ void ll_store(u64* p, float v, unsigned tag) {
  const u64 w = ((u64)tag << 32) | (u64)__float_as_uint(v);
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ u64 ll_load(const u64* p) {
  u64 w;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  return w;
}
__device__ __forceinline__ void ll_load2(const u64* p, u64& a, u64& b) {  // 16-byte aligned pair of words
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
// four words = one full 32-byte L2 sector per request (LDG.E.256.STRONG.GPU; every word carries its own tag)
__device__ __forceinline__ void ll_load4(const u64* p, u64 (&w)[4]) {
  asm volatile("ld.relaxed.gpu.global.v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3]) : "l"(p) : "memory");
}
// system-scope variants for words another GPU writes / reads (tensor-parallel slots)
__device__ __forceinline__ void ll_store_sys(u64* p, float v, unsigned tag) {
  const u64 w = ((u64)tag << 32) | (u64)__float_as_uint(v);
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ u64 ll_load_sys(const u64* p) {
  u64 w;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  return w;
}
__device__ __forceinline__ void ll_load2_sys(const u64* p, u64& a, u64& b) {
  asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ unsigned ll_tag(u64 w) { return (unsigned)(w >> 32); }
__device__ __forceinline__ float ll_val(u64 w) { return __uint_as_float((unsigned)w); }

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

__device__ __noinline__ void mbar_wait_slow(const KParams& p, uint32_t bar, uint32_t parity, int code, int task) {
  const long long t0 = clock64();
  // the Loader's waits (EMPTY / INFLIGHT) time out later than the consumers': the first report names the root cause
  const long long limit = (code == DE_WATCHDOG_EMPTY || code == DE_WATCHDOG_INFLIGHT) ? 2 * kWatchdogCycles : kWatchdogCycles;
  while (!mbar_try_wait_hint(bar, parity, 2000u)) {
    if (clock64() - t0 > limit) dev_fail(p, code, task, (int)bar, (int)parity, 0);
  }
}
__device__ __forceinline__ void mbar_wait(const KParams& p, uint32_t bar, uint32_t parity, int code, int task) {
  if (!mbar_try_wait(bar, parity)) mbar_wait_slow(p, bar, parity, code, task);
}

// slow paths of the tagged-word polls (out of line: they are cold and keep the hot code small)
__device__ __noinline__ u64 ll_spin(const KParams& p, const u64* addr, unsigned tag, int task) {
  const long long t0 = clock64();
  u64 w;
  while (ll_tag(w = ll_load(addr)) != tag) {
    if (clock64() - t0 > kWatchdogCycles) dev_fail(p, DE_WATCHDOG_TAG, task, (int)ll_tag(w), (int)tag, (int)((uintptr_t)addr & 0x7fffffff));
  }
  return w;
}
__device__ __forceinline__ float ll_wait(const KParams& p, const u64* addr, unsigned tag, int task) {
  u64 w = ll_load(addr);
  if (ll_tag(w) != tag) w = ll_spin(p, addr, tag, task);
  return ll_val(w);
}

// ----------------------------------------------------------------------------------
// shared-memory layout
// ----------------------------------------------------------------------------------
struct SmemHdr {
  u64 full[kMaxStages];
  u64 empty[kMaxStages];
  float red[64];
  int misc[32];
  float red2[2][8][32];  // cross-K-group partial sums of a tile: [tile parity][K group][row]
  u64 xbar[8];           // slice barriers of a streamed activation vector (down_streamed)
  // A copy of the kernel parameters.  The out-of-line task bodies take `const KParams&`; a reference to the
  // __grid_constant__ parameter makes every p.field a generic load that misses L1 (the shared-memory carve-out
  // leaves no L1) and pays an L2 round trip under the weight stream -- dozens of them, dependent, at the top of
  // every task.  The copy in shared memory is one LDS away.
  KParams kp;
};
static_assert(sizeof(SmemHdr) <= kSmemReserved, "smem header too large");

struct ConsumerCtx {
  uint32_t slot;      // ring slot of the next stage to drain
  uint32_t ph;        // its mbarrier phase parity
  int cw;             // consumer warp index 0..C-1
  int lane;
  int ctid;           // thread index among consumers
  int nct;            // number of consumer threads
  unsigned epoch;     // step sequence number (tag prefix)
  float rs;           // RMSNorm scale of the current GEMV's input (applied in the epilogue), else 1
  float* act_loc;     // fused down projection: this SM's SwiGLU outputs (shared memory, behind the staged gate/up input)
  float best_val;     // LM-head running argmax (epilogue lanes)
  int best_idx;
};

// "the consumers of this SM are polling for their inputs": the Loader holds its bulk traffic back meanwhile
// (a poll's round trip queues behind every bulk byte in flight to the same SM and to the same L2 slices)
constexpr int kMiscPolling = 24;
__device__ __forceinline__ void set_polling(SmemHdr* hdr, int ctid, int v) {
  if (ctid == 0) *reinterpret_cast<volatile int*>(&hdr->misc[kMiscPolling]) = v;
}
__device__ __forceinline__ unsigned tag_of(const ConsumerCtx& c, int layer) { return c.epoch * kTagStride + (unsigned)layer + 1u; }

__device__ __forceinline__ void stamp(const KParams& p, const ConsumerCtx& c, int task, int k) {
  if (p.trace && c.ctid == 0) p.trace[(size_t)task * 8 + k] = globaltimer_ns();
}

// Split-KV geometry of one decode step, shared by the Loader (which streams the K/V
// blocks of a unit through the ring) and the Consumers (which drain them).
struct AttnGeom {
  int CL, n_active, t0, n, nblk;
};
__device__ __forceinline__ AttnGeom attn_geometry(const KParams& p, int pos, int slot) {
  AttnGeom g;
  const int ctx = pos + 1;
  g.CL = max(p.attn_min_chunk, (ctx + p.attn_chunks - 1) / p.attn_chunks);
  g.CL = (g.CL + 7) & ~7;
  g.n_active = (ctx + g.CL - 1) / g.CL;
  g.t0 = slot * g.CL;
  g.n = min(ctx, g.t0 + g.CL) - g.t0;           // <= 0 for inactive slots
  g.nblk = g.n > 0 ? (g.n + p.attn_block - 1) / p.attn_block : 0;
  return g;
}

// ----------------------------------------------------------------------------------
// gather of a tagged vector into shared memory
// ----------------------------------------------------------------------------------
// Every consumer thread owns the 32-byte word quads i = ctid, ctid + nct, ... of the vector, issues up to
// kGatherBatch sector loads back to back, and re-polls the batch until every tag is current.  NORM: the
// values are multiplied by the RMSNorm gain while staged and sum(x^2) is returned (per thread).
__device__ __noinline__ float ll_gather(const KParams& p, int ctid, int nct, const u64* src, int n, int kpad,
                                        unsigned tag, float* xs, const float* gain, int task, int first = 0) {
  const bool NORM = gain != nullptr;
  const int n4 = n >> 2, kp4 = kpad >> 2;
  float ss = 0.f;
  for (int i0 = first + ctid; i0 < kp4; i0 += kGatherBatch * nct) {
    float4 g[kGatherBatch];
#pragma unroll
    for (int u = 0; u < kGatherBatch; ++u) {  // static operand first: a DRAM miss under the weight stream, overlapped with the poll
      const int i = i0 + u * nct;
      g[u] = (NORM && i < n4) ? ldg_keep_f4(reinterpret_cast<const float4*>(gain) + i) : make_float4(1.f, 1.f, 1.f, 1.f);
    }
    u64 w[kGatherBatch][4];
    long long t0 = 0;
    for (;;) {  // re-issue the whole batch until every tag is current (one round trip per attempt)
      bool ok = true;
#pragma unroll
      for (int u = 0; u < kGatherBatch; ++u) {
        const int i = i0 + u * nct;
        if (i < n4) ll_load4(src + 4 * i, w[u]);
      }
#pragma unroll
      for (int u = 0; u < kGatherBatch; ++u) {
        const int i = i0 + u * nct;
        if (i < n4) ok = ok && ll_tag(w[u][0]) == tag && ll_tag(w[u][1]) == tag && ll_tag(w[u][2]) == tag && ll_tag(w[u][3]) == tag;
      }
      if (ok) break;
      if (p.poll_sleep_ns) __nanosleep(p.poll_sleep_ns);
      if (t0 == 0) t0 = clock64();
      else if (clock64() - t0 > kWatchdogCycles) dev_fail(p, DE_WATCHDOG_TAG, task, (int)ll_tag(w[0][0]), (int)tag, i0);
    }
#pragma unroll
    for (int u = 0; u < kGatherBatch; ++u) {
      const int i = i0 + u * nct;
      if (i < kp4) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < n4) {
          v = make_float4(ll_val(w[u][0]), ll_val(w[u][1]), ll_val(w[u][2]), ll_val(w[u][3]));
          ss = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, ss))));
          v.x *= g[u].x; v.y *= g[u].y; v.z *= g[u].z; v.w *= g[u].w;
        }
        reinterpret_cast<float4*>(xs)[i] = v;
      }
    }
  }
  return ss;
}

// Tensor-parallel gather: the vector is the sum of one slot of partial rows per rank (rank 0's partial carries
// the residual), summed in rank order so every rank computes bit-identical activations.  8 / T words per
// thread are in flight at a time, each with its T slot words; system-scope loads (peers write the slots).
template <int T>
__device__ __noinline__ float ll_gather_tp(const KParams& p, int ctid, int nct, const u64* src, int n, int kpad,
                                           unsigned tag, float* xs, const float* gain, int task) {
  constexpr int WB = 8 / T;  // words per batch
  const bool NORM = gain != nullptr;
  const int n2 = n >> 1, kp2 = kpad >> 1;
  const size_t slot_stride = (size_t)n;  // words per slot
  float ss = 0.f;
  for (int i0 = ctid; i0 < kp2; i0 += WB * nct) {
    float2 g[WB];
#pragma unroll
    for (int w = 0; w < WB; ++w) {
      const int i = i0 + w * nct;
      g[w] = (NORM && i < n2) ? ldg_keep_f2(reinterpret_cast<const float2*>(gain) + i) : make_float2(1.f, 1.f);
    }
    u64 a[8], b[8];
    long long t0 = 0;
    for (;;) {
      bool ok = true;
#pragma unroll
      for (int u = 0; u < WB * T; ++u) {
        const int i = i0 + (u / T) * nct;
        if (i < n2) ll_load2_sys(src + (size_t)(u % T) * slot_stride + 2 * i, a[u], b[u]);
      }
#pragma unroll
      for (int u = 0; u < WB * T; ++u) {
        const int i = i0 + (u / T) * nct;
        if (i < n2) ok = ok && ll_tag(a[u]) == tag && ll_tag(b[u]) == tag;
      }
      if (ok) break;
      if (t0 == 0) t0 = clock64();
      else if (clock64() - t0 > kWatchdogCycles) dev_fail(p, DE_WATCHDOG_TAG, task, (int)ll_tag(a[0]), (int)tag, i0);
    }
#pragma unroll
    for (int w = 0; w < WB; ++w) {
      const int i = i0 + w * nct;
      if (i < kp2) {
        float2 v = make_float2(0.f, 0.f);
        if (i < n2) {
#pragma unroll
          for (int sl = 0; sl < T; ++sl) { v.x += ll_val(a[w * T + sl]); v.y += ll_val(b[w * T + sl]); }
          ss = fmaf(v.x, v.x, fmaf(v.y, v.y, ss));
          v.x *= g[w].x; v.y *= g[w].y;
        }
        reinterpret_cast<float2*>(xs)[i] = v;
      }
    }
  }
  return ss;
}
__device__ __forceinline__ float ll_gather_slots(const KParams& p, int ctid, int nct, const u64* src, int n, int kpad,
                                                 unsigned tag, float* xs, const float* gain, int task) {
  switch (p.tp_size) {
    case 1: return ll_gather(p, ctid, nct, src, n, kpad, tag, xs, gain, task);
    case 2: return ll_gather_tp<2>(p, ctid, nct, src, n, kpad, tag, xs, gain, task);
    case 4: return ll_gather_tp<4>(p, ctid, nct, src, n, kpad, tag, xs, gain, task);
    default: return ll_gather_tp<8>(p, ctid, nct, src, n, kpad, tag, xs, gain, task);
  }
}
// one element of a slotted vector (residual operand of an epilogue): sum over the rank slots in rank order.
// The tensor-parallel parts of the GEMV task body are out of line so the single-GPU body keeps its registers.
__device__ __noinline__ float ll_wait_slots_tp(const KParams& p, const u64* src, int n, int idx, unsigned tag, int task) {
  float v = 0.f;
  for (int sl = 0; sl < p.tp_size; ++sl) {
    const u64* a = src + (size_t)sl * n + idx;
    u64 w = ll_load_sys(a);
    const long long t0 = clock64();
    while (ll_tag(w) != tag) {
      w = ll_load_sys(a);
      if (clock64() - t0 > kWatchdogCycles) dev_fail(p, DE_WATCHDOG_TAG, task, (int)ll_tag(w), (int)tag, idx);
    }
    v += ll_val(w);
  }
  return v;
}
// publish one partial row to slot tp_rank of every rank (peer-mapped memory over NVLink): which = 0 -> hm, 1 -> hx[parity]
__device__ __noinline__ void tp_publish(const KParams& p, int which, int parity, int row, float v, unsigned tag) {
  for (int r = 0; r < p.tp_size; ++r) {
    u64* dst = which == 0 ? p.peer_hm[r] + (size_t)p.tp_rank * p.H + row
                          : p.peer_hx[r] + ((size_t)parity * p.tp_size + p.tp_rank) * p.H + row;
    ll_store_sys(dst, v, tag);
  }
}
// every rank publishes (value, index) of its LM-head argmax to every rank and takes the best of all, ties to the
// lowest index; called by one warp of the rank's last CTA
__device__ __noinline__ void tp_argmax_exchange(const KParams& p, int lane, unsigned xtag, float& best, int& idx) {
  if (lane < p.tp_size) {
    ll_store_sys(p.peer_lmx[lane] + 2 * p.tp_rank, best, xtag);
    ll_store_sys(p.peer_lmx[lane] + 2 * p.tp_rank + 1, __int_as_float(idx), xtag);
  }
  best = -INFINITY; idx = 0x7fffffff;
  if (lane < p.tp_size) {
    const u64* rec = p.ll_lmx + 2 * lane;
    u64 wv = ll_load_sys(rec), wi = ll_load_sys(rec + 1);
    const long long t0 = clock64();
    while (ll_tag(wv) != xtag || ll_tag(wi) != xtag) {
      wv = ll_load_sys(rec); wi = ll_load_sys(rec + 1);
      if (clock64() - t0 > kWatchdogCycles) dev_fail(p, DE_WATCHDOG_TAG, -2, (int)ll_tag(wv), (int)xtag, lane);
    }
    best = ll_val(wv); idx = __float_as_int(ll_val(wi));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > best || (ov == best && oi < idx)) { best = ov; idx = oi; }
  }
}

// N words base[0], base[stride], ... gathered by one thread: all loads in flight together, re-polled as a batch.
template <int N>
__device__ __forceinline__ void ll_wait_strided(const KParams& p, const u64* base, int stride, unsigned tag, float (&out)[N],
                                                int task) {
  u64 w[N];
  long long t0 = 0;
  for (;;) {
    bool ok = true;
#pragma unroll
    for (int j = 0; j < N; ++j) w[j] = ll_load(base + (size_t)j * stride);
#pragma unroll
    for (int j = 0; j < N; ++j) ok = ok && ll_tag(w[j]) == tag;
    if (ok) break;
    if (p.poll_sleep_ns) __nanosleep(p.poll_sleep_ns);
    if (t0 == 0) t0 = clock64();
    else if (clock64() - t0 > kWatchdogCycles) dev_fail(p, DE_WATCHDOG_TAG, task, (int)ll_tag(w[0]), (int)tag, -1);
  }
#pragma unroll
  for (int j = 0; j < N; ++j) out[j] = ll_val(w[j]);
}

// ----------------------------------------------------------------------------------
// GEMV task
// ----------------------------------------------------------------------------------
__device__ __forceinline__ float silu(float g) { return g / (1.0f + expf(-g)); }

__device__ __forceinline__ const float* gemv_gain(const KParams& p, const Task& t) {
  if (t.type == T_LMHEAD) return p.fparams + p.fp_final;
  return p.fparams + (size_t)t.layer * p.fp_layer_stride + (t.type == T_GATEUP ? p.fp_ln2 : p.fp_ln1);
}

// The input vector of a GEMV: where its tagged words are, its length, the tag that marks it current and, for the
// RMSNorm-fused operators (QKV: ln1 over the layer input, GATEUP: ln2 over h_mid, LMHEAD: final norm), the gain.
struct VecSrc {
  const u64* src;
  const float* gain;
  int n;
  unsigned tag;
};
template <bool TP>
__device__ __forceinline__ bool gemv_input(const KParams& p, const ConsumerCtx& c, const Task& t, VecSrc& v) {
  const int type = t.type;
  const size_t cp = blockIdx.x % p.rep;
  v.gain = nullptr;
  if (type == T_OPROJ) { v.src = p.ll_attn + cp * p.q_dim; v.n = p.q_dim; v.tag = tag_of(c, t.layer); return true; }
  if (type == T_DOWN) { v.src = p.ll_act; v.n = p.I; v.tag = tag_of(c, t.layer); return true; }
  if (type == T_QKV && t.layer == 0) return false;   // layer 0 reads the embedding row directly
  const int layer = (type == T_LMHEAD) ? p.L : t.layer;
  v.gain = gemv_gain(p, t); v.n = p.H; v.tag = tag_of(c, layer);
  if constexpr (TP) v.src = (type == T_GATEUP) ? p.ll_hm : p.ll_hx + (size_t)(layer & 1) * p.tp_size * p.H;
  else v.src = (type == T_GATEUP) ? p.ll_hm + cp * p.H : p.ll_hx + (cp * 2 + (size_t)(layer & 1)) * p.H;
  return true;
}
__device__ __forceinline__ bool ll_quad_ok(const u64 (&w)[4], unsigned tag) {
  return ll_tag(w[0]) == tag && ll_tag(w[1]) == tag && ll_tag(w[2]) == tag && ll_tag(w[3]) == tag;
}

// Stage the activation vector of a GEMV in shared memory (fp32, zero padded to kpad).  The first two sectors of
// every thread (w0, w1: quads ctid and ctid + nct) were requested at the very top of the task (`early`), before
// any other work of the task: ~2000 clocks of task preamble used to sit between the task start and its first poll.
template <bool TP>
__device__ __forceinline__ void gemv_prologue(const KParams& p, ConsumerCtx& c, const Task& t, int ti, float* xs,
                                              SmemHdr* hdr, int tok, const VecSrc& vs, bool have, bool early,
                                              u64 (&w0)[4], u64 (&w1)[4]) {
  const int kpad = t.kchunks * kChunk;
  const int type = t.type;
  c.rs = 1.0f;
  float ss = 0.f;
  if (!have) {  // QKV of layer 0: the embedding row (bf16), RMSNorm-fused
    const float* gain = gemv_gain(p, t);
    const int h2 = p.H >> 1, kp2 = kpad >> 1;
    for (int i = c.ctid; i < kp2; i += c.nct) {
      float2 v = make_float2(0.f, 0.f);
      if (i < h2) {
        const uint32_t raw = __ldg(reinterpret_cast<const uint32_t*>(p.embed + (size_t)tok * p.H) + i);
        v.x = bf_lo(raw); v.y = bf_hi(raw);
        ss = fmaf(v.x, v.x, fmaf(v.y, v.y, ss));
        const float2 g = ldg_keep_f2(reinterpret_cast<const float2*>(gain) + i);
        v.x *= g.x; v.y *= g.y;
      }
      reinterpret_cast<float2*>(xs)[i] = v;
    }
  } else if (!early) {
    if (TP && vs.gain) ss = ll_gather_slots(p, c.ctid, c.nct, vs.src, vs.n, kpad, vs.tag, xs, vs.gain, ti);
    else ss = ll_gather(p, c.ctid, c.nct, vs.src, vs.n, kpad, vs.tag, xs, vs.gain, ti);
  } else {
    const int n4 = vs.n >> 2, kp4 = kpad >> 2, ia = c.ctid, ib = c.ctid + c.nct;
    float4 ga = make_float4(1.f, 1.f, 1.f, 1.f), gb = ga;
    if (vs.gain) {
      if (ia < n4) ga = ldg_keep_f4(reinterpret_cast<const float4*>(vs.gain) + ia);
      if (ib < n4) gb = ldg_keep_f4(reinterpret_cast<const float4*>(vs.gain) + ib);
    }
    long long t0 = 0;
    while (!((ia >= n4 || ll_quad_ok(w0, vs.tag)) && (ib >= n4 || ll_quad_ok(w1, vs.tag)))) {
      if (ia < n4) ll_load4(vs.src + 4 * ia, w0);
      if (ib < n4) ll_load4(vs.src + 4 * ib, w1);
      if (t0 == 0) t0 = clock64();
      else if (clock64() - t0 > kWatchdogCycles) dev_fail(p, DE_WATCHDOG_TAG, ti, (int)ll_tag(w0[0]), (int)vs.tag, ia);
    }
    if (ia < kp4) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (ia < n4) {
        v = make_float4(ll_val(w0[0]), ll_val(w0[1]), ll_val(w0[2]), ll_val(w0[3]));
        ss = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, ss))));
        v.x *= ga.x; v.y *= ga.y; v.z *= ga.z; v.w *= ga.w;
      }
      reinterpret_cast<float4*>(xs)[ia] = v;
    }
    if (ib < kp4) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (ib < n4) {
        v = make_float4(ll_val(w1[0]), ll_val(w1[1]), ll_val(w1[2]), ll_val(w1[3]));
        ss = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, ss))));
        v.x *= gb.x; v.y *= gb.y; v.z *= gb.z; v.w *= gb.w;
      }
      reinterpret_cast<float4*>(xs)[ib] = v;
    }
    if (kp4 > 2 * c.nct) ss += ll_gather(p, c.ctid, c.nct, vs.src, vs.n, kpad, vs.tag, xs, vs.gain, ti, 2 * c.nct);
  }
  if (type == T_OPROJ || type == T_DOWN) {
    consumer_sync(c.nct);
    set_polling(hdr, c.ctid, 0);
    return;
  }
  // RMSNorm: h * gain was staged and sum(h^2) accumulated in one pass; the scalar rsqrt(mean + eps) commutes
  // with the dot products and is applied to each output row in the epilogue.
  ss = warp_sum(ss);
  float* red = hdr->red + (ti & 1) * 16;  // by task parity: a warp that runs ahead writes the other half
  if (c.lane == 0) red[c.cw] = ss;
  consumer_sync(c.nct);
  set_polling(hdr, c.ctid, 0);
  float tot = 0.f;
  for (int w = 0; w < p.C; ++w) tot += red[w];
  c.rs = rsqrtf(tot / (float)p.H + p.eps);
}

// Epilogue operand of one output row (bias, residual input).  Residuals are tagged words of a
// vector this step has already completed; the tag is still checked (cheap) rather than assumed.
template <bool TP>
__device__ __forceinline__ float load_eop(const KParams& p, const ConsumerCtx& c, const Task& t, int ti, int vrow, int tok) {
  switch (t.type) {
    case T_QKV: return p.has_bias ? ldg_keep_f1(p.fparams + (size_t)t.layer * p.fp_layer_stride + p.fp_bias + vrow) : 0.f;
    case T_OPROJ:
      if (TP && p.tp_rank != 0) return 0.f;  // rank 0's partial rows carry the residual
      if (t.layer == 0) return __bfloat162float(p.embed[(size_t)tok * p.H + vrow]);
      if constexpr (TP) return ll_wait_slots_tp(p, p.ll_hx + (size_t)(t.layer & 1) * p.tp_size * p.H, p.H, vrow, tag_of(c, t.layer), ti);
      else return ll_wait(p, p.ll_hx + ((size_t)(blockIdx.x % p.rep) * 2 + (size_t)(t.layer & 1)) * p.H + vrow, tag_of(c, t.layer), ti);
    case T_DOWN:
      if (TP && p.tp_rank != 0) return 0.f;
      if constexpr (TP) return ll_wait_slots_tp(p, p.ll_hm, p.H, vrow, tag_of(c, t.layer), ti);
      else return ll_wait(p, p.ll_hm + (size_t)(blockIdx.x % p.rep) * p.H + vrow, tag_of(c, t.layer), ti);
    default: return 0.f;
  }
}

template <bool TP>
__device__ __forceinline__ void gemv_epilogue(const KParams& p, ConsumerCtx& c, const Task& t, int vrow, float v,
                                              float v_pair, float eop) {
  switch (t.type) {
    case T_QKV: ll_store(p.ll_qkv + vrow, v + eop, tag_of(c, t.layer)); break;
    case T_OPROJ:
      if constexpr (TP) tp_publish(p, 0, 0, vrow, eop + v, tag_of(c, t.layer));
      else for (int r = 0; r < p.rep; ++r) ll_store(p.ll_hm + (size_t)r * p.H + vrow, eop + v, tag_of(c, t.layer));
      break;
    case T_GATEUP:   // vrow even = gate, pair = up
      if (t.aux & 1) c.act_loc[(vrow - t.a) >> 1] = silu(v) * v_pair;   // fused down projection: the value stays on this SM
      else ll_store(p.ll_act + (vrow >> 1), silu(v) * v_pair, tag_of(c, t.layer));
      break;
    case T_DOWN:
      if constexpr (TP) tp_publish(p, 1, (t.layer + 1) & 1, vrow, eop + v, tag_of(c, t.layer + 1));
      else for (int r = 0; r < p.rep; ++r) ll_store(p.ll_hx + ((size_t)r * 2 + (size_t)((t.layer + 1) & 1)) * p.H + vrow, eop + v, tag_of(c, t.layer + 1));
      break;
    case T_LMHEAD: {
      const int gvrow = TP ? vrow + p.vocab_off : vrow;
      if (p.logits) p.logits[gvrow] = v;
      if (v > c.best_val) { c.best_val = v; c.best_idx = gvrow; }  // rows ascend: first max wins ties
    } break;
    default: break;
  }
}

// Sum eight per-lane partials over the warp with 9 shuffles: after the call every lane holds the
// total of row  4*bit4(lane) + 2*bit3(lane) + bit2(lane).
__device__ __forceinline__ float reduce8(const float (&v)[kRW], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  float u[4], w[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float keep = b4 ? v[i + 4] : v[i], send = b4 ? v[i] : v[i + 4];
    u[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float keep = b3 ? u[i + 2] : u[i], send = b3 ? u[i] : u[i + 2];
    w[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  const float keep = b2 ? w[1] : w[0], send = b2 ? w[0] : w[1];
  float s = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  return s;
}

// One ring stage of a warp: its K group's chunks (every WK-th) of RW rows.  No predication inside:
// all RW weight loads of a chunk are issued back to back ahead of the convert / FFMA2 chains.
template <int RW>
__device__ __forceinline__ void gemv_stage(uint32_t wa, uint32_t row_stride, uint32_t xa_addr, int nch, int WK,
                                           float2 (&acc)[kRW]) {
  const uint32_t wstep = (uint32_t)WK * 512u, xstep = (uint32_t)WK * (kChunk * 4);
#pragma unroll 1
  for (int j = 0; j < nch; ++j, wa += wstep, xa_addr += xstep) {
    const float4 xa = lds128f(xa_addr);
    const float4 xb = lds128f(xa_addr + 512);
    uint4 w[RW];
#pragma unroll
    for (int i = 0; i < RW; ++i) w[i] = lds128u(wa + i * row_stride);
#pragma unroll
    for (int i = 0; i < RW; ++i) {
      acc[i] = __ffma2_rn(make_float2(bf_lo(w[i].x), bf_hi(w[i].x)), make_float2(xa.x, xa.y), acc[i]);
      acc[i] = __ffma2_rn(make_float2(bf_lo(w[i].y), bf_hi(w[i].y)), make_float2(xa.z, xa.w), acc[i]);
      acc[i] = __ffma2_rn(make_float2(bf_lo(w[i].z), bf_hi(w[i].z)), make_float2(xb.x, xb.y), acc[i]);
      acc[i] = __ffma2_rn(make_float2(bf_lo(w[i].w), bf_hi(w[i].w)), make_float2(xb.z, xb.w), acc[i]);
    }
  }
}

// Per-task constants of the stage loop, computed once (nothing but the ring cursor changes per stage).
struct StageGeom {
  uint32_t wofs_full, wofs_last;      // byte offset of this warp's first block inside a full / the last k-tile stage
  uint32_t rstride_full, rstride_last;
  int nch_full, nch_last;             // chunks of this warp's K group in a full / the last k-tile stage
};

// All k-tiles of one row tile.  wait = false: consumer-only probe (no Loader, no barriers).
// The ring cursor lives in registers here (slot, ph) and is written back by the caller.
template <int RW>
__device__ __forceinline__ void gemv_ktiles(const KParams& p, uint32_t& slot, uint32_t& ph, int lane, int ktc, int n_ktiles,
                                            int task_idx, const StageGeom& sg, uint32_t ring_addr, uint32_t xs_addr,
                                            uint32_t full0, uint32_t empty0, int WK, float2 (&acc)[kRW], bool active,
                                            bool wait) {
  const uint32_t n_stage = (uint32_t)p.n_stage, stage_bytes = (uint32_t)p.stage_bytes;
  const uint32_t xtile = (uint32_t)ktc * (kChunk * 4);
  uint32_t xa = xs_addr;
  uint32_t sbase = ring_addr + slot * stage_bytes;
  const int last = n_ktiles - 1;
#pragma unroll 1
  for (int kt = 0; kt <= last; ++kt, xa += xtile) {
    if (wait) mbar_wait(p, full0 + slot * 8, ph, DE_WATCHDOG_FULL, task_idx);
    if (active) {
      const bool is_last = kt == last;
      gemv_stage<RW>(sbase + (is_last ? sg.wofs_last : sg.wofs_full), is_last ? sg.rstride_last : sg.rstride_full, xa,
                     is_last ? sg.nch_last : sg.nch_full, WK, acc);
    }
    if (wait) {
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + slot * 8);
    }
    sbase += stage_bytes;
    if (++slot == n_stage) { slot = 0; ph ^= 1u; sbase = ring_addr; }
  }
}

// The wide operators (gate/up, LM head) in the profiled schedules: WK == 1, RW rows per warp and the
// same KTC chunks in every stage.  Every stride is a compile-time immediate and the chunk loop is
// unrolled, so a stage costs ~110 instructions per chunk instead of ~170 (the loop is issue-bound with
// two warps per scheduler).
template <int RW, int KTC>
__device__ __forceinline__ void gemv_ktiles_wide(const KParams& p, uint32_t& slot, uint32_t& ph, int lane, int n_ktiles,
                                                 int task_idx, uint32_t wofs, uint32_t ring_addr, uint32_t xs_addr,
                                                 uint32_t full0, uint32_t empty0, float2 (&acc)[kRW], bool wait) {
  const uint32_t n_stage = (uint32_t)p.n_stage, stage_bytes = (uint32_t)p.stage_bytes;
  uint32_t xa = xs_addr;
  uint32_t sbase = ring_addr + slot * stage_bytes + wofs;
#pragma unroll 1
  for (int kt = 0; kt < n_ktiles; ++kt, xa += KTC * (kChunk * 4)) {
    if (wait) mbar_wait(p, full0 + slot * 8, ph, DE_WATCHDOG_FULL, task_idx);
#pragma unroll
    for (int j = 0; j < KTC; ++j) {
      const float4 x0 = lds128f(xa + j * (kChunk * 4));
      const float4 x1 = lds128f(xa + j * (kChunk * 4) + 512);
      uint4 w[RW];
#pragma unroll
      for (int i = 0; i < RW; ++i) w[i] = lds128u(sbase + (i * KTC + j) * 512);
#pragma unroll
      for (int i = 0; i < RW; ++i) {
        acc[i] = __ffma2_rn(make_float2(bf_lo(w[i].x), bf_hi(w[i].x)), make_float2(x0.x, x0.y), acc[i]);
        acc[i] = __ffma2_rn(make_float2(bf_lo(w[i].y), bf_hi(w[i].y)), make_float2(x0.z, x0.w), acc[i]);
        acc[i] = __ffma2_rn(make_float2(bf_lo(w[i].z), bf_hi(w[i].z)), make_float2(x1.x, x1.y), acc[i]);
        acc[i] = __ffma2_rn(make_float2(bf_lo(w[i].w), bf_hi(w[i].w)), make_float2(x1.z, x1.w), acc[i]);
      }
    }
    if (wait) {
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + slot * 8);
    }
    sbase += stage_bytes;
    if (++slot == n_stage) { slot = 0; ph ^= 1u; sbase = ring_addr + wofs; }
  }
}

// ---- W4A16 (GPTQ-format int4 weights, fp16 group scales; reference byte model graph_ir.py:296-318) ----------------
// A task whose aux field has bit 1 set streams its weights as 4-bit codes: value = (code - 8) * scale[row][k / 128].
// Ring stage of `rows x chunks`: rows * chunks blocks of 128 bytes (a 256-element chunk of one row: lane l owns 4 bytes =
// the codes of elements 4l..4l+3 and 128+4l..128+4l+3, the elements its two activation LDS.128 hold), then rows * chunks
// pairs of fp16 scales (the chunk's two groups of 128).  Dequantisation without integer conversions: the fp32 word
// 0x41800000 | code << 19 IS 16 + code, so a code costs one shift, one LOP3 and half a packed add (minus 24, exact).
constexpr int kI4ChunkBytes = 128, kI4ScaleBytes = 4, kI4Group = 128;
// groups of 128 reduction elements touched by columns k0 .. k0 + nk of the down projection
__host__ __device__ __forceinline__ int downk_i4_groups(int k0, int nk) { return (k0 + nk - 1) / kI4Group - k0 / kI4Group + 1; }
constexpr int kDownkGroupsMax = 3;
__host__ __device__ __forceinline__ uint32_t i4_stage_bytes(int rows, int chunks) {
  return ((uint32_t)rows * (uint32_t)chunks * (kI4ChunkBytes + kI4ScaleBytes) + 15u) & ~15u;
}
__device__ __forceinline__ void i4_unpack(uint32_t w, float (&lo)[4], float (&hi)[4]) {   // codes 0-3 / 4-7 as code - 8, exactly
  // 0x41800000 | code << 19 is the fp32 number 16 + code; minus 24 (exact) leaves code - 8
  const float2 m24 = make_float2(-24.f, -24.f);
  const float2 a = __fadd2_rn(make_float2(__uint_as_float(((w << 19) & 0x00780000u) | 0x41800000u),
                                          __uint_as_float(((w << 15) & 0x00780000u) | 0x41800000u)), m24);
  const float2 b = __fadd2_rn(make_float2(__uint_as_float(((w << 11) & 0x00780000u) | 0x41800000u),
                                          __uint_as_float(((w << 7) & 0x00780000u) | 0x41800000u)), m24);
  const float2 c = __fadd2_rn(make_float2(__uint_as_float(((w << 3) & 0x00780000u) | 0x41800000u),
                                          __uint_as_float(((w >> 1) & 0x00780000u) | 0x41800000u)), m24);
  const float2 d = __fadd2_rn(make_float2(__uint_as_float(((w >> 5) & 0x00780000u) | 0x41800000u),
                                          __uint_as_float(((w >> 9) & 0x00780000u) | 0x41800000u)), m24);
  lo[0] = a.x; lo[1] = a.y; lo[2] = b.x; lo[3] = b.y;
  hi[0] = c.x; hi[1] = c.y; hi[2] = d.x; hi[3] = d.y;
}
__device__ __forceinline__ float2 h2_to_f2(uint32_t h2) {
  const __half2 h = *reinterpret_cast<const __half2*>(&h2);
  return __half22float2(h);
}

// All k-tiles of one row tile of an int4 task.  acc[i].x / .y accumulate the two groups of every chunk.
template <int RW>
__device__ __forceinline__ void gemv_ktiles_i4(const KParams& p, uint32_t& slot, uint32_t& ph, int lane, int ktc, int chunks_last,
                                               int n_ktiles, int rows, int my_r0, int wk, int WK, int task_idx, uint32_t ring0,
                                               uint32_t xs_addr, uint32_t full0, uint32_t empty0, float2 (&acc)[kRW], bool active, bool wait) {
  const uint32_t n_stage = (uint32_t)p.n_stage, stage_bytes = (uint32_t)p.stage_bytes;
  uint32_t xa0 = xs_addr;   // lane's 16 bytes of the k-tile's first chunk (already offset by wk chunks)
#pragma unroll 1
  for (int kt = 0; kt < n_ktiles; ++kt, xa0 += (uint32_t)ktc * (kChunk * 4)) {
    if (wait) mbar_wait(p, full0 + slot * 8, ph, DE_WATCHDOG_FULL, task_idx);
    const int chunks = kt == n_ktiles - 1 ? chunks_last : ktc;
    if (active) {
      const uint32_t sbase = ring0 + slot * stage_bytes;
      const uint32_t sc_base = sbase + (uint32_t)rows * (uint32_t)chunks * kI4ChunkBytes;
      uint32_t xa = xa0;
#pragma unroll 1
      for (int j = wk; j < chunks; j += WK, xa += (uint32_t)WK * (kChunk * 4)) {
        const float4 x0 = lds128f(xa), x1 = lds128f(xa + 512);
        uint32_t w[RW], sc[RW];
#pragma unroll
        for (int i = 0; i < RW; ++i) {
          const uint32_t blk = (uint32_t)((my_r0 + i) * chunks + j);
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w[i]) : "r"(sbase + blk * kI4ChunkBytes + lane * 4));
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(sc[i]) : "r"(sc_base + blk * kI4ScaleBytes));
        }
#pragma unroll
        for (int i = 0; i < RW; ++i) {
          float lo[4], hi[4];
          i4_unpack(w[i], lo, hi);
          float2 a = __ffma2_rn(make_float2(lo[0], hi[0]), make_float2(x0.x, x1.x), make_float2(0.f, 0.f));
          a = __ffma2_rn(make_float2(lo[1], hi[1]), make_float2(x0.y, x1.y), a);
          a = __ffma2_rn(make_float2(lo[2], hi[2]), make_float2(x0.z, x1.z), a);
          a = __ffma2_rn(make_float2(lo[3], hi[3]), make_float2(x0.w, x1.w), a);
          acc[i] = __ffma2_rn(h2_to_f2(sc[i]), a, acc[i]);
        }
      }
    }
    if (wait) {
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + slot * 8);
    }
    if (++slot == n_stage) { slot = 0; ph ^= 1u; }
  }
}

template <int RW, bool TP, bool I4>
__device__ __forceinline__ void gemv_tiles_t(const KParams& p, ConsumerCtx& c, const Task& t, int task_idx,
                                             const float* xs, SmemHdr* hdr, uint8_t* ring, int tok, float eop0, int probe) {
  const int WK = (t.geom >> 8) & 0xff, rw = (t.geom >> 16) & 0xff, lgWK = 31 - __clz(WK);
  const int wr = c.cw >> lgWK, wk = c.cw & (WK - 1);
  const uint32_t ring_addr = smem_u32(ring) + c.lane * 16;
  const uint32_t full0 = smem_u32(&hdr->full[0]);
  const uint32_t empty0 = smem_u32(&hdr->empty[0]);
  const int my_r0 = wr * rw;
  const int rsel = ((c.lane >> 4) & 1) * 4 + ((c.lane >> 3) & 1) * 2 + ((c.lane >> 2) & 1);  // row held after reduce8
  const int chunks_last = t.kchunks - (t.n_ktiles - 1) * t.ktc;
  StageGeom sg;
  sg.rstride_full = (uint32_t)t.ktc * 512u; sg.rstride_last = (uint32_t)chunks_last * 512u;
  sg.wofs_full = (uint32_t)my_r0 * sg.rstride_full + (uint32_t)wk * 512u;
  sg.wofs_last = (uint32_t)my_r0 * sg.rstride_last + (uint32_t)wk * 512u;
  sg.nch_full = (t.ktc - wk + WK - 1) >> lgWK; sg.nch_last = max(0, (chunks_last - wk + WK - 1) >> lgWK);
  const uint32_t xs_addr = smem_u32(xs) + c.lane * 16 + (uint32_t)wk * (kChunk * 4);
  for (int tile = 0; tile < t.n_tiles; ++tile) {
    const int rows = min(t.rt, t.b - tile * t.rt);
    const int my_n = max(0, min(rw, rows - my_r0));  // rows of this tile owned by this warp
    const int vrow0 = t.a + tile * t.rt;
    // the thread that will run the epilogue of a row loads its operand ahead of the K loop
    int erow = -1;
    if (WK == 1) { if ((c.lane & 3) == 0 && rsel < my_n) erow = my_r0 + rsel; }
    else if (c.ctid < rows) erow = c.ctid;
    float eop = eop0;
    if (tile > 0 && erow >= 0 && !probe) eop = load_eop<TP>(p, c, t, task_idx, vrow0 + erow, tok);
    float2 acc[kRW];
#pragma unroll
    for (int i = 0; i < kRW; ++i) acc[i] = make_float2(0.f, 0.f);
    // rows past my_n read stale bytes of the slot and are discarded by the epilogue (no predication in the loop)
    const bool active = my_n > 0 && probe != 2;
    {
      uint32_t slot = c.slot, ph = c.ph;
      const bool wide = RW >= 4 && WK == 1 && rw == RW && chunks_last == t.ktc && probe != 2;
      if constexpr (I4)
        gemv_ktiles_i4<RW>(p, slot, ph, c.lane, t.ktc, chunks_last, t.n_ktiles, rows, my_r0, wk, WK, task_idx, smem_u32(ring), xs_addr,
                           full0, empty0, acc, active, probe != 4);
      else if (wide && t.ktc == 2)
        gemv_ktiles_wide<RW, 2>(p, slot, ph, c.lane, t.n_ktiles, task_idx, sg.wofs_full, ring_addr, xs_addr, full0, empty0, acc, probe != 4);
      else if (wide && t.ktc == 1)
        gemv_ktiles_wide<RW, 1>(p, slot, ph, c.lane, t.n_ktiles, task_idx, sg.wofs_full, ring_addr, xs_addr, full0, empty0, acc, probe != 4);
      else if (wide && t.ktc == 3)
        gemv_ktiles_wide<RW, 3>(p, slot, ph, c.lane, t.n_ktiles, task_idx, sg.wofs_full, ring_addr, xs_addr, full0, empty0, acc, probe != 4);
      else
        gemv_ktiles<RW>(p, slot, ph, c.lane, t.ktc, t.n_ktiles, task_idx, sg, ring_addr, xs_addr, full0, empty0, WK, acc, active, probe != 4);
      c.slot = slot; c.ph = ph;
    }
    float v[kRW];
#pragma unroll
    for (int i = 0; i < kRW; ++i) v[i] = acc[i].x + acc[i].y;
    float s = reduce8(v, c.lane);
    if (probe) {
      if (s == 1.2345678e-30f) p.probe_sink[blockIdx.x * 64] = s;  // keep the math alive
      continue;
    }
    if (WK == 1) {
      s *= c.rs;
      const float partner = __shfl_xor_sync(0xffffffffu, s, 4);  // row rsel ^ 1 (the `up` row of a gate row)
      if (erow >= 0) {
        if (t.type != T_GATEUP) gemv_epilogue<TP>(p, c, t, vrow0 + erow, s, 0.f, eop);
        else if (!(erow & 1)) gemv_epilogue<TP>(p, c, t, vrow0 + erow, s, partner, 0.f);
      }
    } else {
      float* rb = &hdr->red2[tile & 1][0][0];
      if ((c.lane & 3) == 0 && rsel < my_n) rb[wk * 32 + my_r0 + rsel] = s;
      consumer_sync(c.nct);
      if (erow >= 0) {
        float tot = 0.f, tot2 = 0.f;
        for (int k = 0; k < WK; ++k) tot += rb[k * 32 + erow];
        if (t.type != T_GATEUP) gemv_epilogue<TP>(p, c, t, vrow0 + erow, tot * c.rs, 0.f, eop);
        else if (!(erow & 1)) {
          for (int k = 0; k < WK; ++k) tot2 += rb[k * 32 + erow + 1];
          gemv_epilogue<TP>(p, c, t, vrow0 + erow, tot * c.rs, tot2 * c.rs, 0.f);
        }
      }
    }
  }
  // every warp is done reading the staged activation vector before the next task overwrites the
  // scratch region (K-split tiles already synchronised after their last stage)
  if (WK == 1 && !probe) consumer_sync(c.nct);
}

template <bool TP, bool I4>
__device__ __forceinline__ void gemv_tiles(const KParams& p, ConsumerCtx& c, const Task& t, int task_idx,
                                           const float* xs, SmemHdr* hdr, uint8_t* ring, int tok, float eop0, int probe) {
  switch ((((t.geom >> 16) & 0xff) + 1) >> 1) {  // rows per warp, rounded up to even
    case 1: gemv_tiles_t<2, TP, I4>(p, c, t, task_idx, xs, hdr, ring, tok, eop0, probe); break;
    case 2: gemv_tiles_t<4, TP, I4>(p, c, t, task_idx, xs, hdr, ring, tok, eop0, probe); break;
    case 3: gemv_tiles_t<6, TP, I4>(p, c, t, task_idx, xs, hdr, ring, tok, eop0, probe); break;
    default: gemv_tiles_t<8, TP, I4>(p, c, t, task_idx, xs, hdr, ring, tok, eop0, probe); break;
  }
}

template <bool TP>
__device__ __forceinline__ void lm_finish(const KParams& p, ConsumerCtx& c, SmemHdr* hdr) {
  // per-lane best -> per-warp best -> CTA best -> global partial -> last CTA reduces, publishes, bumps the epoch
  float bv = c.best_val;
  int bi = c.best_idx < 0 ? 0x7fffffff : c.best_idx;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  if (c.lane == 0) { hdr->red[32 + c.cw] = bv; hdr->misc[c.cw] = bi; }
  consumer_sync(c.nct);
  if (c.ctid == 0) {
    float best = hdr->red[32];
    int idx = hdr->misc[0];
    for (int w = 1; w < p.C; ++w) {
      const float v = hdr->red[32 + w];
      const int i = hdr->misc[w];
      if (v > best || (v == best && i < idx)) { best = v; idx = i; }
    }
    p.lm_val[blockIdx.x] = best;
    p.lm_idx[blockIdx.x] = idx;
    __threadfence();
    const unsigned old = atom_acqrel_add(p.sync + 1, 1u);
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
      if (i >= 0 && i != 0x7fffffff && (v > best || (v == best && i < idx))) { best = v; idx = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      if (ov > best || (ov == best && oi < idx)) { best = ov; idx = oi; }
    }
    if constexpr (TP) tp_argmax_exchange(p, c.lane, tag_of(c, p.L + 1), best, idx);
    if (c.lane == 0) {
      p.next_tokens[0] = idx;
      if (p.auto_advance) { p.tokens[0] = idx; p.positions[0] = p.positions[0] + 1; }
      // every CTA is past its last poll of this step: open the next epoch
      p.sync[1] = 0u;
      p.sync[0] = c.epoch + 1u;
    }
  }
}

// The fp32 gains / biases an operator multiplies while it gathers are loaded on the critical path of its hop,
// and under the weight stream they do not stay in L2 from one step to the next: an operator that runs well
// before them asks for their lines (evict-last), one line per SM in turn.
__device__ __forceinline__ void prefetch_fparams(const KParams& p, const ConsumerCtx& c, const float* ptr, int nfloats) {
  const char* base = reinterpret_cast<const char*>(ptr);
  const int nlines = (nfloats * 4 + 127) >> 7;
  for (int i = blockIdx.x + c.ctid * gridDim.x; i < nlines; i += c.nct * gridDim.x)
    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(base + (size_t)i * 128));
}

template <bool TP, bool I4>
__device__ __forceinline__ void run_gemv(const KParams& p, ConsumerCtx& c, const Task& t, int task_idx, float* xs,
                                         SmemHdr* hdr, uint8_t* ring, int tok, int probe) {
  // ---- first of all: ask for the first words of the input vector (the round trip overlaps the rest of the preamble) ----
  VecSrc vs;
  vs.src = nullptr; vs.gain = nullptr; vs.n = 0; vs.tag = 0;
  const bool have = !probe && gemv_input<TP>(p, c, t, vs);
  const bool early = have && !TP;
  u64 w0[4] = {0, 0, 0, 0}, w1[4] = {0, 0, 0, 0};
  if (early) {
    const int n4 = vs.n >> 2;
    if (c.ctid < n4) ll_load4(vs.src + 4 * c.ctid, w0);
    if (c.ctid + c.nct < n4) ll_load4(vs.src + 4 * (c.ctid + c.nct), w1);
  }
  stamp(p, c, task_idx, 0);
  if (!probe) {
    if (t.type == T_QKV) {          // this layer's second norm (gate/up runs three operators later)
      prefetch_fparams(p, c, p.fparams + (size_t)t.layer * p.fp_layer_stride + p.fp_ln2, p.H);
    } else if (t.type == T_GATEUP) {  // the next layer's first norm, biases and q/k-norm gains (or the final norm)
      if (t.layer + 1 < p.L) prefetch_fparams(p, c, p.fparams + (size_t)(t.layer + 1) * p.fp_layer_stride, p.fp_layer_stride);
      else prefetch_fparams(p, c, p.fparams + p.fp_final, p.H);
    }
  }
  // ---- before the inputs are awaited: the epilogue operand of the first tile (bias rows are DRAM
  // misses under the weight stream; residual words were completed earlier in this step) ----
  float eop0 = 0.f;
  if (!probe) {
    const int WK = (t.geom >> 8) & 0xff, rw = (t.geom >> 16) & 0xff;
    const int rows0 = min(t.rt, t.b);
    int erow = -1;
    if (WK == 1) {
      const int rsel = ((c.lane >> 4) & 1) * 4 + ((c.lane >> 3) & 1) * 2 + ((c.lane >> 2) & 1);
      if ((c.lane & 3) == 0 && rsel < rw && c.cw * rw + rsel < rows0) erow = c.cw * rw + rsel;
    } else if (c.ctid < rows0) erow = c.ctid;
    set_polling(hdr, c.ctid, 1);
    if (erow >= 0) eop0 = load_eop<TP>(p, c, t, task_idx, t.a + erow, tok);
    gemv_prologue<TP>(p, c, t, task_idx, xs, hdr, tok, vs, have, early, w0, w1);
  }
  stamp(p, c, task_idx, 1);
  gemv_tiles<TP, I4>(p, c, t, task_idx, xs, hdr, ring, tok, eop0, probe);
  if (probe) { stamp(p, c, task_idx, 7); return; }
  stamp(p, c, task_idx, 2);
  if (t.type == T_LMHEAD) lm_finish<TP>(p, c, hdr);
  stamp(p, c, task_idx, 7);
}

// ----------------------------------------------------------------------------------
// attention unit = (q head, context chunk)
// ----------------------------------------------------------------------------------
// Scratch layout (floats), must fit task_table.scratch_bytes:
//   qs[D + 16] | knew[D] | vnew[D] | comb[kAttnWarps][D + 2] | sw[kAttnWarps]
//
// Decode attention is latency, not throughput: a layer's K/V is a few hundred KB but every later
// operator waits for it.  So the work is spread as widely as it goes -- one unit per (q head, chunk
// of the context), the q heads of a group re-reading their K/V blocks from L2 -- and the code of a
// unit is a short loop nest (it runs once per layer per SM; its instruction footprint matters more
// than its FLOPs).  The K and V rows of the chunk arrive through the weight ring (the paper's
// "KV-cache loads advanced into the pipeline window"): per block of 64 positions one K
// stage and one V stage, issued by the Loader long before this layer's QKV projections are done;
// the row of the new token is patched into the staged copy.  Each of the (up to 8) attention warps
// owns 8 positions of a block (4 lanes per position in the score step, lanes over the head dim in
// P.V) with its online-softmax state in registers; the warps are merged once at the end.  The unit
// publishes one partial record (o[D], m, l); the T_MERGE task of the head combines the records of
// its units.  With a single active unit the normalised output is published directly.
template <int D>
__device__ __forceinline__ void run_attn(const KParams& p, ConsumerCtx& c, const Task& t, int task_idx, float* scratch,
                                         SmemHdr* hdr, uint8_t* ring, int pos) {
  constexpr int DL = D / 4;      // dims per lane in the score step (4 lanes per position)
  constexpr int QS = D + 16;     // padded q row: 4 segments of DL floats, 4 floats apart (conflict-free)
  constexpr int DPL = D / 32;    // output dims per lane
  constexpr int RS = D + 2;      // record: o[D], m, l
  const int G = p.G, h = t.a, slot = t.b, kvh = h / G;
  const AttnGeom ge = attn_geometry(p, pos, slot);
  if (slot >= ge.n_active) return;  // no context for this slot at this length
  stamp(p, c, task_idx, 0);
  const int n = ge.n, t0 = ge.t0, nblk = ge.nblk;
  const bool owns_new = (slot == ge.n_active - 1);  // this chunk contains position `pos`
  const bool writes_cache = owns_new && h == kvh * G;  // one unit per kv head appends K/V to the cache
  const unsigned tag = tag_of(c, t.layer);
  const int AW = min(p.C, kAttnWarps);

  float* qs = scratch;
  float* knew = qs + QS;
  float* vnew = knew + D;
  float* comb = vnew + D;                 // [AW][RS]
  float* sw = comb + kAttnWarps * RS;     // [AW]

  const float* lay_fp = p.fparams + (size_t)t.layer * p.fp_layer_stride;
  const size_t head_base = ((size_t)(t.layer * p.batch + t.aux) * p.nkv + kvh) * (size_t)p.max_ctx * D;
  __nv_bfloat16* Kc = p.kcache + head_base;
  __nv_bfloat16* Vc = p.vcache + head_base;
  const uint32_t ring_addr = smem_u32(ring);
  const uint32_t full0 = smem_u32(&hdr->full[0]);
  const uint32_t empty0 = smem_u32(&hdr->empty[0]);
  const uint32_t n_stage = (uint32_t)p.n_stage;

  // ---- q row (+ k, v of the new token in the owner units): gather, (norm), RoPE ----
  // one warp per row of D elements; lane holds elements lane + 32 j so rotate-half partners share a lane
  set_polling(hdr, c.ctid, 1);
  if (c.cw < (owns_new ? 3 : 1)) {
    constexpr int PER = D / 32, HALF = D / 2;
    const bool is_q = c.cw == 0, is_k = c.cw == 1;
    // first of all: ask for the row's words (the round trip overlaps the loads of the static operands)
    const u64* src = p.ll_qkv + (is_q ? (size_t)h * D : (size_t)p.q_dim + (is_k ? 0 : p.kv_dim) + (size_t)kvh * D) + c.lane;
    u64 wr[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) wr[j] = ll_load(src + 32 * j);
    float cs[PER / 2], sn[PER / 2];
#pragma unroll
    for (int j = 0; j < PER / 2; ++j) {  // static operands: DRAM misses the first time a position is used
      cs[j] = __ldg(p.rope_cos + (size_t)pos * HALF + c.lane + 32 * j);
      sn[j] = __ldg(p.rope_sin + (size_t)pos * HALF + c.lane + 32 * j);
    }
    float gn[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) gn[j] = (p.qk_norm && (is_q || is_k)) ? ldg_keep_f1(lay_fp + (is_q ? p.fp_qn : p.fp_kn) + c.lane + 32 * j) : 1.f;
    float v[PER];
    {
      long long t0 = 0;
      for (;;) {
        bool ok = true;
#pragma unroll
        for (int j = 0; j < PER; ++j) ok = ok && ll_tag(wr[j]) == tag;
        if (ok) break;
#pragma unroll
        for (int j = 0; j < PER; ++j) wr[j] = ll_load(src + 32 * j);
        if (t0 == 0) t0 = clock64();
        else if (clock64() - t0 > kWatchdogCycles) dev_fail(p, DE_WATCHDOG_TAG, task_idx, (int)ll_tag(wr[0]), (int)tag, -1);
      }
#pragma unroll
      for (int j = 0; j < PER; ++j) v[j] = ll_val(wr[j]);
    }
    if (!is_q && !is_k) {  // v row: staged patch value (+ cache)
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        vnew[c.lane + 32 * j] = v[j];
        if (writes_cache) Vc[(size_t)pos * D + c.lane + 32 * j] = __float2bfloat16_rn(v[j]);
      }
    } else {
      if (p.qk_norm) {
        float ss = 0.f;
#pragma unroll
        for (int j = 0; j < PER; ++j) ss += v[j] * v[j];
        ss = warp_sum(ss);
        const float rs = rsqrtf(ss / (float)D + p.eps);
#pragma unroll
        for (int j = 0; j < PER; ++j) v[j] = v[j] * rs * gn[j];
      }
      const float scale = is_q ? rsqrtf((float)D) : 1.f;
#pragma unroll
      for (int j = 0; j < PER / 2; ++j) {
        const int d1 = c.lane + 32 * j;  // < HALF
        const float x1 = v[j], x2 = v[j + PER / 2];
        const float y1 = (x1 * cs[j] - x2 * sn[j]) * scale, y2 = (x2 * cs[j] + x1 * sn[j]) * scale;
        if (is_q) {
          qs[d1 + (d1 / DL) * 4] = y1;
          qs[d1 + HALF + ((d1 + HALF) / DL) * 4] = y2;
        } else {
          knew[d1] = y1; knew[d1 + HALF] = y2;
          if (writes_cache) {
            Kc[(size_t)pos * D + d1] = __float2bfloat16_rn(y1);
            Kc[(size_t)pos * D + d1 + HALF] = __float2bfloat16_rn(y2);
          }
        }
      }
    }
  }
  consumer_sync(c.nct);
  set_polling(hdr, c.ctid, 0);
  stamp(p, c, task_idx, 1);

  const int lsub = c.lane & 3, lpos = c.lane >> 2;
  float qf[DL];  // this lane's quarter of the q row
#pragma unroll
  for (int e = 0; e < DL; e += 4) {
    const float4 q4 = *reinterpret_cast<const float4*>(qs + lsub * (DL + 4) + e);
    qf[e] = q4.x; qf[e + 1] = q4.y; qf[e + 2] = q4.z; qf[e + 3] = q4.w;
  }
  float m_run = -INFINITY, l_run = 0.f, o[DPL];
#pragma unroll
  for (int e = 0; e < DPL; ++e) o[e] = 0.f;

#pragma unroll 1
  for (int blk = 0; blk < nblk; ++blk) {
    const bool patch = owns_new && blk == nblk - 1;
    const int new_row = (pos - t0) - blk * p.attn_block;  // row of the new token inside this block (if patch)
    const int nblkpos = min(p.attn_block, n - blk * p.attn_block);
    mbar_wait(p, full0 + c.slot * 8, c.ph, DE_WATCHDOG_FULL, task_idx);   // K stage
    const uint32_t kb = ring_addr + c.slot * (uint32_t)p.stage_bytes;
    const uint32_t kslot = c.slot;
    if (++c.slot == n_stage) { c.slot = 0; c.ph ^= 1u; }
    mbar_wait(p, full0 + c.slot * 8, c.ph, DE_WATCHDOG_FULL, task_idx);   // V stage
    const uint32_t vb = ring_addr + c.slot * (uint32_t)p.stage_bytes;
    const uint32_t vslot = c.slot;
    if (++c.slot == n_stage) { c.slot = 0; c.ph ^= 1u; }
    if (patch) {  // the staged copies predate this step's K / V row: overwrite them (bf16, as the cache holds them)
      for (int d = c.ctid; d < 2 * D; d += c.nct) {
        const bool isv = d >= D;
        const int dd = isv ? d - D : d;
        const unsigned short bits = __bfloat16_as_ushort(__float2bfloat16_rn(isv ? vnew[dd] : knew[dd]));
        asm volatile("st.shared.u16 [%0], %1;" ::"r"((isv ? vb : kb) + (uint32_t)(new_row * D + dd) * 2u), "h"(bits) : "memory");
      }
      consumer_sync(c.nct);
    }
    if (blk == 0) stamp(p, c, task_idx, 4);
    if (c.cw < AW) {
#pragma unroll 1
      for (int j0 = c.cw * 8; j0 < nblkpos; j0 += AW * 8) {  // groups of 8 positions
        const int tl = j0 + lpos;
        const bool valid = tl < nblkpos;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
        {
          const uint32_t krow = kb + (uint32_t)(tl * D + lsub * DL) * 2u;
#pragma unroll
          for (int e = 0; e < DL; e += 8) {
            const uint4 raw = lds128u(krow + e * 2);
            s0 = fmaf(qf[e + 0], bf_lo(raw.x), s0); s1 = fmaf(qf[e + 1], bf_hi(raw.x), s1);
            s2 = fmaf(qf[e + 2], bf_lo(raw.y), s2); s3 = fmaf(qf[e + 3], bf_hi(raw.y), s3);
            s0 = fmaf(qf[e + 4], bf_lo(raw.z), s0); s1 = fmaf(qf[e + 5], bf_hi(raw.z), s1);
            s2 = fmaf(qf[e + 6], bf_lo(raw.w), s2); s3 = fmaf(qf[e + 7], bf_hi(raw.w), s3);
          }
        }
        float sdot = (s0 + s1) + (s2 + s3);
        sdot += __shfl_xor_sync(0xffffffffu, sdot, 1);
        sdot += __shfl_xor_sync(0xffffffffu, sdot, 2);
        sdot = valid ? sdot : -INFINITY;
        float mb = sdot;  // position j0 of the group is always valid -> finite
        mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 4));
        mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 8));
        mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 16));
        const float m_new = fmaxf(m_run, mb);
        const float resc = __expf(m_run - m_new);       // exp(-inf) = 0 on the first group
        const float pj = valid ? __expf(sdot - m_new) : 0.f;
        m_run = m_new;
        l_run = l_run * resc + (lsub == 0 ? pj : 0.f);
#pragma unroll
        for (int e = 0; e < DPL; ++e) o[e] *= resc;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float pg = __shfl_sync(0xffffffffu, pj, 4 * j);
          const int row = min(j0 + j, nblkpos - 1);   // rows past the end carry pg = 0
          if constexpr (DPL == 4) {
            uint2 raw;
            asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(raw.x), "=r"(raw.y) : "r"(vb + (uint32_t)(row * D + c.lane * 4) * 2u));
            o[0] = fmaf(pg, bf_lo(raw.x), o[0]); o[1] = fmaf(pg, bf_hi(raw.x), o[1]);
            o[2] = fmaf(pg, bf_lo(raw.y), o[2]); o[3] = fmaf(pg, bf_hi(raw.y), o[3]);
          } else {
            uint32_t raw;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(raw) : "r"(vb + (uint32_t)(row * D + c.lane * 2) * 2u));
            o[0] = fmaf(pg, bf_lo(raw), o[0]); o[1] = fmaf(pg, bf_hi(raw), o[1]);
          }
        }
      }
    }
    __syncwarp();
    if (c.lane == 0) { mbar_arrive(empty0 + kslot * 8); mbar_arrive(empty0 + vslot * 8); }
  }
  stamp(p, c, task_idx, 3);
  // ---- merge the attention warps ----
  if (c.cw < AW) {
    float l = l_run;
    l += __shfl_xor_sync(0xffffffffu, l, 4);
    l += __shfl_xor_sync(0xffffffffu, l, 8);
    l += __shfl_xor_sync(0xffffffffu, l, 16);
    float* rec = comb + c.cw * RS;
#pragma unroll
    for (int e = 0; e < DPL; ++e) rec[c.lane * DPL + e] = o[e];
    if (c.lane == 0) { rec[D] = m_run; rec[D + 1] = l; }
  }
  consumer_sync(c.nct);
  stamp(p, c, task_idx, 5);
  if (c.ctid < D) {
    const int d = c.ctid;
    float M = -INFINITY;
    for (int w = 0; w < AW; ++w) M = fmaxf(M, comb[w * RS + D]);
    float ov = 0.f, lv = 0.f;
    for (int w = 0; w < AW; ++w) {
      const float wgt = __expf(comb[w * RS + D] - M);   // warps without positions: m = -inf -> weight 0
      ov = fmaf(wgt, comb[w * RS + d], ov);
      lv = fmaf(wgt, comb[w * RS + D + 1], lv);
    }
    if (ge.n_active == 1) {
      for (int r = 0; r < p.rep; ++r) ll_store(p.ll_attn + (size_t)r * p.q_dim + (size_t)h * D + d, ov / lv, tag);
    } else {
      u64* part = p.ll_part + ((size_t)(t.aux * p.nq + h) * p.attn_chunks + slot) * (size_t)RS;
      ll_store(part + d, ov, tag);
      if (d == 0) { ll_store(part + D, M, tag); ll_store(part + D + 1, lv, tag); }
    }
  }
  (void)sw;
  consumer_sync(c.nct);  // the next task overwrites the scratch region
  stamp(p, c, task_idx, 7);
}

// Flash-decoding merge of the split-KV records of one q head: out[d] = sum_s w_s o_s[d] / sum_s w_s l_s,
// w_s = exp(m_s - M).  Thread d (< D) walks the active units with eight independent loads in flight.
__device__ __forceinline__ void run_merge(const KParams& p, ConsumerCtx& c, const Task& t, int task_idx, int pos) {
  if (p.probe) return;
  const AttnGeom ge = attn_geometry(p, pos, 0);
  if (ge.n_active <= 1) return;  // the single unit published the output itself
  stamp(p, c, task_idx, 0);
  const int D = p.D, RS = D + 2, h = t.a;
  const unsigned tag = tag_of(c, t.layer);
  const u64* base = p.ll_part + ((size_t)(t.aux * p.nq + h) * p.attn_chunks) * (size_t)RS;
  const size_t cs = (size_t)RS;
  if (c.ctid < D) {
    const int d = c.ctid;
    float M = -INFINITY, L = 0.f, O = 0.f;
    for (int s0 = 0; s0 < ge.n_active; s0 += 4) {
      u64 wo[4], wm[4], wl[4];
      long long t0 = 0;
      for (;;) {
        bool ok = true;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (s0 + u < ge.n_active) {
            const u64* rec = base + (size_t)(s0 + u) * cs;
            wo[u] = ll_load(rec + d);
            ll_load2(rec + D, wm[u], wl[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (s0 + u < ge.n_active) ok = ok && ll_tag(wo[u]) == tag && ll_tag(wm[u]) == tag && ll_tag(wl[u]) == tag;
        if (ok) break;
        if (p.poll_sleep_ns) __nanosleep(p.poll_sleep_ns);
        if (t0 == 0) t0 = clock64();
        else if (clock64() - t0 > kWatchdogCycles) dev_fail(p, DE_WATCHDOG_TAG, task_idx, (int)ll_tag(wo[0]), (int)tag, s0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (s0 + u < ge.n_active) {
          const float m = ll_val(wm[u]);
          const float Mn = fmaxf(M, m);
          const float a = __expf(M - Mn), b = __expf(m - Mn);
          O = O * a + ll_val(wo[u]) * b;
          L = L * a + ll_val(wl[u]) * b;
          M = Mn;
        }
      }
    }
    for (int r = 0; r < p.rep; ++r) ll_store(p.ll_attn + (size_t)r * p.q_dim + (size_t)h * D + d, O / L, tag);
  }
  stamp(p, c, task_idx, 7);
}

struct WarpArgs {  // passed by value to the out-of-line task bodies so the consumer context stays in registers
  int cw, lane, ctid, nct;
  unsigned epoch;
  uint32_t slot, ph;
  int layer, a, b, aux, task_idx, pos;
};
// ---- fused down projection ---------------------------------------------------------------------------
// T_DOWNK: the SwiGLU outputs of this SM's gate/up rows (act_loc, nk = 60-61 values for Qwen2.5-1.5B) never leave
// the SM: they multiply the SM's own K-slice of the down projection -- columns k0 .. k0 + nk, stored column-major,
// all H rows each -- and the SM publishes H partial rows.  A lane owns eight consecutive rows of a 256-row block
// (one LDS.128 per column), a warp owns the blocks cw, cw + C, ...: no shuffles, no gather, nothing to wait for.
constexpr int kDownkBlocks = 3;   // 256-row blocks per warp at most (H <= 768 C)

__device__ __forceinline__ void st_quad(u64* dst, const float (&v)[4], unsigned tag) {   // one 32-byte sector, two 16-byte stores
  const u64 t = (u64)tag << 32;
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(dst), "l"(t | (u64)__float_as_uint(v[0])), "l"(t | (u64)__float_as_uint(v[1])) : "memory");
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(dst + 2), "l"(t | (u64)__float_as_uint(v[2])), "l"(t | (u64)__float_as_uint(v[3])) : "memory");
}

// `cols` columns of one stage for the NB row blocks of this warp: four columns per iteration, every LDS.128 of
// an iteration issued before the first FFMA2 (the loop is latency-bound otherwise: one warp or two per scheduler).
template <int NB>
__device__ __forceinline__ void downk_stage(uint32_t cb, uint32_t col_bytes, uint32_t blk_step, const float* act, int cols,
                                            bool probe, float2 (&acc)[kDownkBlocks][4]) {
  int j = 0;
#pragma unroll 1
  for (; j + 4 <= cols; j += 4, cb += 4 * col_bytes) {
    uint4 q[4][NB];
    float a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = probe ? 1.f : act[j + u];
#pragma unroll
      for (int i = 0; i < NB; ++i) q[u][i] = lds128u(cb + u * col_bytes + i * blk_step);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float2 a2 = make_float2(a[u], a[u]);
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        acc[i][0] = __ffma2_rn(make_float2(bf_lo(q[u][i].x), bf_hi(q[u][i].x)), a2, acc[i][0]);
        acc[i][1] = __ffma2_rn(make_float2(bf_lo(q[u][i].y), bf_hi(q[u][i].y)), a2, acc[i][1]);
        acc[i][2] = __ffma2_rn(make_float2(bf_lo(q[u][i].z), bf_hi(q[u][i].z)), a2, acc[i][2]);
        acc[i][3] = __ffma2_rn(make_float2(bf_lo(q[u][i].w), bf_hi(q[u][i].w)), a2, acc[i][3]);
      }
    }
  }
#pragma unroll 1
  for (; j < cols; ++j, cb += col_bytes) {
    const float av = probe ? 1.f : act[j];
    const float2 a2 = make_float2(av, av);
    uint4 q[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) q[i] = lds128u(cb + i * blk_step);
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      acc[i][0] = __ffma2_rn(make_float2(bf_lo(q[i].x), bf_hi(q[i].x)), a2, acc[i][0]);
      acc[i][1] = __ffma2_rn(make_float2(bf_lo(q[i].y), bf_hi(q[i].y)), a2, acc[i][1]);
      acc[i][2] = __ffma2_rn(make_float2(bf_lo(q[i].z), bf_hi(q[i].z)), a2, acc[i][2]);
      acc[i][3] = __ffma2_rn(make_float2(bf_lo(q[i].w), bf_hi(q[i].w)), a2, acc[i][3]);
    }
  }
}

// int4 columns (W4A16): a lane's eight rows of a column are one 32-bit word of codes; the caller folds scale * acc into
// its output rows at the end of every group of 128 columns.
template <int NB>
__device__ __forceinline__ void downk_stage_i4(uint32_t cb, uint32_t col_bytes, uint32_t blk_step, const float* act, int cols,
                                               bool probe, float2 (&acc)[kDownkBlocks][4]) {
  int j = 0;
#pragma unroll 1
  for (; j + 4 <= cols; j += 4, cb += 4 * col_bytes) {
    uint32_t q[4][NB];
    float a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = probe ? 1.f : act[j + u];
#pragma unroll
      for (int i = 0; i < NB; ++i) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(q[u][i]) : "r"(cb + u * col_bytes + i * blk_step));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float2 a2 = make_float2(a[u], a[u]);
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        float lo[4], hi[4];
        i4_unpack(q[u][i], lo, hi);
        acc[i][0] = __ffma2_rn(make_float2(lo[0], lo[1]), a2, acc[i][0]);
        acc[i][1] = __ffma2_rn(make_float2(lo[2], lo[3]), a2, acc[i][1]);
        acc[i][2] = __ffma2_rn(make_float2(hi[0], hi[1]), a2, acc[i][2]);
        acc[i][3] = __ffma2_rn(make_float2(hi[2], hi[3]), a2, acc[i][3]);
      }
    }
  }
#pragma unroll 1
  for (; j < cols; ++j, cb += col_bytes) {
    const float av = probe ? 1.f : act[j];
    const float2 a2 = make_float2(av, av);
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      uint32_t q;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(q) : "r"(cb + i * blk_step));
      float lo[4], hi[4];
      i4_unpack(q, lo, hi);
      acc[i][0] = __ffma2_rn(make_float2(lo[0], lo[1]), a2, acc[i][0]);
      acc[i][1] = __ffma2_rn(make_float2(lo[2], lo[3]), a2, acc[i][1]);
      acc[i][2] = __ffma2_rn(make_float2(hi[0], hi[1]), a2, acc[i][2]);
      acc[i][3] = __ffma2_rn(make_float2(hi[2], hi[3]), a2, acc[i][3]);
    }
  }
}

template <bool I4>
__device__ __noinline__ uint32_t run_downk_nl(const KParams& p, WarpArgs w, int nk, int cps, int n_st, float* scratch,
                                              SmemHdr* hdr, uint8_t* ring) {
  const int H = p.H, nblk = H >> 8;
  if (p.trace && w.ctid == 0) p.trace[(size_t)w.task_idx * 8 + 0] = globaltimer_ns();
  const float* act = scratch + ((H + kChunk - 1) / kChunk) * kChunk;
  if (!p.probe) consumer_sync(w.nct);   // every warp's SwiGLU outputs are in act_loc (K-split gate/up tiles end without a barrier)
  const uint32_t full0 = smem_u32(&hdr->full[0]), empty0 = smem_u32(&hdr->empty[0]);
  const uint32_t ring_addr = smem_u32(ring), n_stage = (uint32_t)p.n_stage, stage_bytes = (uint32_t)p.stage_bytes;
  uint32_t slot = w.slot, ph = w.ph;
  float2 acc[kDownkBlocks][4];
#pragma unroll
  for (int i = 0; i < kDownkBlocks; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
  const int probe_mode = p.probe, C = p.C;
  constexpr bool i4 = I4;
  constexpr uint32_t ebits = I4 ? 4u : 16u;   // bits per weight
  const uint32_t lane_off = (uint32_t)(w.cw * 256 + w.lane * 8) * ebits / 8u, blk_step = (uint32_t)C * 32u * ebits, col_bytes = (uint32_t)H * ebits / 8u;
  const bool probe = probe_mode != 0;
  const int nmine = w.cw < nblk ? (nblk - w.cw + C - 1) / C : 0;   // row blocks cw, cw + C, ... of this warp
  int col = 0;
  // W4A16: the slice's fp16 scales [group][H] arrive as a stage of their own and stay in registers (packed pairs);
  // out[] collects scale * acc at the end of every group, acc restarts
  uint4 sc[kDownkBlocks][kDownkGroupsMax];
  float2 out[kDownkBlocks][4];
  int grp = 0;
  if (i4) {
#pragma unroll
    for (int i = 0; i < kDownkBlocks; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) out[i][j] = make_float2(0.f, 0.f);
    const int ng = downk_i4_groups(w.a, nk);
    if (probe_mode != 4) mbar_wait(p, full0 + slot * 8, ph, DE_WATCHDOG_FULL, w.task_idx);
#pragma unroll
    for (int i = 0; i < kDownkBlocks; ++i)
#pragma unroll
      for (int g = 0; g < kDownkGroupsMax; ++g) {
        sc[i][g] = make_uint4(0, 0, 0, 0);
        if (i < nmine && g < ng && probe_mode != 2)
          sc[i][g] = lds128u(ring_addr + slot * stage_bytes + (uint32_t)((g * H + (w.cw + i * C) * 256 + w.lane * 8) * 2));
      }
    if (probe_mode != 4) {
      __syncwarp();
      if (w.lane == 0) mbar_arrive(empty0 + slot * 8);
    }
    if (++slot == n_stage) { slot = 0; ph ^= 1u; }
  }
  auto fold = [&]() {   // end of a group of 128 columns (or of the slice)
#pragma unroll
    for (int i = 0; i < kDownkBlocks; ++i) {
      uint4 s4 = sc[i][0];
#pragma unroll
      for (int g = 1; g < kDownkGroupsMax; ++g) if (grp == g) s4 = sc[i][g];
      const uint32_t sw[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        out[i][j] = __ffma2_rn(h2_to_f2(sw[j]), acc[i][j], out[i][j]);
        acc[i][j] = make_float2(0.f, 0.f);
      }
    }
    ++grp;
  };
#pragma unroll 1
  for (int st = 0; st < n_st; ++st) {
    if (probe_mode != 4) mbar_wait(p, full0 + slot * 8, ph, DE_WATCHDOG_FULL, w.task_idx);
    const int cols = min(cps, nk - col);
    if (probe_mode != 2) {
      const uint32_t cb = ring_addr + slot * stage_bytes + lane_off;
      if (!i4) {
        if (nmine == 1) downk_stage<1>(cb, col_bytes, blk_step, act + col, cols, probe, acc);
        else if (nmine == 2) downk_stage<2>(cb, col_bytes, blk_step, act + col, cols, probe, acc);
        else if (nmine == 3) downk_stage<3>(cb, col_bytes, blk_step, act + col, cols, probe, acc);
      } else {
        int c0 = 0;
        while (c0 < cols) {   // runs of columns inside one group of 128
          const int k_abs = w.a + col + c0;
          const int run = min(cols - c0, kI4Group - (k_abs & (kI4Group - 1)));
          const uint32_t cbr = cb + (uint32_t)c0 * col_bytes;
          if (nmine == 1) downk_stage_i4<1>(cbr, col_bytes, blk_step, act + col + c0, run, probe, acc);
          else if (nmine == 2) downk_stage_i4<2>(cbr, col_bytes, blk_step, act + col + c0, run, probe, acc);
          else if (nmine == 3) downk_stage_i4<3>(cbr, col_bytes, blk_step, act + col + c0, run, probe, acc);
          c0 += run;
          if (((k_abs + run) & (kI4Group - 1)) == 0 || col + c0 == nk) fold();
        }
      }
    }
    col += cols;
    if (probe_mode != 4) {
      __syncwarp();
      if (w.lane == 0) mbar_arrive(empty0 + slot * 8);
    }
    if (++slot == n_stage) { slot = 0; ph ^= 1u; }
  }
  if (i4) {
#pragma unroll
    for (int i = 0; i < kDownkBlocks; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = out[i][j];
  }
  if (probe) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < kDownkBlocks; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) s += acc[i][j].x + acc[i][j].y;
    if (s == 1.2345678e-30f) p.probe_sink[blockIdx.x * 64] = s;
    return slot | (ph << 8);
  }
  // publish: row quad q of SM s lives at part2[(q * n_sms + s) * 4]: a T_HRED task reads its quads of all SMs contiguously
  const unsigned tag = w.epoch * kTagStride + (unsigned)w.layer + 1u;
#pragma unroll
  for (int i = 0; i < kDownkBlocks; ++i) {
    if (i < nmine) {
      const size_t q0 = (size_t)(w.cw + i * C) * 64 + (size_t)w.lane * 2;
      const float lo4[4] = {acc[i][0].x, acc[i][0].y, acc[i][1].x, acc[i][1].y};
      const float hi4[4] = {acc[i][2].x, acc[i][2].y, acc[i][3].x, acc[i][3].y};
      st_quad(p.ll_part2 + (q0 * gridDim.x + blockIdx.x) * 4, lo4, tag);
      st_quad(p.ll_part2 + ((q0 + 1) * gridDim.x + blockIdx.x) * 4, hi4, tag);
    }
  }
  if (p.trace && w.ctid == 0) p.trace[(size_t)w.task_idx * 8 + 2] = globaltimer_ns();
  consumer_sync(w.nct);   // act_loc / the staged gate/up input may be overwritten by the next task
  if (p.trace && w.ctid == 0) p.trace[(size_t)w.task_idx * 8 + 7] = globaltimer_ns();
  return slot | (ph << 8);
}

// T_HRED: rows 4 q0 .. 4 (q0 + nq) of the next layer's input = residual (h_mid) + the sum of every SM's partial
// row, in a fixed order (SMs 32 apart per lane, then the xor tree) -- the result does not depend on timing.
constexpr int kHredQuadsMax = 16;
__device__ __noinline__ void run_hred_nl(const KParams& p, WarpArgs w, int q0, int nq, float* stage) {
  const int S = (int)gridDim.x, SP = S + 1, items = nq * S;
  const unsigned tag = w.epoch * kTagStride + (unsigned)w.layer + 1u;
  const u64* base = p.ll_part2 + (size_t)q0 * S * 4;   // [nq][S][4] contiguous
  // first of all: ask for the first two sectors of this thread and for its residual word
  u64 wa[4] = {0, 0, 0, 0}, wb[4] = {0, 0, 0, 0};
  const int ia = w.ctid, ib = w.ctid + w.nct;
  if (ia < items) ll_load4(base + 4 * (size_t)ia, wa);
  if (ib < items) ll_load4(base + 4 * (size_t)ib, wb);
  const int nrows = nq * 4, C = p.C;
  const u64* res = p.ll_hm + (size_t)(blockIdx.x % p.rep) * p.H + (size_t)q0 * 4;
  // lane k of warp cw finishes row cw + k C (k < 4): its residual word is requested now as well
  const int my_row = w.cw + w.lane * C;
  const bool has_res = w.lane < 4 && my_row < nrows;
  u64 rw0 = 0;
  if (has_res) rw0 = ll_load(res + my_row);
  if (p.trace && w.ctid == 0) p.trace[(size_t)w.task_idx * 8 + 0] = globaltimer_ns();
  for (int i0 = w.ctid; i0 < items; i0 += 2 * w.nct) {
    const int i1 = i0 + w.nct;
    if (i0 != w.ctid) {
      ll_load4(base + 4 * (size_t)i0, wa);
      if (i1 < items) ll_load4(base + 4 * (size_t)i1, wb);
    }
    long long t0 = 0;
    while (!(ll_quad_ok(wa, tag) && (i1 >= items || ll_quad_ok(wb, tag)))) {
      ll_load4(base + 4 * (size_t)i0, wa);
      if (i1 < items) ll_load4(base + 4 * (size_t)i1, wb);
      if (t0 == 0) t0 = clock64();
      else if (clock64() - t0 > kWatchdogCycles) dev_fail(p, DE_WATCHDOG_TAG, w.task_idx, (int)ll_tag(wa[0]), (int)tag, i0);
    }
    {
      const int q = i0 / S, s = i0 - q * S;
#pragma unroll
      for (int j = 0; j < 4; ++j) stage[(q * 4 + j) * SP + s] = ll_val(wa[j]);
    }
    if (i1 < items) {
      const int q = i1 / S, s = i1 - q * S;
#pragma unroll
      for (int j = 0; j < 4; ++j) stage[(q * 4 + j) * SP + s] = ll_val(wb[j]);
    }
  }
  consumer_sync(w.nct);
  if (p.trace && w.ctid == 0) p.trace[(size_t)w.task_idx * 8 + 1] = globaltimer_ns();
  const unsigned tag_out = w.epoch * kTagStride + (unsigned)(w.layer + 1) + 1u;
  float mine = 0.f;
  for (int k = 0; w.cw + k * C < nrows; ++k) {   // rows cw, cw + C, ...: the total of row cw + k C ends up in lane k
    const int r = w.cw + k * C;
    float s = 0.f;
    for (int j = w.lane; j < S; j += 32) s += stage[r * SP + j];
    s = warp_sum(s);
    if (w.lane == (k & 3)) mine = s;
    if ((k & 3) == 3 || r + C >= nrows) {        // lanes 0..3 publish up to four finished rows
      const int kr = (k & ~3) + w.lane, row_l = w.cw + kr * C;
      if (w.lane < 4 && row_l < nrows) {
        u64 rw = (kr == w.lane) ? rw0 : ll_load(res + row_l);
        const long long t0 = clock64();
        while (ll_tag(rw) != tag) {
          rw = ll_load(res + row_l);
          if (clock64() - t0 > kWatchdogCycles) dev_fail(p, DE_WATCHDOG_TAG, w.task_idx, (int)ll_tag(rw), (int)tag, row_l);
        }
        const float v = ll_val(rw) + mine;
        const int row = q0 * 4 + row_l;
        for (int c2 = 0; c2 < p.rep; ++c2)
          ll_store(p.ll_hx + ((size_t)c2 * 2 + (size_t)((w.layer + 1) & 1)) * p.H + row, v, tag_out);
      }
    }
  }
  if (p.trace && w.ctid == 0) p.trace[(size_t)w.task_idx * 8 + 2] = globaltimer_ns();
  consumer_sync(w.nct);   // the next task overwrites the staging array
  if (p.trace && w.ctid == 0) p.trace[(size_t)w.task_idx * 8 + 7] = globaltimer_ns();
}

template <int D>
__device__ __noinline__ uint32_t run_attn_nl(const KParams& p, WarpArgs w, float* scratch, SmemHdr* hdr, uint8_t* ring) {
  ConsumerCtx c;
  c.cw = w.cw; c.lane = w.lane; c.ctid = w.ctid; c.nct = w.nct; c.epoch = w.epoch; c.slot = w.slot; c.ph = w.ph;
  c.rs = 1.f; c.best_val = 0.f; c.best_idx = 0;
  Task t{};
  t.type = T_ATTN; t.layer = w.layer; t.a = w.a; t.b = w.b; t.aux = w.aux;
  run_attn<D>(p, c, t, w.task_idx, scratch, hdr, ring, w.pos);
  return c.slot | (c.ph << 8);
}
// The GEMV task body is out of line as well: its register allocation and instruction schedule then
// depend only on its own code (the hot loop is sensitive to both), not on what else the kernel inlines.
struct GemvArgs {
  int cw, lane, ctid, nct;
  unsigned epoch;
  uint32_t slot, ph;
  int type, layer, a, b, k, kchunks, rt, ktc, n_tiles, n_ktiles, geom, aux;
  int task_idx, tok, probe;
};
template <bool TP, bool I4>
__device__ __noinline__ uint32_t run_gemv_nl(const KParams& p, GemvArgs g, float* xs, SmemHdr* hdr, uint8_t* ring) {
  ConsumerCtx c;
  c.cw = g.cw; c.lane = g.lane; c.ctid = g.ctid; c.nct = g.nct; c.epoch = g.epoch; c.slot = g.slot; c.ph = g.ph;
  c.rs = 1.f; c.best_val = -INFINITY; c.best_idx = -1;
  Task t{};
  t.type = g.type; t.layer = g.layer; t.a = g.a; t.b = g.b; t.k = g.k; t.kchunks = g.kchunks; t.rt = g.rt; t.ktc = g.ktc;
  t.n_tiles = g.n_tiles; t.n_ktiles = g.n_ktiles; t.geom = g.geom; t.aux = g.aux;
  c.act_loc = xs + ((p.H + kChunk - 1) / kChunk) * kChunk;
  run_gemv<TP, I4>(p, c, t, g.task_idx, xs, hdr, ring, g.tok, g.probe);
  return c.slot | (c.ph << 8);
}
// ---- down projection with its input streamed in ------------------------------------------------------
// The down projection reads the longest vector of the layer (I = 8960 words = 72 KB of tagged words per SM
// for Qwen2.5-1.5B).  Its k-tiles are consumed in order, so the words of k-tiles kt+1 .. kt+kXSlots are in
// flight as bulk copies (cp.async.bulk: one request instruction per 4 KB slice, full sectors, no registers
// held) into a small ring of raw slices while k-tile kt is multiplied; a landed slice is checked, converted
// to fp32 and staged in the other half of a double buffer.  A word that was still old when its slice was
// copied is polled directly.  Only the first slice's round trip is exposed.
// Scratch layout: xbuf[2][ktc * 256] fp32 | raw[kXSlots][ktc * 256] words.
constexpr int kXSlots = 4;

__device__ __forceinline__ bool down_is_streamable(const KParams& p, const Task& t, int nct) {
  const int WK = (t.geom >> 8) & 0xff;
  return t.type == T_DOWN && WK == 1 && t.n_tiles == 1 && t.n_ktiles > 1 && t.ktc * (kChunk / 4) <= nct &&
         t.ktc * kChunk * (8 + 8 * kXSlots) <= p.scratch_bytes;
}

template <int RW, bool TP>
__device__ __forceinline__ void down_streamed(const KParams& p, ConsumerCtx& c, const Task& t, int task_idx, float* scratch,
                                              SmemHdr* hdr, uint8_t* ring, int tok) {
  stamp(p, c, task_idx, 0);
  const int rw = (t.geom >> 16) & 0xff;
  const uint32_t ring_addr = smem_u32(ring) + c.lane * 16;
  const uint32_t full0 = smem_u32(&hdr->full[0]), empty0 = smem_u32(&hdr->empty[0]);
  const uint32_t n_stage = (uint32_t)p.n_stage, stage_bytes = (uint32_t)p.stage_bytes;
  const int my_r0 = c.cw * rw;
  const int rsel = ((c.lane >> 4) & 1) * 4 + ((c.lane >> 3) & 1) * 2 + ((c.lane >> 2) & 1);
  const int rows = t.b;
  const int my_n = max(0, min(rw, rows - my_r0));
  int erow = -1;
  if ((c.lane & 3) == 0 && rsel < my_n) erow = my_r0 + rsel;
  float eop = 0.f;
  if (erow >= 0) eop = load_eop<TP>(p, c, t, task_idx, t.a + erow, tok);   // residual: complete since this SM's gate/up task

  const unsigned tag = tag_of(c, t.layer);
  const u64* src = p.ll_act;
  const int n4 = p.I >> 2;                       // 32-byte word quads of the vector
  const int qps = t.ktc * (kChunk / 4);          // quads per full k-tile
  const int q_all = t.kchunks * (kChunk / 4);    // quads including the zero padding of the last chunk
  float* xbuf = scratch;                         // [2][ktc * 256]
  u64* raw = reinterpret_cast<u64*>(scratch + 2 * t.ktc * kChunk);   // [kXSlots][ktc * 256]
  const uint32_t raw_addr = smem_u32(raw);
  const uint32_t xbar0 = smem_u32(&hdr->xbar[0]);
  const int last = t.n_ktiles - 1;

  auto issue_raw = [&](int kt) {                 // one thread: bulk copy of slice kt into raw slot kt % kXSlots
    if (c.ctid == 0 && kt <= last) {
      const int qb = kt * qps, qe = min(min(qb + qps, q_all), n4);
      if (qe > qb) {
        const uint32_t bytes = (uint32_t)(qe - qb) * 32u, bar = xbar0 + (uint32_t)(kt % kXSlots) * 8u;
        mbar_arrive_expect_tx(bar, bytes);
        tma_bulk_g2s(raw_addr + (uint32_t)(kt % kXSlots) * (uint32_t)qps * 32u, src + 4 * (size_t)qb, bytes, bar);
      }
    }
  };
  auto finish_raw = [&](int kt) {                // check, convert, stage slice kt into xbuf[kt & 1]
    const int qb = kt * qps, qe = min(qb + qps, q_all);
    if (min(qe, n4) > qb) mbar_wait(p, xbar0 + (uint32_t)(kt % kXSlots) * 8u, (uint32_t)(kt / kXSlots) & 1u, DE_WATCHDOG_FULL, task_idx);
    float4* dst = reinterpret_cast<float4*>(xbuf + (size_t)(kt & 1) * t.ktc * kChunk);
    const u64* rawk = raw + (size_t)(kt % kXSlots) * 4 * qps;
    const int i = qb + c.ctid;
    if (i < qe) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i < n4) {
        u64 w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) w[j] = rawk[4 * (i - qb) + j];
        if (ll_tag(w[0]) != tag || ll_tag(w[1]) != tag || ll_tag(w[2]) != tag || ll_tag(w[3]) != tag) {
          long long t0 = 0;                       // copied before its producer stored it: poll the sector itself
          for (;;) {
            ll_load4(src + 4 * (size_t)i, w);
            if (ll_tag(w[0]) == tag && ll_tag(w[1]) == tag && ll_tag(w[2]) == tag && ll_tag(w[3]) == tag) break;
            if (t0 == 0) t0 = clock64();
            else if (clock64() - t0 > kWatchdogCycles) dev_fail(p, DE_WATCHDOG_TAG, task_idx, (int)ll_tag(w[0]), (int)tag, i);
          }
        }
        v = make_float4(ll_val(w[0]), ll_val(w[1]), ll_val(w[2]), ll_val(w[3]));
      }
      dst[i - qb] = v;
    }
    consumer_sync(c.nct);
  };

  // the slice barriers start every task in phase 0 (no copy is pending between tasks)
  if (c.ctid == 0) {
#pragma unroll
    for (int s2 = 0; s2 < kXSlots; ++s2) mbar_init(xbar0 + s2 * 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  // first slice: wait until its words are current before asking for copies (a copy cannot re-poll)
  set_polling(hdr, c.ctid, 1);
  if (c.ctid < min(qps, n4)) ll_spin(p, src + 4 * (size_t)c.ctid, tag, task_idx);
  consumer_sync(c.nct);
  set_polling(hdr, c.ctid, 0);
#pragma unroll
  for (int s2 = 0; s2 < kXSlots; ++s2) issue_raw(s2);
  finish_raw(0);
  issue_raw(kXSlots);
  stamp(p, c, task_idx, 1);

  const int chunks_last = t.kchunks - last * t.ktc;
  const uint32_t rs_full = (uint32_t)t.ktc * 512u, rs_last = (uint32_t)chunks_last * 512u;
  float2 acc[kRW];
#pragma unroll
  for (int i = 0; i < kRW; ++i) acc[i] = make_float2(0.f, 0.f);
  uint32_t slot = c.slot, ph = c.ph;
#pragma unroll 1
  for (int kt = 0; kt <= last; ++kt) {
    mbar_wait(p, full0 + slot * 8, ph, DE_WATCHDOG_FULL, task_idx);
    if (my_n > 0) {
      const bool is_last = kt == last;
      const uint32_t rs = is_last ? rs_last : rs_full;
      gemv_stage<RW>(ring_addr + slot * stage_bytes + (uint32_t)my_r0 * rs, rs,
                     smem_u32(xbuf + (size_t)(kt & 1) * t.ktc * kChunk) + c.lane * 16, is_last ? chunks_last : t.ktc, 1, acc);
    }
    __syncwarp();
    if (c.lane == 0) mbar_arrive(empty0 + slot * 8);
    if (++slot == n_stage) { slot = 0; ph ^= 1u; }
    if (kt < last) {
      finish_raw(kt + 1);
      issue_raw(kt + 1 + kXSlots);
    }
  }
  c.slot = slot; c.ph = ph;
  float v[kRW];
#pragma unroll
  for (int i = 0; i < kRW; ++i) v[i] = acc[i].x + acc[i].y;
  const float sres = reduce8(v, c.lane);
  if (erow >= 0) gemv_epilogue<TP>(p, c, t, t.a + erow, sres, 0.f, eop);
  stamp(p, c, task_idx, 2);
  consumer_sync(c.nct);   // the next task overwrites the scratch region
  stamp(p, c, task_idx, 7);
}

template <bool TP>
__device__ __noinline__ uint32_t run_down_streamed_nl(const KParams& p, GemvArgs g, float* xs, SmemHdr* hdr, uint8_t* ring) {
  ConsumerCtx c;
  c.cw = g.cw; c.lane = g.lane; c.ctid = g.ctid; c.nct = g.nct; c.epoch = g.epoch; c.slot = g.slot; c.ph = g.ph;
  c.rs = 1.f; c.best_val = -INFINITY; c.best_idx = -1;
  Task t{};
  t.type = g.type; t.layer = g.layer; t.a = g.a; t.b = g.b; t.k = g.k; t.kchunks = g.kchunks; t.rt = g.rt; t.ktc = g.ktc;
  t.n_tiles = g.n_tiles; t.n_ktiles = g.n_ktiles; t.geom = g.geom;
  switch ((((t.geom >> 16) & 0xff) + 1) >> 1) {
    case 1: down_streamed<2, TP>(p, c, t, g.task_idx, xs, hdr, ring, g.tok); break;
    case 2: down_streamed<4, TP>(p, c, t, g.task_idx, xs, hdr, ring, g.tok); break;
    case 3: down_streamed<6, TP>(p, c, t, g.task_idx, xs, hdr, ring, g.tok); break;
    default: down_streamed<8, TP>(p, c, t, g.task_idx, xs, hdr, ring, g.tok); break;
  }
  return c.slot | (c.ph << 8);
}

__device__ __noinline__ void run_merge_nl(const KParams& p, WarpArgs w) {
  ConsumerCtx c;
  c.cw = w.cw; c.lane = w.lane; c.ctid = w.ctid; c.nct = w.nct; c.epoch = w.epoch; c.slot = w.slot; c.ph = w.ph;
  c.rs = 1.f; c.best_val = 0.f; c.best_idx = 0;
  Task t{};
  t.type = T_MERGE; t.layer = w.layer; t.a = w.a; t.aux = w.aux;
  run_merge(p, c, t, w.task_idx, w.pos);
}

// ----------------------------------------------------------------------------------
// the persistent kernel
// ----------------------------------------------------------------------------------
template <int CW, bool TP>
__global__ void __launch_bounds__((CW + 1) * 32, 1) adamk_decode_kernel(const __grid_constant__ KParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  SmemHdr* hdr = reinterpret_cast<SmemHdr*>(smem);
  int4* tcache = reinterpret_cast<int4*>(smem + kSmemReserved);
  float* scratch = reinterpret_cast<float*>(smem + kSmemReserved + p.task_cache_bytes);
  uint8_t* ring = smem + kSmemReserved + p.task_cache_bytes + p.scratch_bytes;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tb = p.sm_begin[blockIdx.x], te = p.sm_begin[blockIdx.x + 1];
  // This SM's task records -> shared memory, packed to 32 bytes (a record in global memory is a DRAM / L2
  // round trip under the weight stream; short tasks would expose it every time).
  for (int i = threadIdx.x; i < te - tb; i += blockDim.x) {
    const int4* tp = reinterpret_cast<const int4*>(p.tasks + tb + i);
    const int4 a = __ldg(tp), b = __ldg(tp + 1), cc = __ldg(tp + 2), d = __ldg(tp + 3);
    // type | layer << 8 | aux << 20, a, b | rt << 16, kchunks | ktc << 16   ;   n_tiles | n_ktiles << 16, w_off, geom, k
    tcache[2 * i] = make_int4(a.x | (a.y << 8) | (d.w << 20), a.z, a.w | (b.z << 16), b.y | (b.w << 16));
    tcache[2 * i + 1] = make_int4(cc.x | (cc.y << 16), cc.z, cc.w, b.x);
  }
  {
    const uint32_t* ksrc = reinterpret_cast<const uint32_t*>(&p);
    uint32_t* kdst = reinterpret_cast<uint32_t*>(&hdr->kp);
    for (int i = threadIdx.x; i < (int)(sizeof(KParams) / 4); i += blockDim.x) kdst[i] = ksrc[i];
  }
  const KParams& kp = hdr->kp;   // what the out-of-line task bodies read
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.n_stage; ++s) {
      mbar_init(smem_u32(&hdr->full[s]), 1);
      mbar_init(smem_u32(&hdr->empty[s]), (uint32_t)p.C);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    hdr->misc[kMiscPolling] = 0;
  }
  __syncthreads();
  auto fetch_task = [&](int ti) {  // ti relative to tb
    const int4 u = tcache[2 * ti], v = tcache[2 * ti + 1];
    Task t;
    t.type = u.x & 0xff; t.layer = (u.x >> 8) & 0xfff; t.aux = (int)((unsigned)u.x >> 20); t.a = u.y;
    t.b = u.z & 0xffff; t.rt = (int)((unsigned)u.z >> 16); t.kchunks = u.w & 0xffff; t.ktc = (int)((unsigned)u.w >> 16);
    t.n_tiles = v.x & 0xffff; t.n_ktiles = (int)((unsigned)v.x >> 16); t.w_off = v.y; t.geom = v.z; t.k = v.w;
    t.r12 = t.r13 = t.r14 = 0;
    return t;
  };

  if (warp == 0) {
    // ------------------------------ Loader ------------------------------
    if (lane == 0 && p.probe != 4) {
      uint32_t slot = 0, ph = 0;          // next slot to fill
      uint32_t wslot = 0, wph = 0;        // oldest stage that may still be in flight
      int issued = 0, retired = 0;
      volatile int* polling = reinterpret_cast<volatile int*>(&hdr->misc[kMiscPolling]);
      const int cap = (p.inflight > 0 && p.inflight < p.n_stage) ? p.inflight : p.n_stage;
      const uint32_t ring_addr = smem_u32(ring);
      const uint32_t n_stage = (uint32_t)p.n_stage;
      const uint64_t pol = l2_evict_first_policy();  // weights are read once per step
      if (!p.probe) {
        // The fp32 gains / biases (a few hundred KB for the whole model) are needed on the critical path of
        // every hop: bring them into L2 now, evict-last, one 128-byte line per SM in turn.
        const char* fpb = reinterpret_cast<const char*>(p.fparams);
        for (unsigned off = blockIdx.x * 128u; off < p.fp_bytes; off += gridDim.x * 128u)
          asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(fpb + off));
      }
      int lpos = 0;
      if (!p.probe) {
        lpos = __ldcg(p.positions);
        if (lpos < 0 || lpos >= p.max_ctx) return;  // the consumers report the error
      }
      // While the ring is full (consumers waiting on another SM) the Loader keeps HBM busy by
      // prefetching its own upcoming weight stages into L2, up to pf_window bytes past the ring.
      const uint8_t* wcur = p.wpacked + (size_t)p.sm_stream[blockIdx.x] * 16u;        // next weight byte the ring will load
      const uint8_t* const wend = p.wpacked + (size_t)p.sm_stream[blockIdx.x + 1] * 16u;
      const uint8_t* pf = wcur;
      unsigned n_pf = 0;  // L2 prefetch granules issued this step (debug counter in sync[4])
      constexpr uint32_t kPfGranule = 8192;
      // Pacing.  Every request that reaches DRAM queues behind the ones already there, and so does every tagged-word
      // poll that shares the L2 slice queues with them: an unpaced Loader (148 SMs x ring + prefetch window, all
      // issued at once) keeps megabytes queued and the loaded L2 round trip of a hop grows from ~0.15 us to > 1 us.
      // So the NEW bytes this SM asks HBM for (the frontier `pf`: L2 prefetch granules, or ring stages the prefetch
      // has not covered) are metered at pace_clk_per_64k clocks per 64 KB -- the SM's share of the HBM rate --
      // with a small burst allowance; ring stages behind the frontier are L2 hits and are not metered.
      const long long pace = p.pace_clk_per_64k;
      constexpr long long kPaceBurstClk = 512;
      long long next_ok = clock64();
      auto pace_charge = [&](uint32_t nb) {
        const long long now = clock64();
        next_ok = max(next_ok, now - kPaceBurstClk) + (((long long)nb * pace) >> 16);
      };
      auto blocked_wait = [&](uint32_t bar, uint32_t parity, int code, int ti) {
        if (mbar_test_wait(bar, parity)) return;   // test, not try: try_wait may suspend the lane for its whole time limit, and that time is the prefetcher's
        if (p.pf_window_bytes > 0 && !p.probe) {
          const long long t0 = clock64();
          if (pf < wcur) pf = wcur;
          while (pf < wend && pf < wcur + p.pf_window_bytes) {
            if (mbar_test_wait(bar, parity)) return;
            if (p.poll_inflight && p.poll_inflight != 9 && *polling) {
              if (clock64() - t0 > kWatchdogCycles) dev_fail(p, code, ti, (int)bar, (int)parity, 0);
              continue;   // the consumers are polling: no new HBM requests from this SM
            }
            if (pace) {
              const long long now = clock64();
              if (now < next_ok) {
                if (now - t0 > kWatchdogCycles) dev_fail(p, code, ti, (int)bar, (int)parity, 0);
                continue;   // budget not open yet: keep watching the barrier
              }
            }
            const uint32_t nb = (uint32_t)min((size_t)kPfGranule, (size_t)(wend - pf));
            l2_prefetch_bulk(pf, nb, pol);
            pf += nb;
            ++n_pf;
            if (pace) pace_charge(nb);
            if (clock64() - t0 > kWatchdogCycles) dev_fail(p, code, ti, (int)bar, (int)parity, 0);
          }
        }
        mbar_wait_slow(p, bar, parity, code, ti);
      };
      auto issue = [&](const void* src, uint32_t bytes, bool hint, int ti) {
        // at most `cap` stages in flight (`poll_inflight` while the consumers poll): wait for the oldest one to land
        if (p.poll_inflight == 9 && !p.probe) {   // ring fills return data to THIS SM ahead of its poll replies: hold them, keep the L2 prefetch going
          const long long t0 = clock64();
          while (*polling) {
            if (p.pf_window_bytes > 0) {
              if (pf < wcur) pf = wcur;
              if (pf < wend && pf < wcur + p.pf_window_bytes) {
                const uint32_t nb = (uint32_t)min((size_t)kPfGranule, (size_t)(wend - pf));
                l2_prefetch_bulk(pf, nb, pol);
                pf += nb;
                ++n_pf;
              }
            }
            if (clock64() - t0 > kWatchdogCycles) dev_fail(p, DE_WATCHDOG_INFLIGHT, ti, 9, 0, 0);
          }
        }
        while (issued - retired >= ((p.poll_inflight && p.poll_inflight != 9 && *polling) ? p.poll_inflight : cap)) {
          blocked_wait(smem_u32(&hdr->full[wslot]), wph, DE_WATCHDOG_INFLIGHT, ti);
          if (++wslot == n_stage) { wslot = 0; wph ^= 1u; }
          ++retired;
        }
        blocked_wait(smem_u32(&hdr->empty[slot]), ph ^ 1u, DE_WATCHDOG_EMPTY, ti);
        if (pace && hint && p.probe != 3) {   // weight stage: meter the part the prefetch frontier has not covered
          const uint8_t* e = static_cast<const uint8_t*>(src) + bytes;
          if (e > pf) {
            while (clock64() < next_ok) {}
            const uint8_t* b0 = static_cast<const uint8_t*>(src);
            pace_charge((uint32_t)(e - (pf > b0 ? pf : b0)));
            pf = e;
          }
        }
        const uint32_t fb = smem_u32(&hdr->full[slot]);
        mbar_arrive_expect_tx(fb, bytes);
        if (hint) tma_bulk_g2s_hint(ring_addr + slot * (uint32_t)p.stage_bytes, src, bytes, fb, pol);
        else tma_bulk_g2s(ring_addr + slot * (uint32_t)p.stage_bytes, src, bytes, fb);
        if (++slot == n_stage) { slot = 0; ph ^= 1u; }
        ++issued;
      };
      for (int ti = tb; ti < te; ++ti) {
        const Task lt = fetch_task(ti - tb);
        const int type = lt.type, nrows = lt.b, kchunks = lt.kchunks, rt = lt.rt, ktc = lt.ktc;
        const int n_tiles = lt.n_tiles, n_ktiles = lt.n_ktiles;
        if (type == T_END || type == T_MERGE || type == T_HRED) continue;
        if (type == T_DOWNK) {   // nrows = columns of the SM's K-slice, kchunks = columns per stage, lt.k = H rows per column
          const uint8_t* src = p.wpacked + (size_t)(uint32_t)lt.w_off * 16u;
          const bool i4 = (lt.aux & 2) != 0;
          if (i4) {              // first the fp16 scales of the groups the slice touches: [group][H]
            const uint32_t bytes = (uint32_t)downk_i4_groups(lt.a, nrows) * (uint32_t)lt.k * 2u;
            issue(src, bytes, true, ti);
            src += bytes;
            wcur = src;
          }
          for (int col = 0; col < nrows; col += kchunks) {
            const uint32_t bytes = (uint32_t)min(kchunks, nrows - col) * (uint32_t)lt.k * (i4 ? 1u : 4u) / 2u;
            issue(src, bytes, true, ti);
            src += bytes;
            wcur = src;
          }
          continue;
        }
        if (type == T_ATTN) {
          // K / V blocks of this unit's context chunk, one ring stage each (skipped in probe mode)
          if (p.probe) continue;
          const AttnGeom ge = attn_geometry(p, lpos, lt.b);
          if (lt.b >= ge.n_active) continue;
          const size_t head_base = ((size_t)(lt.layer * p.batch + lt.aux) * p.nkv + lt.a / p.G) * (size_t)p.max_ctx * p.D;
          for (int blk = 0; blk < ge.nblk; ++blk) {
            const int nb = min(p.attn_block, ge.n - blk * p.attn_block);
            const uint32_t bytes = (uint32_t)nb * (uint32_t)p.D * 2u;
            const size_t off = head_base + (size_t)(ge.t0 + blk * p.attn_block) * p.D;
            issue(p.kcache + off, bytes, false, ti);
            issue(p.vcache + off, bytes, false, ti);
          }
          continue;
        }
        const uint8_t* src = p.wpacked + (size_t)(uint32_t)lt.w_off * 16u;
        for (int tile = 0; tile < n_tiles; ++tile) {
          const int rows = min(rt, nrows - tile * rt);
          for (int kt = 0; kt < n_ktiles; ++kt) {
            const int chunks = min(ktc, kchunks - kt * ktc);
            const uint32_t bytes = (lt.aux & 2) ? i4_stage_bytes(rows, chunks) : (uint32_t)rows * (uint32_t)chunks * 512u;
            const uint8_t* lsrc = src;
            if (p.probe == 3) lsrc = p.wpacked + (size_t)p.sm_stream[blockIdx.x] * 16u + ((size_t)(src - p.wpacked) & 0x3ffffu & ~(size_t)0xffff);
            issue(lsrc, bytes, true, ti);
            src += bytes;
            wcur = src;
          }
        }
      }
      if (n_pf && p.sync) atomicAdd(p.sync + 4, n_pf);
    }
    return;
  }

  // ------------------------------ Consumers ------------------------------
  ConsumerCtx c;
  c.slot = 0; c.ph = 0; c.cw = warp - 1; c.lane = lane; c.ctid = threadIdx.x - 32; c.nct = p.C * 32;
  c.rs = 1.0f; c.best_val = -INFINITY; c.best_idx = -1; c.epoch = 0;
  int tok = 0, pos = 0;
  const int probe = p.probe;
  if (!probe) {
    tok = __ldcg(p.tokens);
    pos = __ldcg(p.positions);
    c.epoch = ld_relaxed_u32(p.sync);
    if (pos < 0 || pos >= p.max_ctx || tok < 0 || tok >= p.V * p.tp_size) {
      if (c.ctid == 0) dev_fail(p, DE_BAD_POS, -1, pos, tok, p.max_ctx);
      return;
    }
  }
  for (int ti = tb; ti < te; ++ti) {
    const Task t = fetch_task(ti - tb);
    if (t.type == T_DOWNK || t.type == T_HRED) {
      if (probe && t.type == T_HRED) continue;
      WarpArgs w;
      w.cw = c.cw; w.lane = c.lane; w.ctid = c.ctid; w.nct = c.nct; w.epoch = c.epoch; w.slot = c.slot; w.ph = c.ph;
      w.layer = t.layer; w.a = t.a; w.b = t.b; w.aux = t.aux; w.task_idx = ti; w.pos = pos;
      if (t.type == T_HRED) {
        set_polling(hdr, c.ctid, 1);
        run_hred_nl(kp, w, t.a, t.b, scratch);
        set_polling(hdr, c.ctid, 0);
      }
      else {
        const uint32_t sp = (t.aux & 2) ? run_downk_nl<true>(kp, w, t.b, t.kchunks, t.n_ktiles, scratch, hdr, ring)
                                        : run_downk_nl<false>(kp, w, t.b, t.kchunks, t.n_ktiles, scratch, hdr, ring);
        c.slot = sp & 0xffu; c.ph = sp >> 8;
      }
    } else if (t.type == T_ATTN || t.type == T_MERGE) {
      if (probe) continue;
      WarpArgs w;
      w.cw = c.cw; w.lane = c.lane; w.ctid = c.ctid; w.nct = c.nct; w.epoch = c.epoch; w.slot = c.slot; w.ph = c.ph;
      w.layer = t.layer; w.a = t.a; w.b = t.b; w.aux = t.aux; w.task_idx = ti; w.pos = pos;
      if (t.type == T_MERGE) run_merge_nl(kp, w);
      else {
        const uint32_t sp = (p.D == 128) ? run_attn_nl<128>(kp, w, scratch, hdr, ring) : run_attn_nl<64>(kp, w, scratch, hdr, ring);
        c.slot = sp & 0xffu; c.ph = sp >> 8;
      }
    } else if (t.type != T_END) {
      GemvArgs g;
      g.cw = c.cw; g.lane = c.lane; g.ctid = c.ctid; g.nct = c.nct; g.epoch = c.epoch; g.slot = c.slot; g.ph = c.ph;
      g.type = t.type; g.layer = t.layer; g.a = t.a; g.b = t.b; g.k = t.k; g.kchunks = t.kchunks; g.rt = t.rt; g.ktc = t.ktc;
      g.n_tiles = t.n_tiles; g.n_ktiles = t.n_ktiles; g.geom = t.geom; g.aux = t.aux; g.task_idx = ti; g.tok = tok; g.probe = probe;
      const uint32_t sp = (!probe && p.stream_down && down_is_streamable(p, t, c.nct)) ? run_down_streamed_nl<TP>(kp, g, scratch, hdr, ring)
                          : (!TP && (t.aux & 2))                                        ? run_gemv_nl<false, true>(kp, g, scratch, hdr, ring)
                                                                                       : run_gemv_nl<TP, false>(kp, g, scratch, hdr, ring);
      c.slot = sp & 0xffu; c.ph = sp >> 8;
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
  const AdamkW4A16Layer* qlayers;   // device copy (W4A16 tables) or nullptr
};

__device__ __forceinline__ bool is_gemv(int type) { return type == T_QKV || type == T_OPROJ || type == T_GATEUP || type == T_DOWN || type == T_LMHEAD; }

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

// W4A16 source of a virtual row: codes, scales, K
__device__ __forceinline__ void resolve_row_i4(const PackParams& pp, const Task& t, int vrow, const uint8_t** q, const __half** sc, int* K) {
  const AdamkW4A16Layer& L = pp.qlayers[t.layer];
  const void* qm; const void* sm; int row, k;
  switch (t.type) {
    case T_QKV:
      k = pp.H;
      if (vrow < pp.q_dim) { qm = L.q_wq; sm = L.s_wq; row = vrow; }
      else if (vrow < pp.q_dim + pp.kv_dim) { qm = L.q_wk; sm = L.s_wk; row = vrow - pp.q_dim; }
      else { qm = L.q_wv; sm = L.s_wv; row = vrow - pp.q_dim - pp.kv_dim; }
      break;
    case T_OPROJ: k = pp.q_dim; qm = L.q_wo; sm = L.s_wo; row = vrow; break;
    default:      // T_GATEUP
      k = pp.H; row = vrow >> 1;
      if (vrow & 1) { qm = L.q_wup; sm = L.s_wup; } else { qm = L.q_wgate; sm = L.s_wgate; }
      break;
  }
  *K = k;
  *q = static_cast<const uint8_t*>(qm) + (size_t)row * (k / 2);
  *sc = static_cast<const __half*>(sm) + (size_t)row * ((k + kI4Group - 1) / kI4Group);
}
__device__ __forceinline__ unsigned code_at(const uint8_t* q, int k, int K) {   // 8 (= zero) past the end of the row
  if (k >= K) return 8u;
  const unsigned b = q[k >> 1];
  return (k & 1) ? (b >> 4) : (b & 15u);
}
__device__ void pack_task_i4(const PackParams& pp, const Task& t) {
  uint8_t* dst = pp.wpacked + (size_t)(uint32_t)t.w_off * 16u;
  if (t.type == T_DOWNK) {
    const AdamkW4A16Layer& L = pp.qlayers[t.layer];
    const uint8_t* qd = static_cast<const uint8_t*>(L.q_wdown);
    const __half* sd = static_cast<const __half*>(L.s_wdown);
    const int H = pp.H, ng_row = (pp.I + kI4Group - 1) / kI4Group, g0 = t.a / kI4Group, ng = downk_i4_groups(t.a, t.b);
    __half* sdst = reinterpret_cast<__half*>(dst);
    for (int e = threadIdx.x; e < ng * H; e += blockDim.x) {   // [group][row]
      const int g = e / H, r = e - g * H;
      sdst[e] = sd[(size_t)r * ng_row + g0 + g];
    }
    uint8_t* cdst = dst + (size_t)ng * H * 2;
    for (int e = threadIdx.x; e < t.b * (H / 2); e += blockDim.x) {   // column j: byte b holds rows 2b (low) and 2b + 1
      const int j = e / (H / 2), b = e - j * (H / 2), k = t.a + j;
      const unsigned lo = code_at(qd + (size_t)(2 * b) * (pp.I / 2), k, pp.I), hi = code_at(qd + (size_t)(2 * b + 1) * (pp.I / 2), k, pp.I);
      cdst[e] = (uint8_t)(lo | (hi << 4));
    }
    return;
  }
  for (int tile = 0; tile < t.n_tiles; ++tile) {
    const int rows = min(t.rt, t.b - tile * t.rt);
    for (int kt = 0; kt < t.n_ktiles; ++kt) {
      const int chunks = min(t.ktc, t.kchunks - kt * t.ktc);
      const int nblk = rows * chunks;
      for (int e = threadIdx.x; e < nblk * kI4ChunkBytes; e += blockDim.x) {
        const int blk = e / kI4ChunkBytes, b = e - blk * kI4ChunkBytes, r = blk / chunks, ch = blk - r * chunks;
        const int lane = b >> 2, pair = b & 3;          // byte `pair` of lane's word: elements 2 pair, 2 pair + 1 of its eight
        const uint8_t* q; const __half* sc; int K;
        resolve_row_i4(pp, t, t.a + tile * t.rt + r, &q, &sc, &K);
        const int kbase = (kt * t.ktc + ch) * kChunk;
        unsigned v = 0;
        for (int h2 = 0; h2 < 2; ++h2) {
          const int el = 2 * pair + h2;                 // 0-3: offsets 4 lane + el; 4-7: 128 + 4 lane + el - 4
          const int k = kbase + (el < 4 ? 4 * lane + el : 128 + 4 * lane + (el - 4));
          v |= code_at(q, k, K) << (4 * h2);
        }
        dst[e] = (uint8_t)v;
      }
      __half* sdst = reinterpret_cast<__half*>(dst + (size_t)nblk * kI4ChunkBytes);
      for (int e = threadIdx.x; e < nblk * 2; e += blockDim.x) {
        const int blk = e >> 1, r = blk / chunks, ch = blk - r * chunks;
        const uint8_t* q; const __half* sc; int K;
        resolve_row_i4(pp, t, t.a + tile * t.rt + r, &q, &sc, &K);
        const int g = ((kt * t.ktc + ch) * kChunk) / kI4Group + (e & 1);
        sdst[e] = g < (K + kI4Group - 1) / kI4Group ? sc[g] : __float2half(0.f);
      }
      for (uint32_t e = (uint32_t)nblk * (kI4ChunkBytes + kI4ScaleBytes) + threadIdx.x; e < i4_stage_bytes(rows, chunks); e += blockDim.x)
        dst[e] = 0;      // alignment padding of the stage
      dst += i4_stage_bytes(rows, chunks);
    }
  }
}

__global__ void adamk_pack_kernel(const PackParams pp) {
  const int ti = blockIdx.x;
  if (ti >= pp.n_tasks) return;
  const Task t = pp.tasks[ti];
  if ((t.aux & 2) && pp.qlayers != nullptr) { pack_task_i4(pp, t); return; }
  if (t.type == T_DOWNK) {   // columns t.a .. t.a + t.b of the down projection [H][I], each as H consecutive rows
    __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(pp.wpacked + (size_t)(uint32_t)t.w_off * 16u);
    const __nv_bfloat16* wd = (const __nv_bfloat16*)pp.layers[t.layer].wdown;
    const int n = t.b * pp.H;
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
      const int j = e / pp.H, r = e - j * pp.H;
      d[e] = wd[(size_t)r * pp.I + t.a + j];
    }
    return;
  }
  if (!is_gemv(t.type)) return;
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

// bytes of the packed weight stream a task owns (keep in sync with task_table.task_weight_bytes)
static size_t task_stream_bytes(const Task& t) {
  const bool i4 = (t.aux & 2) != 0;
  if (t.type == T_DOWNK) return i4 ? (size_t)downk_i4_groups(t.a, t.b) * t.k * 2 + (size_t)t.b * t.k / 2 : (size_t)t.b * t.k * 2;
  if (t.type == T_ATTN || t.type == T_MERGE || t.type == T_HRED) return 0;
  if (!i4) return (size_t)t.b * t.kchunks * 512;
  size_t total = 0;
  for (int tile = 0; tile < t.n_tiles; ++tile) {
    const int rows = std::min(t.rt, t.b - tile * t.rt);
    for (int kt = 0; kt < t.n_ktiles; ++kt) total += i4_stage_bytes(rows, std::min(t.ktc, t.kchunks - kt * t.ktc));
  }
  return total;
}

struct AdamkHandle_ {
  AdamkModelDesc desc{};
  int n_sms = 0, C = 0, n_stage = 0, stage_bytes = 0, n_tasks = 0, batch = 0, inflight = 0;
  int attn_chunks = 0, attn_min_chunk = 0, scratch_bytes = 0, n_lm_tasks = 0, poll_sleep_ns = 0, task_cache_bytes = 0, pf_window_kb = 0, pace = 0, poll_inflight = 0, fuse_down = 0, w4a16 = 0;
  int device = 0, dev_sms = 0;     // the device current at adamk_create owns the handle
  const unsigned* d_sm_stream = nullptr;
  size_t packed_weight_bytes = 0;  // matrix streams only
  size_t fparam_floats = 0;
  int fp_layer_stride = 0, fp_ln1 = 0, fp_ln2 = 0, fp_bias = 0, fp_qn = 0, fp_kn = 0, fp_final = 0;
  std::vector<int> host_table;
  int* d_table = nullptr;  // tasks + sm_begin + sm_stream
  const int* d_sm_begin = nullptr;
  const Task* d_tasks = nullptr;
  bool bound = false;
  const uint8_t* wpacked = nullptr;
  const float* fparams = nullptr;
  AdamkWeightPtrs w{};
  int stream_down = 1;
  int tp_rank = 0, tp_size = 1, rep = 1;
  void* peer_ws[kMaxTP] = {nullptr};
  bool peers_bound = false;
  int* status_host = nullptr;
  int* status_dev = nullptr;
  unsigned long long* trace = nullptr;
  int smem_bytes = 0;
  // workspace layout (byte offsets)
  size_t ws_lmx = 0;
  size_t ws_part2 = 0;
  size_t ws_sync = 0, ws_hx = 0, ws_hm = 0, ws_qkv = 0, ws_attn = 0, ws_act = 0, ws_part = 0, ws_lm_val = 0,
         ws_lm_idx = 0, ws_total = 0;
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
  if ((tp_size != 1 && tp_size != 2 && tp_size != 4 && tp_size != 8) || tp_rank < 0 || tp_rank >= tp_size)
    return fail(ADAMK_E_INVALID, "tp_size must be 1, 2, 4 or 8 and 0 <= tp_rank < tp_size");
  if (task_table_bytes < (size_t)kHeaderInts * 4 || task_table_bytes % 4) return fail(ADAMK_E_INVALID, "task table too small");
  const int* tt = static_cast<const int*>(task_table);
  if (tt[0] != kMagic || tt[1] != kVersion) return fail(ADAMK_E_INVALID, "task table magic/version mismatch");
  auto h = new AdamkHandle_();
  h->desc = *desc;
  h->tp_rank = tp_rank; h->tp_size = tp_size;
  if (cudaGetDevice(&h->device) != cudaSuccess ||
      cudaDeviceGetAttribute(&h->dev_sms, cudaDevAttrMultiProcessorCount, h->device) != cudaSuccess) {
    delete h;
    return fail(ADAMK_E_CUDA, "no current CUDA device");
  }
  h->n_sms = tt[2]; h->C = tt[3]; h->n_stage = tt[4]; h->stage_bytes = tt[5]; h->n_tasks = tt[6]; h->batch = tt[7];
  h->inflight = tt[8]; h->attn_chunks = tt[9]; h->attn_min_chunk = tt[10]; h->scratch_bytes = tt[11];
  h->n_lm_tasks = tt[12]; h->poll_sleep_ns = tt[14] & 0xffff; h->stream_down = !((tt[14] >> 16) & 1); h->pf_window_kb = tt[15] & 0xffff; h->pace = (tt[15] >> 16) & 0x7fff; h->poll_inflight = (tt[14] >> 20) & 0xf; h->fuse_down = (tt[14] >> 24) & 1; h->w4a16 = (tt[14] >> 26) & 1;
  auto bad = [&](const std::string& m) { delete h; return fail(ADAMK_E_INVALID, m); };
  const AdamkModelDesc& d = *desc;
  if (d.head_dim != 64 && d.head_dim != 128) return bad("head_dim must be 64 or 128");
  if (d.n_kv_heads < 1 || d.n_q_heads % d.n_kv_heads) return bad("n_q_heads must be a multiple of n_kv_heads");
  if (d.n_q_heads / d.n_kv_heads > kGMax) return bad("more than 8 q heads per kv head");
  if (d.hidden % 8 || d.intermediate % 8) return bad("hidden/intermediate must be multiples of 8");
  if (d.n_layers + 2 > kTagStride) return bad("too many layers for the tag encoding");
  if (h->batch != 1 || d.max_batch != 1) { delete h; return fail(ADAMK_E_UNSUPPORTED, "batch > 1 is not built yet"); }
  if (h->C != 4 && h->C != 7 && h->C != 8 && h->C != 16) return bad("consumer_warps must be 4, 7, 8 or 16");
  if (h->n_stage < 2 || h->n_stage > kMaxStages) return bad("n_stage out of range");
  if (h->inflight < 0 || h->inflight > h->n_stage) return bad("inflight out of range");
  if (h->stage_bytes <= 0 || h->stage_bytes % 1024) return bad("stage_bytes must be a positive multiple of 1024");
  if (h->n_sms < 1 || h->n_tasks < 1) return bad("empty task table");
  if (h->attn_chunks < 1 || h->attn_chunks > kAttnChunksMax || h->attn_min_chunk < 8)
    return bad("attention chunking out of range");
  if (h->stage_bytes < 8 * std::min(h->C, kAttnWarps) * d.head_dim * 2)
    return bad("stage_bytes too small for one K/V block (8 positions per attention warp)");
  const size_t need = ((size_t)kHeaderInts + (size_t)h->n_sms + 1 + (size_t)h->n_tasks * kTaskInts) * 4;
  if (task_table_bytes != need) return bad("task table size does not match its header");
  {
    const int* sb = tt + kHeaderInts;
    int most = 0;
    for (int s2 = 0; s2 < h->n_sms; ++s2) most = std::max(most, sb[s2 + 1] - sb[s2]);
    h->task_cache_bytes = (int)align_up((size_t)most * 32, 512);
  }
  h->smem_bytes = kSmemReserved + h->task_cache_bytes + h->scratch_bytes + h->n_stage * h->stage_bytes;
  if (h->smem_bytes > kSmemMax) return bad("ring + scratch + task cache exceed 227 KB shared memory");
  {  // the scratch region must hold the widest activation vector, and the attention buffers
    const int kmax = std::max(std::max(d.hidden, d.n_q_heads * d.head_dim), h->fuse_down ? 0 : d.intermediate);
    size_t xb = align_up((size_t)kmax, kChunk) * 4;
    if (h->fuse_down) {   // staged gate/up input + this SM's SwiGLU outputs; the [rows][n_sms + 1] staging array of T_HRED
      if (tp_size != 1) return bad("fuse_down is a single-GPU schedule");
      if (d.hidden % 256 || (d.hidden / 256 + h->C - 1) / h->C > kDownkBlocks) return bad("fuse_down: hidden must be a multiple of 256, at most 3 row blocks per warp");
      const size_t act_loc = (size_t)(d.intermediate + h->n_sms - 1) / h->n_sms + 1;
      const size_t quads = (size_t)(d.hidden / 4 + h->n_sms - 1) / h->n_sms;
      xb = std::max(align_up((size_t)d.hidden, kChunk) * 4 + act_loc * 4, std::max(xb, quads * 4 * (size_t)(h->n_sms + 1) * 4));
    }
    const size_t ab = ((size_t)(d.head_dim + 16) + 2 * (size_t)d.head_dim + (size_t)kAttnWarps * (d.head_dim + 2) + kAttnWarps) * 4;
    if ((size_t)h->scratch_bytes < std::max(xb, ab)) return bad("scratch_bytes too small for this model");
  }
  const int* sm_begin = tt + kHeaderInts;
  const Task* tasks = reinterpret_cast<const Task*>(tt + kHeaderInts + h->n_sms + 1);
  if (sm_begin[0] != 0 || sm_begin[h->n_sms] != h->n_tasks) return bad("sm_begin does not cover the task list");
  size_t wbytes = 0;
  int lm_seen = 0;
  for (int s = 0; s < h->n_sms; ++s)
    if (sm_begin[s] > sm_begin[s + 1]) return bad("sm_begin not monotone");
  const int qkv_rows = (d.n_q_heads + 2 * d.n_kv_heads) * d.head_dim;
  for (int i = 0; i < h->n_tasks; ++i) {
    const Task& t = tasks[i];
    if (t.type == T_ATTN) {
      if (t.a < 0 || t.a >= d.n_q_heads || t.b < 0 || t.b >= h->attn_chunks || t.layer < 0 || t.layer >= d.n_layers || t.aux != 0)
        return bad("attention task out of range");
      continue;
    }
    if (t.type == T_MERGE) {
      if (t.a < 0 || t.a >= d.n_q_heads || t.layer < 0 || t.layer >= d.n_layers || t.aux != 0) return bad("merge task out of range");
      continue;
    }
    if (t.type == T_DOWNK || t.type == T_HRED) {
      if (!h->fuse_down) return bad("fused down-projection task in a table without the fuse_down flag");
      if (t.layer < 0 || t.layer >= d.n_layers || t.k != d.hidden) return bad("fused down-projection task out of range");
      if (t.type == T_HRED) {
        if (t.a < 0 || t.b < 1 || t.b > kHredQuadsMax || (t.a + t.b) * 4 > d.hidden) return bad("T_HRED rows out of range");
        continue;
      }
      // T_DOWNK must follow the gate/up task of the same SM whose SwiGLU outputs it multiplies
      if (i == 0 || tasks[i - 1].type != T_GATEUP || !(tasks[i - 1].aux & 1) || tasks[i - 1].layer != t.layer ||
          tasks[i - 1].a != 2 * t.a || tasks[i - 1].b != 2 * t.b)
        return bad("T_DOWNK does not match the preceding gate/up task");
      if (t.a < 0 || t.b < 1 || t.a + t.b > d.intermediate || t.b > 0xffff) return bad("T_DOWNK columns out of range");
      if (t.kchunks < 1 || (size_t)t.kchunks * d.hidden * ((t.aux & 2) ? 1 : 4) / 2 > (size_t)h->stage_bytes || t.n_ktiles != (t.b + t.kchunks - 1) / t.kchunks)
        return bad("T_DOWNK staging inconsistent");
      if (t.aux & ~2) return bad("T_DOWNK aux field out of range");
      if (t.aux & 2) {
        if (!h->w4a16) return bad("int4 task in a table without the W4A16 flag");
        const int ng = downk_i4_groups(t.a, t.b);
        if (ng > kDownkGroupsMax || (size_t)ng * d.hidden * 2 > (size_t)h->stage_bytes) return bad("T_DOWNK: too many scale groups for one stage");
      }
      const size_t off = (size_t)(uint32_t)t.w_off * 16;
      wbytes = std::max(wbytes, off + task_stream_bytes(t));
      continue;
    }
    if (t.type < T_QKV || t.type > T_LMHEAD) return bad("unknown task type");
    if (t.type == T_LMHEAD) ++lm_seen;
    if (t.b > 0xffff || t.rt > 0xffff || t.kchunks > 0xffff || t.ktc > 0xffff || t.n_tiles > 0xffff || t.n_ktiles > 0xffff)
      return bad("task field exceeds the packed 16-bit range");
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
    const int WR = t.geom & 0xff, WK = (t.geom >> 8) & 0xff, rw = (t.geom >> 16) & 0xff;
    if (WR < 1 || WK < 1 || WR * WK != h->C) return bad("warp grid WR x WK must equal consumer_warps");
    if (rw < 2 || rw > kRW || (rw & 1) || t.rt != WR * rw) return bad("rows per warp must be 2, 4, 6 or 8 and rows_per_tile == WR * rw");
    if (WK > 1 && t.rt > 32) return bad("K-split tiles hold at most 32 rows");
    if (t.type == T_GATEUP && ((t.a | t.b | rw) & 1)) return bad("gate/up rows must come in pairs");
    if ((t.aux & 1) && !(t.type == T_GATEUP && h->fuse_down)) return bad("task aux field out of range");
    if (t.aux & 2) {
      if (!h->w4a16) return bad("int4 task in a table without the W4A16 flag");
      if (t.type != T_QKV && t.type != T_OPROJ && t.type != T_GATEUP) return bad("W4A16 covers the QKV / O / gate-up / fused down projections only");
      if (i4_stage_bytes(t.rt, t.ktc) > (uint32_t)h->stage_bytes) return bad("int4 stage larger than stage_bytes");
    }
    if (t.aux & ~3) return bad("task aux field out of range");
    if (t.type == T_DOWN && h->fuse_down) return bad("T_DOWN in a fuse_down table");
    if (t.ktc < 1 || t.n_ktiles != (t.kchunks + t.ktc - 1) / t.ktc || t.n_tiles != (t.b + t.rt - 1) / t.rt)
      return bad("task tiling inconsistent");
    if (!(t.aux & 2) && (size_t)t.rt * t.ktc * 512 > (size_t)h->stage_bytes) return bad("stage larger than stage_bytes");
    if (t.type != T_LMHEAD && (t.layer < 0 || t.layer >= d.n_layers)) return bad("task layer out of range");
    const size_t off = (size_t)(uint32_t)t.w_off * 16;
    wbytes = std::max(wbytes, off + task_stream_bytes(t));
  }
  // lm_finish() publishes the token and bumps the epoch when its counter reaches n_lm_tasks - 1: a header that
  // disagrees with the table would hang the step until the watchdog or end it early
  if (lm_seen != h->n_lm_tasks) return bad("n_lm_tasks in the header differs from the number of LM-head tasks");
  h->packed_weight_bytes = align_up(wbytes, 256);
  // fp32 parameter tail
  h->fp_ln1 = 0; h->fp_ln2 = d.hidden; h->fp_bias = 2 * d.hidden; h->fp_qn = h->fp_bias + qkv_rows;
  h->fp_kn = h->fp_qn + d.head_dim; h->fp_layer_stride = (int)align_up((size_t)h->fp_kn + d.head_dim, 4);
  h->fp_final = h->fp_layer_stride * d.n_layers;
  h->fparam_floats = (size_t)h->fp_final + d.hidden;
  // workspace layout
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes, 256); return r; };
  h->ws_sync = take(64);
  h->rep = tp_size == 1 ? kRep : 1;
  h->ws_hx = take((size_t)h->rep * 2 * tp_size * d.hidden * 8);
  h->ws_hm = take((size_t)h->rep * tp_size * d.hidden * 8);
  h->ws_lmx = take((size_t)kMaxTP * 2 * 8);
  h->ws_qkv = take((size_t)qkv_rows * 8);
  h->ws_attn = take((size_t)h->rep * d.n_q_heads * d.head_dim * 8);
  h->ws_act = take((size_t)d.intermediate * 8);
  h->ws_part = take((size_t)d.n_q_heads * h->attn_chunks * (d.head_dim + 2) * 8);
  h->ws_part2 = take(h->fuse_down ? (size_t)d.hidden * h->n_sms * 8 : 0);
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
        if (t.type == T_ATTN || t.type == T_MERGE || t.type == T_HRED) continue;
        if ((unsigned)t.w_off != cursor) return bad("packed streams must be contiguous per SM, SM-major");
        if (task_stream_bytes(t) % 16) return bad("a task's weight stream is not a multiple of 16 bytes");
        cursor += (unsigned)(task_stream_bytes(t) / 16);
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
  for (const void* fn : {(const void*)adamk_decode_kernel<4, false>, (const void*)adamk_decode_kernel<7, false>,
                         (const void*)adamk_decode_kernel<8, false>, (const void*)adamk_decode_kernel<16, false>,
                         (const void*)adamk_decode_kernel<4, true>, (const void*)adamk_decode_kernel<7, true>,
                         (const void*)adamk_decode_kernel<8, true>, (const void*)adamk_decode_kernel<16, true>})
    if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
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
  CUDA_TRY(cudaMemsetAsync(static_cast<uint8_t*>(workspace) + h->ws_lm_idx, 0xff, (size_t)h->n_sms * 4, (cudaStream_t)stream));
  const unsigned first_epoch = 1u;  // tags of epoch 0 (the zeroed workspace) never match
  CUDA_TRY(cudaMemcpyAsync(static_cast<uint8_t*>(workspace) + h->ws_sync, &first_epoch, 4, cudaMemcpyHostToDevice,
                           (cudaStream_t)stream));
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  return ADAMK_OK;
}

static int bind_weights_impl(adamk_handle h, const AdamkWeightPtrs* w, const AdamkW4A16Layer* qlayers, void* packed, adamk_stream stream_) {
  if (!h || !w || !packed) return fail(ADAMK_E_INVALID, "NULL argument");
  if ((qlayers != nullptr) != (h->w4a16 != 0)) return fail(ADAMK_E_INVALID, "W4A16 task tables bind through adamk_bind_weights_w4a16, bf16 ones through adamk_bind_weights");
  if (!w->embed || !w->final_norm || !w->layers || !w->rope_cos || !w->rope_sin) return fail(ADAMK_E_INVALID, "missing weight pointer");
  if ((uintptr_t)packed % 256) return fail(ADAMK_E_INVALID, "packed buffer must be 256-byte aligned");
  const AdamkModelDesc& d = h->desc;
  cudaStream_t stream = (cudaStream_t)stream_;
  for (int l = 0; l < d.n_layers; ++l) {
    const AdamkLayerWeights& lw = w->layers[l];
    if (!lw.ln1 || !lw.ln2) return fail(ADAMK_E_INVALID, "layer " + std::to_string(l) + ": missing norm pointer");
    if (!qlayers && (!lw.wq || !lw.wk || !lw.wv || !lw.wo || !lw.wgate || !lw.wup || !lw.wdown))
      return fail(ADAMK_E_INVALID, "layer " + std::to_string(l) + ": missing matrix pointer");
    if (qlayers) {
      const AdamkW4A16Layer& q = qlayers[l];
      if (!q.q_wq || !q.s_wq || !q.q_wk || !q.s_wk || !q.q_wv || !q.s_wv || !q.q_wo || !q.s_wo || !q.q_wgate || !q.s_wgate || !q.q_wup ||
          !q.s_wup || !q.q_wdown || !q.s_wdown)
        return fail(ADAMK_E_INVALID, "layer " + std::to_string(l) + ": missing W4A16 code / scale pointer");
    }
    if (d.qkv_bias && (!lw.bq || !lw.bk || !lw.bv)) return fail(ADAMK_E_INVALID, "qkv_bias set but bias pointer missing");
    if (d.qk_norm && (!lw.q_norm || !lw.k_norm)) return fail(ADAMK_E_INVALID, "qk_norm set but norm pointer missing");
  }
  AdamkLayerWeights* d_layers = nullptr;
  CUDA_TRY(cudaMalloc(&d_layers, sizeof(AdamkLayerWeights) * d.n_layers));
  cudaError_t e = cudaMemcpyAsync(d_layers, w->layers, sizeof(AdamkLayerWeights) * d.n_layers, cudaMemcpyHostToDevice, stream);
  if (e != cudaSuccess) { cudaFree(d_layers); return fail(ADAMK_E_CUDA, cudaGetErrorString(e)); }
  AdamkW4A16Layer* d_qlayers = nullptr;
  if (qlayers) {
    e = cudaMalloc(&d_qlayers, sizeof(AdamkW4A16Layer) * d.n_layers);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_qlayers, qlayers, sizeof(AdamkW4A16Layer) * d.n_layers, cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) { cudaFree(d_layers); if (d_qlayers) cudaFree(d_qlayers); return fail(ADAMK_E_CUDA, cudaGetErrorString(e)); }
  }
  PackParams pp{};
  pp.qlayers = d_qlayers;
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
  if (d_qlayers) cudaFree(d_qlayers);
  if (e != cudaSuccess) return fail(ADAMK_E_CUDA, std::string("adamk_bind_weights: ") + cudaGetErrorString(e));
  h->w = *w;
  h->w.layers = nullptr;
  h->wpacked = static_cast<const uint8_t*>(packed);
  h->fparams = fp;
  h->bound = true;
  return ADAMK_OK;
}

int adamk_bind_weights(adamk_handle h, const AdamkWeightPtrs* w, void* packed, adamk_stream stream) {
  return bind_weights_impl(h, w, nullptr, packed, stream);
}

int adamk_bind_weights_w4a16(adamk_handle h, const AdamkWeightPtrs* w, const AdamkW4A16Layer* qlayers, void* packed, adamk_stream stream) {
  if (!qlayers) return fail(ADAMK_E_INVALID, "NULL W4A16 layer array");
  return bind_weights_impl(h, w, qlayers, packed, stream);
}

int adamk_share_weights(adamk_handle h, adamk_handle owner, const AdamkWeightPtrs* w) {
  if (!h || !owner || !w) return fail(ADAMK_E_INVALID, "NULL argument");
  if (!owner->bound) return fail(ADAMK_E_STATE, "the owner handle has no weights bound");
  // identical task tables <=> identical packed layout
  if (h->host_table != owner->host_table || h->packed_weight_bytes != owner->packed_weight_bytes ||
      h->fparam_floats != owner->fparam_floats)
    return fail(ADAMK_E_INVALID, "handles must be built from identical task tables to share packed weights");
  h->w = *w;
  h->w.layers = nullptr;
  h->wpacked = owner->wpacked;
  h->fparams = owner->fparams;
  h->bound = true;
  return ADAMK_OK;
}

int adamk_bind_peers(adamk_handle h, void* const* peer_workspaces, int n_peers) {
  if (!h) return fail(ADAMK_E_INVALID, "NULL handle");
  if (n_peers != h->tp_size) return fail(ADAMK_E_INVALID, "n_peers must equal tp_size");
  if (h->tp_size == 1) return ADAMK_OK;
  if (!peer_workspaces) return fail(ADAMK_E_INVALID, "NULL peer list");
  for (int r = 0; r < n_peers; ++r) {
    if (!peer_workspaces[r]) return fail(ADAMK_E_INVALID, "NULL peer workspace");
    h->peer_ws[r] = peer_workspaces[r];
  }
  h->peers_bound = true;
  return ADAMK_OK;
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
  p.task_cache_bytes = h->task_cache_bytes; p.pf_window_bytes = h->pf_window_kb * 1024; p.pace_clk_per_64k = h->pace; p.poll_inflight = h->poll_inflight;
  p.attn_block = 8 * std::min(h->C, kAttnWarps);
  p.stream_down = h->stream_down;
  p.inflight = h->inflight; p.poll_sleep_ns = (unsigned)h->poll_sleep_ns;
  p.tasks = h->d_tasks; p.sm_begin = h->d_sm_begin; p.sm_stream = h->d_sm_stream;
  p.wpacked = h->wpacked; p.fparams = h->fparams;
  p.fp_layer_stride = h->fp_layer_stride; p.fp_ln1 = h->fp_ln1; p.fp_ln2 = h->fp_ln2; p.fp_bias = h->fp_bias;
  p.fp_qn = h->fp_qn; p.fp_kn = h->fp_kn; p.fp_final = h->fp_final; p.fp_bytes = (unsigned)(h->fparam_floats * 4);
  p.embed = (const __nv_bfloat16*)h->w.embed; p.rope_cos = h->w.rope_cos; p.rope_sin = h->w.rope_sin;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  if (ws) {
    p.sync = (unsigned*)(ws + h->ws_sync);
    p.ll_hx = (u64*)(ws + h->ws_hx); p.ll_hm = (u64*)(ws + h->ws_hm); p.ll_qkv = (u64*)(ws + h->ws_qkv);
    p.ll_attn = (u64*)(ws + h->ws_attn); p.ll_act = (u64*)(ws + h->ws_act); p.ll_part = (u64*)(ws + h->ws_part);
    p.lm_val = (float*)(ws + h->ws_lm_val); p.lm_idx = (int*)(ws + h->ws_lm_idx);
    p.ll_lmx = (u64*)(ws + h->ws_lmx);
    p.ll_part2 = (u64*)(ws + h->ws_part2);
  }
  p.rep = h->rep;
  p.tp_rank = h->tp_rank; p.tp_size = h->tp_size; p.vocab_off = h->tp_rank * d.vocab;
  for (int r = 0; r < h->tp_size; ++r) {
    uint8_t* pw = h->tp_size == 1 ? ws : static_cast<uint8_t*>(h->peer_ws[r]);
    if (!pw) continue;
    p.peer_hx[r] = (u64*)(pw + h->ws_hx); p.peer_hm[r] = (u64*)(pw + h->ws_hm); p.peer_lmx[r] = (u64*)(pw + h->ws_lmx);
  }
  p.status = h->status_dev;
  p.trace = h->trace;
  return ADAMK_OK;
}

static int launch(adamk_handle h, const KParams& p, cudaStream_t stream) {
  // The handle belongs to the device that was current at adamk_create (its task table, status block and SM count):
  // a caller whose thread has another device current is switched for the launch and switched back.
  if (h->dev_sms < h->n_sms) return fail(ADAMK_E_INVALID, "task table was built for more SMs than this device has");
  int cur = 0;
  CUDA_TRY(cudaGetDevice(&cur));
  struct DeviceGuard {
    int back;
    ~DeviceGuard() { if (back >= 0) cudaSetDevice(back); }
  } guard{cur != h->device ? cur : -1};
  if (cur != h->device) CUDA_TRY(cudaSetDevice(h->device));
  void* args[] = {(void*)&p};
  // cooperative launch: all CTAs must be co-resident (they poll each other's outputs)
  const bool tp = h->tp_size > 1;
  const void* fn = h->C == 4 ? (tp ? (const void*)adamk_decode_kernel<4, true> : (const void*)adamk_decode_kernel<4, false>)
                   : h->C == 7 ? (tp ? (const void*)adamk_decode_kernel<7, true> : (const void*)adamk_decode_kernel<7, false>)
                   : h->C == 8 ? (tp ? (const void*)adamk_decode_kernel<8, true> : (const void*)adamk_decode_kernel<8, false>)
                               : (tp ? (const void*)adamk_decode_kernel<16, true> : (const void*)adamk_decode_kernel<16, false>);
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
  if (h->tp_size > 1 && !h->peers_bound) return fail(ADAMK_E_STATE, "adamk_bind_peers has not been called");
  if (h->tp_size > 1 && h->peer_ws[h->tp_rank] != workspace) return fail(ADAMK_E_INVALID, "workspace is not this rank's entry of the peer list");
  if (h->status_host[0] != 0) return fail(ADAMK_E_DEVICE, "a previous step reported a device error; see adamk_device_status");
  KParams p;
  fill_params(h, p, workspace);
  p.kcache = (__nv_bfloat16*)k_cache; p.vcache = (__nv_bfloat16*)v_cache;
  p.logits = logits_out; p.tokens = token_ids; p.positions = positions; p.next_tokens = next_token_out;
  p.auto_advance = auto_advance;
  return launch(h, p, (cudaStream_t)stream);
}

int adamk_decode_step_host(adamk_handle h, const int32_t* token_ids_host, const int32_t* positions_host, int batch,
                           int32_t* token_ids, int32_t* positions, void* k_cache, void* v_cache, void* workspace,
                           float* logits_out, int32_t* next_token_out, int32_t* next_token_host, adamk_stream stream) {
  if (!token_ids_host || !positions_host || !next_token_host || !token_ids || !positions || !next_token_out)
    return fail(ADAMK_E_INVALID, "NULL argument");
  if (!h || batch != h->batch) return fail(ADAMK_E_INVALID, "batch does not match the task table");
  // Host buffers: what the device would answer with a trap (sticky CUDA error) is refused here, before anything is
  // copied or launched.  The device-resident loop (adamk_decode_step with auto_advance) is bounded by its driver.
  for (int b = 0; b < batch; ++b) {
    if (positions_host[b] < 0 || positions_host[b] >= h->desc.max_ctx)
      return fail(ADAMK_E_INVALID, "position outside [0, max_ctx): the step would leave the KV cache");
    if (token_ids_host[b] < 0 || token_ids_host[b] >= h->desc.vocab * h->tp_size)
      return fail(ADAMK_E_INVALID, "token id outside the vocabulary");
  }
  cudaStream_t st = (cudaStream_t)stream;
  const size_t nb = (size_t)batch * sizeof(int32_t);
  if (positions == token_ids + batch && positions_host == token_ids_host + batch) {   // adjacent state: one copy
    CUDA_TRY(cudaMemcpyAsync(token_ids, token_ids_host, 2 * nb, cudaMemcpyHostToDevice, st));
  } else {
    CUDA_TRY(cudaMemcpyAsync(token_ids, token_ids_host, nb, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(positions, positions_host, nb, cudaMemcpyHostToDevice, st));
  }
  const int rc = adamk_decode_step(h, token_ids, positions, batch, k_cache, v_cache, workspace, logits_out, next_token_out, 0, stream);
  if (rc != ADAMK_OK) return rc;
  CUDA_TRY(cudaMemcpyAsync(next_token_host, next_token_out, nb, cudaMemcpyDeviceToHost, st));
  // the caller needs the token to form the next step's input: spin on the stream rather than block (a blocking wait
  // adds the scheduler's wake-up latency to every token)
  cudaError_t q;
  while ((q = cudaStreamQuery(st)) == cudaErrorNotReady) {}
  if (q != cudaSuccess) return fail(ADAMK_E_CUDA, cudaGetErrorString(q));
  if (h->status_host[0] != 0) return fail(ADAMK_E_DEVICE, "the step reported a device error; see adamk_device_status");
  return ADAMK_OK;
}

int adamk_stream_probe(adamk_handle h, float* sink, int mode, adamk_stream stream) {
  if (!h || !sink) return fail(ADAMK_E_INVALID, "NULL argument");
  if (!h->bound) return fail(ADAMK_E_STATE, "adamk_bind_weights has not been called");
  KParams p;
  fill_params(h, p, nullptr);
  p.probe = (mode >= 2 && mode <= 4) ? mode : 1; p.probe_sink = sink;
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
