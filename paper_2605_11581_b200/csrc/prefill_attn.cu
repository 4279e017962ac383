// prefill_attn.cu -- causal flash attention for Prefill on the sm_100a tensor cores (tcgen05 / TMEM / TMA).
//
// The paper runs Prefill on the serving engine's fused operators; this is the attention operator of
// this repository's own Prefill (prefill.TensorCorePrefill), replacing the library call the first round used.
// One CTA = one (q head, 128-row q tile); it walks the K / V blocks of 128 positions up to the causal diagonal:
//
//   warp 0     TMA producer: the Q tile once, then K_j and V^T_j blocks into a two-stage ring
//              (cp.async.bulk.tensor.2d, 128-byte swizzle, K-major boxes of 64 elements)
//   warp 1     one lane issues tcgen05.mma: S_j = Q K_j^T into one of two S accumulators in tensor memory,
//              O_j = P_j V_j into a third; tcgen05.commit publishes them and frees the ring stage
//   warps 2-9  two softmax warpgroups: threads r of both own q row r (= TMEM lane r), one half of its columns each:
//              tcgen05.ld of its half of the S row, causal mask, running
//              maximum / sum (exp2 with the scale folded in), P_j written as bf16 into shared memory in the swizzled
//              K-major layout the PV MMA reads, the O row (fp32, registers) rescaled and accumulated from tensor memory
//
// S_{j+1} is issued before P_j is awaited (two S buffers), so QK^T of the next block overlaps the softmax of this one.
// K comes straight from the KV cache the decode kernel uses ([kv head][max_ctx][D] bf16: rows are K-major); V is
// needed K-major over positions, i.e. transposed: adamk_prefill_vt writes V^T [kv head][D][ctx_pad] (zero padded)
// once per layer -- 2 x ctx x kv_dim bytes, noise next to the GEMMs.  GQA: the q heads of a group are separate CTAs
// that re-read the same K / V^T blocks from L2.
//
// Numerics: bf16 Q, K, V and P, fp32 scores / softmax state / output -- the usual flash-attention contract.
// Output: the bf16 plane(s) [parts][T][n_q * D] the O-projection GEMM takes as its activation operand.

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <mutex>

#include "../../include/adamk_prefill.h"

namespace fa {

constexpr int BQ = 128;    // q rows per tile = TMEM lanes
constexpr int BKV = 128;   // positions per K / V block
constexpr int KB = 64;     // bf16 elements per 128-byte swizzle row
constexpr int kThreads = 320;   // TMA warp, MMA warp, two softmax warpgroups

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
               "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
               : "memory");
}
// K-major operand tile stored as rows of 128 bytes with the 128-byte swizzle; 8-row groups 1024 bytes apart
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t addr) {
  uint64_t d = (addr >> 4) & 0x3fffu;
  d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}
// fp32 accumulate, bf16 x bf16, both operands K-major, M x N
__host__ __device__ constexpr uint32_t instr_desc(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}
__device__ __forceinline__ void umma(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// the same with the A operand in tensor memory (K-major: lane = row, two bf16 per 32-bit column along K)
__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
      "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]),
      "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]),
      "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]),
      "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct Args {
  int T, pos0, n_q, n_kv, max_ctx, parts;
  float sl2e;                 // softmax scale * log2(e)
  __nv_bfloat16* out;         // [parts][T][n_q * D]
  long long plane_stride;
};

// shared memory: Q | 2 x (K | V^T) | barriers, exchange buffers   (P lives in tensor memory)
template <int D>
struct Smem {
  static constexpr int kQ = BQ * D * 2;
  static constexpr int kK = BKV * D * 2;
  static constexpr int kV = D * BKV * 2;
  static constexpr int kStage = kK + kV;
  static constexpr int kBars = 256 + 3 * 1024;   // mbarriers + tensor-memory slot | row-maximum exchange [2][2][128] | row-sum exchange [2][128]
  static constexpr int kTotal = kQ + 2 * kStage + kBars + 1024;
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
flash_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
             const __grid_constant__ CUtensorMap map_vt, const Args a) {
  using S = Smem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* q_s = smem;
  uint8_t* kv_s = smem + S::kQ;
  uint64_t* bars = reinterpret_cast<uint64_t*>(kv_s + 2 * S::kStage);
  uint64_t* q_full = bars;            // 1
  uint64_t* k_full = bars + 1;        // 2   K and V^T blocks travel in separate two-stage rings: a K stage is free as soon
  uint64_t* k_empty = bars + 3;       // 2   as its QK^T product is done, long before the PV product of the same block
  uint64_t* s_full = bars + 5;        // 2
  uint64_t* p_full = bars + 7;        // 1 (256 arrivals)
  uint64_t* o_full = bars + 8;        // 1
  uint64_t* v_full = bars + 9;        // 2
  uint64_t* v_empty = bars + 11;      // 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 13);
  float* mx = reinterpret_cast<float*>(bars) + 64;     // [block parity][warpgroup][row]
  float* lx = mx + 512;                                // [warpgroup][row]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.y, kvh = h / (a.n_q / a.n_kv);
  const int qt = (int)gridDim.x - 1 - (int)blockIdx.x;   // the long tiles (late q rows) are scheduled first
  const int q0 = qt * BQ;
  const int ctx = a.pos0 + a.T;
  const int kv_end = min(ctx, a.pos0 + q0 + BQ);          // causal: nothing past the tile's last row
  const int n_blk = (kv_end + BKV - 1) / BKV;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_q)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_k)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_vt)) : "memory");
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
      mbar_init(&s_full[s], 1);
    }
    mbar_init(p_full, 256);
    mbar_init(o_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "n"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tm_s0 = tmem_base, tm_o = tmem_base + 2 * BKV;   // S buffers at columns 0 and 128, O_j at 256

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, S::kQ);
      for (int kb = 0; kb < D / KB; ++kb) tma_load_2d(&map_q, q_full, q_s + kb * (BQ * 128), kb * KB, h * a.T + q0);
      for (int j = 0; j < n_blk; ++j) {
        const int st = j & 1;
        uint8_t* ks = kv_s + st * S::kStage;
        uint8_t* vs = ks + S::kK;
        mbar_wait(&k_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&k_full[st], S::kK);
        for (int kb = 0; kb < D / KB; ++kb) tma_load_2d(&map_k, &k_full[st], ks + kb * (BKV * 128), kb * KB, kvh * a.max_ctx + j * BKV);
        mbar_wait(&v_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&v_full[st], S::kV);
        for (int kb = 0; kb < BKV / KB; ++kb) tma_load_2d(&map_vt, &v_full[st], vs + kb * (D * 128), j * BKV + kb * KB, kvh * D);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = instr_desc(BQ, BKV), idesc_o = instr_desc(BQ, D);
      auto issue_s = [&](int j) {   // S_j = Q K_j^T into S buffer j & 1
        const int st = j & 1;
        mbar_wait(&k_full[st], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t qa = smem_u32(q_s), ka = smem_u32(kv_s + st * S::kStage);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off_q = (k / 4) * (BQ * 128) + (k % 4) * 32, off_k = (k / 4) * (BKV * 128) + (k % 4) * 32;
          umma(tm_s0 + st * BKV, smem_desc_sw128(qa + off_q), smem_desc_sw128(ka + off_k), idesc_s, k != 0);
        }
        umma_commit(&s_full[st]);
        umma_commit(&k_empty[st]);              // K_j may be overwritten
      };
      mbar_wait(q_full, 0);
      issue_s(0);
      for (int j = 0; j < n_blk; ++j) {
        const int st = j & 1;
        if (j + 1 < n_blk) issue_s(j + 1);      // the next block's scores while this block's softmax runs
        mbar_wait(p_full, j & 1);               // P_j is in tensor memory (over the first half of S_j), O is rescaled if it had to be
        mbar_wait(&v_full[st], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t va = smem_u32(kv_s + st * S::kStage + S::kK);
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k) {    // O += P_j V_j: A from tensor memory (8 columns per 16 positions), accumulating across blocks
          const uint32_t off_v = (k / 4) * (D * 128) + (k % 4) * 32;
          umma_ts(tm_o, tm_s0 + st * BKV + k * 8, smem_desc_sw128(va + off_v), idesc_o, (j | k) != 0);
        }
        umma_commit(&v_empty[st]);              // V^T_j may be overwritten
        umma_commit(o_full);
      }
    }
  } else {
    // Two softmax warpgroups share every q row: warpgroup g owns columns 64 g .. 64 g + 63 of each S block (its half of
    // the maximum, of the exponentials and of P) and columns g D/2 .. of the output row.  The two threads of a row
    // exchange their half maxima through shared memory once per block and their half sums once at the end; everything
    // else (reference maximum, rescale decisions) they compute identically.
    //
    // O accumulates in tensor memory across blocks (the PV MMAs add into it), so the softmax of block j + 1 does not wait
    // for the PV product of block j.  The exponentials are taken against a REFERENCE maximum that is only raised -- and O
    // and the running sum rescaled, in tensor memory -- when the row maximum has grown by more than 2^8 since (P stays
    // below 256, far inside bf16 / fp32 range; the final division by the sum taken against the same reference makes the
    // result independent of it).  P_j goes to tensor memory as well, over the first 64 columns of the S_j it was
    // computed from: it is the A operand of the PV MMA, and no shared-memory round trip is left in the loop.
    const int wg = (warp - 2) >> 2;
    const int quarter = warp & 3;               // the TMEM lanes this warp may access
    const int row = quarter * 32 + lane;        // q row of the tile = TMEM lane
    const int q_pos = a.pos0 + q0 + row;
    const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
    constexpr int DH = D / 2;
    constexpr int NC = BKV / 64;                // 32-column groups of S per thread
    constexpr float kRaise = 8.f;               // log2 of the largest P tolerated before the reference is raised
    float m_ref = -INFINITY, l_run = 0.f;       // reference maximum (raw score units), this thread's half of the sum
    const int c0 = wg * NC;
    const uint32_t to = tm_o + lane_addr + wg * DH;
    for (int j = 0; j < n_blk; ++j) {
      const int st = j & 1, kv0 = j * BKV;
      const bool diag = kv0 + BKV - 1 > a.pos0 + q0;   // some row of the tile masks part of this block
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t ts = tm_s0 + st * BKV + lane_addr;
      // this thread's half of the S row: one trip to tensor memory, kept in registers for the maximum and the exponentials
      uint32_t sr[NC][32];
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) tmem_ld32(ts + (c0 + cc) * 32, sr[cc]);
      tmem_ld_wait();
      if (diag) {
        const int lim = q_pos - kv0 - c0 * 32;            // columns 0 .. lim of this half are visible to the row
#pragma unroll
        for (int cc = 0; cc < NC; ++cc)
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (cc * 32 + i > lim) sr[cc][i] = 0xff800000u;   // -inf: exp2 gives exactly 0 below
      }
      float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};   // four independent chains: a single one is 64 dependent FMNMX
#pragma unroll
      for (int cc = 0; cc < NC; ++cc)
#pragma unroll
        for (int i = 0; i < 32; ++i) mq[i & 3] = fmaxf(mq[i & 3], __uint_as_float(sr[cc][i]));
      float m_blk = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
      mx[(st * 2 + wg) * BQ + row] = m_blk;
      tc_fence_before();                                  // the S loads of this thread are done before its partner may write P over them
      asm volatile("bar.sync 1, 256;" ::: "memory");
      tc_fence_after();
      m_blk = fmaxf(m_blk, mx[(st * 2 + (wg ^ 1)) * BQ + row]);
      if (j == 0) {
        m_ref = m_blk;                                    // column 0 of block 0 is visible to every row: finite
      } else {
        const bool raise = (m_blk - m_ref) * a.sl2e > kRaise;
        if (__any_sync(0xffffffffu, raise)) {             // rare: rescale this warp's rows of O in tensor memory
          mbar_wait(o_full, (j - 1) & 1);                 // every PV product issued so far has been added
          tc_fence_after();
          const float alpha = raise ? ex2((m_ref - m_blk) * a.sl2e) : 1.f;
#pragma unroll
          for (int c = 0; c < DH / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(to + c * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
            tmem_st32(to + c * 32, r);
          }
          tmem_st_wait();
          if (raise) { l_run *= alpha; m_ref = m_blk; }
        }
      }
      // P = exp2((s - m_ref) * scale * log2e) as bf16 pairs, straight into tensor memory: the K-major A operand of the PV MMA
      const float mb = m_ref * a.sl2e;
      const float2 sc2 = make_float2(a.sl2e, a.sl2e), mb2 = make_float2(-mb, -mb);   // packed FFMA2 / FADD2 around the MUFU.EX2
      float2 lq[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        uint32_t packed[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float2 x = __ffma2_rn(make_float2(__uint_as_float(sr[cc][i]), __uint_as_float(sr[cc][i + 1])), sc2, mb2);
          const float2 pp = make_float2(ex2(x.x), ex2(x.y));
          lq[(i >> 1) & 3] = __fadd2_rn(lq[(i >> 1) & 3], pp);       // row sum over the fp32 exponentials
          const __nv_bfloat162 b = __floats2bfloat162_rn(pp.x, pp.y);
          packed[i >> 1] = *reinterpret_cast<const uint32_t*>(&b);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) sr[cc >> 1][(cc & 1) * 16 + i] = packed[i];   // gather the pairs of both groups into one 32-column store
      }
      {
        const float2 s01 = __fadd2_rn(lq[0], lq[1]), s23 = __fadd2_rn(lq[2], lq[3]);
        l_run += (s01.x + s01.y) + (s23.x + s23.y);
      }
      static_assert(NC == 2, "one 32-column tcgen05.st per thread carries its 64 probabilities");
      tmem_st32(tm_s0 + st * BKV + lane_addr + wg * 32, sr[0]);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    mbar_wait(o_full, (n_blk - 1) & 1);
    tc_fence_after();
    lx[wg * BQ + row] = l_run;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    const float inv = 1.f / (l_run + lx[(wg ^ 1) * BQ + row]);
    const int t = q0 + row;
#pragma unroll
    for (int c = 0; c < DH / 32; ++c) {
      uint32_t r[32];
      tmem_ld32(to + c * 32, r);
      tmem_ld_wait();
      if (t < a.T) {
        __nv_bfloat16* dst = a.out + (long long)t * a.n_q * D + h * D + wg * DH + c * 32;
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint32_t hi[4], lo[4];
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            const float v0 = __uint_as_float(r[i + e]) * inv;
            const float v1 = __uint_as_float(r[i + e + 1]) * inv;
            const __nv_bfloat162 b = __floats2bfloat162_rn(v0, v1);
            hi[e >> 1] = *reinterpret_cast<const uint32_t*>(&b);
            const __nv_bfloat162 b2 = __floats2bfloat162_rn(v0 - __low2float(b), v1 - __high2float(b));
            lo[e >> 1] = *reinterpret_cast<const uint32_t*>(&b2);
          }
          *reinterpret_cast<uint4*>(dst + i) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
          if (a.parts > 1) *reinterpret_cast<uint4*>(dst + a.plane_stride + i) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(512) : "memory");
  }
}

// ---- two q tiles per CTA ----------------------------------------------------------------------------------------------
// The kernel above keeps one 128-row q tile per CTA and splits every row between two softmax warpgroups, which then hit
// their exponentials (the MUFU pipe: 16 ex2 per clock per SM = 1024 clocks per 128 x 128 block) at the same time and
// leave it idle the rest of the block.  Here a CTA owns TWO adjacent q tiles of one head; warpgroup t is the softmax of
// tile t (a thread = a whole row: no exchange, no CTA barrier in the loop) and the single MMA lane interleaves the two
// tiles -- PV_A(j), QK_A(j + 1), PV_B(j), QK_B(j + 1) -- so that one tile's softmax runs under the other's MMAs and
// the two warpgroups drift out of phase.  Both tiles multiply the same K / V^T blocks (half the shared-memory traffic
// per q row).  Tensor memory: S_A | S_B | O_A | O_B, 128 columns each; P_t overwrites the first 64 columns of S_t.
template <int D>
struct Smem2 {
  static constexpr int kQt = BQ * D * 2;          // one q tile
  static constexpr int kK = BKV * D * 2;
  static constexpr int kV = D * BKV * 2;
  static constexpr int kBars = 256;
  static constexpr int kTotal = 2 * kQt + 2 * kK + 2 * kV + kBars + 1024;
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
flash2_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
              const __grid_constant__ CUtensorMap map_vt, const Args a) {
  using S = Smem2<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* q_s = smem;                          // tile t at q_s + t * kQt
  uint8_t* k_s = smem + 2 * S::kQt;             // two stages
  uint8_t* v_s = k_s + 2 * S::kK;               // two stages
  uint64_t* bars = reinterpret_cast<uint64_t*>(v_s + 2 * S::kV);
  uint64_t* q_full = bars;            // 1
  uint64_t* k_full = bars + 1;        // 2 stages
  uint64_t* k_empty = bars + 3;
  uint64_t* v_full = bars + 5;
  uint64_t* v_empty = bars + 7;
  uint64_t* s_full = bars + 9;        // per tile
  uint64_t* p_full = bars + 11;       // per tile, 128 arrivals
  uint64_t* o_full = bars + 13;       // per tile
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 15);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.y, kvh = h / (a.n_q / a.n_kv);
  const int qp = (int)gridDim.x - 1 - (int)blockIdx.x;   // the long tile pairs (late q rows) are scheduled first
  const int q0 = qp * 2 * BQ;
  const int ctx = a.pos0 + a.T;
  int nb[2];                                             // K / V blocks each tile attends to (0: the tile lies past T)
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int q0t = q0 + t * BQ;
    nb[t] = q0t < a.T ? (min(ctx, a.pos0 + q0t + BQ) + BKV - 1) / BKV : 0;
  }
  const int n_blk = max(nb[0], nb[1]);

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_q)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_k)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_vt)) : "memory");
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], 128);
      mbar_init(&o_full[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "n"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, (nb[1] > 0 ? 2 : 1) * S::kQt);
      for (int t = 0; t < 2; ++t)
        if (nb[t] > 0)
          for (int kb = 0; kb < D / KB; ++kb) tma_load_2d(&map_q, q_full, q_s + t * S::kQt + kb * (BQ * 128), kb * KB, h * a.T + q0 + t * BQ);
      for (int j = 0; j < n_blk; ++j) {
        const int st = j & 1;
        mbar_wait(&k_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&k_full[st], S::kK);
        for (int kb = 0; kb < D / KB; ++kb)
          tma_load_2d(&map_k, &k_full[st], k_s + st * S::kK + kb * (BKV * 128), kb * KB, kvh * a.max_ctx + j * BKV);
        mbar_wait(&v_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&v_full[st], S::kV);
        for (int kb = 0; kb < BKV / KB; ++kb)
          tma_load_2d(&map_vt, &v_full[st], v_s + st * S::kV + kb * (D * 128), j * BKV + kb * KB, kvh * D);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = instr_desc(BQ, BKV), idesc_o = instr_desc(BQ, D);
      auto qk = [&](int t, int j) {   // S_t = Q_t K_j^T
        const uint32_t qa = smem_u32(q_s + t * S::kQt), ka = smem_u32(k_s + (j & 1) * S::kK);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off_q = (k / 4) * (BQ * 128) + (k % 4) * 32, off_k = (k / 4) * (BKV * 128) + (k % 4) * 32;
          umma(tmem_base + t * BKV, smem_desc_sw128(qa + off_q), smem_desc_sw128(ka + off_k), idesc_s, k != 0);
        }
        umma_commit(&s_full[t]);
      };
      auto pv = [&](int t, int j) {   // O_t += P_t V_j, P_t from tensor memory (over the first half of S_t)
        mbar_wait(&p_full[t], j & 1);
        tc_fence_after();
        const uint32_t va = smem_u32(v_s + (j & 1) * S::kV);
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k) {
          const uint32_t off_v = (k / 4) * (D * 128) + (k % 4) * 32;
          umma_ts(tmem_base + (2 + t) * BKV, tmem_base + t * BKV + k * 8, smem_desc_sw128(va + off_v), idesc_o, (j | k) != 0);
        }
        umma_commit(&o_full[t]);
      };
      mbar_wait(q_full, 0);
      mbar_wait(&k_full[0], 0);
      tc_fence_after();
      for (int t = 0; t < 2; ++t)
        if (nb[t] > 0) qk(t, 0);
      umma_commit(&k_empty[0]);
      for (int j = 0; j < n_blk; ++j) {
        const int st = j & 1;
        const bool next = j + 1 < n_blk;
        mbar_wait(&v_full[st], (j >> 1) & 1);
        if (next) mbar_wait(&k_full[st ^ 1], ((j + 1) >> 1) & 1);
        tc_fence_after();
        for (int t = 0; t < 2; ++t) {
          if (j < nb[t]) pv(t, j);
          if (j + 1 < nb[t]) qk(t, j + 1);
        }
        umma_commit(&v_empty[st]);               // V^T_j may be overwritten
        if (next) umma_commit(&k_empty[st ^ 1]); // and K_{j+1}
      }
    }
  } else {
    const int t = (warp - 2) >> 2;              // the q tile of this warpgroup
    if (nb[t] > 0) {
      const int quarter = warp & 3;             // the TMEM lanes this warp may access
      const int row = quarter * 32 + lane;      // q row of the tile = TMEM lane
      const int q0t = q0 + t * BQ;
      const int q_pos = a.pos0 + q0t + row;
      const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
      const uint32_t ts = tmem_base + t * BKV + lane_addr, to = tmem_base + (2 + t) * BKV + lane_addr;
      constexpr float kRaise = 8.f;             // log2 of the largest P tolerated before the reference maximum is raised
      float m_ref = -INFINITY, l_run = 0.f;
      for (int j = 0; j < nb[t]; ++j) {
        const int kv0 = j * BKV;
        const bool diag = kv0 + BKV - 1 > a.pos0 + q0t;
        mbar_wait(&s_full[t], j & 1);
        tc_fence_after();
        uint32_t sr[4][32];                     // the whole S row: one trip to tensor memory
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(ts + c * 32, sr[c]);
        tmem_ld_wait();
        if (diag) {
          const int lim = q_pos - kv0;          // columns 0 .. lim are visible to the row
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c * 32 + i > lim) sr[c][i] = 0xff800000u;   // -inf: exp2 gives exactly 0 below
        }
        float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i) mq[i & 3] = fmaxf(mq[i & 3], __uint_as_float(sr[c][i]));
        const float m_blk = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
        if (j == 0) {
          m_ref = m_blk;                        // column 0 of block 0 is visible to every row: finite
        } else {
          const bool raise = (m_blk - m_ref) * a.sl2e > kRaise;
          if (__any_sync(0xffffffffu, raise)) { // rare: rescale this warp's rows of O in tensor memory
            mbar_wait(&o_full[t], (j - 1) & 1); // every PV product issued so far has been added
            tc_fence_after();
            const float alpha = raise ? ex2((m_ref - m_blk) * a.sl2e) : 1.f;
#pragma unroll 1
            for (int c = 0; c < D / 32; ++c) {
              uint32_t r[32];
              tmem_ld32(to + c * 32, r);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
              tmem_st32(to + c * 32, r);
            }
            tmem_st_wait();
            if (raise) { l_run *= alpha; m_ref = m_blk; }
          }
        }
        // P = exp2((s - m_ref) * scale * log2e) as bf16 pairs, gathered into the first two register groups
        const float mb = m_ref * a.sl2e;
        // packed arithmetic (FFMA2 / FADD2) around the 128 MUFU.EX2 of the row: the exponentials alone keep this warp's
        // SFU busy for 1024 clocks per block, everything else in the loop is issue slots the warp loses on top of that.
        // The row sum is taken over the fp32 exponentials (the usual flash-attention choice), not their bf16 roundings.
        const float2 sc2 = make_float2(a.sl2e, a.sl2e), mb2 = make_float2(-mb, -mb);
        float2 lq[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t packed[16];
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float2 x = __ffma2_rn(make_float2(__uint_as_float(sr[c][i]), __uint_as_float(sr[c][i + 1])), sc2, mb2);
            const float2 pp = make_float2(ex2(x.x), ex2(x.y));
            lq[(i >> 1) & 3] = __fadd2_rn(lq[(i >> 1) & 3], pp);
            const __nv_bfloat162 b = __floats2bfloat162_rn(pp.x, pp.y);
            packed[i >> 1] = *reinterpret_cast<const uint32_t*>(&b);
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) sr[c >> 1][(c & 1) * 16 + i] = packed[i];
        }
        {
          const float2 s01 = __fadd2_rn(lq[0], lq[1]), s23 = __fadd2_rn(lq[2], lq[3]);
          l_run += (s01.x + s01.y) + (s23.x + s23.y);
        }
        tmem_st32(ts, sr[0]);
        tmem_st32(ts + 32, sr[1]);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_full[t]);
      }
      mbar_wait(&o_full[t], (nb[t] - 1) & 1);
      tc_fence_after();
      const float inv = 1.f / l_run;
      const int tok = q0t + row;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(to + c * 32, r);
        tmem_ld_wait();
        if (tok < a.T) {
          __nv_bfloat16* dst = a.out + (long long)tok * a.n_q * D + h * D + c * 32;
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint32_t hi[4], lo[4];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              const float v0 = __uint_as_float(r[i + e]) * inv;
              const float v1 = __uint_as_float(r[i + e + 1]) * inv;
              const __nv_bfloat162 b = __floats2bfloat162_rn(v0, v1);
              hi[e >> 1] = *reinterpret_cast<const uint32_t*>(&b);
              const __nv_bfloat162 b2 = __floats2bfloat162_rn(v0 - __low2float(b), v1 - __high2float(b));
              lo[e >> 1] = *reinterpret_cast<const uint32_t*>(&b2);
            }
            *reinterpret_cast<uint4*>(dst + i) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
            if (a.parts > 1) *reinterpret_cast<uint4*>(dst + a.plane_stride + i) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
          }
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(512) : "memory");
  }
}

// V^T [n_kv][D][ctx_pad] bf16 from the cache layout [n_kv][max_ctx][D]; columns >= ctx are zero.  grid (ctx_pad / 64, n_kv)
template <int D>
__global__ void vt_kernel(const __nv_bfloat16* __restrict__ v, __nv_bfloat16* __restrict__ vt, int max_ctx, int ctx, int ctx_pad) {
  __shared__ __nv_bfloat16 tile[64][D + 2];
  const int p0 = blockIdx.x * 64, kvh = blockIdx.y;
  for (int i = threadIdx.x; i < 64 * D; i += blockDim.x) {
    const int p = i / D, d = i - p * D;
    tile[p][d] = (p0 + p < ctx) ? v[((long long)kvh * max_ctx + p0 + p) * D + d] : __float2bfloat16(0.f);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 64 * D; i += blockDim.x) {
    const int d = i / 64, p = i - d * 64;
    vt[((long long)kvh * D + d) * ctx_pad + p0 + p] = tile[p][d];
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                  const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}
static thread_local char g_err[256] = "";
static int g_one_tile = 0;   // adamk_prefill_attention_set_kernel(): 1 = always the one-tile kernel (A/B measurements, tests)

// 2-D bf16 tensor [rows, cols] row-major, box [box_rows, 64 columns], 128-byte swizzle
static bool make_map(CUtensorMap* m, const void* base, long long rows, long long cols, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) {
    snprintf(g_err, sizeof g_err, "cuTensorMapEncodeTiled is not available from this driver");
    return false;
  }
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(cols) * 2};
  cuuint32_t box[2] = {cuuint32_t(KB), cuuint32_t(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(g_err, sizeof g_err, "cuTensorMapEncodeTiled failed with %d (rows %lld cols %lld box %d)", int(r), rows, cols, box_rows);
    return false;
  }
  return true;
}

template <int D>
static int run(const void* q, const void* k_cache, const void* vt, const Args& a, int ctx_pad, cudaStream_t stream) {
  CUtensorMap mq, mk, mv;
  if (!make_map(&mq, q, (long long)a.n_q * a.T, D, BQ)) return ADAMK_PF_E_CUDA;
  if (!make_map(&mk, k_cache, (long long)a.n_kv * a.max_ctx, D, BKV)) return ADAMK_PF_E_CUDA;
  if (!make_map(&mv, vt, (long long)a.n_kv * D, ctx_pad, D)) return ADAMK_PF_E_CUDA;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(flash_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<D>::kTotal) != cudaSuccess) return ADAMK_PF_E_CUDA;
    if (cudaFuncSetAttribute(flash2_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem2<D>::kTotal) != cudaSuccess) return ADAMK_PF_E_CUDA;
    configured = true;
  }
  // one q tile per CTA for a pass of at most one tile (a second tile would idle half the CTA), tile pairs otherwise
  if (a.T <= BQ || g_one_tile)
    flash_kernel<D><<<dim3((a.T + BQ - 1) / BQ, a.n_q), kThreads, Smem<D>::kTotal, stream>>>(mq, mk, mv, a);
  else
    flash2_kernel<D><<<dim3((a.T + 2 * BQ - 1) / (2 * BQ), a.n_q), kThreads, Smem2<D>::kTotal, stream>>>(mq, mk, mv, a);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof g_err, "prefill attention launch: %s", cudaGetErrorString(e));
    return ADAMK_PF_E_CUDA;
  }
  return ADAMK_PF_OK;
}

}  // namespace fa

extern "C" {

const char* adamk_prefill_attention_last_error(void) { return fa::g_err; }

void adamk_prefill_attention_set_kernel(int one_tile) { fa::g_one_tile = one_tile ? 1 : 0; }

int adamk_prefill_vt(const void* v_cache, int n_kv, int D, int max_ctx, int ctx, int ctx_pad, void* vt, adamk_pf_stream stream) {
  if (v_cache == nullptr || vt == nullptr || n_kv < 1 || (D != 64 && D != 128) || ctx < 1 || ctx > max_ctx || ctx_pad < ctx || ctx_pad % 64)
    return ADAMK_PF_E_INVALID;
  const dim3 grid(ctx_pad / 64, n_kv);
  if (D == 128) fa::vt_kernel<128><<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const __nv_bfloat16*>(v_cache), static_cast<__nv_bfloat16*>(vt), max_ctx, ctx, ctx_pad);
  else fa::vt_kernel<64><<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const __nv_bfloat16*>(v_cache), static_cast<__nv_bfloat16*>(vt), max_ctx, ctx, ctx_pad);
  return cudaGetLastError() == cudaSuccess ? ADAMK_PF_OK : ADAMK_PF_E_CUDA;
}

int adamk_prefill_attention(const void* q, const void* k_cache, const void* vt, int T, int pos0, int n_q, int n_kv, int D, int max_ctx,
                            int ctx_pad, void* out_planes, int parts, adamk_pf_stream stream) {
  if (q == nullptr || k_cache == nullptr || vt == nullptr || out_planes == nullptr) return ADAMK_PF_E_INVALID;
  if (T < 1 || pos0 < 0 || pos0 + T > max_ctx || n_kv < 1 || n_q % n_kv || (D != 64 && D != 128) || (parts != 1 && parts != 2) ||
      ctx_pad < pos0 + T || ctx_pad % 64)
    return ADAMK_PF_E_INVALID;
  fa::Args a{};
  a.T = T; a.pos0 = pos0; a.n_q = n_q; a.n_kv = n_kv; a.max_ctx = max_ctx; a.parts = parts;
  a.sl2e = 1.4426950408889634f / sqrtf(float(D));
  a.out = static_cast<__nv_bfloat16*>(out_planes);
  a.plane_stride = (long long)T * n_q * D;
  return D == 128 ? fa::run<128>(q, k_cache, vt, a, ctx_pad, static_cast<cudaStream_t>(stream))
                  : fa::run<64>(q, k_cache, vt, a, ctx_pad, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
