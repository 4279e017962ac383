// prefill_gemm.cu -- token-parallel projections of the Prefill phase on the 5th-generation tensor cores.
//
// The paper keeps Prefill on the serving engine's own operators and switches to the MegaKernel for Decode
// (/root/reference/PAPER.md:244-249); SURVEY.md section 8(f) row 2 asks for that Prefill half as hand-written
// sm_100a code.  This file is its GEMM:   D[T, N] = X[T, K] . W[N, K]^T   with the decode kernel's numerical
// contract -- bf16 weights used exactly, activations carried in fp32.  An fp32 activation is fed to the
// tensor cores as `parts` bf16 planes (parts = 2: x = hi + lo, |x - hi - lo| <= 2^-17 |x|; parts = 1: plain
// bf16 rounding), every plane multiplies the same weight tile and all of them accumulate into one fp32
// accumulator in tensor memory, so the result matches the decode kernel's fp32 FMA chain to ~1e-6 relative
// at twice the tensor work, or runs at bf16 cost when parts = 1.
//
// Kernel anatomy (persistent, 192 threads per CTA):
//   warp 0      TMA producer: cp.async.bulk.tensor 2-D tiles (128 x 64 of X, 64-row boxes of W, 128-byte swizzle)
//               into an n-stage shared-memory ring, full/empty mbarriers.
//   warp 1      allocates tensor memory; one elected lane issues tcgen05.mma.kind::f16 (A and B from shared memory
//               through matrix descriptors, D in TMEM), tcgen05.commit releases ring slots and publishes finished
//               accumulators.
//   warps 2-5   epilogue: tcgen05.ld 32 lanes x 32 columns at a time through a padded shared-memory patch (4 rows x 128
//               contiguous bytes per global instruction), fused store+bias / residual add / SwiGLU + bf16-plane split /
//               fp32 atomics.  Two accumulators (2 x 256 TMEM columns) let the tensor pipe start tile i+1 while tile i
//               drains.
// Two kernels share these roles: gemm_kernel<BN, EPI> -- one CTA per 128 x BN tile (4 stages x 48 KB at BN 256) -- and
// gemm_pair_kernel<EPI> -- a cluster of two CTAs per 256 x 256 tile with tcgen05.mma.cta_group::2, each SM staging its
// own 128 token rows and half of the weight tile (6 stages x 32 KB).  plan_gemm() (host, exported as
// adamk_prefill_gemm_plan) picks the shape and cuts the problem into work items: whole tiles walked token-block fastest
// (the CTAs running at any moment share a few weight tiles out of L2 and every weight byte leaves HBM once), the tiles
// of a last partial wave as 64/128-column slices, and -- for decode-sized T with the atomic epilogue -- K ranges
// spread over the idle SMs with all activation planes stacked in the one token tile.

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <mutex>

#include "../../include/adamk_prefill.h"

namespace pf {

constexpr int BM = 128;       // tokens per tile = TMEM lanes
constexpr int BK = 64;        // bf16 elements per k block = one 128-byte swizzle row
constexpr int UK = 16;        // K of one tcgen05.mma (bf16)
constexpr int kThreads = 192;

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
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// Shared-memory matrix descriptor of a K-major tile stored as rows of 128 bytes with the 128-byte swizzle
// (what the TMA box above writes): 8-row groups 1024 bytes apart (stride byte offset), descriptor version 1.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t addr) {
  uint64_t d = (addr >> 4) & 0x3fffu;
  d |= uint64_t(1) << 16;                 // leading byte offset (unused for swizzled K-major), 16-byte units
  d |= uint64_t(1024 >> 4) << 32;         // stride byte offset
  d |= uint64_t(1) << 46;                 // version
  d |= uint64_t(2) << 61;                 // SWIZZLE_128B
  return d;
}

// Instruction descriptor: fp32 accumulate, bf16 x bf16, both operands K-major, M x N.
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
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Programmatic dependent launch: let the next kernel of the stream start its prologue now, and wait for the previous
// kernel's results before touching global memory (both are no-ops for a launch without the attribute).
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int x, int y) {   // box -> L2 only
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y)
               : "memory");
}
constexpr int kEarlyL2Blocks = 96;   // k blocks per CTA requested into L2 ahead of griddepcontrol.wait (8-32 KB each)
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// stamps (CTA 0 only): 0 start, 1 prologue done, 2 first operands landed, 3 accumulator complete (MMA lane),
// 4 epilogue warp 0 done, 5 before exit, 6 accumulator seen by epilogue warp 0
#define PF_STAMP(i) do { if (g.trace != nullptr && blockIdx.x == 0) g.trace[i] = gtime(); } while (0)

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
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

struct GemmArgs {
  int T, N, K, parts;
  int ldo;              // row stride of `out` in elements
  const float* bias;    // [N] or null (EPI_STORE)
  void* out;            // fp32 [T, ldo] (STORE / RESID) or bf16 [parts_out][T, ldo] (SWIGLU)
  int parts_out;
  long long part_stride;  // elements between output planes (SWIGLU)
  int main_items;       // work items [0, main_items) are whole BM x BN tiles ...
  int tail_split;       // ... the remaining tiles are cut into tail_split column slices each (last-wave balance)
  int n_items;
  int ksplit;           // split-K (EPI_ATOMIC only): every tile item becomes ksplit items over disjoint k-block ranges
  int kb_per_split;
  const uint8_t* pf_ptr;       // adamk_prefill_prefetch_next(): bytes the NEXT kernel will stream, pulled into L2 by this
  long long pf_bytes;          // launch's otherwise idle epilogue warps while its own operands are in flight
  unsigned long long* trace;   // debug: %globaltimer stamps of CTA 0 (adamk_prefill_set_trace), or null
  int col_fast;         // walk order of the tiles: 0 = token block fastest (CTAs of a wave share a weight tile: the weight
                        // leaves HBM once, right when it is the large operand), 1 = tile column fastest (CTAs of a wave
                        // share a token block and the whole weight sits in L2: right when the ACTIVATION is the large
                        // operand, e.g. the down projection of a 4096-token pass: 73 MB of activations against 27 MB)
  int n_tiles_n;        // tile columns
  int stacked;          // EPI_ATOMIC with parts * T <= 128: the planes are consecutive rows of ONE token tile, K is walked
                        // once (the weight is read once), accumulator row r adds into output row r % T
                        // 2 = the same with plane p at rows [32 p, 32 p + T) (T <= 32; 3-D tensor map of the token
                        // operand): output row r % 32, every plane's rows in their own tensor-memory lane quarter
  int quarters;         // host: this call's token map is the 3-D plane map (apply_plan turns stacked into 2)
  int w_early;          // programmatic dependent launch: first ring pass of weight boxes issued ahead of griddepcontrol.wait
};

constexpr int BOXN = 64;            // weight rows per TMA box: the slice granularity of a tile
constexpr int kStagePitch = 36;     // floats per staged row (32 + 4: conflict-free 16-byte accesses)
constexpr int kStageFloats = 32 * kStagePitch;

template <int BN>
struct Smem {
  static constexpr int kStageA = BM * BK * 2;
  static constexpr int kStageB = BN * BK * 2;
  static constexpr int kStage = kStageA + kStageB;
  static constexpr int kStages = (BN == 256) ? 4 : 6;
  static constexpr int kEpi = 4 * kStageFloats * 4;
  static constexpr int kBytes = kStages * kStage + kEpi + 1024 /*align slack*/ + 256 /*barriers*/;
};

// One unit of work: rows [m0, m0 + BM) x a slice of `w` accumulator columns of tile column n_blk.
struct Item {
  int m0, n_blk, sub, w;
  int kb_lo, kb_len;    // k blocks [kb_lo, kb_lo + kb_len) of every plane
};

template <int BN>
__device__ __forceinline__ Item decode_item(int idx_k, const GemmArgs& g, int m_tiles, int kb_per_part) {
  const int idx = idx_k / g.ksplit, ks = idx_k - idx * g.ksplit;
  const int kb_lo = ks * g.kb_per_split;
  const int kb_len = min(g.kb_per_split, kb_per_part - kb_lo);
  int tile = idx, sub = 0, w = BN;
  if (idx >= g.main_items) {
    const int t = idx - g.main_items;
    tile = g.main_items + t / g.tail_split;
    sub = t % g.tail_split;
    w = BN / g.tail_split;
  }
  if (g.col_fast) return Item{(tile / g.n_tiles_n) * BM, tile % g.n_tiles_n, sub, w, kb_lo, kb_len};
  return Item{(tile % m_tiles) * BM, tile / m_tiles, sub, w, kb_lo, kb_len};
}

// Weight row of the j-th 64-row box of an item.  SwiGLU tiles hold BN/2 gate rows then the BN/2 up rows of the
// same features; a slice takes w/2 of each so that gate and up of a feature stay in one accumulator.
template <int BN, int EPI>
__device__ __forceinline__ int box_row(const Item& it, int j) {
  if constexpr (EPI == ADAMK_PF_EPI_SWIGLU) {
    const int half_boxes = it.w / (2 * BOXN);
    return j < half_boxes ? it.n_blk * BN + it.sub * (it.w / 2) + j * BOXN
                          : it.n_blk * BN + BN / 2 + it.sub * (it.w / 2) + (j - half_boxes) * BOXN;
  } else {
    return it.n_blk * BN + it.sub * it.w + j * BOXN;
  }
}

__device__ __forceinline__ uint2 split4(const float4 v, uint2* lo) {
  const __nv_bfloat16 h0 = __float2bfloat16_rn(v.x), h1 = __float2bfloat16_rn(v.y), h2 = __float2bfloat16_rn(v.z),
                      h3 = __float2bfloat16_rn(v.w);
  const __nv_bfloat16 l0 = __float2bfloat16_rn(v.x - __bfloat162float(h0)), l1 = __float2bfloat16_rn(v.y - __bfloat162float(h1)),
                      l2 = __float2bfloat16_rn(v.z - __bfloat162float(h2)), l3 = __float2bfloat16_rn(v.w - __bfloat162float(h3));
  auto pack = [](__nv_bfloat16 a, __nv_bfloat16 b) { return uint32_t(__bfloat16_as_ushort(a)) | (uint32_t(__bfloat16_as_ushort(b)) << 16); };
  *lo = make_uint2(pack(l0, l1), pack(l2, l3));
  return make_uint2(pack(h0, h1), pack(h2, h3));
}

// Drain one accumulator slice (this warp's 32 rows x w columns at t_addr) with the fused epilogue.
template <int BN, int EPI>
__device__ __forceinline__ void epilogue_tile(const GemmArgs& g, uint32_t t_addr, float* patch, int row0, int n_blk, int sub, int w,
                                              int lane, int sub_row, int cg, bool first_split) {
  if constexpr (EPI == ADAMK_PF_EPI_SWIGLU) {
    const int halfw = w / 2;
    const int f0 = n_blk * (BN / 2) + sub * halfw;
    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(g.out);
#pragma unroll 1
    for (int c = 0; c < halfw; c += 32) {
      uint32_t ga[32], up[32];
      tmem_ld32(t_addr + c, ga);
      tmem_ld32(t_addr + halfw + c, up);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float a = __uint_as_float(ga[j + i]);
          v[i] = __fdividef(a, 1.0f + __expf(-a)) * __uint_as_float(up[j + i]);   // fast divide: the IEEE slow path costs more than the tile
        }
        *reinterpret_cast<float4*>(patch + lane * kStagePitch + j) = make_float4(v[0], v[1], v[2], v[3]);
      }
      __syncwarp();
      const int f = f0 + c + cg;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = i * 4 + sub_row, row = row0 + r;
        const float4 v = *reinterpret_cast<const float4*>(patch + r * kStagePitch + cg);
        if (row < g.T && f < g.N / 2) {
          uint2 lo;
          const uint2 hi = split4(v, &lo);
          __nv_bfloat16* dst = out + (long long)row * g.ldo + f;
          *reinterpret_cast<uint2*>(dst) = hi;
          if (g.parts_out == 2) *reinterpret_cast<uint2*>(dst + g.part_stride) = lo;
        }
      }
      __syncwarp();
    }
  } else if constexpr (EPI == ADAMK_PF_EPI_ATOMIC) {
    // Decode-sized tiles: a handful of live rows per warp, so the warp's instruction latency is the cost
    // (tools/gemm_trace.py: 4.9 us per 256-column tile for the general path, 3.3 us for this one).  Row bookkeeping is
    // done once per tile and only live rows are staged and sent.  The stacked planes of a token go out as separate
    // atomics: summing them in the patch first was measured slower (2.55 vs 2.31 ms per batch-8 step).
    const int n0 = n_blk * BN + sub * w;
    float* out = static_cast<float*>(g.out);
    // rows of this patch that hold data (stacked == 2: plane q sits in rows [32 q, 32 q + T), one TMEM lane quarter and
    // therefore one epilogue warp per plane instead of one warp for all of them)
    const int live = g.stacked == 2 ? min(32, g.T) : min(32, (g.stacked ? g.parts * g.T : g.T) - row0);
    const int n_it = (live + 3) >> 2;
    long long roff[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = row0 + i * 4 + sub_row;
      roff[i] = (i * 4 + sub_row < live) ? (long long)(g.stacked == 2 ? (row & 31) : g.stacked ? row % g.T : row) * g.ldo : -1;
    }
#pragma unroll 1
    for (int c = 0; c < w; c += 64) {   // two tensor-memory loads in flight per wait (w is a multiple of 64)
      uint32_t acc[2][32];
      tmem_ld32(t_addr + c, acc[0]);
      tmem_ld32(t_addr + c + 32, acc[1]);
      tmem_ld_wait();
#pragma unroll
      for (int hc = 0; hc < 2; ++hc) {
        const int col = n0 + c + hc * 32 + cg;
        const bool col_ok = col < g.N;
        const float4 b = (g.bias != nullptr && col_ok && first_split) ? *reinterpret_cast<const float4*>(g.bias + col) : make_float4(0, 0, 0, 0);
        if (lane < live) {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(patch + lane * kStagePitch + j) = make_float4(
                __uint_as_float(acc[hc][j]), __uint_as_float(acc[hc][j + 1]), __uint_as_float(acc[hc][j + 2]), __uint_as_float(acc[hc][j + 3]));
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i < n_it && roff[i] >= 0 && col_ok) {
            const int r = i * 4 + sub_row;
            float4 v = *reinterpret_cast<const float4*>(patch + r * kStagePitch + cg);
            if (row0 + r < g.T) { v.x += b.x; v.y += b.y; v.z += b.z; v.w += b.w; }   // bias: once per output row
            atomicAdd(reinterpret_cast<float4*>(out + roff[i] + col), v);
          }
        }
        __syncwarp();
      }
    }
  } else {
    const int n0 = n_blk * BN + sub * w;
    float* out = static_cast<float*>(g.out);
#pragma unroll 1
    for (int c = 0; c < w; c += 32) {
      uint32_t acc[32];
      tmem_ld32(t_addr + c, acc);
      const int col = n0 + c + cg;
      const bool col_ok = col < g.N;
      float4 o[8];
      if constexpr (EPI == ADAMK_PF_EPI_RESID) {   // residual rows: in flight while the accumulator arrives
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int row = row0 + i * 4 + sub_row;
          o[i] = (row < g.T && col_ok) ? *reinterpret_cast<const float4*>(out + (long long)row * g.ldo + col) : make_float4(0, 0, 0, 0);
        }
      } else {
        const float4 b = (g.bias != nullptr && col_ok) ? *reinterpret_cast<const float4*>(g.bias + col) : make_float4(0, 0, 0, 0);
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = b;
      }
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(patch + lane * kStagePitch + j) =
            make_float4(__uint_as_float(acc[j]), __uint_as_float(acc[j + 1]), __uint_as_float(acc[j + 2]), __uint_as_float(acc[j + 3]));
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = i * 4 + sub_row, row = row0 + r;
        float4 v = *reinterpret_cast<const float4*>(patch + r * kStagePitch + cg);
        v.x += o[i].x; v.y += o[i].y; v.z += o[i].z; v.w += o[i].w;
        if (row < g.T && col_ok) *reinterpret_cast<float4*>(out + (long long)row * g.ldo + col) = v;
      }
      __syncwarp();
    }
  }
}

template <int BN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
gemm_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w, const GemmArgs g) {
  using S = Smem<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* epi_stage = reinterpret_cast<float*>(smem + S::kStages * S::kStage);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kStages * S::kStage + S::kEpi);
  uint64_t* empty = full + S::kStages;
  uint64_t* acc_full = empty + S::kStages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  griddep_launch();
  if (threadIdx.x == 0) PF_STAMP(0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_tiles = (g.T + BM - 1) / BM;
  const int kb_per_part = (g.K + BK - 1) / BK;
  const int n_work = g.n_items * g.ksplit;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_x)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_w)) : "memory");
    for (int s = 0; s < S::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "n"(2 * BN) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch: the weight operand is constant data, so the producer lane fills the (empty) ring
  // with the weight boxes of its first kStages k blocks BEFORE waiting for the previous kernel; only the token
  // rows, the accumulator targets and the bias wait.  A decode-sized launch otherwise spends 2.8-3.8 us on its
  // first operands from cold HBM (tools/gemm_trace.py) with nothing in flight.
  const bool producer = warp == 0 && lane == 0;
  int pre = 0;   // ring stages whose weight boxes (and transaction count) were issued ahead of the wait
  if (producer && g.w_early) {
    int ahead = 0;   // k blocks past the ring whose weight boxes were requested into L2 (w_early >= 2)
    const int ahead_max = g.w_early >= 2 ? kEarlyL2Blocks : 0;
    for (int idx = blockIdx.x; idx < n_work && (pre < S::kStages || ahead < ahead_max); idx += gridDim.x) {
      const Item it = decode_item<BN>(idx, g, m_tiles, kb_per_part);
      const int boxes = it.w / BOXN;
      const int n_kb = it.kb_len * (g.stacked ? 1 : g.parts);
      for (int kb = 0; kb < n_kb && (pre < S::kStages || ahead < ahead_max); ++kb) {
        const int part = kb / it.kb_len, k0 = (it.kb_lo + kb - part * it.kb_len) * BK;
        if (pre < S::kStages) {
          uint8_t* sa = smem + pre * S::kStage;
          mbar_expect_tx(&full[pre], S::kStageA + boxes * BOXN * BK * 2);
          for (int j = 0; j < boxes; ++j)
            tma_load_2d(&map_w, &full[pre], sa + S::kStageA + j * (BOXN * BK * 2), k0, box_row<BN, EPI>(it, j));
          ++pre;
        } else {
          if (part == 0 || g.stacked)   // the planes of an unstacked pass walk the same weight again
            for (int j = 0; j < boxes; ++j) tma_prefetch_2d(&map_w, k0, box_row<BN, EPI>(it, j));
          ++ahead;
        }
      }
    }
  }
  griddep_wait();   // everything above overlapped the previous kernel's tail
  if (threadIdx.x == 0) PF_STAMP(1);

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int issued = 0;
      for (int idx = blockIdx.x; idx < n_work; idx += gridDim.x) {
        const Item it = decode_item<BN>(idx, g, m_tiles, kb_per_part);
        const int boxes = it.w / BOXN;
        const uint32_t bytes = S::kStageA + boxes * BOXN * BK * 2;
        const int n_kb = it.kb_len * (g.stacked ? 1 : g.parts);
        for (int kb = 0; kb < n_kb; ++kb, ++issued) {
          const int part = kb / it.kb_len, k0 = (it.kb_lo + kb - part * it.kb_len) * BK;
          uint8_t* sa = smem + stage * S::kStage;
          if (issued < pre) {   // first pass over the ring: the weights are already on their way
            if (g.stacked == 2) tma_load_3d(&map_x, &full[stage], sa, k0, 0, 0);
            else tma_load_2d(&map_x, &full[stage], sa, k0, part * g.T + it.m0);
          } else {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_expect_tx(&full[stage], bytes);
            if (g.stacked == 2) tma_load_3d(&map_x, &full[stage], sa, k0, 0, 0);   // plane p -> rows [32 p, 32 p + T)
            else tma_load_2d(&map_x, &full[stage], sa, k0, part * g.T + it.m0);
            for (int j = 0; j < boxes; ++j)
              tma_load_2d(&map_w, &full[stage], sa + S::kStageA + j * (BOXN * BK * 2), k0, box_row<BN, EPI>(it, j));
          }
          if (++stage == S::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int n = 0;
      for (int idx = blockIdx.x; idx < n_work; idx += gridDim.x, ++n) {
        const Item it = decode_item<BN>(idx, g, m_tiles, kb_per_part);
        const uint32_t idesc = instr_desc(BM, it.w);
        const int as = n & 1;
        mbar_wait(&acc_empty[as], ((n >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * BN;
        const int n_kb = it.kb_len * (g.stacked ? 1 : g.parts);
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (n == 0 && kb == 0) PF_STAMP(2);
          const uint32_t a_addr = smem_u32(smem + stage * S::kStage);
          const uint64_t a_desc = smem_desc_sw128(a_addr), b_desc = smem_desc_sw128(a_addr + S::kStageA);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)
            umma(d_tmem, a_desc + uint64_t(k * UK * 2 >> 4), b_desc + uint64_t(k * UK * 2 >> 4), idesc, (kb | k) != 0);
          umma_commit(&empty[stage]);
          if (++stage == S::kStages) { stage = 0; phase ^= 1; }
        }
        umma_commit(&acc_full[as]);
        if (n == 0) PF_STAMP(3);
      }
    }
  } else {
    if (g.pf_bytes > 0 && warp == 2) {
      // L2 prefetch of the next kernel's weights: this CTA's 1/gridDim share, 4 KB per request, one lane per request
      const long long per = ((g.pf_bytes / gridDim.x) + 4095) & ~4095ll;
      const long long lo = per * blockIdx.x, hi = min(lo + per, g.pf_bytes & ~15ll);
      for (long long off = lo + lane * 4096ll; off < hi; off += 32 * 4096ll) {
        const uint32_t sz = uint32_t(min(4096ll, hi - off));
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g.pf_ptr + off), "r"(sz) : "memory");
      }
    }
    // Epilogue.  tcgen05.ld hands each lane one accumulator row; a row-per-lane store would touch 32 lines per
    // instruction, so every 32 x 32 block goes through a padded shared-memory patch and leaves as 4 rows x 128
    // contiguous bytes per instruction (8 lanes per row).
    const int quarter = warp & 3;   // the TMEM lanes this warp may read: 32 * (warp id % 4)
    float* patch = epi_stage + quarter * kStageFloats;
    const int sub_row = lane >> 3, cg = (lane & 7) * 4;
    int n = 0;
    for (int idx = blockIdx.x; idx < n_work; idx += gridDim.x, ++n) {
      const Item it = decode_item<BN>(idx, g, m_tiles, kb_per_part);
      const int as = n & 1;
      const int row0 = it.m0 + quarter * 32;
      mbar_wait(&acc_full[as], (n >> 1) & 1);
      tc_fence_after();
      if (n == 0 && quarter == 0 && lane == 0) PF_STAMP(6);
      const uint32_t t_addr = tmem_base + as * BN + (uint32_t(quarter * 32) << 16);
      const int rows_live = (EPI == ADAMK_PF_EPI_ATOMIC && g.stacked) ? (g.stacked == 2 ? g.parts * 32 : g.parts * g.T) : g.T;
      if (row0 < rows_live)   // decode-sized T: most warps own no live row and only hand the accumulator back
        epilogue_tile<BN, EPI>(g, t_addr, patch, row0, it.n_blk, it.sub, it.w, lane, sub_row, cg, it.kb_lo == 0);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[as]);
      if (n == 0 && quarter == 0 && lane == 0) PF_STAMP(4);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) PF_STAMP(5);
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(2 * BN) : "memory");
  }
}

// ---------------------------------------------------------------------------------------------------------
// CTA-pair variant: two CTAs of one cluster (the two SMs of a TPC) share a 256 x 256 tile.  Each CTA stages its
// own 128 token rows and HALF of the weight tile (128 rows), tcgen05.mma.cta_group::2 issued by the leader reads
// both halves, and each CTA keeps the accumulator of its own 128 rows in its own tensor memory.  Per SM that is
// 32 KB of operands per k block instead of 48 KB for the same tensor work, and six ring stages instead of four:
// the single-CTA kernel is bound by the bytes it can keep in flight from L2, this one is not.

constexpr uint32_t kPeerMask = 0xFEFFFFFFu;   // shared::cluster address of the same offset in the pair's leader CTA

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, uint64_t* leader_bar, void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(leader_bar) & kPeerMask)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {   // arrive on the leader CTA's copy of `bar`
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, 0;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void umma_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  const uint32_t z = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(z)
      : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {   // arrive on `bar` in both CTAs of the pair
  const uint16_t both = 3;
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "h"(both)
               : "memory");
}

struct PairSmem {
  static constexpr int BN = 256;
  static constexpr int kStageA = BM * BK * 2;
  static constexpr int kStageB = (BN / 2) * BK * 2;
  static constexpr int kStage = kStageA + kStageB;
  static constexpr int kStages = 6;
  static constexpr int kEpi = 4 * kStageFloats * 4;
  static constexpr int kBytes = kStages * kStage + kEpi + 1024 + 256;
};

template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
gemm_pair_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w, const GemmArgs g) {
  using S = PairSmem;
  constexpr int BN = S::BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* epi_stage = reinterpret_cast<float*>(smem + S::kStages * S::kStage);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kStages * S::kStage + S::kEpi);
  uint64_t* empty = full + S::kStages;
  uint64_t* acc_full = empty + S::kStages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  griddep_launch();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int m_tiles = (g.T + 2 * BM - 1) / (2 * BM);
  const int kb_per_part = (g.K + BK - 1) / BK;
  const int n_kb = kb_per_part * g.parts;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_x)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_w)) : "memory");
    for (int s = 0; s < S::kStages; ++s) {
      mbar_init(&full[s], 2);    // leader: arrive.expect_tx of both CTAs' bytes; peer: plain remote arrive
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 8);   // the four epilogue warps of each CTA
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "n"(2 * BN) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();

  // item -> (row block of 256 tokens, tile column, column slice); slices of the last wave are w = 128 wide
  auto decode = [&](int idx, int& m0, int& n_blk, int& sub, int& w) {
    int tile = idx;
    sub = 0;
    w = BN;
    if (idx >= g.main_items) {
      const int t = idx - g.main_items;
      tile = g.main_items + t / g.tail_split;
      sub = t % g.tail_split;
      w = BN / g.tail_split;
    }
    if (g.col_fast) {
      m0 = (tile / g.n_tiles_n) * 2 * BM;
      n_blk = tile % g.n_tiles_n;
    } else {
      m0 = (tile % m_tiles) * 2 * BM;
      n_blk = tile / m_tiles;
    }
  };

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int idx = pair; idx < g.n_items; idx += n_pairs) {
        int m0, n_blk, sub, w;
        decode(idx, m0, n_blk, sub, w);
        const int boxes = w / (2 * BOXN);   // this CTA's half of the slice
        const uint32_t bytes = S::kStageA + boxes * BOXN * BK * 2;
        const int wrow0 = (EPI == ADAMK_PF_EPI_SWIGLU) ? n_blk * BN + int(rank) * (BN / 2) + sub * (w / 2)
                                                       : n_blk * BN + sub * w + int(rank) * (w / 2);
        for (int kb = 0; kb < n_kb; ++kb) {
          const int part = kb / kb_per_part, k0 = (kb - part * kb_per_part) * BK;
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * S::kStage;
          if (rank == 0) mbar_expect_tx(&full[stage], 2 * bytes);
          else mbar_arrive_leader(&full[stage]);
          tma_load_2d_pair(&map_x, &full[stage], sa, k0, part * g.T + m0 + int(rank) * BM);
          for (int j = 0; j < boxes; ++j)
            tma_load_2d_pair(&map_w, &full[stage], sa + S::kStageA + j * (BOXN * BK * 2), k0, wrow0 + j * BOXN);
          if (++stage == S::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int n = 0;
      for (int idx = pair; idx < g.n_items; idx += n_pairs, ++n) {
        int m0, n_blk, sub, w;
        decode(idx, m0, n_blk, sub, w);
        const uint32_t idesc = instr_desc(2 * BM, w);
        const int as = n & 1;
        mbar_wait(&acc_empty[as], ((n >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * BN;
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + stage * S::kStage);
          const uint64_t a_desc = smem_desc_sw128(a_addr), b_desc = smem_desc_sw128(a_addr + S::kStageA);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)
            umma_pair(d_tmem, a_desc + uint64_t(k * UK * 2 >> 4), b_desc + uint64_t(k * UK * 2 >> 4), idesc, (kb | k) != 0);
          umma_commit_pair(&empty[stage]);
          if (++stage == S::kStages) { stage = 0; phase ^= 1; }
        }
        umma_commit_pair(&acc_full[as]);
      }
    }
  } else {
    const int quarter = warp & 3;
    float* patch = epi_stage + quarter * kStageFloats;
    const int sub_row = lane >> 3, cg = (lane & 7) * 4;
    int n = 0;
    for (int idx = pair; idx < g.n_items; idx += n_pairs, ++n) {
      int m0, n_blk, sub, w;
      decode(idx, m0, n_blk, sub, w);
      const int as = n & 1;
      const int row0 = m0 + int(rank) * BM + quarter * 32;
      mbar_wait(&acc_full[as], (n >> 1) & 1);
      tc_fence_after();
      const uint32_t t_addr = tmem_base + as * BN + (uint32_t(quarter * 32) << 16);
      epilogue_tile<BN, EPI>(g, t_addr, patch, row0, n_blk, sub, w, lane, sub_row, cg, true);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) mbar_arrive(&acc_empty[as]);
        else mbar_arrive_leader(&acc_empty[as]);
      }
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(2 * BN) : "memory");
  }
}

// ---------------------------------------------------------------------------------------------------------
// host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                  const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static thread_local char g_err[256] = "";
char* err_buf() { return g_err; }

static unsigned long long* g_trace = nullptr;   // adamk_prefill_set_trace()
static const uint8_t* g_pf_ptr = nullptr;        // adamk_prefill_prefetch_next(): consumed by the next GEMM launch
static long long g_pf_bytes = 0;
static int g_pdl = 0;   // adamk_prefill_set_pdl(): launch with programmatic stream serialization
static int g_walk = -1;  // adamk_prefill_set_walk(): -1 = choose per call, 0 = token block fastest, 1 = tile column fastest
int pdl_enabled() { return g_pdl; }

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

// 2-D bf16 tensor [rows, cols] row-major, box [box_rows, 64 columns], 128-byte swizzle, zero fill outside.
static bool make_map(CUtensorMap* m, const void* base, long long rows, long long cols, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) {
    snprintf(g_err, sizeof g_err, "cuTensorMapEncodeTiled is not available from this driver");
    return false;
  }
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(cols) * 2};
  cuuint32_t box[2] = {cuuint32_t(BK), cuuint32_t(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(g_err, sizeof g_err, "cuTensorMapEncodeTiled failed with %d (rows %lld cols %lld box %d)", int(r), rows, cols, box_rows);
    return false;
  }
  return true;
}

// The token operand of a stacked decode-sized call as bf16 [parts][T][cols]: box [4 planes][32 rows][64 columns], so
// that plane p lands in rows [32 p, 32 p + T) of the 128-row tile (rows and planes outside the tensor are zero filled).
static bool make_map_planes(CUtensorMap* m, const void* base, int parts, long long T, long long cols) {
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) {
    snprintf(g_err, sizeof g_err, "cuTensorMapEncodeTiled is not available from this driver");
    return false;
  }
  cuuint64_t dims[3] = {cuuint64_t(cols), cuuint64_t(T), cuuint64_t(parts)};
  cuuint64_t strides[2] = {cuuint64_t(cols) * 2, cuuint64_t(T) * cuuint64_t(cols) * 2};
  cuuint32_t box[3] = {cuuint32_t(BK), 32, 4};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(g_err, sizeof g_err, "cuTensorMapEncodeTiled (planes) failed with %d (parts %d T %lld cols %lld)", int(r), parts, T, cols);
    return false;
  }
  return true;
}

static int g_quarters = 1;   // adamk_prefill_set_plane_quarters()

// How one GEMM call is cut into work: tile shape, work items (whole tiles + column slices of the last wave), split-K.
// Pure host arithmetic (adamk_prefill_gemm_plan exposes it; tests/test_prefill_plan.py checks it without a GPU).
struct Plan {
  int tile;   // ADAMK_PF_TILE_128 / _256 / _PAIR
  int tiles, main_items, tail_split, n_items, ksplit, kb_per_split, stacked, grid;
};

static double waves_of(long long tiles, int units, int max_split) {
  const long long full = tiles / units, rem = tiles % units;
  int split = 1;
  while (rem > 0 && split * 2 <= max_split && rem * split * 2 <= units) split *= 2;
  return double(full) + (rem ? 1.0 / split : 0.0);
}

static Plan plan_gemm(int T, int N, int K, int parts, int epilogue, int tile, int n_sms) {
  Plan p = {};
  if (tile == ADAMK_PF_TILE_AUTO) {
    // 256-wide tiles for wide outputs; between one CTA per tile and a CTA pair per 256 x 256 tile take the one whose
    // last wave is fuller (tile times are equal: a pair does twice the work on twice the SMs), pairs on a tie.
    if (N < 1024 && epilogue != ADAMK_PF_EPI_SWIGLU) {
      tile = ADAMK_PF_TILE_128;
    } else if (epilogue == ADAMK_PF_EPI_ATOMIC && T <= BM && (long long)N * K * 2 <= (32ll << 20)) {
      // decode-sized and short: the one-warp epilogue (1.8 us per 128 columns) outweighs the k loop, which a
      // 128-wide tile lengthens (tools/gemm_trace.py: 12.1 vs 13.3 us for QKV, 16.3 vs 17.4 for down, but 24.8 vs
      // 24.3 for the 55 MB gate/up matrix, which therefore stays on 256)
      tile = ADAMK_PF_TILE_128;
    } else {
      const long long n_t = (N + 255) / 256;
      const double single = waves_of((long long)((T + BM - 1) / BM) * n_t, n_sms, epilogue == ADAMK_PF_EPI_SWIGLU ? 2 : 4);
      const double paired = waves_of((long long)((T + 2 * BM - 1) / (2 * BM)) * n_t, n_sms / 2, 2);
      tile = (T > BM && paired <= single && epilogue != ADAMK_PF_EPI_ATOMIC && n_sms >= 2) ? ADAMK_PF_TILE_PAIR : ADAMK_PF_TILE_256;
    }
  }
  p.tile = tile;
  const int kb_per_part = (K + BK - 1) / BK;
  p.ksplit = 1;
  p.kb_per_split = kb_per_part;
  p.tail_split = 1;
  if (tile == ADAMK_PF_TILE_PAIR) {
    p.tiles = ((T + 2 * BM - 1) / (2 * BM)) * ((N + 255) / 256);
    const int max_pairs = n_sms / 2;
    const int pairs = p.tiles < max_pairs ? p.tiles : max_pairs;
    const int rem = p.tiles % pairs;
    p.tail_split = (rem > 0 && rem * 2 <= pairs) ? 2 : 1;   // a slice is at least one 64-row weight box per CTA
    p.main_items = p.tiles - rem;
    p.n_items = p.main_items + rem * p.tail_split;
    p.grid = 2 * pairs;
    return p;
  }
  // One CTA per tile.  Whole tiles, except that the tiles of a last partial wave are cut into column slices so that
  // the wave keeps every SM busy for a fraction of a tile time; with fewer tiles than SMs every tile is sliced.
  const int BN = tile;
  p.tiles = ((T + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int max_split = (epilogue == ADAMK_PF_EPI_SWIGLU) ? BN / (2 * BOXN) : BN / BOXN;
  int split = 1;
  if (epilogue == ADAMK_PF_EPI_ATOMIC) {
    // decode-sized: whole weight boxes per stage and as many K ranges as there are idle SMs keep the most bytes in
    // flight; all planes ride in one token tile when they fit
    p.main_items = p.tiles;
    p.n_items = p.tiles;
    p.stacked = (parts * T <= BM) ? 1 : 0;
    if (p.tiles * 2 <= n_sms) {
      int want = n_sms / p.tiles;
      if (want > kb_per_part) want = kb_per_part;
      p.kb_per_split = (kb_per_part + want - 1) / want;
      p.ksplit = (kb_per_part + p.kb_per_split - 1) / p.kb_per_split;
    }
  } else if (p.tiles < n_sms) {
    while (split * 2 <= max_split && p.tiles * split * 2 <= n_sms) split *= 2;
    p.main_items = 0;
    p.n_items = p.tiles * split;
  } else {
    const int rem = p.tiles % n_sms;
    while (rem > 0 && split * 2 <= max_split && rem * split * 2 <= n_sms) split *= 2;
    p.main_items = p.tiles - rem;
    p.n_items = p.main_items + rem * split;
  }
  p.tail_split = split;
  const long long work = (long long)p.n_items * p.ksplit;
  p.grid = work < n_sms ? int(work) : n_sms;
  return p;
}

static void apply_plan(GemmArgs& g, const Plan& p) {
  g.main_items = p.main_items;
  g.tail_split = p.tail_split;
  g.n_items = p.n_items;
  g.ksplit = p.ksplit;
  g.kb_per_split = p.kb_per_split;
  g.stacked = (p.stacked && g.quarters) ? 2 : p.stacked;
  g.w_early = g_pdl >= 2 ? g_pdl - 1 : 0;
}

template <int BN, int EPI>
static int launch(const CUtensorMap& mx, const CUtensorMap& mw, const GemmArgs& g_in, const Plan& plan, cudaStream_t stream) {
  static bool configured = false;
  auto kern = gemm_kernel<BN, EPI>;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<BN>::kBytes);
    if (e != cudaSuccess) {
      snprintf(g_err, sizeof g_err, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
      return ADAMK_PF_E_CUDA;
    }
    configured = true;
  }
  GemmArgs g = g_in;
  apply_plan(g, plan);
  const int grid = plan.grid;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(kThreads);
  lc.dynamicSmemBytes = Smem<BN>::kBytes;
  lc.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = g_pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&lc, kern, mx, mw, g);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof g_err, "prefill gemm launch: %s", cudaGetErrorString(e));
    return ADAMK_PF_E_CUDA;
  }
  return ADAMK_PF_OK;
}

template <int EPI>
static int launch_pair(const CUtensorMap& mx, const CUtensorMap& mw, const GemmArgs& g_in, const Plan& plan, cudaStream_t stream) {
  static bool configured = false;
  auto kern = gemm_pair_kernel<EPI>;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, PairSmem::kBytes);
    if (e != cudaSuccess) {
      snprintf(g_err, sizeof g_err, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
      return ADAMK_PF_E_CUDA;
    }
    configured = true;
  }
  GemmArgs g = g_in;
  apply_plan(g, plan);
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(plan.grid);
  lc.blockDim = dim3(kThreads);
  lc.dynamicSmemBytes = PairSmem::kBytes;
  lc.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = g_pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&lc, kern, mx, mw, g);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof g_err, "prefill gemm (CTA pair) launch: %s", cudaGetErrorString(e));
    return ADAMK_PF_E_CUDA;
  }
  return ADAMK_PF_OK;
}

}  // namespace pf

extern "C" {

const char* adamk_prefill_last_error(void) { return pf::g_err; }

void adamk_prefill_set_walk(int mode) { pf::g_walk = mode < 0 ? -1 : (mode ? 1 : 0); }
void adamk_prefill_set_plane_quarters(int on) { pf::g_quarters = on ? 1 : 0; }
void adamk_prefill_set_pdl(int on) { pf::g_pdl = on < 0 ? 0 : (on > 3 ? 3 : on); }

void adamk_prefill_prefetch_next(const void* ptr, long long bytes) {
  pf::g_pf_ptr = static_cast<const uint8_t*>(ptr);
  pf::g_pf_bytes = (ptr != nullptr && bytes > 0) ? bytes : 0;
}

void adamk_prefill_set_trace(void* stamps) { pf::g_trace = static_cast<unsigned long long*>(stamps); }

// Argument checks shared by the planner and the launcher (no device access).
static int check_shape(int parts, int T, int K, int N, int ldo, int epilogue, int parts_out, int tile_n) {
  using namespace pf;
  if (T <= 0 || N <= 0 || K <= 0 || parts < 1 || parts > 3) {
    snprintf(g_err, sizeof g_err, "prefill gemm: bad argument (T %d N %d K %d parts %d)", T, N, K, parts);
    return ADAMK_PF_E_INVALID;
  }
  if (K % 8 != 0 || N % 8 != 0 || ldo % 8 != 0) {
    snprintf(g_err, sizeof g_err, "prefill gemm: K, N and ldo must be multiples of 8 (K %d N %d ldo %d)", K, N, ldo);
    return ADAMK_PF_E_INVALID;
  }
  if (epilogue < ADAMK_PF_EPI_STORE || epilogue > ADAMK_PF_EPI_ATOMIC) {
    snprintf(g_err, sizeof g_err, "prefill gemm: unknown epilogue %d", epilogue);
    return ADAMK_PF_E_INVALID;
  }
  if (tile_n != ADAMK_PF_TILE_AUTO && tile_n != ADAMK_PF_TILE_128 && tile_n != ADAMK_PF_TILE_256 && tile_n != ADAMK_PF_TILE_PAIR) {
    snprintf(g_err, sizeof g_err, "prefill gemm: tile must be 0, 128, 256 or ADAMK_PF_TILE_PAIR");
    return ADAMK_PF_E_INVALID;
  }
  if (tile_n == ADAMK_PF_TILE_PAIR && epilogue == ADAMK_PF_EPI_ATOMIC) {
    snprintf(g_err, sizeof g_err, "prefill gemm: the atomic (split-K) epilogue runs on one-CTA tiles only");
    return ADAMK_PF_E_INVALID;
  }
  if (epilogue == ADAMK_PF_EPI_SWIGLU) {
    const int width = tile_n == ADAMK_PF_TILE_128 ? 128 : 256;
    if (N % width != 0 || (parts_out != 1 && parts_out != 2)) {
      snprintf(g_err, sizeof g_err, "prefill gemm: SwiGLU epilogue needs N %% tile width == 0 and 1 or 2 output planes");
      return ADAMK_PF_E_INVALID;
    }
  }
  return ADAMK_PF_OK;
}

int adamk_prefill_gemm_plan(int parts, int T, int K, int N, int epilogue, int tile_n, int n_sms, int32_t plan_out[9]) {
  if (plan_out == nullptr || n_sms <= 0) return ADAMK_PF_E_INVALID;
  const int rc = check_shape(parts, T, K, N, 8, epilogue, 2, tile_n);
  if (rc != ADAMK_PF_OK) return rc;
  const pf::Plan p = pf::plan_gemm(T, N, K, parts, epilogue, tile_n, n_sms);
  const int32_t v[9] = {p.tile, p.tiles, p.main_items, p.tail_split, p.n_items, p.ksplit, p.kb_per_split, p.stacked, p.grid};
  for (int i = 0; i < 9; ++i) plan_out[i] = v[i];
  return ADAMK_PF_OK;
}

int adamk_prefill_gemm(const void* x_planes, int parts, int T, int K, const void* w, int N, const float* bias, void* out, int ldo,
                       int epilogue, int parts_out, long long part_stride, int tile_n, adamk_pf_stream stream) {
  using namespace pf;
  if (x_planes == nullptr || w == nullptr || out == nullptr) {
    snprintf(g_err, sizeof g_err, "prefill gemm: null operand");
    return ADAMK_PF_E_INVALID;
  }
  const int rc = check_shape(parts, T, K, N, ldo, epilogue, parts_out, tile_n);
  if (rc != ADAMK_PF_OK) return rc;
  if ((reinterpret_cast<uintptr_t>(x_planes) | reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(out)) & 15) {
    snprintf(g_err, sizeof g_err, "prefill gemm: operands must be 16-byte aligned");
    return ADAMK_PF_E_INVALID;
  }
  int dev = 0, n_sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    snprintf(g_err, sizeof g_err, "prefill gemm: no CUDA device");
    return ADAMK_PF_E_CUDA;
  }
  const Plan plan = plan_gemm(T, N, K, parts, epilogue, tile_n, n_sms);
  CUtensorMap mx, mw;
  // a stacked decode-sized call with several planes of at most 32 tokens: one tensor-memory lane quarter per plane
  const bool quarters = g_quarters && plan.stacked && plan.tile != ADAMK_PF_TILE_PAIR && epilogue == ADAMK_PF_EPI_ATOMIC && T <= 32 &&
                        parts >= 2 && parts <= 4;
  if (!(quarters ? make_map_planes(&mx, x_planes, parts, T, K) : make_map(&mx, x_planes, (long long)parts * T, K, BM)) ||
      !make_map(&mw, w, N, K, BOXN))
    return ADAMK_PF_E_CUDA;
  GemmArgs g{T, N, K, parts, ldo, bias, out, parts_out, part_stride, 0, 1, 0, 1, 0, g_pf_ptr, g_pf_bytes, g_trace, 0};
  g.quarters = quarters ? 1 : 0;
  g_pf_ptr = nullptr;
  g_pf_bytes = 0;
  {
    // walk order: tile column fastest when the activation is the larger operand and the weight fits L2 with room to spare
    const long long xb = (long long)parts * T * K * 2, wb = (long long)N * K * 2;
    const int bn = plan.tile == ADAMK_PF_TILE_PAIR ? 256 : plan.tile;
    g.n_tiles_n = (N + bn - 1) / bn;
    g.col_fast = g_walk >= 0 ? g_walk : (epilogue != ADAMK_PF_EPI_ATOMIC && xb > wb && wb <= (48ll << 20));
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (plan.tile == ADAMK_PF_TILE_PAIR) {
    switch (epilogue) {
      case ADAMK_PF_EPI_STORE: return launch_pair<ADAMK_PF_EPI_STORE>(mx, mw, g, plan, s);
      case ADAMK_PF_EPI_RESID: return launch_pair<ADAMK_PF_EPI_RESID>(mx, mw, g, plan, s);
      default: return launch_pair<ADAMK_PF_EPI_SWIGLU>(mx, mw, g, plan, s);
    }
  }
  switch (epilogue * 1000 + plan.tile) {
    case ADAMK_PF_EPI_STORE * 1000 + 128: return launch<128, ADAMK_PF_EPI_STORE>(mx, mw, g, plan, s);
    case ADAMK_PF_EPI_STORE * 1000 + 256: return launch<256, ADAMK_PF_EPI_STORE>(mx, mw, g, plan, s);
    case ADAMK_PF_EPI_RESID * 1000 + 128: return launch<128, ADAMK_PF_EPI_RESID>(mx, mw, g, plan, s);
    case ADAMK_PF_EPI_RESID * 1000 + 256: return launch<256, ADAMK_PF_EPI_RESID>(mx, mw, g, plan, s);
    case ADAMK_PF_EPI_ATOMIC * 1000 + 128: return launch<128, ADAMK_PF_EPI_ATOMIC>(mx, mw, g, plan, s);
    case ADAMK_PF_EPI_ATOMIC * 1000 + 256: return launch<256, ADAMK_PF_EPI_ATOMIC>(mx, mw, g, plan, s);
    case ADAMK_PF_EPI_SWIGLU * 1000 + 128: return launch<128, ADAMK_PF_EPI_SWIGLU>(mx, mw, g, plan, s);
    default: return launch<256, ADAMK_PF_EPI_SWIGLU>(mx, mw, g, plan, s);
  }
}

}  // extern "C"
