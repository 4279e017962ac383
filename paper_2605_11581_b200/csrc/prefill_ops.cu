// prefill_ops.cu -- the element-wise operators between the Prefill GEMMs (prefill_gemm.cu): embedding gather,
// RMSNorm fused with the bf16-plane split the tensor-core GEMM consumes, q/k head norm + rotary embedding fused
// with the KV-cache write, and the plain plane split.  All HBM-bound row kernels: one CTA per token row, 16-byte
// accesses, fp32 arithmetic in the order of the decode kernel (adamk.cu) / the oracle (oracle/decode_ref.py)
// so that a cache filled here is the cache the decode kernel would have produced.

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

#include "../../include/adamk_prefill.h"

namespace pf {
char* err_buf();   // prefill_gemm.cu: the thread-local message adamk_prefill_last_error() returns
int pdl_enabled(); // prefill_gemm.cu: adamk_prefill_set_pdl()
}

namespace pfo {

// Programmatic dependent launch (see prefill_gemm.cu): every kernel here starts with griddep_sync().
__device__ __forceinline__ void griddep_sync() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <typename... KArgs, typename... Args>
static void launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = pf::pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&lc, kern, KArgs(args)...);
}

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < nw; ++i) t += red[i];   // same order in every thread
  __syncthreads();
  return t;
}

// v as the sum of `parts` bf16 values, plane p at dst[p * stride]: 1 = plain rounding, 2 = hi + lo (2^-17 relative),
// 3 = hi + mid + lo (below fp32 resolution).
__device__ __forceinline__ void put_split(__nv_bfloat16* dst, long long stride, int parts, float v) {
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  dst[0] = h;
  if (parts > 1) {
    const float r1 = v - __bfloat162float(h);
    const __nv_bfloat16 m = __float2bfloat16_rn(r1);
    dst[stride] = m;
    if (parts > 2) dst[2 * stride] = __float2bfloat16_rn(r1 - __bfloat162float(m));
  }
}

// Four consecutive values at once: one 8-byte store per plane.
__device__ __forceinline__ void put_split4(__nv_bfloat16* dst, long long stride, int parts, const float (&v)[4]) {
  float r[4] = {v[0], v[1], v[2], v[3]};
  for (int p = 0; p < parts; ++p) {
    __nv_bfloat16 b[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      b[j] = __float2bfloat16_rn(r[j]);
      r[j] -= __bfloat162float(b[j]);
    }
    const uint32_t lo = uint32_t(__bfloat16_as_ushort(b[0])) | (uint32_t(__bfloat16_as_ushort(b[1])) << 16);
    const uint32_t hi = uint32_t(__bfloat16_as_ushort(b[2])) | (uint32_t(__bfloat16_as_ushort(b[3])) << 16);
    *reinterpret_cast<uint2*>(dst + p * stride) = make_uint2(lo, hi);
  }
}

// `vocab` > 0: token ids outside [0, vocab) read row 0 instead of memory outside the table (a device-resident
// decode loop feeds tokens the host never sees)
__global__ void embed_kernel(const int32_t* __restrict__ tokens, const __nv_bfloat16* __restrict__ embed, float* __restrict__ h, int H, int vocab) {
  griddep_sync();
  const int t = blockIdx.x;
  int tok = tokens[t];
  if (vocab > 0 && (tok < 0 || tok >= vocab)) tok = 0;
  const __nv_bfloat16* src = embed + (long long)tok * H;
  float* dst = h + (long long)t * H;
  for (int i = threadIdx.x * 2; i < H; i += blockDim.x * 2) {
    const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(src + i);
    *reinterpret_cast<float2*>(dst + i) = make_float2(__low2float(v), __high2float(v));
  }
}

// planes[p][t][:] = split(h[t] * rsqrt(mean(h[t]^2) + eps) * gain)
constexpr int kNormKeep = 4;   // float4 pieces of a row a thread keeps in registers (256 threads: rows up to 4096 wide)
__global__ void rmsnorm_split_kernel(const float* __restrict__ h, const __nv_bfloat16* __restrict__ gain, float eps, int H,
                                     __nv_bfloat16* __restrict__ planes, long long plane_stride, int parts, float4* zero, long long zero_n4,
                                     int rows) {
  // The kernel is a chain of L2 round trips between two GEMMs.  The gain is constant data: it is requested ahead of
  // griddepcontrol.wait (under the previous kernel's tail), and the row stays in registers between the two passes.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const long long t = blockIdx.x;
  const int step = blockDim.x * 4;
  uint2 gk[kNormKeep];
#pragma unroll
  for (int n = 0; n < kNormKeep; ++n) {
    const int i = threadIdx.x * 4 + n * step;
    gk[n] = (t < rows && i < H) ? *reinterpret_cast<const uint2*>(gain + i) : make_uint2(0, 0);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ float red[32];
  // batched decode: clear the fp32 targets of the atomic GEMMs that follow (saves a memset launch per layer).  The grid
  // may hold more CTAs than rows: a handful of rows would otherwise clear megabytes (the logits) by themselves.
  for (long long i = t * blockDim.x + threadIdx.x; i < zero_n4; i += (long long)gridDim.x * blockDim.x) zero[i] = make_float4(0, 0, 0, 0);
  if (t >= rows) return;
  const float* row = h + t * H;
  float4 vk[kNormKeep];
  float ss = 0.f;
#pragma unroll
  for (int n = 0; n < kNormKeep; ++n) {
    const int i = threadIdx.x * 4 + n * step;
    vk[n] = i < H ? *reinterpret_cast<const float4*>(row + i) : make_float4(0, 0, 0, 0);
  }
#pragma unroll
  for (int n = 0; n < kNormKeep; ++n) ss += vk[n].x * vk[n].x + vk[n].y * vk[n].y + vk[n].z * vk[n].z + vk[n].w * vk[n].w;
  for (int i = threadIdx.x * 4 + kNormKeep * step; i < H; i += step) {   // rows wider than the register window
    const float4 v = *reinterpret_cast<const float4*>(row + i);
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  const float inv = rsqrtf(block_sum(ss, red) / float(H) + eps);
  __nv_bfloat16* hi = planes + t * H;
#pragma unroll
  for (int n = 0; n < kNormKeep; ++n) {
    const int i = threadIdx.x * 4 + n * step;
    if (i < H) {
      const float x[4] = {vk[n].x * inv * __uint_as_float(gk[n].x << 16), vk[n].y * inv * __uint_as_float(gk[n].x & 0xffff0000u),
                          vk[n].z * inv * __uint_as_float(gk[n].y << 16), vk[n].w * inv * __uint_as_float(gk[n].y & 0xffff0000u)};
      put_split4(hi + i, plane_stride, parts, x);
    }
  }
  for (int i = threadIdx.x * 4 + kNormKeep * step; i < H; i += step) {
    const float4 v = *reinterpret_cast<const float4*>(row + i);
    const uint2 graw = *reinterpret_cast<const uint2*>(gain + i);
    const float x[4] = {v.x * inv * __uint_as_float(graw.x << 16), v.y * inv * __uint_as_float(graw.x & 0xffff0000u),
                        v.z * inv * __uint_as_float(graw.y << 16), v.w * inv * __uint_as_float(graw.y & 0xffff0000u)};
    put_split4(hi + i, plane_stride, parts, x);
  }
}

__global__ void split_kernel(const float* __restrict__ x, long long n, __nv_bfloat16* __restrict__ planes, long long plane_stride, int parts) {
  griddep_sync();
  const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i >= n) return;
  const float4 v = *reinterpret_cast<const float4*>(x + i);
  const float a[4] = {v.x, v.y, v.z, v.w};
  put_split4(planes + i, plane_stride, parts, a);
}

// One CTA per token, one warp per head (q heads, then k heads, then v heads).  D <= 256.
//   q_out    fp32 or bf16 [n_q][T][D]        (head-major, what the attention operator reads)
//   k/v      bf16 [n_kv][max_ctx][D] of this layer, written at positions pos0 .. pos0 + T - 1
struct RopeArgs {
  const float* qkv;   // [T][(n_q + 2 n_kv) D]
  const __nv_bfloat16 *q_gain, *k_gain;   // [D] or null
  const float *cos, *sin;                 // [max_ctx][D/2]
  void* q_out;
  __nv_bfloat16 *k_cache, *v_cache;
  int T, n_q, n_kv, D, max_ctx, pos0, q_is_bf16;
  float eps;
  const int32_t* positions;   // batched decode: token t sits at positions[t] of sequence t (null: pos0 + t of one sequence)
  long long seq_stride;       // cache elements between the sequences of consecutive tokens (0 for one sequence)
};

__global__ void rope_store_kernel(const RopeArgs a) {
  griddep_sync();
  const int t = blockIdx.x, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int heads = a.n_q + 2 * a.n_kv, half = a.D / 2;
  const float* row = a.qkv + (long long)t * heads * a.D;
  const int pos = a.positions != nullptr ? a.positions[t] : a.pos0 + t;
  if (pos < 0 || pos >= a.max_ctx) return;   // a sequence past its cache: nothing is written (no out-of-bounds K / V / table access)
  __nv_bfloat16* k_cache = a.k_cache + t * a.seq_stride;
  __nv_bfloat16* v_cache = a.v_cache + t * a.seq_stride;
  // gridDim.y spreads the heads of a token over CTAs (batched decode: a few tokens, latency- not work-bound)
  for (int hd = blockIdx.y * nw + (threadIdx.x >> 5); hd < heads; hd += nw * gridDim.y) {
    const float* x = row + hd * a.D;
    if (hd >= a.n_q + a.n_kv) {   // value head: plain bf16 store
      __nv_bfloat16* dst = v_cache + ((long long)(hd - a.n_q - a.n_kv) * a.max_ctx + pos) * a.D;
      for (int i = lane; i < a.D; i += 32) dst[i] = __float2bfloat16_rn(x[i]);
      continue;
    }
    const bool is_q = hd < a.n_q;
    const __nv_bfloat16* gain = is_q ? a.q_gain : a.k_gain;
    float inv = 1.f;
    if (gain != nullptr) {
      float ss = 0.f;
      for (int i = lane; i < a.D; i += 32) ss += x[i] * x[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      inv = rsqrtf(ss / float(a.D) + a.eps);
    }
    for (int i = lane; i < half; i += 32) {
      float x1 = x[i], x2 = x[i + half];
      if (gain != nullptr) {
        x1 = x1 * inv * __bfloat162float(gain[i]);
        x2 = x2 * inv * __bfloat162float(gain[i + half]);
      }
      const float c = a.cos[(long long)pos * half + i], s = a.sin[(long long)pos * half + i];
      const float r1 = x1 * c - x2 * s, r2 = x2 * c + x1 * s;
      if (is_q) {
        const long long o = ((long long)hd * a.T + t) * a.D;
        if (a.q_is_bf16) {
          __nv_bfloat16* q = static_cast<__nv_bfloat16*>(a.q_out) + o;
          q[i] = __float2bfloat16_rn(r1);
          q[i + half] = __float2bfloat16_rn(r2);
        } else {
          float* q = static_cast<float*>(a.q_out) + o;
          q[i] = r1;
          q[i + half] = r2;
        }
      } else {
        __nv_bfloat16* k = k_cache + ((long long)(hd - a.n_q) * a.max_ctx + pos) * a.D;
        k[i] = __float2bfloat16_rn(r1);
        k[i + half] = __float2bfloat16_rn(r2);
      }
    }
  }
}

// ---------------------------------------------------------------------------------------------------------
// Batched decode (one new token per sequence): attention over each sequence's cache, and the greedy pick.

constexpr int kAttnChunk = 64;    // cache positions per CTA: small chunks = many CTAs = many loads in flight
constexpr int kAttnThreads = 128;   // 2 threads per cache position (4 per position with 256 threads measured 38 % slower)
constexpr int kMaxGroup = 8;      // q heads per kv head

__device__ __forceinline__ void bf16x8_to_float(const uint4 u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    f[2 * j] = __uint_as_float(w[j] << 16);
    f[2 * j + 1] = __uint_as_float(w[j] & 0xffff0000u);
  }
}

// Scores in shared memory are stored per consuming warp: position p belongs to warp p % 4 in the value phase, which
// reads its 16 positions as four 16-byte words.
__device__ __forceinline__ int sc_slot(int p) { return (p & 3) * (kAttnChunk / 4) + (p >> 2); }

// grid (splits, n_kv, B).  Partial softmax of the G q heads of one kv head over positions [s * 64, s * 64 + 64) of
// sequence b:  part[b][q head][s][0..D) = sum_p exp(score_p - m) v_p,  [D] = m,  [D + 1] = sum_p exp(score_p - m).
// Every global load of a phase is issued before the first use (the kernel is latency-, not bandwidth-limited).
template <int D, int G>
__global__ void __launch_bounds__(kAttnThreads, 5)
batch_attn_partial_kernel(const float* __restrict__ q, const __nv_bfloat16* __restrict__ k_cache, const __nv_bfloat16* __restrict__ v_cache,
                          const int32_t* __restrict__ positions, float* __restrict__ part, int B, int n_q, int n_kv, int max_ctx,
                          long long seq_stride, int splits, float scale) {
  griddep_sync();
  const int s = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int ctx = min(positions[b] + 1, max_ctx);   // the new token's K / V are already in the cache; never past the cache
  const int p0 = s * kAttnChunk;
  if (p0 >= ctx) return;              // the merge kernel derives the live split count from positions, too
  const int n_pos = min(kAttnChunk, ctx - p0);
  constexpr int NW = kAttnThreads / 32;
  __shared__ __align__(16) float q_s[G][D + 12];   // each quarter of a row shifted by 16 more bytes: the four threads of a
                                                   // position pair read different banks (ncu: a third of all shared wavefronts
                                                   // were conflicts without the shift)
  __shared__ __align__(16) float sc[G][kAttnChunk];   // position p at sc_slot(p): a warp's positions are contiguous
  __shared__ float ml[G][2];
  __shared__ __align__(16) float ored[NW][G][D];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const __nv_bfloat16* kb = k_cache + b * seq_stride + ((long long)kvh * max_ctx + p0) * D;
  const __nv_bfloat16* vb = v_cache + b * seq_stride + ((long long)kvh * max_ctx + p0) * D;

  // scores: four threads share two positions -- a quarter of each K row per thread, so that every 16-byte q read from
  // shared memory feeds the products of two positions (all global loads in flight before the first use)
  constexpr int QC = D / 32;                 // 16-byte pieces of a quarter row
  const int pi = tid >> 2, qd = tid & 3;     // position pair, quarter
  uint4 kraw[2][QC];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int pp = 2 * pi + r;
    if (pp < n_pos) {
      const uint4* row = reinterpret_cast<const uint4*>(kb + (long long)pp * D) + qd * QC;
#pragma unroll
      for (int c = 0; c < QC; ++c) kraw[r][c] = row[c];
    } else {
#pragma unroll
      for (int c = 0; c < QC; ++c) kraw[r][c] = make_uint4(0, 0, 0, 0);
    }
  }
  for (int i = tid; i < G * D; i += kAttnThreads) {
    const int g = i / D, d = i - g * D;
    q_s[g][d + (d / (D / 4)) * 4] = q[((long long)(kvh * G + g) * B + b) * D + d] * scale;   // quarter q at a 16-byte bank shift
  }
  __syncthreads();
  {
    float2 acc[2][G];   // even / odd feature sums, packed fp32 FMAs (FFMA2): half the issue slots of scalar FMAs
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int g = 0; g < G; ++g) acc[r][g] = make_float2(0.f, 0.f);
#pragma unroll
    for (int c = 0; c < QC; ++c) {
      float k0[8], k1[8];
      bf16x8_to_float(kraw[0][c], k0);
      bf16x8_to_float(kraw[1][c], k1);
      const int d0 = qd * (D / 4) + c * 8 + qd * 4;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float4 qa = *reinterpret_cast<const float4*>(&q_s[g][d0]), qb = *reinterpret_cast<const float4*>(&q_s[g][d0 + 4]);
        const float2 q01 = make_float2(qa.x, qa.y), q23 = make_float2(qa.z, qa.w), q45 = make_float2(qb.x, qb.y), q67 = make_float2(qb.z, qb.w);
        acc[0][g] = __ffma2_rn(q01, make_float2(k0[0], k0[1]), acc[0][g]);
        acc[0][g] = __ffma2_rn(q23, make_float2(k0[2], k0[3]), acc[0][g]);
        acc[0][g] = __ffma2_rn(q45, make_float2(k0[4], k0[5]), acc[0][g]);
        acc[0][g] = __ffma2_rn(q67, make_float2(k0[6], k0[7]), acc[0][g]);
        acc[1][g] = __ffma2_rn(q01, make_float2(k1[0], k1[1]), acc[1][g]);
        acc[1][g] = __ffma2_rn(q23, make_float2(k1[2], k1[3]), acc[1][g]);
        acc[1][g] = __ffma2_rn(q45, make_float2(k1[4], k1[5]), acc[1][g]);
        acc[1][g] = __ffma2_rn(q67, make_float2(k1[6], k1[7]), acc[1][g]);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float t = acc[r][g].x + acc[r][g].y;
        t += __shfl_xor_sync(0xffffffffu, t, 1);
        t += __shfl_xor_sync(0xffffffffu, t, 2);
        if (qd == 0) sc[g][sc_slot(2 * pi + r)] = (2 * pi + r < n_pos) ? t : -INFINITY;
      }
  }
  // values: warp w owns positions w, w + 4, ...; issue all of its (coalesced) V rows now, use them after the softmax
  constexpr int E = D / 32, NV = kAttnChunk / NW;
  uint32_t vraw[NV][E / 2];   // kept as bf16 pairs until used (registers decide how many CTAs share an SM)
#pragma unroll
  for (int u = 0; u < NV; ++u) {
    const int pp = warp + u * NW;
    if (pp < n_pos) {
      if constexpr (E == 4) {
        const uint2 raw = *reinterpret_cast<const uint2*>(vb + (long long)pp * D + lane * 4);
        vraw[u][0] = raw.x;
        vraw[u][1] = raw.y;
      } else {
        vraw[u][0] = *reinterpret_cast<const uint32_t*>(vb + (long long)pp * D + lane * 2);
      }
    } else {
#pragma unroll
      for (int e = 0; e < E / 2; ++e) vraw[u][e] = 0u;
    }
  }
  __syncthreads();
  // chunk softmax: warp w handles heads w, w + 4; a lane covers positions lane and lane + 32
  for (int g = warp; g < G; g += NW) {
    const float s0 = sc[g][sc_slot(lane)], s1 = sc[g][sc_slot(lane + 32)];
    float m = fmaxf(s0, s1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const float e0 = __expf(s0 - m), e1 = __expf(s1 - m);   // exp(-inf) = 0 for the positions past the end
    sc[g][sc_slot(lane)] = e0;
    sc[g][sc_slot(lane + 32)] = e1;
    float l = e0 + e1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) { ml[g][0] = m; ml[g][1] = l; }
  }
  __syncthreads();
  {
    float2 o[G][E / 2];
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int e = 0; e < E / 2; ++e) o[g][e] = make_float2(0.f, 0.f);
#pragma unroll
    for (int u4 = 0; u4 < NV; u4 += 4) {
      float2 vf[4][E / 2];
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int e = 0; e < E / 2; ++e)
          vf[k][e] = make_float2(__uint_as_float(vraw[u4 + k][e] << 16), __uint_as_float(vraw[u4 + k][e] & 0xffff0000u));
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float4 w4 = *reinterpret_cast<const float4*>(&sc[g][warp * NV + u4]);   // this warp's four next positions
        const float w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int e = 0; e < E / 2; ++e) o[g][e] = __ffma2_rn(make_float2(w[k], w[k]), vf[k][e], o[g][e]);
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if constexpr (E == 4) *reinterpret_cast<float4*>(&ored[warp][g][lane * 4]) = make_float4(o[g][0].x, o[g][0].y, o[g][1].x, o[g][1].y);
      else *reinterpret_cast<float2*>(&ored[warp][g][lane * 2]) = o[g][0];
    }
  }
  __syncthreads();
  for (int i = tid; i < G * D; i += kAttnThreads) {
    const int g = i / D, d = i - g * D;
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) t += ored[w][g][d];
    part[(((long long)b * n_q + kvh * G + g) * splits + s) * (D + 2) + d] = t;
  }
  if (tid < G) {
    float* dst = part + (((long long)b * n_q + kvh * G + tid) * splits + s) * (D + 2);
    dst[D] = ml[tid][0];
    dst[D + 1] = ml[tid][1];
  }
}

// grid (n_q, B), 4 D threads: merge the live splits and emit the attention output as bf16 planes [P][B][n_q * D].
// The kernel is a chain of dependent L2 round trips, not work: thread group q = tid / D takes the splits
// s = 8 (q + 4 k) .. + 7 (eight loads in flight each), so a 2K context is two round trips instead of five, and the four
// partial (numerator, denominator) pairs meet in shared memory in a fixed order.
constexpr int kMergeGroups = 4;
template <int D>
__global__ void __launch_bounds__(kMergeGroups * D)
batch_attn_merge_kernel(const float* __restrict__ part, const int32_t* __restrict__ positions, __nv_bfloat16* __restrict__ planes,
                        int B, int n_q, int splits, int parts) {
  griddep_sync();
  const int h = blockIdx.x, b = blockIdx.y, d = threadIdx.x % D, q = threadIdx.x / D;
  const int live = min(max((positions[b] + kAttnChunk) / kAttnChunk, 1), splits);   // ceil((pos + 1) / chunk), inside the records that exist
  const float* src = part + ((long long)b * n_q + h) * splits * (D + 2);
  // the splits' maxima through shared memory (one load each, all in flight), then the weighted sums eight splits at a time
  extern __shared__ float m_s[];
  __shared__ float num_s[kMergeGroups][D], den_s[kMergeGroups];
  for (int s = threadIdx.x; s < live; s += kMergeGroups * D) m_s[s] = src[s * (D + 2) + D];
  __syncthreads();
  float M = -INFINITY;
  for (int s = 0; s < live; ++s) M = fmaxf(M, m_s[s]);
  float num = 0.f, den = 0.f;
  for (int s0 = 8 * q; s0 < live; s0 += 8 * kMergeGroups) {
    float ov[8], lv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int s = min(s0 + u, live - 1);
      ov[u] = src[s * (D + 2) + d];
      lv[u] = src[s * (D + 2) + D + 1];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float w = (s0 + u < live) ? __expf(m_s[s0 + u] - M) : 0.f;
      num = fmaf(w, ov[u], num);
      den = fmaf(w, lv[u], den);
    }
  }
  num_s[q][d] = num;
  if (d == 0) den_s[q] = den;
  __syncthreads();
  if (q == 0) {
#pragma unroll
    for (int g = 1; g < kMergeGroups; ++g) {
      num += num_s[g][d];
      den += den_s[g];
    }
    const long long o = (long long)b * n_q * D + h * D + d;
    put_split(planes + o, (long long)B * n_q * D, parts, num / den);
  }
}

// grid B: greedy pick (lowest index on ties), written to next[b]; tokens / positions advanced in place when asked.
__global__ void batch_argmax_kernel(const float* __restrict__ logits, int V, int32_t* __restrict__ next, int32_t* tokens, int32_t* positions) {
  griddep_sync();
  const int b = blockIdx.x;
  const float* row = logits + (long long)b * V;
  float best = -INFINITY;
  int idx = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const float v = row[i];
    if (v > best) { best = v; idx = i; }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > best || (ov == best && oi < idx)) { best = ov; idx = oi; }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sv[warp] = best; si[warp] = idx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (blockDim.x >> 5); ++w)
      if (sv[w] > best || (sv[w] == best && si[w] < idx)) { best = sv[w]; idx = si[w]; }
    if (idx < 0 || idx >= V) idx = 0;   // a row of NaN / -inf has no maximum: a valid token id, not the 0x7fffffff sentinel
    next[b] = idx;
    if (tokens != nullptr) tokens[b] = idx;
    if (positions != nullptr) positions[b] += 1;
  }
}

// The same pick with every row cut into kArgmaxSlices slices (grid (slices, B)): a row of 150 K logits scanned by ONE
// CTA took 73 us -- a whole GEMM's worth of a decode step.  Each CTA leaves (value, index) of its slice in `scratch`
// [B][slices]; the last CTA of a row to finish (a counter per row, zero before the first call and reset by that CTA)
// reduces the slices in slice order, so ties still go to the lowest index.
constexpr int kArgmaxSlices = 64;
__global__ void batch_argmax_sliced_kernel(const float* __restrict__ logits, int V, unsigned long long* __restrict__ scratch,
                                           int32_t* __restrict__ next, int32_t* tokens, int32_t* positions) {
  griddep_sync();
  const int b = blockIdx.y, sl = blockIdx.x, S = gridDim.x;
  const int per = (V + S - 1) / S, lo = sl * per, hi = min(V, lo + per);
  const float* row = logits + (long long)b * V;
  float best = -INFINITY;
  int idx = 0x7fffffff;
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const float v = row[i];
    if (v > best) { best = v; idx = i; }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
  __shared__ int last;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > best || (ov == best && oi < idx)) { best = ov; idx = oi; }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sv[warp] = best; si[warp] = idx; }
  __syncthreads();
  unsigned long long* part = scratch + (long long)b * (S + 1);   // S partial records, then the row's counter
  if (threadIdx.x == 0) {
    for (int w = 1; w < (blockDim.x >> 5); ++w)
      if (sv[w] > best || (sv[w] == best && si[w] < idx)) { best = sv[w]; idx = si[w]; }
    part[sl] = ((unsigned long long)__float_as_uint(best) << 32) | (unsigned)idx;
    __threadfence();
    last = atomicAdd(reinterpret_cast<unsigned*>(part + S), 1u) == (unsigned)(S - 1);
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  best = -INFINITY;
  idx = 0x7fffffff;
  for (int k = 0; k < S; ++k) {
    const unsigned long long rec = *reinterpret_cast<volatile unsigned long long*>(part + k);
    const float v = __uint_as_float((unsigned)(rec >> 32));
    const int i = (int)(unsigned)rec;
    if (v > best || (v == best && i < idx)) { best = v; idx = i; }
  }
  if (idx < 0 || idx >= V) idx = 0;   // a row of NaN / -inf has no maximum: a valid token id, not the sentinel
  next[b] = idx;
  if (tokens != nullptr) tokens[b] = idx;
  if (positions != nullptr) positions[b] += 1;
  *reinterpret_cast<unsigned*>(part + S) = 0u;   // ready for the next step
}

// act planes [P][B][I] = split(silu(gate) * up) from gu fp32 [B][2 I] whose columns interleave gate and up in blocks of
// `block` features (the layout of the fused-SwiGLU GEMM weight).  grid (feature blocks, tokens).
__global__ void swiglu_split_kernel(const float* __restrict__ gu, int I, int block, __nv_bfloat16* __restrict__ planes, long long plane_stride,
                                    int parts) {
  griddep_sync();
  const long long t = blockIdx.y;
  const float* row = gu + t * 2 * I;
  __nv_bfloat16* hi = planes + t * I;
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < I; f += gridDim.x * blockDim.x) {
    const int blk = f / block, j = f - blk * block;
    const float g = row[blk * 2 * block + j], u = row[blk * 2 * block + block + j];
    put_split(hi + f, plane_stride, parts, __fdividef(g, 1.0f + __expf(-g)) * u);
  }
}

static int done(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(pf::err_buf(), 256, "%s: %s", what, cudaGetErrorString(e));
    return ADAMK_PF_E_CUDA;
  }
  return ADAMK_PF_OK;
}

}  // namespace pfo

extern "C" {

int adamk_prefill_embed(const int32_t* tokens, int T, const void* embed, int H, float* h, adamk_pf_stream stream) {
  if (tokens == nullptr || embed == nullptr || h == nullptr || T <= 0 || H <= 0 || H % 2) return ADAMK_PF_E_INVALID;
  pfo::launch(pfo::embed_kernel, dim3(T), dim3(256), 0, static_cast<cudaStream_t>(stream), tokens, static_cast<const __nv_bfloat16*>(embed), h, H, 0);
  return pfo::done("prefill embed");
}

int adamk_batch_embed(const int32_t* tokens, int T, const void* embed, int H, int vocab, float* h, adamk_pf_stream stream) {
  if (tokens == nullptr || embed == nullptr || h == nullptr || T <= 0 || H <= 0 || H % 2 || vocab <= 0) return ADAMK_PF_E_INVALID;
  pfo::launch(pfo::embed_kernel, dim3(T), dim3(256), 0, static_cast<cudaStream_t>(stream), tokens, static_cast<const __nv_bfloat16*>(embed), h, H, vocab);
  return pfo::done("batch embed");
}

int adamk_prefill_rmsnorm_split(const float* h, const void* gain, float eps, int T, int H, void* planes, int parts, adamk_pf_stream stream) {
  if (h == nullptr || gain == nullptr || planes == nullptr || T <= 0 || H <= 0 || H % 4 || (parts < 1 || parts > 3)) return ADAMK_PF_E_INVALID;
  pfo::launch(pfo::rmsnorm_split_kernel, dim3(T), dim3(256), 0, static_cast<cudaStream_t>(stream), h, static_cast<const __nv_bfloat16*>(gain), eps, H,
                                                                             static_cast<__nv_bfloat16*>(planes), (long long)T * H, parts, nullptr, 0, T);
  return pfo::done("prefill rmsnorm");
}

int adamk_batch_rmsnorm_split(const float* h, const void* gain, float eps, int B, int H, void* planes, int parts, float* zero, long long zero_n,
                              adamk_pf_stream stream) {
  if (h == nullptr || gain == nullptr || planes == nullptr || B <= 0 || H <= 0 || H % 4 || (parts < 1 || parts > 3) || zero_n % 4 ||
      (reinterpret_cast<uintptr_t>(zero) & 15))
    return ADAMK_PF_E_INVALID;
  // one CTA per row, plus CTAs that only clear: ~16 KB of the zeroed region per CTA, at most one CTA per SM
  long long grid = (zero != nullptr ? zero_n * 4 / 16384 : 0);
  grid = grid > 148 ? 148 : grid;
  grid = grid < B ? B : grid;
  pfo::launch(pfo::rmsnorm_split_kernel, dim3((unsigned)grid), dim3(256), 0, static_cast<cudaStream_t>(stream), h, static_cast<const __nv_bfloat16*>(gain), eps, H,
                                                                             static_cast<__nv_bfloat16*>(planes), (long long)B * H, parts,
                                                                             reinterpret_cast<float4*>(zero), zero_n / 4, B);
  return pfo::done("batch rmsnorm");
}

int adamk_prefill_split(const float* x, long long n, void* planes, int parts, adamk_pf_stream stream) {
  if (x == nullptr || planes == nullptr || n <= 0 || n % 4 || (parts < 1 || parts > 3)) return ADAMK_PF_E_INVALID;
  const long long blocks = (n / 4 + 255) / 256;
  pfo::launch(pfo::split_kernel, dim3((unsigned)blocks), dim3(256), 0, static_cast<cudaStream_t>(stream), x, n, static_cast<__nv_bfloat16*>(planes), n, parts);
  return pfo::done("prefill split");
}

int adamk_prefill_rope_store(const float* qkv, int T, int n_q, int n_kv, int D, const void* q_gain, const void* k_gain, float eps,
                             const float* cos, const float* sin, int pos0, int max_ctx, void* q_out, int q_is_bf16, void* k_cache,
                             void* v_cache, adamk_pf_stream stream) {
  if (qkv == nullptr || cos == nullptr || sin == nullptr || q_out == nullptr || k_cache == nullptr || v_cache == nullptr || T <= 0 ||
      D % 2 || pos0 < 0 || pos0 + T > max_ctx || (q_gain == nullptr) != (k_gain == nullptr))
    return ADAMK_PF_E_INVALID;
  pfo::RopeArgs a{qkv, static_cast<const __nv_bfloat16*>(q_gain), static_cast<const __nv_bfloat16*>(k_gain), cos, sin, q_out,
                  static_cast<__nv_bfloat16*>(k_cache), static_cast<__nv_bfloat16*>(v_cache), T, n_q, n_kv, D, max_ctx, pos0, q_is_bf16, eps,
                  nullptr, 0};
  pfo::launch(pfo::rope_store_kernel, dim3(T), dim3(256), 0, static_cast<cudaStream_t>(stream), a);
  return pfo::done("prefill rope");
}

int adamk_batch_rope_store(const float* qkv, int B, int n_q, int n_kv, int D, const void* q_gain, const void* k_gain, float eps,
                           const float* cos, const float* sin, const int32_t* positions, long long seq_stride, int max_ctx, float* q_out,
                           void* k_cache, void* v_cache, adamk_pf_stream stream) {
  if (qkv == nullptr || cos == nullptr || sin == nullptr || q_out == nullptr || k_cache == nullptr || v_cache == nullptr || positions == nullptr ||
      B <= 0 || D % 2 || (q_gain == nullptr) != (k_gain == nullptr))
    return ADAMK_PF_E_INVALID;
  pfo::RopeArgs a{qkv, static_cast<const __nv_bfloat16*>(q_gain), static_cast<const __nv_bfloat16*>(k_gain), cos, sin, q_out,
                  static_cast<__nv_bfloat16*>(k_cache), static_cast<__nv_bfloat16*>(v_cache), B, n_q, n_kv, D, max_ctx, 0, 0, eps,
                  positions, seq_stride};
  // one head per warp, two warps per CTA: 8 sequences x 16 heads are 64 CTAs instead of 8
  pfo::launch(pfo::rope_store_kernel, dim3(B, (n_q + 2 * n_kv + 1) / 2), dim3(64), 0, static_cast<cudaStream_t>(stream), a);
  return pfo::done("batch rope");
}

size_t adamk_batch_attention_workspace(int B, int n_q, int D, int max_ctx) {
  const size_t splits = (size_t(max_ctx) + pfo::kAttnChunk - 1) / pfo::kAttnChunk;
  return size_t(B) * n_q * splits * (D + 2) * sizeof(float);
}

int adamk_batch_attention(const float* q, const void* k_cache, const void* v_cache, const int32_t* positions, int B, int n_q, int n_kv, int D,
                          int max_ctx, long long seq_stride, float* workspace, void* out_planes, int parts, adamk_pf_stream stream) {
  if (q == nullptr || k_cache == nullptr || v_cache == nullptr || positions == nullptr || workspace == nullptr || out_planes == nullptr || B <= 0 ||
      n_kv <= 0 || n_q % n_kv || n_q / n_kv > pfo::kMaxGroup || (parts < 1 || parts > 3))
    return ADAMK_PF_E_INVALID;
  if (D != 64 && D != 128) {
    snprintf(pf::err_buf(), 256, "batch attention: head_dim %d is not built (64, 128)", D);
    return ADAMK_PF_E_INVALID;
  }
  const int splits = (max_ctx + pfo::kAttnChunk - 1) / pfo::kAttnChunk;
  const float scale = 1.0f / sqrtf(float(D));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const dim3 grid(splits, n_kv, B), mgrid(n_q, B);
  const auto* kc = static_cast<const __nv_bfloat16*>(k_cache);
  const auto* vc = static_cast<const __nv_bfloat16*>(v_cache);
  auto* planes = static_cast<__nv_bfloat16*>(out_planes);
  const int G = n_q / n_kv;
  bool ok = true;
#define ADAMK_ATTN_CASE(DD, GG)                                                                                                          \
  pfo::launch(pfo::batch_attn_partial_kernel<DD, GG>, dim3(grid), dim3(pfo::kAttnThreads), 0, s, q, kc, vc, positions, workspace, B, n_q, \
              n_kv, max_ctx, seq_stride, splits, scale)
  if (D == 128) {
    switch (G) {
      case 1: ADAMK_ATTN_CASE(128, 1); break;
      case 2: ADAMK_ATTN_CASE(128, 2); break;
      case 4: ADAMK_ATTN_CASE(128, 4); break;
      case 6: ADAMK_ATTN_CASE(128, 6); break;
      case 7: ADAMK_ATTN_CASE(128, 7); break;
      case 8: ADAMK_ATTN_CASE(128, 8); break;
      default: ok = false;
    }
    if (ok) pfo::launch(pfo::batch_attn_merge_kernel<128>, dim3(mgrid), dim3(pfo::kMergeGroups * 128), splits * sizeof(float), s, workspace, positions, planes, B, n_q, splits, parts);
  } else {
    switch (G) {
      case 1: ADAMK_ATTN_CASE(64, 1); break;
      case 2: ADAMK_ATTN_CASE(64, 2); break;
      case 4: ADAMK_ATTN_CASE(64, 4); break;
      case 6: ADAMK_ATTN_CASE(64, 6); break;
      case 7: ADAMK_ATTN_CASE(64, 7); break;
      case 8: ADAMK_ATTN_CASE(64, 8); break;
      default: ok = false;
    }
    if (ok) pfo::launch(pfo::batch_attn_merge_kernel<64>, dim3(mgrid), dim3(pfo::kMergeGroups * 64), splits * sizeof(float), s, workspace, positions, planes, B, n_q, splits, parts);
  }
#undef ADAMK_ATTN_CASE
  if (!ok) {
    snprintf(pf::err_buf(), 256, "batch attention: %d q heads per kv head at head_dim %d is not built", G, D);
    return ADAMK_PF_E_INVALID;
  }
  return pfo::done("batch attention");
}

int adamk_batch_swiglu_split(const float* gu, int B, int I, int block, void* planes, int parts, adamk_pf_stream stream) {
  if (gu == nullptr || planes == nullptr || B <= 0 || I <= 0 || block <= 0 || I % block || (parts < 1 || parts > 3)) return ADAMK_PF_E_INVALID;
  pfo::launch(pfo::swiglu_split_kernel, dim3(dim3((I + 511) / 512, B)), dim3(512), 0, static_cast<cudaStream_t>(stream), gu, I, block, static_cast<__nv_bfloat16*>(planes), (long long)B * I, parts);
  return pfo::done("batch swiglu");
}

size_t adamk_batch_argmax_workspace(int B) { return B > 0 ? (size_t)B * (pfo::kArgmaxSlices + 1) * sizeof(unsigned long long) : 0; }

int adamk_batch_argmax_sliced(const float* logits, int B, int V, void* scratch, int32_t* next, int32_t* tokens, int32_t* positions,
                              adamk_pf_stream stream) {
  if (logits == nullptr || next == nullptr || scratch == nullptr || B <= 0 || V <= 0) return ADAMK_PF_E_INVALID;
  pfo::launch(pfo::batch_argmax_sliced_kernel, dim3(pfo::kArgmaxSlices, B), dim3(256), 0, static_cast<cudaStream_t>(stream), logits, V,
              static_cast<unsigned long long*>(scratch), next, tokens, positions);
  return pfo::done("batch argmax (sliced)");
}

int adamk_batch_argmax(const float* logits, int B, int V, int32_t* next, int32_t* tokens, int32_t* positions, adamk_pf_stream stream) {
  if (logits == nullptr || next == nullptr || B <= 0 || V <= 0) return ADAMK_PF_E_INVALID;
  pfo::launch(pfo::batch_argmax_kernel, dim3(B), dim3(1024), 0, static_cast<cudaStream_t>(stream), logits, V, next, tokens, positions);
  return pfo::done("batch argmax");
}

}  // extern "C"
