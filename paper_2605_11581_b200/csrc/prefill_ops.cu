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
}

namespace pfo {

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

__device__ __forceinline__ void put_split(__nv_bfloat16* hi, __nv_bfloat16* lo, float v) {
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  *hi = h;
  if (lo != nullptr) *lo = __float2bfloat16_rn(v - __bfloat162float(h));
}

__global__ void embed_kernel(const int32_t* __restrict__ tokens, const __nv_bfloat16* __restrict__ embed, float* __restrict__ h, int H) {
  const int t = blockIdx.x;
  const __nv_bfloat16* src = embed + (long long)tokens[t] * H;
  float* dst = h + (long long)t * H;
  for (int i = threadIdx.x * 2; i < H; i += blockDim.x * 2) {
    const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(src + i);
    *reinterpret_cast<float2*>(dst + i) = make_float2(__low2float(v), __high2float(v));
  }
}

// planes[p][t][:] = split(h[t] * rsqrt(mean(h[t]^2) + eps) * gain)
__global__ void rmsnorm_split_kernel(const float* __restrict__ h, const __nv_bfloat16* __restrict__ gain, float eps, int H,
                                     __nv_bfloat16* __restrict__ planes, long long plane_stride, int parts) {
  __shared__ float red[32];
  const long long t = blockIdx.x;
  const float* row = h + t * H;
  float ss = 0.f;
  for (int i = threadIdx.x * 4; i < H; i += blockDim.x * 4) {
    const float4 v = *reinterpret_cast<const float4*>(row + i);
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  const float inv = rsqrtf(block_sum(ss, red) / float(H) + eps);
  __nv_bfloat16* hi = planes + t * H;
  __nv_bfloat16* lo = parts == 2 ? hi + plane_stride : nullptr;
  for (int i = threadIdx.x * 4; i < H; i += blockDim.x * 4) {
    const float4 v = *reinterpret_cast<const float4*>(row + i);
    const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) put_split(hi + i + j, lo ? lo + i + j : nullptr, x[j] * inv * __bfloat162float(gain[i + j]));
  }
}

__global__ void split_kernel(const float* __restrict__ x, long long n, __nv_bfloat16* __restrict__ planes, long long plane_stride, int parts) {
  const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i >= n) return;
  const float4 v = *reinterpret_cast<const float4*>(x + i);
  const float a[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) put_split(planes + i + j, parts == 2 ? planes + plane_stride + i + j : nullptr, a[j]);
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
};

__global__ void rope_store_kernel(const RopeArgs a) {
  const int t = blockIdx.x, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int heads = a.n_q + 2 * a.n_kv, half = a.D / 2;
  const float* row = a.qkv + (long long)t * heads * a.D;
  const int pos = a.pos0 + t;
  for (int hd = threadIdx.x >> 5; hd < heads; hd += nw) {
    const float* x = row + hd * a.D;
    if (hd >= a.n_q + a.n_kv) {   // value head: plain bf16 store
      __nv_bfloat16* dst = a.v_cache + ((long long)(hd - a.n_q - a.n_kv) * a.max_ctx + pos) * a.D;
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
        __nv_bfloat16* k = a.k_cache + ((long long)(hd - a.n_q) * a.max_ctx + pos) * a.D;
        k[i] = __float2bfloat16_rn(r1);
        k[i + half] = __float2bfloat16_rn(r2);
      }
    }
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
  pfo::embed_kernel<<<T, 256, 0, static_cast<cudaStream_t>(stream)>>>(tokens, static_cast<const __nv_bfloat16*>(embed), h, H);
  return pfo::done("prefill embed");
}

int adamk_prefill_rmsnorm_split(const float* h, const void* gain, float eps, int T, int H, void* planes, int parts, adamk_pf_stream stream) {
  if (h == nullptr || gain == nullptr || planes == nullptr || T <= 0 || H <= 0 || H % 4 || (parts != 1 && parts != 2)) return ADAMK_PF_E_INVALID;
  pfo::rmsnorm_split_kernel<<<T, 256, 0, static_cast<cudaStream_t>(stream)>>>(h, static_cast<const __nv_bfloat16*>(gain), eps, H,
                                                                             static_cast<__nv_bfloat16*>(planes), (long long)T * H, parts);
  return pfo::done("prefill rmsnorm");
}

int adamk_prefill_split(const float* x, long long n, void* planes, int parts, adamk_pf_stream stream) {
  if (x == nullptr || planes == nullptr || n <= 0 || n % 4 || (parts != 1 && parts != 2)) return ADAMK_PF_E_INVALID;
  const long long blocks = (n / 4 + 255) / 256;
  pfo::split_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(x, n, static_cast<__nv_bfloat16*>(planes), n, parts);
  return pfo::done("prefill split");
}

int adamk_prefill_rope_store(const float* qkv, int T, int n_q, int n_kv, int D, const void* q_gain, const void* k_gain, float eps,
                             const float* cos, const float* sin, int pos0, int max_ctx, void* q_out, int q_is_bf16, void* k_cache,
                             void* v_cache, adamk_pf_stream stream) {
  if (qkv == nullptr || cos == nullptr || sin == nullptr || q_out == nullptr || k_cache == nullptr || v_cache == nullptr || T <= 0 ||
      D % 2 || pos0 < 0 || pos0 + T > max_ctx || (q_gain == nullptr) != (k_gain == nullptr))
    return ADAMK_PF_E_INVALID;
  pfo::RopeArgs a{qkv, static_cast<const __nv_bfloat16*>(q_gain), static_cast<const __nv_bfloat16*>(k_gain), cos, sin, q_out,
                  static_cast<__nv_bfloat16*>(k_cache), static_cast<__nv_bfloat16*>(v_cache), T, n_q, n_kv, D, max_ctx, pos0, q_is_bf16, eps};
  pfo::rope_store_kernel<<<T, 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return pfo::done("prefill rope");
}

}  // extern "C"
