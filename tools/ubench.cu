// Micro-benchmarks for the GEMV consumer inner loop on sm_100a (run under gpurun).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ float4 lds128f(uint32_t a) { float4 v; asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a)); return v; }
__device__ __forceinline__ uint4 lds128u(uint32_t a) { uint4 v; asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a)); return v; }

// MODE 0: FFMA2 path, 1: scalar FFMA path, 2: loads only, 3: cvt+FFMA2 without loads (registers)
template <int MODE, int RW>
__global__ void __launch_bounds__(288, 1) body(float* out, int iters, int stage_bytes, int n_stage) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (stage_bytes * n_stage + 40960) / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3f803f80u + i;
  __syncthreads();
  if (warp == 0) return;
  const int cw = warp - 1;
  const uint32_t xs = (uint32_t)__cvta_generic_to_shared(smem) + lane * 16;
  const uint32_t ring = xs + 40960;
  float2 acc[8];
  for (int i = 0; i < 8; ++i) acc[i] = make_float2(0.f, 0.f);
  long long t0 = clock64();
  int slot = 0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t wa = ring + slot * stage_bytes + cw * RW * 512;
    const uint32_t xa_addr = xs + (it % 6) * 1024;
    const float4 xa = lds128f(xa_addr), xb = lds128f(xa_addr + 512);
    uint4 w[RW];
#pragma unroll
    for (int i = 0; i < RW; ++i) w[i] = lds128u(wa + i * 512);
    if (MODE == 2) {
#pragma unroll
      for (int i = 0; i < RW; ++i) acc[i].x += __uint_as_float(w[i].x ^ w[i].y ^ w[i].z ^ w[i].w) + xa.x + xb.x;
    } else if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < RW; ++i) {
        acc[i] = __ffma2_rn(make_float2(bf_lo(w[i].x), bf_hi(w[i].x)), make_float2(xa.x, xa.y), acc[i]);
        acc[i] = __ffma2_rn(make_float2(bf_lo(w[i].y), bf_hi(w[i].y)), make_float2(xa.z, xa.w), acc[i]);
        acc[i] = __ffma2_rn(make_float2(bf_lo(w[i].z), bf_hi(w[i].z)), make_float2(xb.x, xb.y), acc[i]);
        acc[i] = __ffma2_rn(make_float2(bf_lo(w[i].w), bf_hi(w[i].w)), make_float2(xb.z, xb.w), acc[i]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < RW; ++i) {
        acc[i].x = fmaf(bf_lo(w[i].x), xa.x, acc[i].x); acc[i].y = fmaf(bf_hi(w[i].x), xa.y, acc[i].y);
        acc[i].x = fmaf(bf_lo(w[i].y), xa.z, acc[i].x); acc[i].y = fmaf(bf_hi(w[i].y), xa.w, acc[i].y);
        acc[i].x = fmaf(bf_lo(w[i].z), xb.x, acc[i].x); acc[i].y = fmaf(bf_hi(w[i].z), xb.y, acc[i].y);
        acc[i].x = fmaf(bf_lo(w[i].w), xb.z, acc[i].x); acc[i].y = fmaf(bf_hi(w[i].w), xb.w, acc[i].y);
      }
    }
    if (++slot == n_stage) slot = 0;
  }
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y;
  out[blockIdx.x * 288 + threadIdx.x] = s;
  if (threadIdx.x == 32) out[148 * 288 + blockIdx.x] = (float)(t1 - t0);
}

template <int K>
__global__ void __launch_bounds__(256, 1) alu(float* out, int iters) {
  float2 a[8]; uint32_t u[8];
  for (int i = 0; i < 8; ++i) { a[i] = make_float2(threadIdx.x * 1e-3f + i, 1.f); u[i] = threadIdx.x * 7919u + i; }
  const float2 m = make_float2(1.0001f, 0.9999f), c = make_float2(1e-6f, 1e-6f);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (K == 0) a[i] = __ffma2_rn(a[i], m, c);
      if (K == 1) { a[i].x = fmaf(a[i].x, m.x, c.x); a[i].y = fmaf(a[i].y, m.y, c.y); }
      if (K == 2) u[i] = (u[i] << 16) ^ (u[i] >> 3);                  // shift pair
      if (K == 3) u[i] = (u[i] & 0xffff0000u) + 0x10001u;            // lop + add
      if (K == 4) asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(u[i]) : "r"(u[(i + 1) & 7]));
    }
  }
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y + __uint_as_float(u[i] & 0x3fffffff);
  out[blockIdx.x * 256 + threadIdx.x] = s;
  if (threadIdx.x == 0) out[148 * 288 + blockIdx.x] = (float)(t1 - t0);
}

int main() {
  float* out; cudaMalloc(&out, (148 * 288 + 148) * 4);
  std::vector<float> h(148);
  auto report = [&](const char* name, double per_iter_work, const char* unit) {
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), out + 148 * 288, 148 * 4, cudaMemcpyDeviceToHost);
    double mean = 0; for (float v : h) mean += v; mean /= 148;
    printf("%-44s %10.0f cycles  -> %.2f %s\n", name, mean, mean / per_iter_work, unit);
  };
  const int iters = 20000;
  const int smem = 40960 + 5 * 32768 + 1024;
#define RUN_BODY(MODE, RW, name) do { cudaFuncSetAttribute(body<MODE, RW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
    body<MODE, RW><<<148, 288, smem>>>(out, iters, 32768, 5); cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e)); \
    report(name, (double)iters * RW, "cycles per row-chunk per warp (8 warps/SM)"); } while (0)
  RUN_BODY(0, 8, "body FFMA2 RW=8");
  RUN_BODY(1, 8, "body FFMA  RW=8");
  RUN_BODY(2, 8, "body loads only RW=8");
  RUN_BODY(0, 4, "body FFMA2 RW=4");
  RUN_BODY(0, 2, "body FFMA2 RW=2");
  RUN_BODY(1, 2, "body FFMA  RW=2");
#define RUN_ALU(K, name) do { alu<K><<<148, 256>>>(out, iters); report(name, (double)iters * 8, "cycles per op per warp (2 warps/SMSP)"); } while (0)
  RUN_ALU(0, "FFMA2 dependent x8 chains");
  RUN_ALU(1, "2xFFMA dependent x8 chains");
  RUN_ALU(2, "shl+shr+xor");
  RUN_ALU(3, "and+add");
  RUN_ALU(4, "prmt");
  return 0;
}
