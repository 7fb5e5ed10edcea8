// Pipe throughput microbenchmarks on sm_100a (not product code): long loops
// of independent chains of one instruction class, or two classes mixed, so
// the measured rate is the pipe's issue/throughput limit.
#include <cuda_runtime.h>
#include <stdint.h>
#define ITERS 2048
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float sinap(float x) { float r; asm volatile("sin.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ float rcpap(float x) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ float ex2(float x) { float r; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }

extern "C" __global__ void k_ffma2(float* out, float s) {
  float2 a[8]; for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x + i, s * i);
  const float2 b = make_float2(0.999f, 0.998f), c = make_float2(0.001f, 0.002f);
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = ffma2(a[i], b, c);
  float r = 0; for (int i = 0; i < 8; ++i) r += a[i].x + a[i].y;
  if (r == 1.2345f) out[threadIdx.x] = r;
}
extern "C" __global__ void k_ffma(float* out, float s) {
  float a[16]; for (int i = 0; i < 16; ++i) a[i] = threadIdx.x + i * s;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], 0.999f, 0.001f);
  float r = 0; for (int i = 0; i < 16; ++i) r += a[i];
  if (r == 1.2345f) out[threadIdx.x] = r;
}
extern "C" __global__ void k_mufu(float* out, float s) {
  float a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * s;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = rcpap(a[i] + 1.0f);
  float r = 0; for (int i = 0; i < 8; ++i) r += a[i];
  if (r == 1.2345f) out[threadIdx.x] = r;
}
extern "C" __global__ void k_dfma(float* out, float s) {
  double a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i * (double)s;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], 0.999, 0.001);
  double r = 0; for (int i = 0; i < 8; ++i) r += a[i];
  if (r == 1.2345) out[threadIdx.x] = (float)r;
}
extern "C" __global__ void k_f2f(float* out, float s) {
  double a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i * (double)s;
  float acc[8] = {0};
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) { float f; asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f) : "d"(a[i])); acc[i] = f; a[i] = (double)__int_as_float(__float_as_int(f) ^ it); }
  float r = 0; for (int i = 0; i < 8; ++i) r += acc[i];
  if (r == 1.2345f) out[threadIdx.x] = r;
}
// mixes: per iteration 8 FFMA2 + k of the other class
extern "C" __global__ void k_ffma2_dfma(float* out, float s) {
  float2 a[8]; for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x + i, s * i);
  double d[4]; for (int i = 0; i < 4; ++i) d[i] = threadIdx.x + i * (double)s;
  const float2 b = make_float2(0.999f, 0.998f), c = make_float2(0.001f, 0.002f);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = ffma2(a[i], b, c);
#pragma unroll
    for (int i = 0; i < 4; ++i) d[i] = fma(d[i], 0.999, 0.001);
  }
  float r = 0; for (int i = 0; i < 8; ++i) r += a[i].x + a[i].y;
  for (int i = 0; i < 4; ++i) r += (float)d[i];
  if (r == 1.2345f) out[threadIdx.x] = r;
}
extern "C" __global__ void k_ffma2_mufu(float* out, float s) {
  float2 a[8]; for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x + i, s * i);
  float m[2]; for (int i = 0; i < 2; ++i) m[i] = threadIdx.x * 1e-3f + i * s;
  const float2 b = make_float2(0.999f, 0.998f), c = make_float2(0.001f, 0.002f);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = ffma2(a[i], b, c);
#pragma unroll
    for (int i = 0; i < 2; ++i) m[i] = rcpap(m[i] + 1.0f);
  }
  float r = 0; for (int i = 0; i < 8; ++i) r += a[i].x + a[i].y;
  for (int i = 0; i < 2; ++i) r += m[i];
  if (r == 1.2345f) out[threadIdx.x] = r;
}
extern "C" __global__ void k_ffma_ffma2(float* out, float s) {
  float2 a[8]; for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x + i, s * i);
  float f[8]; for (int i = 0; i < 8; ++i) f[i] = threadIdx.x + i * s;
  const float2 b = make_float2(0.999f, 0.998f), c = make_float2(0.001f, 0.002f);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = ffma2(a[i], b, c);
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = fmaf(f[i], 0.999f, 0.001f);
  }
  float r = 0; for (int i = 0; i < 8; ++i) r += a[i].x + a[i].y + f[i];
  if (r == 1.2345f) out[threadIdx.x] = r;
}
typedef void (*kfn)(float*, float);
extern "C" int run(int which, float* out, int blocks, int threads, void* stream) {
  kfn ks[] = {k_ffma2, k_ffma, k_mufu, k_dfma, k_f2f, k_ffma2_dfma, k_ffma2_mufu, k_ffma_ffma2};
  ks[which]<<<blocks, threads, 0, (cudaStream_t)stream>>>(out, 1.0f);
  return (int)cudaGetLastError();
}
