// FP64 pipe microbenchmarks on sm_100a (analysis, not product code): does an
// fp64 warp-instruction take one issue slot or two, what does mixing ALU /
// LDS / FSEL work into a DFMA stream cost, and DFMA latency.
#include <cuda_runtime.h>
#include <stdint.h>
#define ITERS 1024

extern "C" __global__ void k_dfma(float* out, float s) {            // 8 DFMA
  double a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i * (double)s;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], 0.999, 0.001);
  double r = 0; for (int i = 0; i < 8; ++i) r += a[i];
  if (r == 1.2345) out[threadIdx.x] = (float)r;
}
extern "C" __global__ void k_dfma_alu(float* out, float s) {        // 8 DFMA + 8 IADD3/LOP3
  double a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i * (double)s;
  unsigned u[8]; for (int i = 0; i < 8; ++i) u[i] = threadIdx.x * 7 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = fma(a[i], 0.999, 0.001); u[i] = (u[i] ^ it) + 0x9e37u; }
  }
  double r = 0; unsigned x = 0; for (int i = 0; i < 8; ++i) { r += a[i]; x ^= u[i]; }
  if (r == 1.2345 || x == 77u) out[threadIdx.x] = (float)r;
}
extern "C" __global__ void k_dfma_alu2(float* out, float s) {       // 8 DFMA + 16 ALU
  double a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i * (double)s;
  unsigned u[8], w[8]; for (int i = 0; i < 8; ++i) { u[i] = threadIdx.x * 7 + i; w[i] = i; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = fma(a[i], 0.999, 0.001); u[i] = (u[i] ^ it) + 0x9e37u; w[i] = (w[i] | it) + u[i]; }
  }
  double r = 0; unsigned x = 0; for (int i = 0; i < 8; ++i) { r += a[i]; x ^= u[i] ^ w[i]; }
  if (r == 1.2345 || x == 77u) out[threadIdx.x] = (float)r;
}
extern "C" __global__ void k_dfma_lds(float* out, float s) {        // 8 DFMA + 4 LDS.64 (broadcast)
  __shared__ double sh[64];
  if (threadIdx.x < 64) sh[threadIdx.x] = 1.0 + threadIdx.x * 1e-9;
  __syncthreads();
  double a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i * (double)s;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], sh[(it + (i >> 1)) & 63], 0.001);
  }
  double r = 0; for (int i = 0; i < 8; ++i) r += a[i];
  if (r == 1.2345) out[threadIdx.x] = (float)r;
}
extern "C" __global__ void k_dfma_ffma(float* out, float s) {       // 8 DFMA + 8 FFMA
  double a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i * (double)s;
  float f[8]; for (int i = 0; i < 8; ++i) f[i] = threadIdx.x + i * s;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = fma(a[i], 0.999, 0.001); f[i] = fmaf(f[i], 0.999f, 0.001f); }
  }
  double r = 0; for (int i = 0; i < 8; ++i) r += a[i] + f[i];
  if (r == 1.2345) out[threadIdx.x] = (float)r;
}
extern "C" __global__ void k_dfma_lat(float* out, float s) {        // 1 dependent chain
  double a = threadIdx.x * (double)s;
  for (int it = 0; it < ITERS * 8; ++it) a = fma(a, 0.999, 0.001);
  if (a == 1.2345) out[threadIdx.x] = (float)a;
}
typedef void (*kfn)(float*, float);
extern "C" int run(int which, float* out, int blocks, int threads, void* stream) {
  kfn ks[] = {k_dfma, k_dfma_alu, k_dfma_alu2, k_dfma_lds, k_dfma_ffma, k_dfma_lat};
  ks[which]<<<blocks, threads, 0, (cudaStream_t)stream>>>(out, 1.0f);
  return (int)cudaGetLastError();
}

// occupancy/ILP sweep: each thread runs ILP independent dependent chains
template <int ILP>
__global__ void k_chains(float* out, float s) {
  double a[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x + i * (double)s;
  for (int it = 0; it < ITERS * 8 / ILP; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = fma(a[i], 0.999, 0.001);
  double r = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) r += a[i];
  if (r == 1.2345) out[threadIdx.x] = (float)r;
}
__global__ void k_dmul(float* out, float s) {           // 8 independent DMUL chains
  double a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i * (double)s;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = a[i] * 0.999;
  double r = 0; for (int i = 0; i < 8; ++i) r += a[i];
  if (r == 1.2345) out[threadIdx.x] = (float)r;
}
__global__ void k_dfma_reg(float* out, float s) {       // 8 DFMA, all-register operands
  double a[8], b = 0.999 + threadIdx.x * 1e-12, c = 0.001 + s * 1e-12;
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i * (double)s;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  double r = 0; for (int i = 0; i < 8; ++i) r += a[i];
  if (r == 1.2345) out[threadIdx.x] = (float)r;
}
extern "C" int run2(int which, float* out, int blocks, int threads, void* stream) {
  kfn ks[] = {k_chains<1>, k_chains<2>, k_chains<3>, k_chains<4>, k_dmul, k_dfma_reg};
  ks[which]<<<blocks, threads, 0, (cudaStream_t)stream>>>(out, 1.0f);
  return (int)cudaGetLastError();
}
