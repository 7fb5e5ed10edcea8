// Store-path ceilings for the grid kernel's output layout: persistent warps
// issuing 7 streaming v4 stores per lane per chunk (6 planes + codes) with no
// cell math.  mode 0: each warp walks a contiguous item range (grid_kernel);
// mode 1: items dealt round-robin over all warps (global write front);
// mode 2: each block walks a contiguous range, its warps interleaved
// (block-local write front).  Not product code.
#include <cuda_runtime.h>
#include <stdint.h>
template <int ST>
__device__ __forceinline__ void stv(float* p, float4 v) {
  if constexpr (ST == 0) __stcs(reinterpret_cast<float4*>(p), v);
  else if constexpr (ST == 1) *reinterpret_cast<float4*>(p) = v;
  else if constexpr (ST == 2) __stwt(reinterpret_cast<float4*>(p), v);
  else asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
template <int ST = 0>
__device__ __forceinline__ void do_item(float* planes, int32_t* codes, int64_t gi, int64_t chunks,
                                        int64_t m, int64_t ps, int lane) {
  const int64_t sat = gi / chunks, c = gi - sat * chunks;
  const int64_t j0 = c * 128 + lane * 4;
  if (j0 + 4 > m) return;
  float* row = planes + sat * m + j0;
  const float x = (float)gi;
#pragma unroll
  for (int p = 0; p < 6; ++p) stv<ST>(row + p * ps, make_float4(x, x + p, x, x));
  stv<ST>(reinterpret_cast<float*>(codes + sat * m + j0), make_float4(0, 0, 0, 0));
}
extern "C" __global__ void store_kernel(float* planes, int32_t* codes, int64_t n, int64_t m,
                                        int64_t chunks, int64_t ps, int mode) {
  const int wpb = blockDim.x / 32;
  const int64_t nwarps = (int64_t)gridDim.x * wpb;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t total = n * chunks;
  if (mode == 0) {
    const int64_t g0 = total * w / nwarps, g1 = total * (w + 1) / nwarps;
    for (int64_t gi = g0; gi < g1; ++gi) do_item(planes, codes, gi, chunks, m, ps, lane);
  } else if (mode >= 10) {
    const int64_t g0 = total * w / nwarps, g1 = total * (w + 1) / nwarps;
    for (int64_t gi = g0; gi < g1; ++gi) {
      if (mode == 11) do_item<1>(planes, codes, gi, chunks, m, ps, lane);
      else if (mode == 12) do_item<2>(planes, codes, gi, chunks, m, ps, lane);
      else do_item<3>(planes, codes, gi, chunks, m, ps, lane);
    }
  } else if (mode == 1) {
    for (int64_t gi = w; gi < total; gi += nwarps) do_item(planes, codes, gi, chunks, m, ps, lane);
  } else {
    const int64_t b0 = total * blockIdx.x / gridDim.x, b1 = total * (blockIdx.x + 1) / gridDim.x;
    for (int64_t gi = b0 + (threadIdx.x >> 5); gi < b1; gi += wpb) do_item(planes, codes, gi, chunks, m, ps, lane);
  }
}
extern "C" int launch_store(float* planes, int32_t* codes, int64_t n, int64_t m, int blocks, int threads,
                            int mode, void* stream) {
  const int64_t chunks = (m + 127) / 128;
  store_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(planes, codes, n, m, chunks, n * m, mode);
  return (int)cudaGetLastError();
}

// mode 3/4: one contiguous stream, v4 (3) or v8 256-bit (4) stores, grid-stride
// mode 5: grid_kernel mapping with 8 steps per lane and v8 stores
__device__ __forceinline__ void st8(float* p, float x) {
  asm volatile("st.global.cs.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" :: "l"(p), "f"(x) : "memory");
}
extern "C" __global__ void stream_kernel(float* buf, int64_t nfloats, int mode) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  const float x = (float)tid;
  if (mode == 3) {
    for (int64_t i = tid * 4; i + 4 <= nfloats; i += nt * 4) __stcs(reinterpret_cast<float4*>(buf + i), make_float4(x, x, x, x));
  } else {
    for (int64_t i = tid * 8; i + 8 <= nfloats; i += nt * 8) st8(buf + i, x);
  }
}
extern "C" __global__ void store8_kernel(float* planes, int32_t* codes, int64_t n, int64_t m,
                                         int64_t chunks, int64_t ps) {
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x / 32);
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t total = n * chunks;
  const int64_t g0 = total * w / nwarps, g1 = total * (w + 1) / nwarps;
  for (int64_t gi = g0; gi < g1; ++gi) {
    const int64_t sat = gi / chunks, c = gi - sat * chunks;
    const int64_t j0 = c * 256 + lane * 8;
    if (j0 + 8 > m) continue;
    float* row = planes + sat * m + j0;
    const float x = (float)gi;
#pragma unroll
    for (int p = 0; p < 6; ++p) st8(row + p * ps, x + p);
    st8(reinterpret_cast<float*>(codes + sat * m + j0), 0.0f);
  }
}
extern "C" int launch_stream(float* buf, int64_t nfloats, int blocks, int threads, int mode, void* stream) {
  stream_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(buf, nfloats, mode);
  return (int)cudaGetLastError();
}
extern "C" int launch_store8(float* planes, int32_t* codes, int64_t n, int64_t m, int blocks, int threads,
                             void* stream) {
  const int64_t chunks = (m + 255) / 256;
  store8_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(planes, codes, n, m, chunks, n * m);
  return (int)cudaGetLastError();
}

// mode 20/21: stage each chunk's 7 x 512 B in shared memory and write it with
// TMA bulk stores (cp.async.bulk.global.shared::cta), double-buffered per warp;
// 21 stages two consecutive chunks of a row (1 KB per bulk store).
template <int CH>
__global__ void tma_store_kernel(float* planes, int32_t* codes, int64_t n, int64_t m, int64_t chunks,
                                 int64_t ps) {
  extern __shared__ __align__(128) float smem[];
  const int wpb = blockDim.x / 32;
  const int wib = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * wpb;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  constexpr int SEG = 128 * CH;                  // floats per plane segment
  float* wbuf = smem + (size_t)wib * 2 * 7 * SEG;
  const int64_t items = n * (chunks / CH);       // items of CH chunks (m multiple of 128*CH assumed)
  const int64_t g0 = items * w / nwarps, g1 = items * (w + 1) / nwarps;
  int buf = 0;
  for (int64_t gi = g0; gi < g1; ++gi, buf ^= 1) {
    const int64_t per = chunks / CH;
    const int64_t sat = gi / per, c = gi - sat * per;
    const int64_t j0 = c * SEG;
    float* sb = wbuf + buf * 7 * SEG;
    // make sure the bulk stores that read this buffer two items ago are done
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
    const float x = (float)gi;
#pragma unroll
    for (int k = 0; k < CH; ++k) {
#pragma unroll
      for (int p = 0; p < 7; ++p)
        *reinterpret_cast<float4*>(sb + p * SEG + k * 128 + lane * 4) = make_float4(x, x + p, x, x);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
#pragma unroll
      for (int p = 0; p < 7; ++p) {
        float* g = p < 6 ? planes + p * ps + sat * m + j0 : reinterpret_cast<float*>(codes + sat * m + j0);
        const unsigned s = (unsigned)__cvta_generic_to_shared(sb + p * SEG);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     :: "l"(g), "r"(s), "r"(SEG * 4) : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
extern "C" int launch_tma(float* planes, int32_t* codes, int64_t n, int64_t m, int blocks, int threads,
                          int ch, void* stream) {
  const int64_t chunks = (m + 127) / 128;
  const size_t smem = (size_t)(threads / 32) * 2 * 7 * 128 * ch * 4;
  if (ch == 1) {
    cudaFuncSetAttribute(tma_store_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    tma_store_kernel<1><<<blocks, threads, smem, (cudaStream_t)stream>>>(planes, codes, n, m, chunks, n * m);
  } else {
    cudaFuncSetAttribute(tma_store_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    tma_store_kernel<2><<<blocks, threads, smem, (cudaStream_t)stream>>>(planes, codes, n, m, chunks, n * m);
  }
  return (int)cudaGetLastError();
}
