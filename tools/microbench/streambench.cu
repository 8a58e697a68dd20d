// Streaming skeleton of the fused forward (3 planar f32 planes in, 3 out) on
// sm_100a: which structure reaches the HBM copy peak?
//   A  grid-stride float4 copy, many CTAs
//   B  persistent CTA/SM, W warps, 128-px chunks (lane = 4 px), DEPTH chunks
//      of register prefetch, streaming cache hints
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o streambench streambench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ float4 ldg_na(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}

__global__ void copyA(const float4* __restrict__ in, float4* __restrict__ out, long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x)
    __stcs(out + i, __ldcs(in + i));
}

// chunks of 128 px per warp; chunk c covers px [128c, 128c+128) of every plane
template <int DEPTH, bool HINT>
__global__ void copyB(const float* __restrict__ in, float* __restrict__ out, long long pl, int nchunks) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int gw = blockIdx.x * nw + warp, stride = gridDim.x * nw;
  float4 buf[DEPTH][3];
  int c = gw;
#pragma unroll
  for (int d = 0; d < DEPTH; ++d) {
    const int cc = c + d * stride;
    if (cc < nchunks)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float4* p = reinterpret_cast<const float4*>(in + k * pl + (long long)cc * 128) + lane;
        buf[d][k] = HINT ? ldg_na(p) : *p;
      }
  }
  for (; c < nchunks; c += stride) {
    float4 v[3] = {buf[0][0], buf[0][1], buf[0][2]};
#pragma unroll
    for (int d = 0; d + 1 < DEPTH; ++d)
#pragma unroll
      for (int k = 0; k < 3; ++k) buf[d][k] = buf[d + 1][k];
    const int cn = c + DEPTH * stride;
    if (cn < nchunks)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float4* p = reinterpret_cast<const float4*>(in + k * pl + (long long)cn * 128) + lane;
        buf[DEPTH - 1][k] = HINT ? ldg_na(p) : *p;
      }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      float4* q = reinterpret_cast<float4*>(out + k * pl + (long long)c * 128) + lane;
      if (HINT) __stcs(q, v[k]); else *q = v[k];
    }
  }
}

template <typename F>
float timeit(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f(i);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f(i);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / reps;
}

int main() {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const long long pl = 3840LL * 2160, n = 3 * pl;  // one 4K frame
  const int SETS = 4;
  float *in, *out;
  CK(cudaMalloc(&in, n * 4 * SETS));
  CK(cudaMalloc(&out, n * 4 * SETS));
  CK(cudaMemset(in, 0, n * 4 * SETS));
  const double bytes = 2.0 * n * 4;
  auto rep = [&](const char* name, float us) {
    printf("%-34s %8.2f us  %7.1f GB/s\n", name, us, bytes / (us * 1e-6) / 1e9);
  };
  const int reps = 50;
  for (int bs : {256, 512}) for (int per : {2, 4, 8}) {
    float us = timeit([&](int i) {
      copyA<<<nsm * per, bs>>>(reinterpret_cast<float4*>(in + (i % SETS) * n),
                               reinterpret_cast<float4*>(out + (i % SETS) * n), n / 4);
    }, reps);
    char nm[64]; snprintf(nm, 64, "A grid-stride bs=%d ctas=%dxSM", bs, per);
    rep(nm, us);
  }
  const int nchunks = (int)(pl / 128);
#define RUNB(D, H, NW)                                                                       \
  {                                                                                          \
    float us = timeit([&](int i) {                                                           \
      copyB<D, H><<<nsm, NW * 32>>>(in + (i % SETS) * n, out + (i % SETS) * n, pl, nchunks); \
    }, reps);                                                                                \
    char nm[64]; snprintf(nm, 64, "B depth=%d hint=%d warps=%d", D, (int)H, NW);           \
    rep(nm, us);                                                                             \
  }
  RUNB(1, true, 15) RUNB(2, true, 15) RUNB(3, true, 15) RUNB(4, true, 15)
  RUNB(1, false, 15) RUNB(2, false, 15)
  RUNB(1, true, 30) RUNB(2, true, 30)
  RUNB(1, true, 8) RUNB(2, true, 8) RUNB(4, true, 8)
  return 0;
}
