// Does SHFL share the shared-memory (LSU/MIO) pipe with LDS.128?  (development tool)
// Kernel: per iteration one random-address LDS.128 and S shuffles; 15 warps x 148 CTAs.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a shflbench.cu -o shflbench
#include <cstdio>
#include <cuda_runtime.h>

template <int S>
__global__ void __launch_bounds__(480, 1) k(float* out, int iters) {
  __shared__ float4 tab[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) tab[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  unsigned x = threadIdx.x * 2654435761u + blockIdx.x;
  float acc = 0.f, r = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    const float4 v = tab[(x >> 8) & 2047];
    acc += v.x + v.y + v.z + v.w;
#pragma unroll
    for (int s = 0; s < S; ++s) r = __shfl_sync(0xffffffffu, r + acc, (x >> (s & 15)) & 31);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + r;
}

template <int S>
float run(float* out, int iters) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<S><<<148, 480>>>(out, iters);
  cudaEventRecord(a);
  k<S><<<148, 480>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 480 * 4);
  const int it = 20000;
  const double n = 148.0 * 15 * it;  // warp-iterations
  float t0 = run<0>(out, it), t4 = run<4>(out, it), t8 = run<8>(out, it), t16 = run<16>(out, it);
  printf("LDS.128 only         : %.3f ms  %.2f clk/warp-iter/SM\n", t0, t0 * 1e-3 * 1.965e9 / (n / 148));
  printf("LDS.128 +  4 SHFL    : %.3f ms\n", t4);
  printf("LDS.128 +  8 SHFL    : %.3f ms\n", t8);
  printf("LDS.128 + 16 SHFL    : %.3f ms  (SHFL alone est. %.2f clk per SHFL per SM)\n", t16,
         (t16 - t0) * 1e-3 * 1.965e9 / (n / 148) / 16);
  return 0;
}
