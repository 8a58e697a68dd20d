// Shared-memory atomic add throughput by operand type: u32 (fixed point),
// u64 (wide fixed point), f32.  32 lanes on pseudo-random words of a 48 KB
// table (the backward's scatter pattern), cycles per warp instruction per SM.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atomswidth atomswidth.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;
constexpr int WORDS = 12288;  // 48 KB of u32

template <int MODE>  // 0 u32, 1 u64, 2 f32
__global__ void kern(uint32_t seed, long long* cyc, uint32_t* out) {
  extern __shared__ uint32_t tab[];
  for (int i = threadIdx.x; i < WORDS; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  uint32_t h = seed ^ (threadIdx.x * 2654435761u);
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    h = h * 1664525u + 1013904223u;
    const uint32_t w = (h >> 8) % (WORDS / 2);
    if (MODE == 0) atomicAdd(&tab[2 * w], h & 0xffu);
    if (MODE == 1) atomicAdd(reinterpret_cast<unsigned long long*>(tab) + w, (unsigned long long)(h & 0xffu));
    if (MODE == 2) atomicAdd(reinterpret_cast<float*>(tab) + 2 * w, 1.0f);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (threadIdx.x < 32) out[blockIdx.x * 32 + threadIdx.x] = tab[threadIdx.x];
}

template <int M>
double run(int nsm, long long* c, uint32_t* o, long long* h) {
  cudaFuncSetAttribute(kern<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, WORDS * 4);
  kern<M><<<nsm, 512, WORDS * 4>>>(1u, c, o);
  kern<M><<<nsm, 512, WORDS * 4>>>(2u, c, o);
  cudaDeviceSynchronize();
  cudaMemcpy(h, c, sizeof(long long) * nsm, cudaMemcpyDeviceToHost);
  double a = 0;
  for (int i = 0; i < nsm; ++i) a += (double)h[i];
  return a / nsm / ((double)ITERS * 16);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long* c;
  uint32_t* o;
  cudaMalloc(&c, sizeof(long long) * nsm);
  cudaMalloc(&o, 4 * 32 * nsm);
  long long* h = new long long[nsm];
  printf("u32 atomicAdd: %.3f cycles per warp instruction per SM\n", run<0>(nsm, c, o, h));
  printf("u64 atomicAdd: %.3f\n", run<1>(nsm, c, o, h));
  printf("f32 atomicAdd: %.3f\n", run<2>(nsm, c, o, h));
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
