// Shared int32 ATOMS.ADD cost vs. the number of active lanes (distinct,
// bank-spread addresses): does a partially masked warp instruction cost less?
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atomsmask atomsmask.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 1024;

template <typename T>
__global__ void k(int active_every, long long* cyc, int* out) {
  __shared__ T si[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) si[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool on = (lane % active_every) == 0;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    const int a = (((warp * 97 + i * 131) & 127) * 32 + lane) & 4095;
    if (on) atomicAdd(&si[a], (T)(lane + i));
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = (int)si[threadIdx.x];
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long *c, h;
  int* o;
  cudaMalloc(&c, nsm * 8);
  cudaMalloc(&o, nsm * 512 * 4);
  for (int every : {1, 4, 32, 101, 104}) {
    const bool wide = every > 100;
    if (wide) every -= 100;
    if (wide) { k<unsigned long long><<<nsm, 512>>>(every, c, o); k<unsigned long long><<<nsm, 512>>>(every, c, o); }
    else { k<int><<<nsm, 512>>>(every, c, o); k<int><<<nsm, 512>>>(every, c, o); }
    printf("%s ", wide ? "u64" : "i32");
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    const double warp_instr = 16.0 * ITERS;  // per SM (16 warps)
    printf("active lanes %2d: %.2f cycles per warp ATOMS, %.2f lane-ops/clk\n", 32 / every,
           h / warp_instr, warp_instr * (32 / every) / h);
  }
  return 0;
}
