// Shared int32 ATOMS.ADD cost per warp instruction vs. the lane->address
// pattern: distinct banks, same address, groups of same address, bank
// conflicts (same bank, distinct addresses).  Guides the backward's scatter.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atomspattern atomspattern.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 1024;

__global__ void k(int mode, long long* cyc, int* out) {
  __shared__ int si[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) si[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int off;
  switch (mode) {
    case 0: off = lane; break;                 // 32 banks, distinct
    case 1: off = 0; break;                    // all same address
    case 2: off = (lane >> 3) * 33; break;     // 4 groups of 8 same-address, distinct banks
    case 3: off = (lane >> 2) * 33; break;     // 8 groups of 4
    case 4: off = lane * 32; break;            // 32-way bank conflict, distinct addresses
    case 5: off = (lane & 3) * 32 + (lane >> 2); break;  // 4-way bank conflict
    default: off = (lane * 97) & 255; break;   // pseudo-random spread
  }
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    const int a = (((warp * 7 + i) & 7) * 1024 + off) & 8191;
    atomicAdd(&si[a], lane + i);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = si[threadIdx.x];
}

int main() {
  long long *c, h;
  int* o;
  cudaMalloc(&c, 148 * 8);
  cudaMalloc(&o, 148 * 512 * 4);
  const char* names[] = {"distinct banks", "all same address", "4 groups x 8 same", "8 groups x 4 same",
                         "32-way bank conflict", "4-way bank conflict", "pseudo-random"};
  for (int m = 0; m < 7; ++m) {
    k<<<148, 512>>>(m, c, o);
    k<<<148, 512>>>(m, c, o);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-22s %6.2f cycles per warp ATOMS (SM-wide)\n", names[m], h / (16.0 * ITERS));
  }
  return 0;
}
