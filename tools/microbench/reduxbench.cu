// Warp aggregation primitives on sm_100a: MATCH.ANY + REDUX.SUM with
// per-group member masks (labeled partitions), cycles per warp instruction.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o reduxbench reduxbench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 1024;

template <int MODE>
__global__ void k(int groups, long long* cyc, int* out) {
  const int lane = threadIdx.x & 31;
  int acc = 0;
  int key = lane % groups;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    if (MODE == 0) {  // 12 REDUX with the group mask (mask computed once)
      const unsigned m = __match_any_sync(0xffffffffu, key);
#pragma unroll
      for (int v = 0; v < 12; ++v) acc += __reduce_add_sync(m, acc + v + i);
    } else if (MODE == 1) {  // MATCH.ANY alone (key changes every iteration)
      acc += (int)__match_any_sync(0xffffffffu, key ^ (i & 1));
    } else {  // 12 full-mask REDUX
#pragma unroll
      for (int v = 0; v < 12; ++v) acc += __reduce_add_sync(0xffffffffu, acc + v + i);
    }
    key ^= acc & 1;
  }
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5)] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  long long *c, h[16];
  int* o;
  cudaMalloc(&c, 148 * 16 * 8);
  cudaMalloc(&o, 148 * 512 * 4);
  for (int g : {1, 4, 9, 32}) {
    k<0><<<148, 512>>>(g, c, o); k<0><<<148, 512>>>(g, c, o);
    cudaMemcpy(h, c, 16 * 8, cudaMemcpyDeviceToHost);
    printf("groups %2d: match+12 redux(group mask): %.1f cycles/iter per warp (16 warps/SM)\n", g, h[0] / (double)ITERS);
  }
  k<1><<<148, 512>>>(9, c, o); k<1><<<148, 512>>>(9, c, o);
  cudaMemcpy(h, c, 16 * 8, cudaMemcpyDeviceToHost);
  printf("match.any alone: %.1f cycles/iter per warp\n", h[0] / (double)ITERS);
  k<2><<<148, 512>>>(1, c, o); k<2><<<148, 512>>>(1, c, o);
  cudaMemcpy(h, c, 16 * 8, cudaMemcpyDeviceToHost);
  printf("12 full-mask redux: %.1f cycles/iter per warp\n", h[0] / (double)ITERS);
  return 0;
}
