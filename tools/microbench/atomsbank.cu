// Shared-memory u32 atomic add (ATOMS.ADD) cost by bank pattern: is the
// cost of a warp instruction set by the most-loaded bank (like LDS) or is
// there a fixed floor?  16 warps per SM, cycles per warp instruction per SM.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atomsbank atomsbank.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;
constexpr int WORDS = 12288;  // 48 KB

// MODE: 0 conflict-free (lane l -> bank l, random row)
//       1 random words (32 banks)
//       2 2 lanes per bank (lane l -> bank l/2, random rows)
//       3 4 lanes per bank
//       4 all lanes one word
//       5 16 active lanes (even lanes), random words
//       6 8 active lanes, random words
//       7 conflict-free, result used (dependent chain through the returned value)
//       8 random rows of a per-lane bank, every lane on 1 of 8 copies: bank = 4*(e&7) + (l&3)... (see code)
template <int MODE>
__global__ void kern(uint32_t seed, long long* cyc, uint32_t* out) {
  extern __shared__ uint32_t tab[];
  for (int i = threadIdx.x; i < WORDS; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t h = seed ^ (threadIdx.x * 2654435761u);
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    h = h * 1664525u + 1013904223u;
    const uint32_t row = (h >> 8) % (WORDS / 32);
    uint32_t w;
    bool act = true;
    if (MODE == 0 || MODE == 7) w = row * 32 + lane;
    else if (MODE == 1) w = (h >> 8) % WORDS;
    else if (MODE == 2) w = row * 32 + (lane >> 1);
    else if (MODE == 3) w = row * 32 + (lane >> 2);
    else if (MODE == 4) w = 5;
    else if (MODE == 5) { w = (h >> 8) % WORDS; act = (lane & 1) == 0; }
    else if (MODE == 6) { w = (h >> 8) % WORDS; act = (lane & 3) == 0; }
    else w = 0;
    if (act) {
      if (MODE == 7) acc += atomicAdd(&tab[w], (h & 0xffu) + (acc & 1u));
      else atomicAdd(&tab[w], h & 0xffu);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (threadIdx.x < 32) out[blockIdx.x * 32 + threadIdx.x] = tab[threadIdx.x] + acc;
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
  printf("ATOMS u32 conflict-free (lane -> own bank)   %.3f cycles per warp instruction per SM\n", run<0>(nsm, c, o, h));
  printf("ATOMS u32 random words                       %.3f\n", run<1>(nsm, c, o, h));
  printf("ATOMS u32 2 lanes per bank (distinct words)  %.3f\n", run<2>(nsm, c, o, h));
  printf("ATOMS u32 4 lanes per bank (distinct words)  %.3f\n", run<3>(nsm, c, o, h));
  printf("ATOMS u32 all lanes one word                 %.3f\n", run<4>(nsm, c, o, h));
  printf("ATOMS u32 16 active lanes, random            %.3f\n", run<5>(nsm, c, o, h));
  printf("ATOMS u32 8 active lanes, random             %.3f\n", run<6>(nsm, c, o, h));
  printf("ATOMS u32 conflict-free, result used         %.3f\n", run<7>(nsm, c, o, h));
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
