// ATOMS.ADD (u32, shared) throughput for given warp address patterns: per-lane
// word indices from a file (32 integers per line, "# label" starts a group),
// every lane active, eight independent atomics per step (the same pattern
// shifted by multiples of 32 words, so bank structure is kept).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atomspat atomspat.cu
// Run:   atomspat patterns.txt
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

constexpr int ITERS = 512;
constexpr int WORDS = 16384;  // 64 KB

__global__ void __launch_bounds__(512) kern(const int* __restrict__ word, uint32_t* out, long long* cyc) {
  extern __shared__ uint32_t tab[];
  for (int i = threadIdx.x; i < WORDS; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tab) + (uint32_t)word[lane] * 4u;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    const uint32_t w = base + (uint32_t)(it & 1) * 16384u;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(w + (uint32_t)j * 2048u), "r"((uint32_t)(lane + it + j)) : "memory");
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (threadIdx.x < 32) out[blockIdx.x * 32 + threadIdx.x] = tab[threadIdx.x];
}

int main(int argc, char** argv) {
  if (argc < 2) return 1;
  FILE* f = fopen(argv[1], "r");
  if (!f) return 1;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int* dword;
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&dword, 32 * sizeof(int));
  cudaMalloc(&out, sizeof(uint32_t) * nsm * 32);
  cudaMalloc(&cyc, sizeof(long long) * nsm);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, WORDS * 4);
  long long* hc = new long long[nsm];
  char line[4096], label[256] = "";
  double sum = 0;
  int n = 0;
  auto flush = [&]() {
    if (n) printf("%-40s %6.3f cycles per warp ATOMS per SM (%d patterns)\n", label, sum / n, n);
    sum = 0;
    n = 0;
  };
  while (fgets(line, sizeof line, f)) {
    if (line[0] == '#') {
      flush();
      strncpy(label, line + 2, sizeof label - 1);
      label[strcspn(label, "\n")] = 0;
      continue;
    }
    int h[32], k = 0;
    char* p = line;
    for (; k < 32; ++k) {
      char* e;
      h[k] = (int)strtol(p, &e, 10);
      if (e == p) break;
      p = e;
    }
    if (k < 32) continue;
    for (int i = 0; i < 32; ++i) h[i] %= 8192;
    cudaMemcpy(dword, h, sizeof h, cudaMemcpyHostToDevice);
    kern<<<nsm, 512, WORDS * 4>>>(dword, out, cyc);
    kern<<<nsm, 512, WORDS * 4>>>(dword, out, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(hc, cyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost);
    double a = 0;
    for (int i = 0; i < nsm; ++i) a += (double)hc[i];
    sum += a / nsm / ((double)ITERS * 8 * 16);
    ++n;
  }
  flush();
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
