// Clean LDS.128 throughput probe: every lane active, no predicates, no
// branches in the timed loop; eight independent 128-bit loads per step with
// all four words consumed.  Per-lane 16-byte chunk indices come from a file
// (one warp pattern of 32 integers per line; "# label" starts a group), and
// the same kernel is run under ncu for the wavefront counters.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ldsclean ldsclean.cu
// Run:   ldsclean patterns.txt
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

constexpr int ITERS = 1024;
constexpr int CHUNKS = 8192;  // 128 KB

__global__ void __launch_bounds__(512) kern(const int* __restrict__ chunk, uint32_t* out, long long* cyc) {
  extern __shared__ uint4 sm[];
  for (int i = threadIdx.x; i < CHUNKS; i += blockDim.x) sm[i] = make_uint4(i, i * 3, i * 5, i * 7);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm) + (uint32_t)chunk[lane] * 16u;
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    const uint32_t w = base + (uint32_t)(it & 3) * 16384u;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t x, y, z, v;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(x), "=r"(y), "=r"(z), "=r"(v)
                   : "r"(w + (uint32_t)j * 1024u));
      acc ^= x ^ y ^ z ^ v;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main(int argc, char** argv) {
  if (argc < 2) return 1;
  FILE* f = fopen(argv[1], "r");
  if (!f) return 1;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 512;
  int* dchunk;
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&dchunk, 32 * sizeof(int));
  cudaMalloc(&out, sizeof(uint32_t) * nsm * threads);
  cudaMalloc(&cyc, sizeof(long long) * nsm);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CHUNKS * 16);
  long long* hc = new long long[nsm];
  char line[4096], label[256] = "";
  double sum = 0;
  int n = 0;
  auto flush = [&]() {
    if (n) printf("%-34s %.3f cycles per warp LDS.128 per SM (%d patterns)\n", label, sum / n, n);
    sum = 0;
    n = 0;
  };
  while (fgets(line, sizeof(line), f)) {
    if (line[0] == '#') {
      flush();
      strncpy(label, line + 2, sizeof(label) - 1);
      label[strcspn(label, "\n")] = 0;
      continue;
    }
    int ch[32], k = 0;
    char* p = line;
    while (k < 32) {
      char* e;
      long v = strtol(p, &e, 10);
      if (e == p) break;
      ch[k++] = (int)(v % 2048);
      p = e;
    }
    if (k < 32) continue;
    cudaMemcpy(dchunk, ch, sizeof(ch), cudaMemcpyHostToDevice);
    kern<<<nsm, threads, CHUNKS * 16>>>(dchunk, out, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(hc, cyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int s = 0; s < nsm; ++s) avg += (double)hc[s];
    avg /= nsm;
    sum += avg / ((double)ITERS * 8 * (threads / 32));
    ++n;
  }
  flush();
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
