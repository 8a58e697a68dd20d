// Do the texture path or L1-cached global loads add gather bandwidth on top of
// shared memory?  Each warp gathers random 16-byte entries from a 48 KB table
// through one of: LDS.128 (shared), TEX (tex1Dfetch<float4>), LDG.128 (L1
// resident), or a mix in the same warp.  Reports bytes/clk/SM.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pathbench pathbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 2048;
constexpr int ENTRIES = 3072;  // 48 KB of float4

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// mode bits: 1 = LDS, 2 = TEX, 4 = LDG.  `local` = entries per lane neighbourhood (locality)
__global__ void gather(int mode, cudaTextureObject_t tex, const float4* __restrict__ g, float* out,
                       long long* cyc) {
  __shared__ float4 sm[ENTRIES];
  for (int i = threadIdx.x; i < ENTRIES; i += blockDim.x) sm[i] = g[i];
  __syncthreads();
  uint32_t s = hash(threadIdx.x * 7919u + blockIdx.x * 104729u);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    s = s * 1664525u + 1013904223u;
    const uint32_t i1 = (s >> 8) % ENTRIES;
    const uint32_t i2 = (s >> 4) % ENTRIES;
    const uint32_t i3 = (s >> 12) % ENTRIES;
    if (mode & 1) { float4 v = sm[i1]; acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w; }
    if (mode & 2) { float4 v = tex1Dfetch<float4>(tex, (int)i2); acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w; }
    if (mode & 4) { float4 v = __ldg(g + i3); acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w; }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

int main() {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float4* g; float* out; long long* cyc;
  CK(cudaMalloc(&g, sizeof(float4) * ENTRIES));
  CK(cudaMemset(g, 0, sizeof(float4) * ENTRIES));
  CK(cudaMalloc(&out, sizeof(float) * nsm * 1024));
  CK(cudaMalloc(&cyc, sizeof(long long) * nsm));
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = g;
  rd.res.linear.desc = cudaCreateChannelDesc<float4>();
  rd.res.linear.sizeInBytes = sizeof(float4) * ENTRIES;
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex;
  CK(cudaCreateTextureObject(&tex, &rd, &td, nullptr));
  long long* h = new long long[nsm];
  const char* names[] = {"", "LDS", "TEX", "LDS+TEX", "LDG", "LDS+LDG", "TEX+LDG", "LDS+TEX+LDG"};
  for (int threads : {512, 1024}) {
    for (int mode = 1; mode < 8; ++mode) {
      gather<<<nsm, threads>>>(mode, tex, g, out, cyc);
      CK(cudaDeviceSynchronize());
      gather<<<nsm, threads>>>(mode, tex, g, out, cyc);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(h, cyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost));
      double avg = 0;
      for (int i = 0; i < nsm; ++i) avg += h[i];
      avg /= nsm;
      int nfetch = __builtin_popcount(mode);
      double bytes = (double)threads * ITERS * nfetch * 16;
      printf("threads=%4d %-12s bytes/clk/SM = %6.1f  (cycles %.0f)\n", threads, names[mode],
             bytes / avg, avg);
    }
  }
  return 0;
}
