// Throughput-bound gather test: does TEX (tex1Dfetch<float4>) or L1-resident
// LDG.128 add bandwidth on top of LDS.128 when all run in the same warps?
// Indices are precomputed per thread (8 random entries) and perturbed with a
// cheap xor per iteration, so the load pipes — not integer math — saturate.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pathbench2 pathbench2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 1024;
constexpr int ENTRIES = 2048;  // 32 KB of float4 (power of two for xor perturbation)

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int NL, int NT, int NG>  // loads per iteration through LDS / TEX / LDG
__global__ void gather(cudaTextureObject_t tex, const float4* __restrict__ g, float* out,
                       long long* cyc, int spread) {
  __shared__ float4 sm[ENTRIES];
  for (int i = threadIdx.x; i < ENTRIES; i += blockDim.x) sm[i] = g[i];
  __syncthreads();
  uint32_t idx[8];
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    // spread=0: every lane distinct random; spread=S: lanes share cells in groups of S
    const uint32_t key = spread ? (threadIdx.x / spread) : threadIdx.x;
    idx[k] = hash(key * 8 + k + blockIdx.x * 7777u) & (ENTRIES - 1);
  }
  (void)lane;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
    const uint32_t p = (uint32_t)(i * 37) & (ENTRIES - 1) & ~255u;
#pragma unroll
    for (int k = 0; k < NL; ++k) { float4 v = sm[idx[k] ^ p]; acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w; }
#pragma unroll
    for (int k = 0; k < NT; ++k) { float4 v = tex1Dfetch<float4>(tex, (int)(idx[(k + 3) & 7] ^ p)); acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w; }
#pragma unroll
    for (int k = 0; k < NG; ++k) { float4 v = __ldg(g + (idx[(k + 5) & 7] ^ p)); acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w; }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

template <int NL, int NT, int NG>
int run(const char* name, int nsm, int threads, cudaTextureObject_t tex, const float4* g, float* out,
        long long* cyc, long long* h, int spread) {
  gather<NL, NT, NG><<<nsm, threads>>>(tex, g, out, cyc, spread);
  CK(cudaDeviceSynchronize());
  gather<NL, NT, NG><<<nsm, threads>>>(tex, g, out, cyc, spread);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h, cyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost));
  double avg = 0;
  for (int i = 0; i < nsm; ++i) avg += h[i];
  avg /= nsm;
  double warp_loads = (double)(threads / 32) * ITERS * (NL + NT + NG);
  printf("threads=%4d spread=%d %-14s cycles/warp-load = %5.2f   bytes/clk/SM = %6.1f\n", threads,
         spread, name, avg / warp_loads, warp_loads * 512 / avg);
  return 0;
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
  for (int spread : {0, 4}) {
    for (int threads : {512, 1024}) {
      run<8, 0, 0>("LDS x8", nsm, threads, tex, g, out, cyc, h, spread);
      run<0, 8, 0>("TEX x8", nsm, threads, tex, g, out, cyc, h, spread);
      run<0, 0, 8>("LDG x8", nsm, threads, tex, g, out, cyc, h, spread);
      run<6, 2, 0>("LDS6+TEX2", nsm, threads, tex, g, out, cyc, h, spread);
      run<4, 4, 0>("LDS4+TEX4", nsm, threads, tex, g, out, cyc, h, spread);
      run<6, 0, 2>("LDS6+LDG2", nsm, threads, tex, g, out, cyc, h, spread);
    }
  }
  return 0;
}
