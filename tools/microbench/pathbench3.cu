// TEX gathers from a 52 KB table while the CTA holds ~190 KB of shared memory
// (so L1 keeps only what the carve-out leaves), mixed with LDS gathers.
// Mimics the fused kernel's planned split: 2 LUT pairs in shared memory,
// 1 pair through the texture path.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pathbench3 pathbench3.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 512;
constexpr int TEX_ENTRIES = 3360;   // 52.5 KB of float4
constexpr int SM_ENTRIES = 6720;    // 105 KB of float4 (two pairs)

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int NL, int NT>
__global__ void gather(cudaTextureObject_t tex, const float4* __restrict__ g, float* out,
                       long long* cyc, int spread, int smem_floats) {
  extern __shared__ float4 sm[];
  for (int i = threadIdx.x; i < SM_ENTRIES; i += blockDim.x) sm[i] = g[i % TEX_ENTRIES];
  __syncthreads();
  uint32_t idx[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t key = threadIdx.x / spread;
    idx[k] = hash(key * 8 + k + blockIdx.x * 7777u) % (TEX_ENTRIES - 512);
  }
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
    const uint32_t p = (uint32_t)(i * 48) & 511u;
#pragma unroll
    for (int k = 0; k < NL; ++k) { float4 v = sm[idx[k] + p + (k & 1) * TEX_ENTRIES]; acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w; }
#pragma unroll
    for (int k = 0; k < NT; ++k) { float4 v = tex1Dfetch<float4>(tex, (int)(idx[(k + 3) & 7] + p)); acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w; }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w + (float)smem_floats;
}

template <int NL, int NT>
int run(const char* name, int nsm, int threads, int smem, cudaTextureObject_t tex, const float4* g,
        float* out, long long* cyc, long long* h, int spread) {
  CK(cudaFuncSetAttribute(gather<NL, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  gather<NL, NT><<<nsm, threads, smem>>>(tex, g, out, cyc, spread, smem / 4);
  CK(cudaDeviceSynchronize());
  gather<NL, NT><<<nsm, threads, smem>>>(tex, g, out, cyc, spread, smem / 4);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h, cyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost));
  double avg = 0;
  for (int i = 0; i < nsm; ++i) avg += h[i];
  avg /= nsm;
  double warp_loads = (double)(threads / 32) * ITERS * (NL + NT);
  printf("smem=%6d spread=%d %-12s cycles/warp-load = %5.2f   bytes/clk/SM = %6.1f\n", smem,
         spread, name, avg / warp_loads, warp_loads * 512 / avg);
  return 0;
}

int main() {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float4* g; float* out; long long* cyc;
  CK(cudaMalloc(&g, sizeof(float4) * TEX_ENTRIES));
  CK(cudaMemset(g, 0, sizeof(float4) * TEX_ENTRIES));
  CK(cudaMalloc(&out, sizeof(float) * nsm * 1024));
  CK(cudaMalloc(&cyc, sizeof(long long) * nsm));
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = g;
  rd.res.linear.desc = cudaCreateChannelDesc<float4>();
  rd.res.linear.sizeInBytes = sizeof(float4) * TEX_ENTRIES;
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex;
  CK(cudaCreateTextureObject(&tex, &rd, &td, nullptr));
  long long* h = new long long[nsm];
  const int smems[] = {SM_ENTRIES * 16, SM_ENTRIES * 16 + 65536, 200 * 1024};
  for (int smem : smems) {
    for (int spread : {2, 4}) {
      run<8, 0>("LDS x8", nsm, 512, smem, tex, g, out, cyc, h, spread);
      run<0, 8>("TEX x8", nsm, 512, smem, tex, g, out, cyc, h, spread);
      run<6, 2>("LDS6+TEX2", nsm, 512, smem, tex, g, out, cyc, h, spread);
      run<6, 3>("LDS6+TEX3", nsm, 512, smem, tex, g, out, cyc, h, spread);
      run<5, 3>("LDS5+TEX3", nsm, 512, smem, tex, g, out, cyc, h, spread);
    }
  }
  return 0;
}
