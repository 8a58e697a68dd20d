// TLD.128 (tex1Dfetch<float4>) cost per warp instruction vs how many distinct
// texels / 128-byte lines a warp touches; LDS.128 run alongside shows whether
// the two pipes overlap.  Throughput-bound loop (16 independent fetches per
// iteration, the table fits in L1).
//
// With 2 or 3 LDS.128 (4 cycles each) per TLD: if the two pipes have
// separate data paths the loop costs max(8, 4k) cycles per TLD, if they share
// the L1 data SRAM port 4 + 4k.
//
// Question: is the texture path's cost per instruction fixed (~10 cycles, the
// round-1 estimate) or does it drop when a warp's 32 lanes hit few cells
// (decides where LUT pair gb lives).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o texphase texphase.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) {                                                            \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

constexpr int ITERS = 1024;
constexpr int TEXELS = 4096;  // 64 KB

__global__ void kern(cudaTextureObject_t t, const int* __restrict__ idx, int with_lds, float* out,
                     long long* cyc) {
  extern __shared__ float4 sm[];
  for (int i = threadIdx.x; i < 1024 * 3; i += blockDim.x) sm[i] = make_float4(i, i, i, i);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int base = idx[lane];
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm) + (uint32_t)lane * 16u;
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    const int w = base + (it & 3) * 1024;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float4 v;
      asm volatile("tex.1d.v4.f32.s32 {%0,%1,%2,%3}, [%4, {%5}];"
                   : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                   : "l"(t), "r"(w + j * 64));
      acc += v.x;
#pragma unroll
      for (int k = 0; k < 3; ++k)
        if (k < with_lds) {  // with_lds LDS.128 (4 cycles each, distinct chunks) per TLD
          float x, y, z, q;
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                       : "=f"(x), "=f"(y), "=f"(z), "=f"(q)
                       : "r"(sb + (uint32_t)(j * 3 + k) * 512u));
          acc += x + y + z + q;
        }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const int threads = 512;
  float4* buf;
  CK(cudaMalloc(&buf, TEXELS * 16));
  CK(cudaMemset(buf, 0, TEXELS * 16));
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = buf;
  rd.res.linear.desc = cudaCreateChannelDesc<float4>();
  rd.res.linear.sizeInBytes = TEXELS * 16;
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex;
  CK(cudaCreateTextureObject(&tex, &rd, &td, nullptr));
  struct P {
    const char* name;
    int (*f)(int);
  } pats[] = {
      {"32 distinct texels (consecutive)", [](int l) { return l; }},
      {"broadcast (1 texel)", [](int) { return 0; }},
      {"8 distinct texels (4 lanes share)", [](int l) { return l >> 2; }},
      {"4 distinct texels, 4 lines", [](int l) { return (l >> 3) * 8; }},
      {"9 cells x 3 texels apart", [](int l) { return ((l * 7) % 9) * 3; }},
      {"16 distinct (pairs share)", [](int l) { return l >> 1; }},
      {"32 distinct, stride 8 texels", [](int l) { return l * 8; }},
  };
  int* didx;
  float* out;
  long long* cyc;
  CK(cudaMalloc(&didx, 32 * sizeof(int)));
  CK(cudaMalloc(&out, sizeof(float) * nsm * threads));
  CK(cudaMalloc(&cyc, sizeof(long long) * nsm));
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152));
  long long* hc = new long long[nsm];
  for (auto& p : pats) {
    int h[32];
    for (int l = 0; l < 32; ++l) h[l] = p.f(l);
    CK(cudaMemcpy(didx, h, sizeof(h), cudaMemcpyHostToDevice));
    for (int lds = 0; lds < 4; ++lds) {
      if (lds > 1 && p.f != pats[0].f) continue;
      for (int rep = 0; rep < 2; ++rep) {
        kern<<<nsm, threads, 49152>>>(tex, didx, lds, out, cyc);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
      }
      CK(cudaMemcpy(hc, cyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost));
      double avg = 0;
      for (int s = 0; s < nsm; ++s) avg += (double)hc[s];
      avg /= nsm;
      printf("%-36s +%d LDS.128  cycles per warp TLD.128 per SM = %.3f\n", p.name, lds,
             avg / ((double)ITERS * 8 * (threads / 32)));
    }
  }
  return 0;
}
