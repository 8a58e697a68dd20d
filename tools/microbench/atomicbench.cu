// Shared / global atomic throughput on sm_100a (backward scatter design).
// Reports lane-operations per clock per SM for: int32 ATOMS.ADD (distinct
// addresses, 4-lane sharing, all-same), f32 atomicAdd on shared (CAS loop),
// f32 RED to global (distinct, L2-resident).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atomicbench atomicbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 1024;

template <int MODE>
__global__ void k(int share, float* gout, long long* cyc, float* gacc) {
  __shared__ int si[4096];
  __shared__ float sf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) { si[i] = 0; sf[i] = 0.f; }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int key = share ? lane / share : lane;  // lanes sharing an address
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    const int a = ((warp * 97 + i * 131) & 127) * 32 + key;  // spread over banks
    if (MODE == 0) atomicAdd(&si[a & 4095], lane + i);
    if (MODE == 1) atomicAdd(&sf[a & 4095], (float)(lane + 1));
    if (MODE == 2) atomicAdd(&gacc[(blockIdx.x * 8192 + (a & 8191))], (float)(lane + 1));
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  gout[blockIdx.x * blockDim.x + threadIdx.x] = (float)si[threadIdx.x] + sf[threadIdx.x];
}

template <int MODE>
int run(const char* name, int nsm, int share, float* o, long long* c, float* g, long long* h) {
  k<MODE><<<nsm, 512>>>(share, o, c, g);
  CK(cudaDeviceSynchronize());
  k<MODE><<<nsm, 512>>>(share, o, c, g);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h, c, sizeof(long long) * nsm, cudaMemcpyDeviceToHost));
  double avg = 0;
  for (int i = 0; i < nsm; ++i) avg += h[i];
  avg /= nsm;
  const double lane_ops = 512.0 * ITERS;
  printf("%-22s share=%2d  lane-ops/clk/SM = %6.2f   cycles/warp-instr = %6.2f\n", name, share,
         lane_ops / avg, avg / (lane_ops / 32));
  return 0;
}

int main() {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float *o, *g; long long* c;
  CK(cudaMalloc(&o, sizeof(float) * nsm * 512));
  CK(cudaMalloc(&g, sizeof(float) * nsm * 8192));
  CK(cudaMemset(g, 0, sizeof(float) * nsm * 8192));
  CK(cudaMalloc(&c, sizeof(long long) * nsm));
  long long* h = new long long[nsm];
  for (int share : {0, 2, 4, 8, 32}) {
    run<0>("ATOMS.ADD int32", nsm, share, o, c, g, h);
    run<1>("shared f32 (CAS)", nsm, share, o, c, g, h);
    run<2>("global RED f32", nsm, share, o, c, g, h);
  }
  return 0;
}
