// Does SHFL run beside LDS.128 (separate pipe) or share its data path?
// Loops of independent SHFL.IDX (random lane), LDS.128 (distinct chunks),
// and both interleaved; cycles per warp instruction per SM.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o shfllds shfllds.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 1024;

template <int MODE>  // 0 shfl only, 1 lds only, 2 both (1:1), 3 both (2 shfl : 1 lds)
__global__ void kern(uint32_t* out, long long* cyc) {
  __shared__ uint4 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_uint4(i, i, i, i);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t v0 = lane * 7, v1 = lane * 3, v2 = lane, v3 = lane + 5;
  uint32_t acc = 0;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm) + (uint32_t)lane * 16u;
  int src = (lane * 13) & 31;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE != 1) {
        acc ^= __shfl_sync(0xffffffffu, v0 + j, src);
        if (MODE == 3) acc ^= __shfl_sync(0xffffffffu, v1 + j, (src + 7) & 31);
      }
      if (MODE != 0) {
        uint32_t x, y, z, w;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(x), "=r"(y), "=r"(z), "=r"(w)
                     : "r"(sb + (uint32_t)((j + it) & 7) * 512u));
        acc ^= x ^ y ^ z ^ w;
      }
    }
    src = (src + 5) & 31;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + v2 + v3;
}

template <int M>
double run(int nsm, uint32_t* out, long long* cyc, long long* hc, int threads) {
  kern<M><<<nsm, threads>>>(out, cyc);
  kern<M><<<nsm, threads>>>(out, cyc);
  cudaDeviceSynchronize();
  cudaMemcpy(hc, cyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int s = 0; s < nsm; ++s) avg += (double)hc[s];
  return avg / nsm / ((double)ITERS * 8 * (threads / 32));
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out;
  long long* cyc;
  const int threads = 512;
  cudaMalloc(&out, sizeof(uint32_t) * nsm * threads);
  cudaMalloc(&cyc, sizeof(long long) * nsm);
  long long* hc = new long long[nsm];
  printf("cycles per loop step (8 steps/iter) per SM, 16 warps:\n");
  printf("  SHFL only            %.3f\n", run<0>(nsm, out, cyc, hc, threads));
  printf("  LDS.128 only         %.3f\n", run<1>(nsm, out, cyc, hc, threads));
  printf("  SHFL + LDS.128       %.3f\n", run<2>(nsm, out, cyc, hc, threads));
  printf("  2 SHFL + LDS.128     %.3f\n", run<3>(nsm, out, cyc, hc, threads));
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
