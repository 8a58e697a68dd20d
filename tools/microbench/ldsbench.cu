// Shared-memory gather microbenchmark for the fused slice+LUT kernel design.
//
// Question answered: how many cycles does one warp-wide LDS.{32,64,128} cost on
// sm_100a for the access patterns the LUT gather produces (distinct cells,
// few distinct cells, broadcast, partially-predicated warps)?  The fused
// kernel's smem budget per pixel is derived from these numbers.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ldsbench ldsbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;
constexpr int SMEM_FLOATS = 16384;  // 64 KB

// pattern -> per-lane float offset (in floats) inside a 512 B window
__device__ __forceinline__ int lane_off(int pat, int lane, int width) {
  switch (pat) {
    case 0: return lane * width;                 // distinct, conflict-free
    case 1: return 0;                            // broadcast
    case 2: return (lane >> 3) * width;          // 4 distinct (8 consecutive lanes share)
    case 3: return (lane & 7) * width;           // 8 distinct, each quarter-warp identical
    case 4: return (lane >> 2) * width;          // 8 distinct (4 consecutive lanes share)
    case 5: return (lane >> 1) * width;          // 16 distinct (pairs share)
    case 6: return lane * width * 2;             // 2-way bank conflict-ish stride
    case 7: return (lane & 1) ? 0 : lane * width; // half lanes broadcast, half distinct
    default: return 0;
  }
}

template <int W>
__global__ void lds_kernel(int pat, int active_mask_bits, float* out, long long* cycles) {
  extern __shared__ float sm[];
  for (int i = threadIdx.x; i < SMEM_FLOATS; i += blockDim.x) sm[i] = (float)(i & 255) * 0.5f;
  __syncthreads();
  int lane = threadIdx.x & 31;
  int off = lane_off(pat, lane, W);
  bool active = (active_mask_bits >> lane) & 1;
  float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
  uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  long long t0 = clock64();
  if (active) {
#pragma unroll 8
    for (int i = 0; i < ITERS; ++i) {
      int window = ((i * 37) & 63) * 128;  // rotate through 64 windows of 512 B
      uint32_t a = base + (uint32_t)((window + off) & (SMEM_FLOATS - 1)) * 4u;
      if (W == 4) {
        float x, y, z, w;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(a));
        acc0 += x; acc1 += y; acc2 += z; acc3 += w;
      } else if (W == 2) {
        float x, y;
        asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(x), "=f"(y) : "r"(a));
        acc0 += x; acc1 += y;
      } else {
        float x;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(a));
        acc0 += x;
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int clk = 0, memclk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s sms=%d smemPerBlockOptin=%zu smemPerSM=%zu l2=%d regsPerSM=%d clock_khz=%d\n",
         prop.name, prop.multiProcessorCount, prop.sharedMemPerBlockOptin,
         prop.sharedMemPerMultiprocessor, prop.l2CacheSize, prop.regsPerMultiprocessor, clk);
  int nsm = prop.multiProcessorCount;
  int threads = 1024;
  float* out; long long* cyc;
  CK(cudaMalloc(&out, sizeof(float) * nsm * threads));
  CK(cudaMalloc(&cyc, sizeof(long long) * nsm));
  long long* hc = new long long[nsm];
  const char* names[] = {"distinct", "broadcast", "4distinct(8share)", "8distinct(qw-same)",
                         "8distinct(4share)", "16distinct(2share)", "stride2", "half-bcast"};
  struct { int w; void (*k)(int, int, float*, long long*); } ks[] = {
      {1, lds_kernel<1>}, {2, lds_kernel<2>}, {4, lds_kernel<4>}};
  for (auto& kk : ks) {
    CK(cudaFuncSetAttribute(kk.k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_FLOATS * 4));
    for (int pat = 0; pat < 8; ++pat) {
      for (int am = 0; am < 5; ++am) {
        // all / first 16 lanes / even lanes / one quarter-warp (lanes 0-7) /
        // one lane per quarter-warp: do predicated-off 8-lane phases of an
        // LDS.128 cost wavefronts?
        const int masks[5] = {-1, 0x0000FFFF, 0x55555555, 0x000000FF, 0x01010101};
        const char* mnames[5] = {"all ", "lo16", "even", "q0  ", "1/q "};
        int mask = masks[am];
        kk.k<<<nsm, threads, SMEM_FLOATS * 4>>>(pat, mask, out, cyc);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(hc, cyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost));
        double avg = 0; for (int i = 0; i < nsm; ++i) avg += hc[i]; avg /= nsm;
        double per = avg / ((double)ITERS * (threads / 32));
        printf("LDS.%d pat=%-20s mask=%s  cycles/warp-instr/SM=%.3f\n", kk.w * 32, names[pat],
               mnames[am], per);
      }
    }
  }
  return 0;
}
