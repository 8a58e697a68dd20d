// Stream memory-operation pipeline probe (development tool).
//
// Strips of one 4K image cross PCIe on two streams (H2D on s_in, D2H on
// s_out) in four variants, to see what the per-strip handshakes cost:
//   0  plain copies, no dependency between the streams
//   1  + cuStreamWriteValue32 behind every H2D
//   2  + cuStreamWaitValue32 (on the H2D's flag) before every D2H
//   3  as 2, but a spinning relay kernel turns ready[s] into done[s]
// nvcc -O2 -arch=sm_100a memops.cu -lcuda -o memops && ./memops [strips] [MB]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                             \
  do {                                                                    \
    auto e_ = (x);                                                        \
    if (e_ != 0) {                                                        \
      fprintf(stderr, "%s:%d error %d\n", __FILE__, __LINE__, (int)e_);   \
      exit(1);                                                            \
    }                                                                     \
  } while (0)

__global__ void relay(const int* ready, int* done, int n, int gen) {
  for (int s = 0; s < n; ++s) {
    if (threadIdx.x == 0) {
      int v;
      do {
        asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ready + s) : "memory");
      } while (v != gen);
      asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(done + s), "r"(1) : "memory");
    }
  }
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 16;
  const size_t mb = argc > 2 ? atoi(argv[2]) : 100;
  const size_t bytes = mb << 20, sb = bytes / n;
  char *h_in, *h_out, *d_in, *d_out;
  int *ready, *done;
  CK(cudaHostAlloc(&h_in, bytes, 0));
  CK(cudaHostAlloc(&h_out, bytes, 0));
  CK(cudaMalloc(&d_in, bytes));
  CK(cudaMalloc(&d_out, bytes));
  CK(cudaMalloc(&ready, 4 * n));
  CK(cudaMalloc(&done, 4 * n));
  CK(cudaMemset(ready, 0, 4 * n));
  cudaStream_t s_in, s_out, s_k;
  CK(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s_k, cudaStreamNonBlocking));
  cudaEvent_t t0, t1, ev[64][2];
  CK(cudaEventCreate(&t0));
  CK(cudaEventCreate(&t1));
  for (int s = 0; s < n; ++s) {
    CK(cudaEventCreate(&ev[s][0]));
    CK(cudaEventCreate(&ev[s][1]));
  }
  int gen = 0;
  for (int variant = 0; variant < 4; ++variant) {
    for (int rep = 0; rep < 4; ++rep) {
      ++gen;
      CK(cudaMemset(done, 0, 4 * n));
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(t0, s_in));
      CK(cudaStreamWaitEvent(s_out, t0, 0));
      if (variant == 3) {
        CK(cudaStreamWaitEvent(s_k, t0, 0));
        relay<<<1, 32, 0, s_k>>>(ready, done, n, gen);
      }
      for (int s = 0; s < n; ++s) {
        CK(cudaMemcpyAsync(d_in + s * sb, h_in + s * sb, sb, cudaMemcpyHostToDevice, s_in));
        if (variant >= 1) CK(cuStreamWriteValue32(s_in, (CUdeviceptr)(ready + s), gen, 0));
        CK(cudaEventRecord(ev[s][0], s_in));
        if (variant == 2) CK(cuStreamWaitValue32(s_out, (CUdeviceptr)(ready + s), gen, CU_STREAM_WAIT_VALUE_EQ));
        if (variant == 3) CK(cuStreamWaitValue32(s_out, (CUdeviceptr)(done + s), 1, CU_STREAM_WAIT_VALUE_GEQ));
        CK(cudaMemcpyAsync(h_out + s * sb, d_out + s * sb, sb, cudaMemcpyDeviceToHost, s_out));
        CK(cudaEventRecord(ev[s][1], s_out));
      }
      CK(cudaStreamWaitEvent(s_in, ev[n - 1][1], 0));
      CK(cudaEventRecord(t1, s_in));
      CK(cudaDeviceSynchronize());
      float ms;
      CK(cudaEventElapsedTime(&ms, t0, t1));
      if (rep == 3) {
        printf("variant %d: %d strips x %.2f MB each way: %.3f ms\n", variant, n, sb / 1048576.0, ms);
        for (int s = 0; s < n; s += (n > 8 ? n / 8 : 1)) {
          float a, b;
          CK(cudaEventElapsedTime(&a, t0, ev[s][0]));
          CK(cudaEventElapsedTime(&b, t0, ev[s][1]));
          printf("   strip %2d  h2d done %.3f  d2h done %.3f\n", s, a, b);
        }
      }
    }
  }
  return 0;
}
