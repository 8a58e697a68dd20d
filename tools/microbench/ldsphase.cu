// LDS.128 cost per warp instruction vs which lanes are active and how many
// distinct 16-byte chunks each quarter / half warp touches.  Throughput-bound
// loop: 16 independent predicated loads per iteration, one LOP3 per load.
//
// Question: does a predicated-off 8-lane phase cost a shared-memory cycle?
// (decides whether a lane may skip re-loading an unchanged grid slot).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ldsphase ldsphase.cu
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

constexpr int ITERS = 2048;
constexpr int CHUNKS = 8192;  // 128 KB of 16-byte chunks

struct Pat {
  const char* name;
  int chunk[32];  // chunk index per lane
  uint32_t active;
};

__global__ void kern(const int* __restrict__ chunk, uint32_t active, uint32_t* out, long long* cyc) {
  extern __shared__ uint4 sm[];
  for (int i = threadIdx.x; i < CHUNKS; i += blockDim.x) sm[i] = make_uint4(i, i * 3, i * 5, i * 7);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm) + (uint32_t)chunk[lane] * 16u;
  const uint32_t p = (active >> lane) & 1u;
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    // 16 windows of 1 KB (64 chunks) apart: same bank pattern, independent loads
    const uint32_t w = base + (uint32_t)((it & 3) * 16) * 1024u;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      uint32_t x, y, z, v;
      if (active == 0xffffffffu) {  // unpredicated (a predicated LDS.128 measured slower)
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(x), "=r"(y), "=r"(z), "=r"(v)
                     : "r"(w + (uint32_t)j * 1024u));
      } else {
        asm volatile(
            "{ .reg .pred q; setp.ne.u32 q, %5, 0;\n"
            "@q ld.shared.v4.u32 {%0,%1,%2,%3}, [%4]; }"
            : "=r"(x), "=r"(y), "=r"(z), "=r"(v)
            : "r"(w + (uint32_t)j * 1024u), "r"(p));
      }
      acc ^= x ^ y ^ z ^ v;  // all four words live: keeps the 128-bit load
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int run_file(const char* path);
int main(int argc, char** argv) {
  if (argc > 1) return run_file(argv[1]);
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const int threads = 256;
  Pat pats[16];
  int np = 0;
  auto add = [&](const char* n, uint32_t act, auto f) {
    Pat& P = pats[np++];
    P.name = n;
    P.active = act;
    for (int l = 0; l < 32; ++l) P.chunk[l] = f(l);
  };
  add("distinct, all lanes", 0xffffffffu, [](int l) { return l; });
  add("distinct, lanes 0-7 only", 0x000000ffu, [](int l) { return l; });
  add("distinct, lanes 0-15 only", 0x0000ffffu, [](int l) { return l; });
  add("distinct, lanes 8-15 only", 0x0000ff00u, [](int l) { return l; });
  add("distinct, 1 lane per quarter", 0x01010101u, [](int l) { return l; });
  add("distinct, lane 0 only", 0x00000001u, [](int l) { return l; });
  add("broadcast, all lanes", 0xffffffffu, [](int) { return 0; });
  add("quarter: 8 distinct, all quarters same", 0xffffffffu, [](int l) { return l & 7; });
  add("quarter: 1 chunk each (4 distinct)", 0xffffffffu, [](int l) { return l >> 3; });
  add("quarter: 2 chunks (lanes 4 share)", 0xffffffffu, [](int l) { return l >> 2; });
  add("quarter: 4 chunks (pairs share)", 0xffffffffu, [](int l) { return l >> 1; });
  add("half: 16 distinct, halves same", 0xffffffffu, [](int l) { return l & 15; });
  add("2-way bank conflict (stride 8 chunks)", 0xffffffffu, [](int l) { return (l & 7) * 8 + (l >> 3); });
  add("q0: 4 chunks same bank group", 0x000000ffu, [](int l) { return (l & 3) * 8; });
  add("quarters 0,2 active distinct", 0x00ff00ffu, [](int l) { return l; });
  add("all lanes, 8 distinct in q0, rest = lane0", 0xffffffffu, [](int l) { return l < 8 ? l : 0; });
  int* dchunk;
  uint32_t* out;
  long long* cyc;
  CK(cudaMalloc(&dchunk, 32 * sizeof(int)));
  CK(cudaMalloc(&out, sizeof(uint32_t) * nsm * threads));
  CK(cudaMalloc(&cyc, sizeof(long long) * nsm));
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CHUNKS * 16));
  long long* hc = new long long[nsm];
  for (int i = 0; i < np; ++i) {
    CK(cudaMemcpy(dchunk, pats[i].chunk, 32 * sizeof(int), cudaMemcpyHostToDevice));
    for (int rep = 0; rep < 2; ++rep) {
      kern<<<nsm, threads, CHUNKS * 16>>>(dchunk, pats[i].active, out, cyc);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
    }
    CK(cudaMemcpy(hc, cyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost));
    double avg = 0;
    for (int s = 0; s < nsm; ++s) avg += (double)hc[s];
    avg /= nsm;
    const double per = avg / ((double)ITERS * 16 * (threads / 32));
    printf("%-44s active=%08x  cycles per warp LDS.128 per SM = %.3f\n", pats[i].name, pats[i].active, per);
  }
  return 0;
}

// File mode: each line holds 32 chunk indices (< 4096), '# label' lines start groups; prints measured cycles
// per warp LDS.128 and the bank-group model max_g(#distinct chunks in group g).
int run_file(const char* path) {
  FILE* f = fopen(path, "r");
  if (!f) return 1;
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const int threads = 256;
  int* dchunk;
  uint32_t* out;
  long long* cyc;
  CK(cudaMalloc(&dchunk, 32 * sizeof(int)));
  CK(cudaMalloc(&out, sizeof(uint32_t) * nsm * threads));
  CK(cudaMalloc(&cyc, sizeof(long long) * nsm));
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CHUNKS * 16));
  long long* hc = new long long[nsm];
  int ch[32];
  double sum_meas = 0, sum_model = 0;
  int n = 0;
  char label[128] = "";
  while (true) {
    int c0 = fgetc(f);
    while (c0 == '\n' || c0 == ' ' || c0 == '\r') c0 = fgetc(f);
    if (c0 == '#') {
      if (n) printf("%-28s mean measured %.3f mean model %.3f over %d\n", label, sum_meas / n, sum_model / n, n);
      sum_meas = sum_model = 0;
      n = 0;
      if (!fgets(label, sizeof(label), f)) break;
      for (char* p = label; *p; ++p) if (*p == '\n') *p = 0;
      continue;
    }
    if (c0 == EOF) break;
    ungetc(c0, f);
    int ok = 1;
    for (int l = 0; l < 32 && ok; ++l) ok = fscanf(f, "%d", &ch[l]) == 1;
    if (!ok) break;
    int model = 0;
    for (int g = 0; g < 8; ++g) {
      int cnt = 0;
      for (int l = 0; l < 32; ++l) {
        if (ch[l] % 8 != g) continue;
        bool seen = false;
        for (int m = 0; m < l; ++m) seen |= ch[m] == ch[l];
        cnt += !seen;
      }
      model = cnt > model ? cnt : model;
    }
    CK(cudaMemcpy(dchunk, ch, sizeof(ch), cudaMemcpyHostToDevice));
    kern<<<nsm, threads, CHUNKS * 16>>>(dchunk, 0xffffffffu, out, cyc);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(hc, cyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost));
    double avg = 0;
    for (int s = 0; s < nsm; ++s) avg += (double)hc[s];
    avg /= nsm;
    const double per = avg / ((double)ITERS * 16 * (threads / 32));
    sum_meas += per;
    sum_model += model;
    ++n;
  }
  if (n) printf("%-28s mean measured %.3f mean model %.3f over %d\n", label, sum_meas / n, sum_model / n, n);
  return 0;
}
