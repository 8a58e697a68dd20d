// svdlut_naive.cu — the reference's multi-pass "original structure" on the GPU
// (SURVEY.md §8(f) rows 3 and 4), bitwise equal to the reference:
//
//   slice_kernel    transform.slice_grid2d  (transform.py:152-178)  -> (B, K, H, W)
//   lut2d_kernel    transform.apply_lut2d   (transform.py:123-141)  -> (B, 3, H, W)
//   combine_kernel  transform.combine_slices (transform.py:181-193) -> (B, 3, H, W)
//   lut3d_kernel    transform.apply_lut3d   (transform.py:93-120)   -> (B, 3, H, W)
//
// These materialize every intermediate raster (the structure the fused kernel
// removes) and exist to reproduce the paper's multi-stage vs fused runtime
// comparison on B200 with identical numerics.  Numerics follow the numpy
// expressions exactly:
//   * interp.bracket_array (interp.py:114-123): t = f32(clip(p, 0, 1)) *
//     f32(d - 1) rounded to f32, i = min(floor(t), d - 2), delta = f64(t) - i;
//   * _bilinear_arrays (transform.py:79-90): f64, no FMA,
//     v00*((1-da)*(1-db)) + v10*(da*(1-db)) + v01*((1-da)*db) + v11*(da*db)
//     accumulated left to right; weights are f32 scalars promoted to f64;
//   * every stage stores f32 (numpy assigns into float32 rasters);
//   * combine_slices: base + sum over maps j = c, c+3, ... in f32, sequential.
#include "svdlut_common.cuh"
#include "svdlut_internal.h"

namespace svdlut {

#define NM __dmul_rn
#define NA __dadd_rn
#define NS __dsub_rn

// interp.bracket_array (f32 product, f64 delta)
__device__ __forceinline__ void bracket_arr(float p, int d, int& i, double& delta) {
  p = fminf(fmaxf(p, 0.0f), 1.0f);  // np.clip (inputs are finite)
  const float t = __fmul_rn(p, (float)(d - 1));
  const float f = fminf(floorf(t), (float)(d - 2));
  i = (int)f;
  delta = NS((double)t, (double)i);
}

// transform._spatial_brackets (transform.py:144-149): x / (n - 1) in f32
__device__ __forceinline__ void spatial_arr(int x, int n, int d, int& i, double& delta) {
  bracket_arr(__fdiv_rn((float)x, (float)(n - 1)), d, i, delta);
}

// _bilinear_arrays on plane[a][b] (row stride `stride`)
__device__ __forceinline__ double bil(const float* __restrict__ pl, int stride, int ia, double da,
                                      int ib, double db) {
  const double v00 = (double)__ldg(pl + ia * stride + ib);
  const double v10 = (double)__ldg(pl + (ia + 1) * stride + ib);
  const double v01 = (double)__ldg(pl + ia * stride + ib + 1);
  const double v11 = (double)__ldg(pl + (ia + 1) * stride + ib + 1);
  const double ea = NS(1.0, da), eb = NS(1.0, db);
  double out = NM(v00, NM(ea, eb));
  out = NA(out, NM(v10, NM(da, eb)));
  out = NA(out, NM(v01, NM(ea, db)));
  return NA(out, NM(v11, NM(da, db)));
}

__global__ void slice_kernel(const float* __restrict__ rgb, float* __restrict__ fs, int batch, int h,
                             int w, int y0, int h_total, const float* __restrict__ gp,
                             const float* __restrict__ gw, const float* __restrict__ gb, int k, int ds) {
  const long long plane = (long long)h * w;
  const long long total = (long long)batch * plane;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(e / plane);
    const long long o = e - (long long)b * plane;
    const int y = (int)(o / w), x = (int)(o - (long long)y * w);
    const float* X = rgb + (long long)b * 3 * plane;
    int ix, iy, ic[3];
    double dx, dy, dc[3];
    spatial_arr(x, w, ds, ix, dx);
    spatial_arr(y0 + y, h_total, ds, iy, dy);
    for (int c = 0; c < 3; ++c) bracket_arr(__ldg(X + c * plane + o), ds, ic[c], dc[c]);
    for (int kk = 0; kk < k; ++kk) {
      const float* G = gp + ((long long)b * k + kk) * 3 * ds * ds;
      const float* W3 = gw + ((long long)b * k + kk) * 3;
      const int c = kk % 3;
      double acc = NM((double)__ldg(W3 + 0), bil(G, ds, ix, dx, iy, dy));
      acc = NA(acc, NM((double)__ldg(W3 + 1), bil(G + ds * ds, ds, ix, dx, ic[c], dc[c])));
      acc = NA(acc, NM((double)__ldg(W3 + 2), bil(G + 2 * ds * ds, ds, iy, dy, ic[c], dc[c])));
      acc = NA(acc, (double)__ldg(gb + (long long)b * k + kk));
      fs[((long long)b * k + kk) * plane + o] = (float)acc;
    }
  }
}

__global__ void lut2d_kernel(const float* __restrict__ rgb, float* __restrict__ out, int batch, int h,
                             int w, const float* __restrict__ lp, const float* __restrict__ lw,
                             const float* __restrict__ lb, int dt) {
  const long long plane = (long long)h * w;
  const long long total = (long long)batch * plane;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(e / plane);
    const long long o = e - (long long)b * plane;
    const float* X = rgb + (long long)b * 3 * plane;
    int ir, ig, ib;
    double dr, dg, db;
    bracket_arr(__ldg(X + o), dt, ir, dr);
    bracket_arr(__ldg(X + plane + o), dt, ig, dg);
    bracket_arr(__ldg(X + 2 * plane + o), dt, ib, db);
    for (int c = 0; c < 3; ++c) {
      const float* P = lp + ((long long)b * 9 + c * 3) * dt * dt;
      const float* Wc = lw + (long long)b * 9 + c * 3;
      double acc = NM((double)__ldg(Wc + 0), bil(P, dt, ir, dr, ig, dg));
      acc = NA(acc, NM((double)__ldg(Wc + 1), bil(P + dt * dt, dt, ir, dr, ib, db)));
      acc = NA(acc, NM((double)__ldg(Wc + 2), bil(P + 2 * dt * dt, dt, ig, dg, ib, db)));
      acc = NA(acc, (double)__ldg(lb + (long long)b * 3 + c));
      out[((long long)b * 3 + c) * plane + o] = (float)acc;
    }
  }
}

__global__ void combine_kernel(const float* __restrict__ base, const float* __restrict__ fs,
                               float* __restrict__ out, int batch, long long plane, int k) {
  const long long total = (long long)batch * plane;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(e / plane);
    const long long o = e - (long long)b * plane;
    for (int c = 0; c < 3; ++c) {
      float s = __ldg(fs + ((long long)b * k + c) * plane + o);
      for (int j = c + 3; j < k; j += 3) s = __fadd_rn(s, __ldg(fs + ((long long)b * k + j) * plane + o));
      out[((long long)b * 3 + c) * plane + o] = __fadd_rn(__ldg(base + ((long long)b * 3 + c) * plane + o), s);
    }
  }
}

// _gather3 (transform.py:110-120): bilinear over (r, g) on slab ib, f64
__device__ __forceinline__ double gather3(const float* __restrict__ cube, int d, int ir, int ig, int ib,
                                          double dr, double dg) {
  const double v00 = (double)__ldg(cube + ((long long)ir * d + ig) * d + ib);
  const double v10 = (double)__ldg(cube + ((long long)(ir + 1) * d + ig) * d + ib);
  const double v01 = (double)__ldg(cube + ((long long)ir * d + ig + 1) * d + ib);
  const double v11 = (double)__ldg(cube + ((long long)(ir + 1) * d + ig + 1) * d + ib);
  const double er = NS(1.0, dr), eg = NS(1.0, dg);
  double out = NM(v00, NM(er, eg));
  out = NA(out, NM(v10, NM(dr, eg)));
  out = NA(out, NM(v01, NM(er, dg)));
  return NA(out, NM(v11, NM(dr, dg)));
}

__global__ void lut3d_kernel(const float* __restrict__ rgb, float* __restrict__ out, int batch, int h,
                             int w, const float* __restrict__ cubes, int d) {
  const long long plane = (long long)h * w;
  const long long total = (long long)batch * plane;
  const long long cube_n = (long long)d * d * d;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(e / plane);
    const long long o = e - (long long)b * plane;
    const float* X = rgb + (long long)b * 3 * plane;
    int ir, ig, ib;
    double dr, dg, db;
    bracket_arr(__ldg(X + o), d, ir, dr);
    bracket_arr(__ldg(X + plane + o), d, ig, dg);
    bracket_arr(__ldg(X + 2 * plane + o), d, ib, db);
    for (int c = 0; c < 3; ++c) {
      const float* cube = cubes + ((long long)b * 3 + c) * cube_n;
      const double low = gather3(cube, d, ir, ig, ib, dr, dg);
      const double high = gather3(cube, d, ir, ig, ib + 1, dr, dg);
      double acc = NM(low, NS(1.0, db));
      acc = NA(acc, NM(high, db));
      out[((long long)b * 3 + c) * plane + o] = (float)acc;
    }
  }
}

static int grid_for(long long total) {
  long long g = (total + 255) / 256;
  const long long cap = 148LL * 16;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

cudaError_t launch_slice(const float* rgb, float* fs, int batch, int h, int w, int y0, int h_total,
                         const float* gp, const float* gw, const float* gb, int k, int ds,
                         cudaStream_t st) {
  const long long total = (long long)batch * h * w;
  if (total == 0) return cudaSuccess;
  slice_kernel<<<grid_for(total), 256, 0, st>>>(rgb, fs, batch, h, w, y0, h_total, gp, gw, gb, k, ds);
  return cudaGetLastError();
}

cudaError_t launch_lut2d(const float* rgb, float* out, int batch, int h, int w, const float* lp,
                         const float* lw, const float* lb, int dt, cudaStream_t st) {
  const long long total = (long long)batch * h * w;
  if (total == 0) return cudaSuccess;
  lut2d_kernel<<<grid_for(total), 256, 0, st>>>(rgb, out, batch, h, w, lp, lw, lb, dt);
  return cudaGetLastError();
}

cudaError_t launch_combine(const float* base, const float* fs, float* out, int batch, int h, int w,
                           int k, cudaStream_t st) {
  const long long total = (long long)batch * h * w;
  if (total == 0) return cudaSuccess;
  combine_kernel<<<grid_for(total), 256, 0, st>>>(base, fs, out, batch, (long long)h * w, k);
  return cudaGetLastError();
}

cudaError_t launch_lut3d(const float* rgb, float* out, int batch, int h, int w, const float* cubes,
                         int d, cudaStream_t st) {
  const long long total = (long long)batch * h * w;
  if (total == 0) return cudaSuccess;
  lut3d_kernel<<<grid_for(total), 256, 0, st>>>(rgb, out, batch, h, w, cubes, d);
  return cudaGetLastError();
}

// ---- analysis.occurrence_stats (analysis.py:109-122): corner-touch histogram ----
// Every pixel touches the 8 corners of its bracketing cell (left indices of
// interp.bracket_array per channel).  Counts are exact integers: a per-CTA
// shared-memory int32 histogram (d^3 <= kOccSmemMax entries), flushed once to
// the global u64 cube; larger cubes count straight into global memory.  Lane l
// of a warp walks pixels span + l*kOccRun + j (j < kOccRun), so the 32 lanes
// of one atomic instruction sit kOccRun pixels apart and rarely hit the same
// address (shared atomics serialize same-address lanes); a lane's consecutive
// pixels share 32-byte sectors through L1.
constexpr int kOccRun = 32;
constexpr int kOccSmemMax = 48 * 1024;  // int32 entries (192 KB)

__device__ __forceinline__ int left_index(float p, int d) {
  p = fminf(fmaxf(p, 0.0f), 1.0f);
  return (int)fminf(floorf(__fmul_rn(p, (float)(d - 1))), (float)(d - 2));
}

__global__ void occurrence_kernel(const float* __restrict__ rgb, int batch, long long plane, int d,
                                  unsigned long long* __restrict__ cube, int use_smem) {
  extern __shared__ int hist[];
  const int n3 = d * d * d;
  if (use_smem) {
    for (int i = threadIdx.x; i < n3; i += blockDim.x) hist[i] = 0;
    __syncthreads();
  }
  const long long total = (long long)batch * plane;
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const long long span = 32LL * kOccRun;
  for (long long s = (blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5)) * span; s < total;
       s += warps * span) {
    for (int j = 0; j < kOccRun; ++j) {
      const long long e = s + (long long)lane * kOccRun + j;
      if (e >= total) break;
      const long long b = e / plane, o = e - b * plane;
      const float* X = rgb + b * 3 * plane + o;
      const int ir = left_index(__ldg(X), d), ig = left_index(__ldg(X + plane), d),
                ib = left_index(__ldg(X + 2 * plane), d);
      const int base = (ir * d + ig) * d + ib;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int idx = base + ((c >> 2) * d + ((c >> 1) & 1)) * d + (c & 1);
        if (use_smem) atomicAdd(&hist[idx], 1);
        else atomicAdd(&cube[idx], 1ull);
      }
    }
  }
  if (use_smem) {
    __syncthreads();
    for (int i = threadIdx.x; i < n3; i += blockDim.x)
      if (hist[i]) atomicAdd(&cube[i], (unsigned long long)hist[i]);
  }
}

cudaError_t launch_occurrence(const float* rgb, int batch, int h, int w, int d, unsigned long long* cube,
                              cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(cube, 0, sizeof(unsigned long long) * d * d * d, st);
  if (e != cudaSuccess) return e;
  const long long total = (long long)batch * h * w;
  if (total == 0) return cudaSuccess;
  const int n3 = d * d * d;
  const int use_smem = n3 <= kOccSmemMax;
  const size_t smem = use_smem ? (size_t)n3 * 4 : 0;
  if (smem > 48 * 1024) {
    e = cudaFuncSetAttribute(occurrence_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long spans = (total + 32LL * kOccRun * 16 - 1) / (32LL * kOccRun * 16);
  const int grid = (int)(spans < sms ? (spans < 1 ? 1 : spans) : sms);
  occurrence_kernel<<<grid, 512, smem, st>>>(rgb, batch, (long long)h * w, d, cube, use_smem);
  return cudaGetLastError();
}

}  // namespace svdlut
