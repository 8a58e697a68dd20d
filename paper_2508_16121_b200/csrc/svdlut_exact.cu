// svdlut_exact.cu — K2x: f64 op-for-op restatement of the reference kernel
// (transform.py:215-300) whose output is bitwise equal to fused_enhance, plus
// the index-dump kernel used by the bit-exact cell-selection test.
//
// Every product / sum uses __dmul_rn / __dadd_rn so nvcc cannot contract
// into DFMA (the numba reference has no FMA); the left-to-right sum order of
// the Python expressions is kept.  Tables are read through the read-only
// path (≈60 KB per image, L1/L2 resident).  Any d_t, d_s >= 2 and K % 3 == 0.
#include "svdlut_common.cuh"
#include "svdlut_internal.h"

namespace svdlut {

#define DM __dmul_rn
#define DA __dadd_rn
#define DS __dsub_rn

// interp.py:35-45 in f64 (p is an f32 sample promoted to f64).
__device__ __forceinline__ void bracket_f64(double p, int d, int& i, double& delta) {
  // interp.py:37-40 (strict compares); a NaN, which the reference's Image
  // rejects before any compute, is taken as 0 so the cell index stays in range
  if (!(p >= 0.0)) {  // p < 0 or NaN
    p = 0.0;
  } else if (p > 1.0) {
    p = 1.0;
  }
  const double t = DM(p, (double)(d - 1));
  int ii = (int)t;  // trunc == floor for t >= 0
  if (ii > d - 2) ii = d - 2;
  i = ii;
  delta = DS(t, (double)ii);
}

// ((w00*P00 + w10*P10) + w01*P01) + w11*P11, all f64, no FMA.
__device__ __forceinline__ double blend4(double w00, double w10, double w01, double w11,
                                         const float* __restrict__ pl, int stride, int a,
                                         int b) {
  const double p00 = (double)__ldg(pl + a * stride + b);
  const double p10 = (double)__ldg(pl + (a + 1) * stride + b);
  const double p01 = (double)__ldg(pl + a * stride + b + 1);
  const double p11 = (double)__ldg(pl + (a + 1) * stride + b + 1);
  return DA(DA(DA(DM(w00, p00), DM(w10, p10)), DM(w01, p01)), DM(w11, p11));
}

__global__ void fused_exact_kernel(const float* __restrict__ rgb, float* __restrict__ out,
                                   int batch, int h, int w, int y0, int h_total,
                                   const float* __restrict__ lp, const float* __restrict__ lw,
                                   const float* __restrict__ lb, int dt,
                                   const float* __restrict__ gp, const float* __restrict__ gw,
                                   const float* __restrict__ gb, int k, int ds) {
  const long long plane = (long long)h * w;
  const long long total = (long long)batch * plane;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(e / plane);
    const long long o = e - (long long)b * plane;
    const int y = (int)(o / w);
    const int x = (int)(o - (long long)y * w);
    const float* X = rgb + (long long)b * 3 * plane;
    const float* P = lp + (long long)b * 9 * dt * dt;
    const float* LW = lw + b * 9;
    const float* LB = lb + b * 3;
    const float* G = gp + (long long)b * k * 3 * ds * ds;
    const float* GW = gw + (long long)b * k * 3;
    const float* GB = gb + (long long)b * k;

    const SpatialBr cy = spatial_bracket(y0 + y, h_total, ds);
    const SpatialBr cx = spatial_bracket(x, w, ds);
    const int jy = cy.i, jx = cx.i;
    const double ey = (double)cy.d, ex = (double)cx.d;

    const double r = (double)X[o], g = (double)X[plane + o], bl = (double)X[2 * plane + o];
    int ir, ig, ib;
    double dr, dg, db;
    bracket_f64(r, dt, ir, dr);
    bracket_f64(g, dt, ig, dg);
    bracket_f64(bl, dt, ib, db);
    const int dd = dt * dt;
    double a[3];
    double w00 = DM(DS(1.0, dr), DS(1.0, dg)), w10 = DM(dr, DS(1.0, dg));
    double w01 = DM(DS(1.0, dr), dg), w11 = DM(dr, dg);
    for (int c = 0; c < 3; ++c)
      a[c] = DM((double)LW[c * 3 + 0], blend4(w00, w10, w01, w11, P + (c * 3 + 0) * dd, dt, ir, ig));
    w00 = DM(DS(1.0, dr), DS(1.0, db));
    w10 = DM(dr, DS(1.0, db));
    w01 = DM(DS(1.0, dr), db);
    w11 = DM(dr, db);
    for (int c = 0; c < 3; ++c)
      a[c] = DA(a[c], DM((double)LW[c * 3 + 1], blend4(w00, w10, w01, w11, P + (c * 3 + 1) * dd, dt, ir, ib)));
    w00 = DM(DS(1.0, dg), DS(1.0, db));
    w10 = DM(dg, DS(1.0, db));
    w01 = DM(DS(1.0, dg), db);
    w11 = DM(dg, db);
    for (int c = 0; c < 3; ++c)
      a[c] = DA(a[c], DM((double)LW[c * 3 + 2], blend4(w00, w10, w01, w11, P + (c * 3 + 2) * dd, dt, ig, ib)));
    for (int c = 0; c < 3; ++c) a[c] = DA(a[c], (double)LB[c]);

    int jc3[3];
    double ec3[3];
    bracket_f64(r, ds, jc3[0], ec3[0]);
    bracket_f64(g, ds, jc3[1], ec3[1]);
    bracket_f64(bl, ds, jc3[2], ec3[2]);
    const double q00 = DM(DS(1.0, ex), DS(1.0, ey)), q10 = DM(ex, DS(1.0, ey));
    const double q01 = DM(DS(1.0, ex), ey), q11 = DM(ex, ey);
    const int sd = ds * ds;
    for (int kk = 0; kk < k; ++kk) {
      const int ch = kk % 3;
      const int jc = jc3[ch];
      const double ec = ec3[ch];
      const float* Gk = G + kk * 3 * sd;
      double s = DM((double)GW[kk * 3 + 0], blend4(q00, q10, q01, q11, Gk, ds, jx, jy));
      double u0 = DM(DS(1.0, ex), DS(1.0, ec)), u1 = DM(ex, DS(1.0, ec));
      double u2 = DM(DS(1.0, ex), ec), u3 = DM(ex, ec);
      s = DA(s, DM((double)GW[kk * 3 + 1], blend4(u0, u1, u2, u3, Gk + sd, ds, jx, jc)));
      u0 = DM(DS(1.0, ey), DS(1.0, ec));
      u1 = DM(ey, DS(1.0, ec));
      u2 = DM(DS(1.0, ey), ec);
      u3 = DM(ey, ec);
      s = DA(s, DM((double)GW[kk * 3 + 2], blend4(u0, u1, u2, u3, Gk + 2 * sd, ds, jy, jc)));
      s = DA(s, (double)GB[kk]);
      a[ch] = DA(a[ch], s);
    }
    float* O = out + (long long)b * 3 * plane;
    O[o] = (float)a[0];
    O[plane + o] = (float)a[1];
    O[2 * plane + o] = (float)a[2];
  }
}

// Cell selection as the fast kernel computes it (svdlut_common.cuh helpers:
// color_bracket and the table-free col_bracket / row_bracket).
__global__ void indices_kernel(const float* __restrict__ rgb, int batch, int h, int w, int y0,
                               int h_total, int dt, int ds, double rcp_w, double rcp_h,
                               int32_t* __restrict__ idx) {
  const long long plane = (long long)h * w;
  const long long total = (long long)batch * plane;
  const float tdm1 = (float)(dt - 1), tdm2 = (float)(dt - 2);
  const float sdm1 = (float)(ds - 1), sdm2 = (float)(ds - 2);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(e / plane);
    const long long o = e - (long long)b * plane;
    const int y = (int)(o / w);
    const int x = (int)(o - (long long)y * w);
    const float* X = rgb + (long long)b * 3 * plane;
    int32_t* I = idx + (long long)b * 8 * plane;
    for (int c = 0; c < 3; ++c) {
      const float q = clamp01(X[c * plane + o]);
      int i;
      float d;
      color_bracket(q, tdm1, tdm2, i, d);
      I[c * plane + o] = i;
      color_bracket(q, sdm1, sdm2, i, d);
      I[(3 + c) * plane + o] = i;
    }
    float ex, ey;
    I[6 * plane + o] = (int32_t)(col_bracket(x, rcp_w, sdm1, sdm2, ex) - 0x4B000000u);
    I[7 * plane + o] = (int32_t)(row_bracket(y0 + y, rcp_h, sdm1, sdm2, ey) - 0x4B000000u);
  }
}

static int grid_for(long long total, int threads) {
  long long g = (total + threads - 1) / threads;
  if (g > 148LL * 16) g = 148LL * 16;
  if (g < 1) g = 1;
  return (int)g;
}

cudaError_t launch_fused_exact(const float* rgb, float* out, int batch, int h, int w, int y0,
                               int h_total, const float* lp, const float* lw, const float* lb,
                               int dt, const float* gp, const float* gw, const float* gb, int k,
                               int ds, cudaStream_t st) {
  const long long total = (long long)batch * h * w;
  if (total == 0) return cudaSuccess;
  fused_exact_kernel<<<grid_for(total, 256), 256, 0, st>>>(rgb, out, batch, h, w, y0, h_total, lp,
                                                           lw, lb, dt, gp, gw, gb, k, ds);
  return cudaGetLastError();
}

cudaError_t launch_indices(const float* rgb, int batch, int h, int w, int y0, int h_total,
                           int dt, int ds, int32_t* idx, cudaStream_t st) {
  const long long total = (long long)batch * h * w;
  if (total == 0) return cudaSuccess;
  indices_kernel<<<grid_for(total, 256), 256, 0, st>>>(rgb, batch, h, w, y0, h_total, dt, ds,
                                                       1.0 / (double)(w - 1),
                                                       1.0 / (double)(h_total - 1), idx);
  return cudaGetLastError();
}

}  // namespace svdlut
