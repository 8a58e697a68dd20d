// svdlut_prep.cu — table prologue kernels (K1): LUT reconstruction from SVD
// factors and weight folding / grid merging into coefficient cells.  All tiny (≈60 KB of tables per image); launched
// once per call on the caller's stream.
#include "svdlut_common.cuh"
#include "svdlut_internal.h"

namespace svdlut {

// svd.py:210-220: planes[c,p] = f32((f64(u) * f64(s)) @ f64(vt)).
// One CTA per (plane, image); each thread owns output entries.  The f64
// product u*s is exact; the n-term sum runs in index order without FMA.
__global__ void reconstruct_kernel(const float* __restrict__ u, const float* __restrict__ s,
                                   const float* __restrict__ vt, int dt, int ns,
                                   float* __restrict__ planes) {
  const int cp = blockIdx.x;  // 0..8
  const long long b = blockIdx.y;
  const float* U = u + (b * 9 + cp) * (long long)dt * ns;
  const float* S = s + (b * 9 + cp) * (long long)ns;
  const float* V = vt + (b * 9 + cp) * (long long)ns * dt;
  float* P = planes + (b * 9 + cp) * (long long)dt * dt;
  for (int e = threadIdx.x; e < dt * dt; e += blockDim.x) {
    const int i = e / dt, j = e - i * dt;
    double acc = 0.0;
    for (int m = 0; m < ns; ++m) {
      double us = __dmul_rn((double)U[i * ns + m], (double)S[m]);
      acc = __dadd_rn(acc, __dmul_rn(us, (double)V[m * dt + j]));
    }
    P[e] = (float)acc;
  }
}

// Coefficients of the bilinear form on one cell from its 4 corner values.
struct Coef {
  float a, b, c, d;
};
__device__ __forceinline__ Coef cell_coef(double p00, double p10, double p01, double p11) {
  Coef k;
  k.a = (float)p00;
  k.b = (float)(p10 - p00);
  k.c = (float)(p01 - p00);
  k.d = (float)((p11 - p10) - (p01 - p00));
  return k;
}

// One reconstructed LUT entry, identical to reconstruct_kernel's output:
// f32(sum_m (f64 U[i,m] * f64 S[m]) * f64 Vt[m,j]) in index order, no FMA.
__device__ __forceinline__ float lut_entry(const float* __restrict__ U, const float* __restrict__ S,
                                           const float* __restrict__ V, int dt, int ns, int i,
                                           int j) {
  double acc = 0.0;
  for (int m = 0; m < ns; ++m)
    acc = __dadd_rn(acc, __dmul_rn(__dmul_rn((double)U[i * ns + m], (double)S[m]), (double)V[m * dt + j]));
  return (float)acc;
}

constexpr int kPackBand = 4;  // LUT cell rows per pack block

// Packs one image's tables (layout in svdlut_common.cuh).  grid.y = image.
// The LUT planes come either from `lp` (B,3,3,d_t,d_t) or, when lp == NULL,
// straight from the SVD factors (u, s, vt, n_s) — the fused prologue that
// skips materialising the planes.
//   blocks [0, 9*nbands) one band of kPackBand cell rows of LUT plane (c, p):
//                        the band's vertex rows are reconstructed into shared
//                        memory, then channel c's 4 coefficients of each cell
//                        written into the chunk planes
//   remaining blocks     merged grid cells / vertices and padding
__global__ void pack_kernel(const float* __restrict__ lp, const float* __restrict__ fu,
                            const float* __restrict__ fs, const float* __restrict__ fvt, int ns,
                            const float* __restrict__ lw,
                            const float* __restrict__ lb, const float* __restrict__ gp,
                            const float* __restrict__ gw, const float* __restrict__ gb, int k,
                            TableLayout L, float* __restrict__ tables, int stage_factors) {
  extern __shared__ float Ts[];  // vertex rows of one LUT plane band (+ staged factors)
  // let the fused kernel that follows launch and run its prologue (it waits
  // for this grid's completion before reading the tables)
  asm volatile("griddepcontrol.launch_dependents;");
  const long long b = blockIdx.y;
  const int dt = L.dt, ds = L.ds;
  const float* W = lw + b * 9;
  const float* Bl = lb + b * 3;
  const float* G = gp + b * (long long)k * 3 * ds * ds;
  const float* GW = gw + b * (long long)k * 3;
  const float* GB = gb + b * (long long)k;
  float* T = tables + b * (long long)L.total_floats;

  const int nbands = (dt - 1 + kPackBand - 1) / kPackBand;
  if (blockIdx.x < 9 * nbands) {
    // plane (c, p), cell rows [i0, i1): vertex rows [v0, v1] staged in smem
    const int cpi = blockIdx.x / nbands, band = blockIdx.x - cpi * nbands;
    const int c = cpi / 3, p = cpi - 3 * c;
    const int i0 = band * kPackBand, i1 = min(i0 + kPackBand, dt - 1);
    const int v0 = i0, v1 = i1;
    const long long cp = b * 9 + c * 3 + p;
    const int nv = (v1 - v0 + 1) * dt;
    if (!lp && stage_factors) {
      // the band's U rows, S and all of Vt into shared memory first (one
      // round of global latency instead of one per term of every dot product),
      // then the same f64 sums in the same order
      float* Us = Ts + (kPackBand + 1) * dt;
      float* Ss = Us + (kPackBand + 1) * ns;
      float* Vs = Ss + ns;
      const float* U = fu + cp * dt * ns + (long long)v0 * ns;
      for (int e = threadIdx.x; e < (v1 - v0 + 1) * ns; e += blockDim.x) Us[e] = U[e];
      for (int e = threadIdx.x; e < ns; e += blockDim.x) Ss[e] = fs[cp * ns + e];
      for (int e = threadIdx.x; e < ns * dt; e += blockDim.x) Vs[e] = fvt[cp * ns * dt + e];
      __syncthreads();
      for (int e = threadIdx.x; e < nv; e += blockDim.x) {
        const int il = e / dt, j = e - il * dt;
        Ts[e] = lut_entry(Us, Ss, Vs, dt, ns, il, j);
      }
    } else {
      for (int e = threadIdx.x; e < nv; e += blockDim.x) {
        const int i = v0 + e / dt, j = e - (e / dt) * dt;
        if (lp) {
          Ts[e] = lp[cp * dt * dt + i * dt + j];
        } else {
          Ts[e] = lut_entry(fu + cp * dt * ns, fs + cp * ns, fvt + cp * ns * dt, dt, ns, i, j);
        }
      }
    }
    __syncthreads();
    const double w = (double)W[c * 3 + p];
    float* P0 = T + L.plane_off(p, 0);
    const int sA = coef_slot(c, 0), sB = coef_slot(c, 1), sC = coef_slot(c, 2), sD = coef_slot(c, 3);
    for (int e = threadIdx.x; e < (i1 - i0) * L.cst; e += blockDim.x) {
      const int il = e / L.cst, j = e - il * L.cst;
      const int i = i0 + il;
      double q[4] = {0.0, 0.0, 0.0, 0.0};
      if (j < dt - 1) {
        const float* R0 = Ts + (i - v0) * dt;
        const double p00 = w * R0[j], p10 = w * R0[dt + j];
        const double p01 = w * R0[j + 1], p11 = w * R0[dt + j + 1];
        q[0] = p00;                            // A
        q[1] = p10 - p00;                      // B
        q[2] = p01 - p00;                      // C
        q[3] = (p11 - p10) - (p01 - p00);      // D
      }
      const int sl[4] = {sA, sB, sC, sD};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int idx = 3 * p + (sl[t] >> 2);
        if (plane_tiled(idx) && j >= dt - 1) continue;  // tiled planes have no padding columns
        const int cell = L.cell_index(idx, i, j);
        SVDLUT_CHECK(i < dt - 1 && j < L.cst && cell < L.plane_floats / 4);
        P0[(sl[t] >> 2) * L.plane_floats + cell * 4 + (sl[t] & 3)] = (float)q[t];
      }
    }
    return;
  }

  const int n_xc = 3 * (ds - 1) * (ds - 1);
  const int n_gxy = ds * ds;  // vertices (3 floats each)
  const int n_gyc = 3 * ds * ds;
  const int n_tail = L.total_floats - (L.gyc_off + n_gyc);
  const int n_gbpad = L.plane_floats / 4;  // tiled planes: zero the positions that hold no cell
  const int total = n_xc + n_gxy + n_gyc + n_tail + n_gbpad;
  const int gb0 = 9 * nbands;
  for (int e = (blockIdx.x - gb0) * blockDim.x + threadIdx.x; e < total;
       e += (gridDim.x - gb0) * blockDim.x) {
    int r = e;
    if (r < n_xc) {  // merged xc cell (c, jx, jc)
      const int c = r / ((ds - 1) * (ds - 1));
      const int rem = r - c * (ds - 1) * (ds - 1);
      const int ja = rem / (ds - 1), jc = rem - ja * (ds - 1);
      double p00 = 0, p10 = 0, p01 = 0, p11 = 0;
      for (int kk = c; kk < k; kk += 3) {
        const float* pl = G + (kk * 3 + 1) * ds * ds;
        const double w = (double)GW[kk * 3 + 1];
        p00 += w * pl[ja * ds + jc];
        p10 += w * pl[(ja + 1) * ds + jc];
        p01 += w * pl[ja * ds + jc + 1];
        p11 += w * pl[(ja + 1) * ds + jc + 1];
      }
      const Coef q = cell_coef(p00, p10, p01, p11);
      float* dst = T + L.xc_off + r * 4;
      dst[0] = q.a;
      dst[1] = q.b;
      dst[2] = q.c;
      dst[3] = q.d;
      continue;
    }
    r -= n_xc;
    if (r < n_gxy) {  // merged xy vertex (a, b), channels packed
      double acc[3] = {0.0, 0.0, 0.0};
      for (int kk = 0; kk < k; ++kk) acc[kk % 3] += (double)GW[kk * 3 + 0] * G[(kk * 3 + 0) * ds * ds + r];
      float* dst = T + L.gxy_off + r * 3;
      dst[0] = (float)acc[0];
      dst[1] = (float)acc[1];
      dst[2] = (float)acc[2];
      if (r == n_gxy - 1)  // alignment padding up to gyc_off
        for (int t = L.gxy_off + n_gxy * 3; t < L.gyc_off; ++t) T[t] = 0.f;
      continue;
    }
    r -= n_gxy;
    if (r < n_gyc) {  // merged yc vertex (c, a, b) + channel bias
      const int c = r / (ds * ds), ab = r - c * ds * ds;
      double acc = (double)Bl[c];
      for (int kk = c; kk < k; kk += 3) acc += (double)GB[kk];
      for (int kk = c; kk < k; kk += 3) acc += (double)GW[kk * 3 + 2] * G[(kk * 3 + 2) * ds * ds + ab];
      T[L.gyc_off + r] = (float)acc;
      continue;
    }
    r -= n_gyc;
    if (r < n_tail) {
      T[L.gyc_off + n_gyc + r] = 0.f;  // tail padding
      continue;
    }
    r -= n_tail;
    {  // position r of every tiled plane: zero unless it holds a cell (i, j)
      const int tile = r >> 4, tr = (r >> 2) & 3, tc = r & 3;
      const int ti = tile / L.tiles(), tj = tile - ti * L.tiles();
      const int i = ti * 4 + tr, j = tj * 4 + tc;
      if (tile < L.tiles() * L.tiles() && i < dt - 1 && j < dt - 1) continue;
      for (int idx = 0; idx < 9; ++idx)
        if (plane_tiled(idx))
          reinterpret_cast<float4*>(T + L.plane_off(idx / 3, idx % 3))[r] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

cudaError_t launch_reconstruct(const float* u, const float* s, const float* vt, int batch, int dt,
                               int ns, float* planes, cudaStream_t st) {
  dim3 grid(9, batch);
  reconstruct_kernel<<<grid, 256, 0, st>>>(u, s, vt, dt, ns, planes);
  return cudaGetLastError();
}

cudaError_t launch_pack(const float* lp, const float* fu, const float* fs, const float* fvt, int ns,
                        const float* lw, const float* lb, const float* gp, const float* gw,
                        const float* gb, int k, const TableLayout& L, int batch, float* tables,
                        cudaStream_t st) {
  // 9 planes x row bands + enough grid blocks for one item per thread
  const int grid_items = 3 * (L.ds - 1) * (L.ds - 1) + 4 * L.ds * L.ds + 64 + L.plane_floats / 4;
  const int nbands = (L.dt - 1 + kPackBand - 1) / kPackBand;
  dim3 grid(9 * nbands + (grid_items + 255) / 256, batch);
  size_t smem = (size_t)(kPackBand + 1) * L.dt * sizeof(float);
  // factors path: stage U band rows, S and Vt too when that stays small
  const size_t fac = ((size_t)(kPackBand + 1) * ns + ns + (size_t)ns * L.dt) * sizeof(float);
  const int stage = (!lp && smem + fac <= 32 * 1024) ? 1 : 0;
  if (stage) smem += fac;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(pack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  pack_kernel<<<grid, 256, smem, st>>>(lp, fu, fs, fvt, ns, lw, lb, gp, gw, gb, k, L, tables, stage);
  return cudaGetLastError();
}


}  // namespace svdlut
