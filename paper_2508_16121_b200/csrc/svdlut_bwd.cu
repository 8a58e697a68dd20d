// svdlut_bwd.cu — K3/K4: backward of the fused apply and of the LUT
// reconstruction.  The reference has no backward;
// the math follows SURVEY.md Appendix B and is pinned against the f64 oracle
// (oracle_fused_bwd) and finite differences.
//
// Structure
//   pack_vertex_kernel  per image: weight-folded LUT vertices (channel-packed
//                       float4) and per-channel merged grid planes — the
//                       tables the input gradient needs.
//   fused_bwd_kernel    persistent CTA per SM.  Per pixel: recompute the
//                       brackets, gx from the vertex tables, and scatter-add
//                       gY·w_uv into UNWEIGHTED per-CTA shared-memory
//                       accumulators E (LUT: [pair][i][j][c], grids:
//                       [plane][c][a][b]).  Consecutive pixels of a lane that
//                       hit the same cell are merged in registers first
//                       (run-length aggregation), so smooth images issue far
//                       fewer shared atomics than pixels × corners.  At the
//                       end of each image phase the CTA flushes its non-zero
//                       accumulators to a global E with one atomic each.
//   finalize_kernel     dlut = lw·E, dlw = <T, E>, dgrid[k,q] = gw[k,q]·E[q,k%3],
//                       dgw = <G, E>, dlb / dgb from the per-image gY sums.
//   reconstruct_bwd     dU = dT·Vtᵀ·diag S, dS = diag(Uᵀ dT Vtᵀ), dVt = diag S·Uᵀ·dT.
#include <cstdint>
#include "svdlut_common.cuh"
#include "svdlut_internal.h"

namespace svdlut {

constexpr int kBwdThreads = 512;
constexpr int kRun = 8;  // consecutive pixels per lane (run-length window)

struct VtxLayout {
  int dt, ds;
  int lut_off;   // float4 [3][dt][dt]
  int xy_off;    // float4 [ds][ds]
  int xc_off;    // float  [3][ds][ds]
  int yc_off;    // float  [3][ds][ds]
  int total;     // floats (multiple of 4)
  __host__ __device__ static VtxLayout make(int dt, int ds) {
    VtxLayout L;
    L.dt = dt;
    L.ds = ds;
    L.lut_off = 0;
    L.xy_off = 3 * dt * dt * 4;
    L.xc_off = L.xy_off + ds * ds * 4;
    L.yc_off = L.xc_off + 3 * ds * ds;
    L.total = (L.yc_off + 3 * ds * ds + 3) & ~3;
    return L;
  }
};
// E accumulators share the vertex layout (lut [p][i][j][c(4)], xy [a][b][c(4)], xc/yc [c][a][b]).

struct BwdWs {
  float* vtx;     // batch * VtxLayout.total
  float* E;       // batch * VtxLayout.total (global accumulators)
  float* gsum;    // batch * 4 (sum of gY per channel)
  SpatialBr* col;
  SpatialBr* row;
};

static size_t rup(size_t v) { return (v + 255) / 256 * 256; }

size_t bwd_workspace_bytes(int batch, int h, int w, int dt, int ds, int k) {
  (void)k;
  const VtxLayout L = VtxLayout::make(dt, ds);
  return 2 * rup((size_t)batch * L.total * 4) + rup((size_t)batch * 16) +
         rup((size_t)w * sizeof(SpatialBr)) + rup((size_t)h * sizeof(SpatialBr)) + 256;
}

static BwdWs carve(void* ws, int batch, int h, int w, const VtxLayout& L) {
  char* p = (char*)ws;
  BwdWs W;
  W.vtx = (float*)p;
  p += rup((size_t)batch * L.total * 4);
  W.E = (float*)p;
  p += rup((size_t)batch * L.total * 4);
  W.gsum = (float*)p;
  p += rup((size_t)batch * 16);
  W.col = (SpatialBr*)p;
  p += rup((size_t)w * sizeof(SpatialBr));
  W.row = (SpatialBr*)p;
  return W;
}

__global__ void pack_vertex_kernel(const float* __restrict__ lp, const float* __restrict__ lw,
                                   const float* __restrict__ gp, const float* __restrict__ gw,
                                   int k, VtxLayout L, float* __restrict__ vtx) {
  const long long b = blockIdx.y;
  const int dt = L.dt, ds = L.ds;
  const float* P = lp + b * 9LL * dt * dt;
  const float* W = lw + b * 9;
  const float* G = gp + b * (long long)k * 3 * ds * ds;
  const float* GW = gw + b * (long long)k * 3;
  float* V = vtx + b * (long long)L.total;
  const int n_lut = 3 * dt * dt, n_xy = ds * ds, n_c = 3 * ds * ds;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n_lut + n_xy + 2 * n_c;
       e += gridDim.x * blockDim.x) {
    if (e < n_lut) {
      const int p = e / (dt * dt), ij = e - p * dt * dt;
      float4 v;
      v.x = W[0 * 3 + p] * P[(0 * 3 + p) * dt * dt + ij];
      v.y = W[1 * 3 + p] * P[(1 * 3 + p) * dt * dt + ij];
      v.z = W[2 * 3 + p] * P[(2 * 3 + p) * dt * dt + ij];
      v.w = 0.f;
      reinterpret_cast<float4*>(V + L.lut_off)[e] = v;
    } else if (e < n_lut + n_xy) {
      const int ab = e - n_lut;
      float acc[3] = {0.f, 0.f, 0.f};
      for (int kk = 0; kk < k; ++kk) acc[kk % 3] += GW[kk * 3 + 0] * G[(kk * 3 + 0) * ds * ds + ab];
      reinterpret_cast<float4*>(V + L.xy_off)[ab] = make_float4(acc[0], acc[1], acc[2], 0.f);
    } else {
      int r = e - n_lut - n_xy;
      const int q = r < n_c ? 1 : 2;
      if (r >= n_c) r -= n_c;
      const int c = r / (ds * ds), ab = r - c * ds * ds;
      float acc = 0.f;
      for (int kk = c; kk < k; kk += 3) acc += GW[kk * 3 + q] * G[(kk * 3 + q) * ds * ds + ab];
      V[(q == 1 ? L.xc_off : L.yc_off) + r] = acc;
    }
  }
}

// Per-lane run-length accumulator for one bilinear term with C channels.
template <int C>
struct RunAcc {
  int key;           // packed cell id, -1 = empty
  float v[4][C];     // corner accumulators (00, 10, 01, 11)
};

struct BwdParams {
  const float* rgb;
  const float* gy;
  float* gx;
  int h, w;
  VtxLayout L;
  const float* vtx;
  float* E;
  float* gsum;
  const SpatialBr* col;
  const SpatialBr* row;
  int rpr;             // runs per row (row split into kRun-pixel runs)
  long long per_img;   // h * rpr
  long long total;
};

// Flush a run: 4 corners x C channels of shared atomics.  C == 3 tables are
// float4-strided ([a][b][4]); C == 1 tables are scalar ([a][b]).
template <int C>
__device__ __forceinline__ void flush(RunAcc<C>& R, float* base, int stride) {
  if (R.key < 0) return;
  constexpr int S = C == 3 ? 4 : 1;
  const int a = R.key >> 16, b = R.key & 0xffff;
  float* p00 = base + (a * stride + b) * S;
  float* p10 = base + ((a + 1) * stride + b) * S;
  float* p01 = base + (a * stride + b + 1) * S;
  float* p11 = base + ((a + 1) * stride + b + 1) * S;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    atomicAdd(p00 + c, R.v[0][c]);
    atomicAdd(p10 + c, R.v[1][c]);
    atomicAdd(p01 + c, R.v[2][c]);
    atomicAdd(p11 + c, R.v[3][c]);
  }
  R.key = -1;
}

template <int C>
__device__ __forceinline__ void run_add(RunAcc<C>& R, int key, float* base, int stride,
                                        const float* g, float a, float b) {
  if (R.key != key) {
    flush<C>(R, base, stride);
    R.key = key;
#pragma unroll
    for (int c = 0; c < C; ++c) R.v[0][c] = R.v[1][c] = R.v[2][c] = R.v[3][c] = 0.f;
  }
  const float w00 = (1.f - a) * (1.f - b), w10 = a * (1.f - b), w01 = (1.f - a) * b, w11 = a * b;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    R.v[0][c] = __fmaf_rn(g[c], w00, R.v[0][c]);
    R.v[1][c] = __fmaf_rn(g[c], w10, R.v[1][c]);
    R.v[2][c] = __fmaf_rn(g[c], w01, R.v[2][c]);
    R.v[3][c] = __fmaf_rn(g[c], w11, R.v[3][c]);
  }
}

__global__ void __launch_bounds__(kBwdThreads, 1) fused_bwd_kernel(BwdParams p) {
  extern __shared__ __align__(16) float sm[];
  const VtxLayout& L = p.L;
  float* V = sm;             // vertex tables
  float* Es = sm + L.total;  // accumulators
  const int dt = L.dt, ds = L.ds;
  const float tdm1 = (float)(dt - 1), tdm2 = (float)(dt - 2);
  const float sdm1 = (float)(ds - 1), sdm2 = (float)(ds - 2);
  const long long c_begin = (long long)blockIdx.x * p.total / gridDim.x;
  const long long c_end = (long long)(blockIdx.x + 1) * p.total / gridDim.x;
  __shared__ float gs[3];
  const int pa[3] = {0, 0, 1}, pb[3] = {1, 2, 2};

  long long c = c_begin;
  while (c < c_end) {
    const int b = (int)(c / p.per_img);
    const long long phase_end = min(c_end, (long long)(b + 1) * p.per_img);
    __syncthreads();
    const float4* src = reinterpret_cast<const float4*>(p.vtx + (long long)b * L.total);
    for (int i = threadIdx.x; i < L.total / 4; i += blockDim.x) {
      reinterpret_cast<float4*>(V)[i] = __ldg(src + i);
      reinterpret_cast<float4*>(Es)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (threadIdx.x < 3) gs[threadIdx.x] = 0.f;
    __syncthreads();

    const long long plane = (long long)p.h * p.w;
    const float* X = p.rgb + (long long)b * 3 * plane;
    const float* GY = p.gy + (long long)b * 3 * plane;
    float* GX = p.gx ? p.gx + (long long)b * 3 * plane : nullptr;
    float gsum_l[3] = {0.f, 0.f, 0.f};

    for (long long t = c + threadIdx.x; t < phase_end; t += blockDim.x) {
      const long long rem = t - (long long)b * p.per_img;
      const int y = (int)(rem / p.rpr);
      const int x0 = (int)(rem - (long long)y * p.rpr) * kRun;
      const SpatialBr rb = p.row[y];
      const int jy = rb.i;
      const float ey = rb.d;
      RunAcc<3> Rl[3], Rxy;
      RunAcc<1> Rxc[3], Ryc[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        Rl[q].key = -1;
        Rxc[q].key = -1;
        Ryc[q].key = -1;
      }
      Rxy.key = -1;
      for (int u = 0; u < kRun; ++u) {
        const int x = x0 + u;
        if (x >= p.w) break;
        const long long o = (long long)y * p.w + x;
        float Xv[3], g[3], q[3];
        int it[3], is[3];
        float et[3], es[3];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          Xv[ch] = X[ch * plane + o];
          g[ch] = GY[ch * plane + o];
          gsum_l[ch] += g[ch];
          q[ch] = clamp01(Xv[ch]);
          color_bracket(q[ch], tdm1, tdm2, it[ch], et[ch]);
          color_bracket(q[ch], sdm1, sdm2, is[ch], es[ch]);
        }
        float gxa[3] = {0.f, 0.f, 0.f}, gxs[3] = {0.f, 0.f, 0.f};
#pragma unroll
        for (int pr = 0; pr < 3; ++pr) {
          const int A = pa[pr], Bc = pb[pr];
          const int ia = it[A], ib = it[Bc];
          const float da = et[A], db = et[Bc];
          const float4* T4 = reinterpret_cast<const float4*>(V + L.lut_off) + pr * dt * dt;
          const float4 v00 = T4[ia * dt + ib], v10 = T4[(ia + 1) * dt + ib];
          const float4 v01 = T4[ia * dt + ib + 1], v11 = T4[(ia + 1) * dt + ib + 1];
          // sum_c g_c * dv_c/da and dv_c/db
          const float d0a = (1.f - db) * (v10.x - v00.x) + db * (v11.x - v01.x);
          const float d1a = (1.f - db) * (v10.y - v00.y) + db * (v11.y - v01.y);
          const float d2a = (1.f - db) * (v10.z - v00.z) + db * (v11.z - v01.z);
          const float d0b = (1.f - da) * (v01.x - v00.x) + da * (v11.x - v10.x);
          const float d1b = (1.f - da) * (v01.y - v00.y) + da * (v11.y - v10.y);
          const float d2b = (1.f - da) * (v01.z - v00.z) + da * (v11.z - v10.z);
          gxa[A] += g[0] * d0a + g[1] * d1a + g[2] * d2a;
          gxa[Bc] += g[0] * d0b + g[1] * d1b + g[2] * d2b;
          run_add<3>(Rl[pr], (ia << 16) | ib, Es + L.lut_off + pr * dt * dt * 4, dt, g, da, db);
        }
        const SpatialBr cb = p.col[x];
        const int jx = cb.i;
        const float ex = cb.d;
        run_add<3>(Rxy, (jx << 16) | jy, Es + L.xy_off, ds, g, ex, ey);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          const int jc = is[ch];
          const float ec = es[ch];
          const float* Pxc = V + L.xc_off + ch * ds * ds;
          const float* Pyc = V + L.yc_off + ch * ds * ds;
          const float x00 = Pxc[jx * ds + jc], x10 = Pxc[(jx + 1) * ds + jc];
          const float x01 = Pxc[jx * ds + jc + 1], x11 = Pxc[(jx + 1) * ds + jc + 1];
          const float y00 = Pyc[jy * ds + jc], y10 = Pyc[(jy + 1) * ds + jc];
          const float y01 = Pyc[jy * ds + jc + 1], y11 = Pyc[(jy + 1) * ds + jc + 1];
          gxs[ch] += g[ch] * ((1.f - ex) * (x01 - x00) + ex * (x11 - x10) +
                              (1.f - ey) * (y01 - y00) + ey * (y11 - y10));
          const float gc[1] = {g[ch]};
          run_add<1>(Rxc[ch], (jx << 16) | jc, Es + L.xc_off + ch * ds * ds, ds, gc, ex, ec);
          run_add<1>(Ryc[ch], (jy << 16) | jc, Es + L.yc_off + ch * ds * ds, ds, gc, ey, ec);
        }
        if (GX) {
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            const float m = (Xv[ch] < 0.f || Xv[ch] > 1.f) ? 0.f : 1.f;  // strict clamp
            GX[ch * plane + o] = m * (gxa[ch] * tdm1 + gxs[ch] * sdm1);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        flush<3>(Rl[q], Es + L.lut_off + q * dt * dt * 4, dt);
        flush<1>(Rxc[q], Es + L.xc_off + q * ds * ds, ds);
        flush<1>(Ryc[q], Es + L.yc_off + q * ds * ds, ds);
      }
      flush<3>(Rxy, Es + L.xy_off, ds);
    }
    // per-image gY sums
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      float v = gsum_l[ch];
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if ((threadIdx.x & 31) == 0) atomicAdd(&gs[ch], v);
    }
    __syncthreads();
    float* Eg = p.E + (long long)b * L.total;
    for (int i = threadIdx.x; i < L.total; i += blockDim.x) {
      const float v = Es[i];
      if (v != 0.f) atomicAdd(Eg + i, v);
    }
    if (threadIdx.x < 3) atomicAdd(p.gsum + b * 4 + threadIdx.x, gs[threadIdx.x]);
    c = phase_end;
  }
}

// Converts the unweighted accumulators into parameter gradients.  grid.y = image.
__global__ void finalize_kernel(const float* __restrict__ lp, const float* __restrict__ lw,
                                const float* __restrict__ gp, const float* __restrict__ gw, int k,
                                VtxLayout L, const float* __restrict__ E,
                                const float* __restrict__ gsum, float* dlp, float* dlw,
                                float* dlb, float* dgp, float* dgw, float* dgb) {
  const long long b = blockIdx.y;
  const int dt = L.dt, ds = L.ds;
  const float* Eb = E + b * (long long)L.total;
  const int task = blockIdx.x;  // 0..8: LUT planes (c,p); 9..: grid planes (kk, q)
  __shared__ double red[32];
  double acc = 0.0;
  if (task < 9) {
    const int c = task / 3, pr = task - c * 3;
    const float* T = lp + (b * 9 + task) * (long long)dt * dt;
    const float w = lw[b * 9 + task];
    float* D = dlp + (b * 9 + task) * (long long)dt * dt;
    for (int ij = threadIdx.x; ij < dt * dt; ij += blockDim.x) {
      const float e = Eb[L.lut_off + (pr * dt * dt + ij) * 4 + c];
      D[ij] = w * e;
      acc += (double)T[ij] * (double)e;
    }
  } else {
    const int kq = task - 9;
    const int kk = kq / 3, q = kq - kk * 3, c = kk % 3;
    const float* Gp = gp + (b * k * 3 + kq) * (long long)ds * ds;
    const float w = gw[b * k * 3 + kq];
    float* D = dgp + (b * k * 3 + kq) * (long long)ds * ds;
    for (int ab = threadIdx.x; ab < ds * ds; ab += blockDim.x) {
      float e;
      if (q == 0) e = Eb[L.xy_off + ab * 4 + c];
      else e = Eb[(q == 1 ? L.xc_off : L.yc_off) + c * ds * ds + ab];
      D[ab] = w * e;
      acc += (double)Gp[ab] * (double)e;
    }
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    if (task < 9) {
      dlw[b * 9 + task] = (float)s;
      if (task % 3 == 0) dlb[b * 3 + task / 3] = gsum[b * 4 + task / 3];
    } else {
      const int kq = task - 9;
      dgw[b * k * 3 + kq] = (float)s;
      if (kq % 3 == 0) dgb[b * k + kq / 3] = gsum[b * 4 + (kq / 3) % 3];
    }
  }
}

cudaError_t launch_fused_bwd(const float* rgb, const float* gy, int batch, int h, int w, int y0,
                             int h_total, const float* lp, const float* lw, int dt,
                             const float* gp, const float* gw, int k, int ds, float* gx,
                             float* dlp, float* dlw, float* dlb, float* dgp, float* dgw,
                             float* dgb, void* ws, size_t ws_bytes, cudaStream_t st) {
  (void)ws_bytes;
  const VtxLayout L = VtxLayout::make(dt, ds);
  const size_t smem = (size_t)L.total * 4 * 2;
  if (smem > (size_t)fwd_max_smem_bytes()) return cudaErrorInvalidValue;
  BwdWs W = carve(ws, batch, h, w, L);
  cudaError_t e;
  {
    const int items = 3 * dt * dt + 7 * ds * ds;
    dim3 grid((items + 255) / 256, batch);
    pack_vertex_kernel<<<grid, 256, 0, st>>>(lp, lw, gp, gw, k, L, W.vtx);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if ((e = cudaMemsetAsync(W.E, 0, (size_t)batch * L.total * 4, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(W.gsum, 0, (size_t)batch * 16, st)) != cudaSuccess) return e;
  if ((e = launch_spatial(w, h, y0, h_total, ds, W.col, W.row, st)) != cudaSuccess) return e;
  BwdParams p;
  p.rgb = rgb;
  p.gy = gy;
  p.gx = gx;
  p.h = h;
  p.w = w;
  p.L = L;
  p.vtx = W.vtx;
  p.E = W.E;
  p.gsum = W.gsum;
  p.col = W.col;
  p.row = W.row;
  p.rpr = (w + kRun - 1) / kRun;
  p.per_img = (long long)h * p.rpr;
  p.total = (long long)batch * p.per_img;
  if (p.total > 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    long long grid = sms;
    if (grid > (p.total + kBwdThreads - 1) / kBwdThreads) grid = (p.total + kBwdThreads - 1) / kBwdThreads;
    if (grid < 1) grid = 1;
    if ((e = cudaFuncSetAttribute(fused_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem)) != cudaSuccess)
      return e;
    fused_bwd_kernel<<<(int)grid, kBwdThreads, smem, st>>>(p);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  dim3 fg(9 + 3 * k, batch);
  finalize_kernel<<<fg, 256, 0, st>>>(lp, lw, gp, gw, k, L, W.E, W.gsum, dlp, dlw, dlb, dgp, dgw,
                                      dgb);
  return cudaGetLastError();
}

// dU[i,m] = S[m] * sum_j dT[i,j] Vt[m,j]; dS[m] = sum_ij dT[i,j] U[i,m] Vt[m,j];
// dVt[m,j] = S[m] * sum_i U[i,m] dT[i,j].  One CTA per (plane, image).
__global__ void reconstruct_bwd_kernel(const float* __restrict__ u, const float* __restrict__ s,
                                       const float* __restrict__ vt,
                                       const float* __restrict__ dT, int dt, int ns,
                                       float* __restrict__ du, float* __restrict__ ds_,
                                       float* __restrict__ dvt) {
  const long long pl = (long long)blockIdx.y * 9 + blockIdx.x;
  const float* U = u + pl * dt * ns;
  const float* S = s + pl * ns;
  const float* V = vt + pl * ns * dt;
  const float* G = dT + pl * dt * dt;
  for (int e = threadIdx.x; e < dt * ns; e += blockDim.x) {
    const int i = e / ns, m = e - i * ns;
    double acc = 0.0;
    for (int j = 0; j < dt; ++j) acc += (double)G[i * dt + j] * (double)V[m * dt + j];
    du[pl * dt * ns + e] = (float)(acc * (double)S[m]);
  }
  for (int e = threadIdx.x; e < ns * dt; e += blockDim.x) {
    const int m = e / dt, j = e - m * dt;
    double acc = 0.0;
    for (int i = 0; i < dt; ++i) acc += (double)U[i * ns + m] * (double)G[i * dt + j];
    dvt[pl * ns * dt + e] = (float)(acc * (double)S[m]);
  }
  for (int m = threadIdx.x >> 5; m < ns; m += blockDim.x >> 5) {
    double acc = 0.0;
    for (int ij = threadIdx.x & 31; ij < dt * dt; ij += 32) {
      const int i = ij / dt, j = ij - i * dt;
      acc += (double)G[ij] * (double)U[i * ns + m] * (double)V[m * dt + j];
    }
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if ((threadIdx.x & 31) == 0) ds_[pl * ns + m] = (float)acc;
  }
}

cudaError_t launch_reconstruct_bwd(const float* u, const float* s, const float* vt,
                                   const float* dplanes, int batch, int dt, int ns, float* du,
                                   float* ds, float* dvt, cudaStream_t st) {
  dim3 grid(9, batch);
  reconstruct_bwd_kernel<<<grid, 256, 0, st>>>(u, s, vt, dplanes, dt, ns, du, ds, dvt);
  return cudaGetLastError();
}

}  // namespace svdlut
