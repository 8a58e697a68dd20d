// svdlut_bwd.cu — K3/K4: backward of the fused apply and of the LUT
// reconstruction.  The reference has no backward;
// the math follows SURVEY.md Appendix B and is pinned against the f64 oracle
// (oracle_fused_bwd), itself pinned by autograd and finite differences.
//
// fused_bwd_kernel mirrors the forward kernel's structure (svdlut_fwd.cu):
// persistent CTA per SM over a contiguous row range, the same packed
// coefficient tables (BWD_PLANES chunk planes staged in shared memory by TMA,
// the others gathered through the texture path), per-row merged grid slots
// (double buffered, one CTA barrier per row), warps on 128-pixel chunks with
// lane = 4 consecutive pixels.
//   gX    from the coefficient form: d/da (A + B a + C b + D a b) = B + D b,
//         d/db = C + D a; grid slot d/dec = M' + N' ex; the strict clamp of
//         interp.py:37-40 zeroes the gradient outside [0, 1].
//   E     UNWEIGHTED scatter sums  E_lut[p][i][j][c] = sum gY_c w_ij and
//         E_grid[q][c][a][b], accumulated per CTA in shared memory as 32-bit
//         fixed point (native ATOMS.ADD; shared f32 / u64 atomics are CAS
//         loops).  Per pixel: 36 LUT atomics (3 pairs x 4 corners x 3
//         channels) and 12 into the row's xc plane; each lane issues them in
//         a lane-rotated corner x channel order, so up to twelve neighbouring
//         lanes that share a cell hit twelve different words (an ATOMS warp
//         instruction costs ~3.1 cycles conflict-free and one more per extra
//         lane on a word, tools/microbench/atomspat.cu).  The xy and yc
//         planes are derived at the row's end from the row's xc sums
//         (sum_vc wc = sum_vx wx = 1) and take the row's y weights.
//   flush to the global f32 accumulators before any fixed-point partial can
//         pass 2^31, and at the end of each image.
// finalize_kernel: dlut = lw * E, dlw = <T, E>, dgrid[k,q] = gw[k,q] * E[q][k%3],
// dgw = <G, E>, dlb / dgb from the per-image gY sums.
#include <atomic>
#include <cstdint>
#include "svdlut_common.cuh"
#include "svdlut_internal.h"

namespace svdlut {

#ifndef BWD_NW
#define BWD_NW 15
#endif
constexpr int kBwdWarps = BWD_NW;
constexpr int kBPx = 4;
constexpr uint32_t kMagic = 0x4B000000u;
#ifndef BWD_XR_COPIES
#define BWD_XR_COPIES 4
#endif
constexpr int kXRCopies = BWD_XR_COPIES;  // lane-group copies of the row's xc sums
constexpr int kLutPad = 2;  // accumulator vertices per LUT row beyond d_t
constexpr int kBwdL2Rows = 2;  // rows of L2 prefetch distance (X and gY planes)

// LUT chunk planes (bit 3*pair + chunk) staged in shared memory by TMA; the
// others are gathered through the texture path.  Only the input gradient gX
// reads them (B, C, D coefficients of the pixel's cells).
#ifndef BWD_PLANES
#define BWD_PLANES 0x3Fu
#endif
constexpr unsigned kBwdPlanes = BWD_PLANES;
constexpr int bpopc(unsigned m) { return m ? (int)(m & 1u) + bpopc(m >> 1) : 0; }
constexpr int kBwdStaged = bpopc(kBwdPlanes & 0x1FFu);

// Addressing of the chunk planes from 2^23-biased cell index bits
// (ba = kMagic + i): shared-memory byte addresses or texel indices.
struct BAddr {
  uint32_t lutK;   // smem, row-stride cell order: lutK + ba*cst16 + bb*16 + slot*plane_bytes
  uint32_t lutT;   // smem, 4x4-tiled order:      lutT + tiled(ba, bb)*16 + slot*plane_bytes
  uint32_t texR;   // texel, row-stride:          texR + ba*cst + bb + idx*ptex
  uint32_t texT;   // texel, tiled:               texT + tiled(ba, bb) + idx*ptex
  uint32_t cst, cst16, tiles, plane_bytes, ptex;
  cudaTextureObject_t tex;
};

template <int IDX>
__device__ __forceinline__ float4 bfetch(const BAddr& a, uint32_t ba, uint32_t bb) {
  constexpr bool kSmem = (kBwdPlanes >> IDX) & 1u;
  constexpr bool kTiled = plane_tiled(IDX);
  const uint32_t tcell = (((ba >> 2) * a.tiles + (bb >> 2)) << 4) + ((ba & 3u) << 2) + (bb & 3u);
  if constexpr (kSmem) {
    constexpr int kSlot = bpopc(kBwdPlanes & ((1u << IDX) - 1u));
    const uint32_t addr = (kTiled ? tcell * 16u + a.lutT : ba * a.cst16 + bb * 16u + a.lutK) +
                          (uint32_t)kSlot * a.plane_bytes;
    return *reinterpret_cast<const float4*>(__cvta_shared_to_generic(addr));
  } else {
    const uint32_t t = (kTiled ? tcell + a.texT : ba * a.cst + bb + a.texR) + (uint32_t)IDX * a.ptex;
    return tex1Dfetch<float4>(a.tex, (int)t);
  }
}

// Bulk L2 prefetch of row y of three planes (16-byte aligned cover, clipped
// to each plane), no completion tracking.
__device__ __forceinline__ void bprefetch_row(const float* plane0, long long pl, int y, int w) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const float* pc = plane0 + c * pl;
    const uintptr_t lo = reinterpret_cast<uintptr_t>(pc + (long long)y * w) & ~(uintptr_t)15;
    const uintptr_t hi = (reinterpret_cast<uintptr_t>(pc + (long long)(y + 1) * w) + 15) & ~(uintptr_t)15;
    const uintptr_t end = reinterpret_cast<uintptr_t>(pc + pl) & ~(uintptr_t)15;
    const uintptr_t top = hi < end ? hi : end;
    if (top > lo)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((uint32_t)(top - lo))
                   : "memory");
  }
}

// Global accumulator layout per image (floats): lut [p 3][i d_t][j d_t+2][c 3]
// (row stride padded by two vertices: 3(d_t+2) = 105 words = 9 mod 32 at
// d_t = 33 spreads the rotated corners' banks better than one vertex, 6 mod
// 32: 8 x 1080p backward 638 -> 623 us),
// grid [q 3 (xy|xc|yc)][c 3][a d_s][b d_s], then gsum [4].
struct AccLayout {
  int dt, ds, lut_off, grid_off, gsum_off, total;
  __host__ __device__ static AccLayout make(int dt, int ds) {
    AccLayout A;
    A.dt = dt;
    A.ds = ds;
    A.lut_off = 0;
    A.grid_off = 3 * dt * (dt + kLutPad) * 3;
    A.gsum_off = A.grid_off + 9 * ds * ds;
    A.total = (A.gsum_off + 4 + 3) & ~3;
    return A;
  }
};

static size_t rup(size_t v) { return (v + 255) / 256 * 256; }

size_t bwd_workspace_bytes(int batch, int h, int w, int dt, int ds, int k) {
  (void)h;
  (void)w;
  const TableLayout L = TableLayout::make(dt, ds);
  const AccLayout A = AccLayout::make(dt, ds);
  return rup((size_t)batch * L.bytes()) + rup((size_t)batch * A.total * 4) +
         rup((size_t)batch * (3 + k) * 4) + rup((size_t)batch * 4) + rup((size_t)batch * 8) + 256;
}

struct BwdParams {
  const float* rgb;
  const float* gy;
  float* gx;
  int batch, h, w, y0;
  const float* tables;
  TableLayout L;
  AccLayout A;
  cudaTextureObject_t tex;
  int tex_base;
  double rcp_w, rcp_h;
  float* E;            // global accumulators, batch * A.total
  const float* gmax;   // per image max|gY|
  const double* gss;   // per image sum of gY^2 (may be NULL): outlier bound
  // fused L2 step (L2 = true): `gy` is the target T, gY = gscale (Y - T) is
  // formed per pixel from the tables, and sum (Y - T)^2 goes to loss[b]
  float gscale;
  double* loss;
};

// Per-pixel front end shared by the backward and the fused L2 step: the
// colour / spatial brackets and the gathered coefficient cells and slots.
struct PixFront {
  uint32_t br, bg, bb;  // 2^23-biased LUT cell bits
  uint32_t sr, sg, sb;  // 2^23-biased guide cell bits
  int jx;
  float dr, dg, db, er, eg, eb, ex;
  float4 q[9];  // chunk planes: pair rg 0-2, rb 3-5, gb 6-8
  float4 s[3];  // merged grid slots per channel: L2 step {M, M', N, N'}; backward {M', N', -, -}
};

// Y of one pixel from its cells, the forward kernel's arithmetic
// (svdlut_fwd.cu): per pair (A + B a) + (C + D a) b, then the slot term
// (M + N ex) + (M' + N' ex) ec per channel.
__device__ __forceinline__ float3 pix_y(const PixFront& F) {
  float2 acc01;
  float acc2;
#pragma unroll
  for (int pr = 0; pr < 3; ++pr) {
    const float da = pr == 2 ? F.dg : F.dr, dbv = pr == 0 ? F.dg : F.db;
    const float4 k0 = F.q[3 * pr], k1 = F.q[3 * pr + 1], k2 = F.q[3 * pr + 2];
    const float2 s01 = __ffma2_rn(make_float2(k1.z, k1.w), make_float2(da, da), make_float2(k1.x, k1.y));
    const float2 ts2 = __ffma2_rn(make_float2(k2.z, k2.w), make_float2(da, da), make_float2(k2.x, k2.y));
    if (pr == 0) {
      acc01 = __ffma2_rn(s01, make_float2(dbv, dbv),
                         __ffma2_rn(make_float2(k0.z, k0.w), make_float2(da, da), make_float2(k0.x, k0.y)));
      acc2 = __fmaf_rn(ts2.y, dbv, ts2.x);
    } else {
      acc01 = __ffma2_rn(make_float2(k0.z, k0.w), make_float2(da, da), __fadd2_rn(acc01, make_float2(k0.x, k0.y)));
      acc01 = __ffma2_rn(s01, make_float2(dbv, dbv), acc01);
      acc2 = __fmaf_rn(ts2.y, dbv, acc2 + ts2.x);
    }
  }
  const float2 p0 = __ffma2_rn(make_float2(F.s[0].z, F.s[0].w), make_float2(F.ex, F.ex), make_float2(F.s[0].x, F.s[0].y));
  const float2 p1 = __ffma2_rn(make_float2(F.s[1].z, F.s[1].w), make_float2(F.ex, F.ex), make_float2(F.s[1].x, F.s[1].y));
  const float2 p2 = __ffma2_rn(make_float2(F.s[2].z, F.s[2].w), make_float2(F.ex, F.ex), make_float2(F.s[2].x, F.s[2].y));
  const float2 o01 = __fadd2_rn(acc01, make_float2(__fmaf_rn(p0.y, F.er, p0.x), __fmaf_rn(p1.y, F.eg, p1.x)));
  return make_float3(o01.x, o01.y, acc2 + __fmaf_rn(p2.y, F.eb, p2.x));
}

__device__ __forceinline__ uint32_t bsmem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float4 blds4(uint32_t a) {
  return *reinterpret_cast<const float4*>(__cvta_shared_to_generic(a));
}
__device__ __forceinline__ float2 blds2(uint32_t a) {
  return *reinterpret_cast<const float2*>(__cvta_shared_to_generic(a));
}
// Cyclic rotation of a channel triple by the lane's channel offset r (rot1:
// r == 1, rot2: r == 2) with selects: (a, b, c) -> (b, c, a) / (c, a, b).
template <typename T>
__device__ __forceinline__ void rot3(bool rot1, bool rot2, T& a, T& b, T& c) {
  const T a1 = rot1 ? b : (rot2 ? c : a);
  const T b1 = rot1 ? c : (rot2 ? a : b);
  const T c1 = rot1 ? a : (rot2 ? b : c);
  a = a1;
  b = b1;
  c = c1;
}

// Shared-memory fixed-point add at a byte address (ATOMS.ADD, no return).
__device__ __forceinline__ void ared(uint32_t addr, int v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t bbracket(float q, float dm1, float dm2, float& delta) {
  const float t = fminf(__fmul_rz(q, dm1), dm2);
  const float m = __fadd_rz(t, 8388608.0f);
  delta = __fmaf_rn(q, dm1, -(m - 8388608.0f));
  return __float_as_uint(m);
}

// Scatter values are accumulated as 32-bit fixed point: v * S with
// S = 2^16 / B, B = min(max|gY|, kOutlierSigmas * rms(gY)) of the image, so
// one contribution is at most 2^16 in magnitude (resolution 2^-16 B).
// Pixels with some |gY| > B (heavy-tailed residuals) would either overflow
// that bound or, with B = max|gY|, leave the rest of the image with too
// coarse a resolution; they scatter through global f32 atomics instead
// (rare by construction).  Conversion is an add of 1.5*2^23
// (round to nearest even on the FMA pipe).
// Shared sums are flushed to the global f32 accumulators at least every
// row that could take one partial past 2^31: every shared partial is a sum
// of at most one contribution (|v| <= 2^16) per pixel, so at most
// kMaxFlushPx pixels may accumulate between flushes (rows <= kMaxFlushPx px).
constexpr int kMaxFlushPx = 32767;
constexpr float kFixedOne = 65536.0f;
constexpr float kOutlierSigmas = 6.0f;
#ifndef BWD_PROBE_HEADROOM
#define BWD_PROBE_HEADROOM 1.5f
#endif
constexpr float kProbeHeadroom = BWD_PROBE_HEADROOM;  // probe bound = headroom x the row statistic
__device__ __forceinline__ int to_fixed(float v, float S) {
  return __float_as_int(__fmaf_rn(v, S, 12582912.0f)) - 0x4B400000;
}

// Merged grid coefficients of channel c at (row jy/ey, x-cell jx, guide cell
// jc) from the grid block `gsm` (xc first, svdlut_common.cuh).
__device__ __forceinline__ float4 bgrid_entry(const float* gsm, const TableLayout& L, int c, int jx,
                                              int jc, int jy, float ey) {
  const int ds = L.ds;
  const float4 x = __ldg(reinterpret_cast<const float4*>(gsm) + (c * (ds - 1) + jx) * (ds - 1) + jc);
  const float* Y = gsm + (L.gyc_off - L.xc_off) + c * ds * ds;
  const float y00 = __ldg(Y + jy * ds + jc), y01 = __ldg(Y + jy * ds + jc + 1);
  const float y10 = __ldg(Y + (jy + 1) * ds + jc), y11 = __ldg(Y + (jy + 1) * ds + jc + 1);
  const float q0 = __fmaf_rn(ey, y10 - y00, y00), q1 = __fmaf_rn(ey, y11 - y01, y01);
  const float* X = gsm + (L.gxy_off - L.xc_off);
  const float v00 = __ldg(X + (jx * ds + jy) * 3 + c), v01 = __ldg(X + (jx * ds + jy + 1) * 3 + c);
  const float v10 = __ldg(X + ((jx + 1) * ds + jy) * 3 + c), v11 = __ldg(X + ((jx + 1) * ds + jy + 1) * 3 + c);
  const float r0 = __fmaf_rn(ey, v01 - v00, v00), r1 = __fmaf_rn(ey, v11 - v10, v10);
  return make_float4(x.x + q0 + r0, x.z + (q1 - q0), x.y + (r1 - r0), x.w);  // {M, M', N, N'}
}

struct BChunk {
  float r[kBPx], g[kBPx], b[kBPx], y0[kBPx], y1[kBPx], y2[kBPx];
};

__device__ __forceinline__ void bload4(const float* p, float* v, int x, int w, bool vec) {
  if (vec && x + 4 <= w) {
    const float4 t = __ldcs(reinterpret_cast<const float4*>(p + x));
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcs(p + min(x + u, w - 1));
  }
}

__device__ __forceinline__ void bload_chunk(const float* X, const float* GY, long long pl, int y,
                                            int x0, int w, int lane, bool vec, BChunk& c) {
  const long long ro = (long long)y * w;
  const int x = x0 + 4 * lane;
  bload4(X + ro, c.r, x, w, vec);
  bload4(X + pl + ro, c.g, x, w, vec);
  bload4(X + 2 * pl + ro, c.b, x, w, vec);
  bload4(GY + ro, c.y0, x, w, vec);
  bload4(GY + pl + ro, c.y1, x, w, vec);
  bload4(GY + 2 * pl + ro, c.y2, x, w, vec);
}

// L2: the fused training step (gY formed per pixel, implies DYN).  DYN: the
// fixed-point bound comes per CTA from a probe of its first row (and is
// raised on demand) instead of precomputed per-image statistics.
template <int DT, int DS, bool L2, bool DYN>
__global__ void __launch_bounds__(kBwdWarps * 32, 1) fused_bwd_kernel(BwdParams p) {
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t bar_storage;
  // fused L2 step: max |gY|, sum gY^2 and the number of pixels above the
  // bound, of the probe row and of each row (row parity)
  __shared__ float s_max[3], s_ss[3];
  __shared__ int s_nbig[3];
  const int dt = DT ? DT : p.L.dt;
  const int ds = DS ? DS : p.L.ds;
  const TableLayout L = TableLayout::make(dt, ds);
  const AccLayout A = AccLayout::make(dt, ds);
  const uint32_t bar = bsmem_addr(&bar_storage);
  const uint32_t sbase = bsmem_addr(smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned full = 0xffffffffu;
  const int rc0 = lane % 3, rc1 = (lane + 1) % 3, rc2 = (lane + 2) % 3;  // lane's channel order
  const bool rot1 = rc0 == 1, rot2 = rc0 == 2;  // (x0, x1, x2) -> (x_rc0, x_rc1, x_rc2)
  // lane's corner order: k-th corner = (k + lane/3) % 4, bit 0 the first
  // axis (LUT a / grid x), bit 1 the second (LUT b / grid guide)
  bool kqa[4], kqb[4];
  uint32_t kcoff[4], kxoff[4];  // byte offsets of the k-th corner (LUT / grid xc)
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int q = (k + lane / 3) & 3;
    kqa[k] = q & 1;
    kqb[k] = q & 2;
    kcoff[k] = (uint32_t)(((q & 1) ? (dt + kLutPad) * 3 : 0) + ((q & 2) ? 3 : 0)) * 4u;
    kxoff[k] = (uint32_t)(((q & 1) ? ds : 0) + ((q & 2) ? 1 : 0)) * 4u;
  }

  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // staged: the kBwdPlanes chunk planes (in plane order), then the slot rows
  // and the accumulators
  const uint32_t plane_bytes = (uint32_t)L.plane_floats * 4u;
  const uint32_t table_bytes = (uint32_t)kBwdStaged * plane_bytes;
  const int nent = (ds - 1) * 3 * (ds - 1);
  float4* slots = reinterpret_cast<float4*>(reinterpret_cast<char*>(smem) + table_bytes);
  float* Es = reinterpret_cast<float*>(slots + 2 * nent);  // A.total floats
  const float tdm1 = (float)(dt - 1), tdm2 = (float)(dt - 2);
  const float sdm1 = (float)(ds - 1), sdm2 = (float)(ds - 2);
  BAddr ad;
  ad.cst = (uint32_t)L.cst;
  ad.cst16 = ad.cst * 16u;
  ad.ptex = (uint32_t)L.plane_floats / 4u;  // texels per plane
  ad.tiles = (uint32_t)L.tiles();
  ad.plane_bytes = plane_bytes;
  ad.lutK = sbase - kMagic * (ad.cst16 + 16u);
  ad.lutT = sbase - (((kMagic >> 2) * ad.tiles + (kMagic >> 2)) << 8);
  ad.tex = p.tex;
  const uint32_t chan_bytes = (uint32_t)(ds - 1) * 16u;
  const uint32_t jx_bytes = 3u * chan_bytes;
  const uint32_t slot_row_bytes = (uint32_t)nent * 16u;
  const uint32_t slotK0 = bsmem_addr(slots) - kMagic * 16u;
  int* Ei = reinterpret_cast<int*>(Es);
  int* Rrow = Ei + A.total;         // 2 rows x [Rx 3*ds | Rc 3*ds]
  // 2 rows x kXRCopies lane-group copies (4: lanes 0-7, 8-15, ...; lanes
  // with the same corner x channel rotation never share a copy) x the row's
  // xc plane [c 3][vx ds][vc ds]
  int* XRrow = Rrow + 12 * ds;
  const int xr_size = 3 * ds * ds;
  const uint32_t sXR = bsmem_addr(XRrow) + (uint32_t)((kXRCopies == 3 ? lane / 12 : lane / (32 / kXRCopies)) * xr_size) * 4u;
  // byte address of LUT pair pr's cell from 2^23-biased index bits:
  // lutE[pr] + bits_a * (dt+1)*12 + bits_b * 12
  const uint32_t rowB = (uint32_t)(dt + kLutPad) * 12u;
  uint32_t lutE[3];
#pragma unroll
  for (int pr = 0; pr < 3; ++pr)
    lutE[pr] = bsmem_addr(Ei) + (uint32_t)(A.lut_off + pr * dt * (dt + kLutPad) * 3) * 4u - kMagic * (rowB + 12u);
  const uint32_t rcb0 = (uint32_t)rc0 * 4u, rcb1 = (uint32_t)rc1 * 4u, rcb2 = (uint32_t)rc2 * 4u;
  int* E_lut = Ei + A.lut_off;
  int* E_xy = Ei + A.grid_off;
  int* E_xc = E_xy + 3 * ds * ds;
  int* E_yc = E_xc + 3 * ds * ds;

  const long long rows_total = (long long)p.batch * p.h;
  const long long r_begin = (long long)blockIdx.x * rows_total / gridDim.x;
  const long long r_end = (long long)(blockIdx.x + 1) * rows_total / gridDim.x;
  const long long pl = (long long)p.h * p.w;
  const bool vec = ((p.w & 3) == 0) &&
                   (((uintptr_t)p.rgb | (uintptr_t)p.gy | (uintptr_t)p.gx) & 15) == 0;
  uint32_t phase = 0;

  long long r = r_begin;
  while (r < r_end) {
    const int b = (int)(r / p.h);
    const int y_first = (int)(r - (long long)b * p.h);
    const int y_last = (int)(min(r_end, (long long)(b + 1) * p.h) - 1 - (long long)b * p.h);
    const float* tb = p.tables + (long long)b * L.total_floats;
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(table_bytes)
                   : "memory");
      auto copy = [&](uint32_t dst, const char* from, uint32_t bytes) {
        for (uint32_t off = 0; off < bytes; off += 32768u)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  dst + off),
              "l"(from + off), "r"(min(32768u, bytes - off)), "r"(bar)
              : "memory");
      };
      uint32_t dst = sbase;
#pragma unroll
      for (int idx = 0; idx < 9; ++idx)
        if ((kBwdPlanes >> idx) & 1u) {
          copy(dst, reinterpret_cast<const char*>(tb + L.lut_off + idx * L.plane_floats), plane_bytes);
          dst += plane_bytes;
        }
    }
    for (int i = threadIdx.x; i < A.total + 12 * ds + 2 * kXRCopies * xr_size; i += blockDim.x) Ei[i] = 0;
    float gm = 0.f;
    if (!DYN) {
      gm = p.gmax[b];
      if (p.gss) gm = fminf(gm, kOutlierSigmas * (float)sqrt(p.gss[b] / (3.0 * (double)pl)));
    }
    float S = gm > 0.f ? kFixedOne / gm : 1.0f;  // fixed-point scale of this image (segment)
    float bound = gm > 0.f ? gm : 3.4e38f;       // |gY| above: global slow path
    float invS = 1.0f / S;
    float* Eg = p.E + (long long)b * A.total;
    int px_since_flush = 0;
    const float* X = p.rgb + (long long)b * 3 * pl;
    const float* GY = p.gy + (long long)b * 3 * pl;
    float* GX = p.gx ? p.gx + (long long)b * 3 * pl : nullptr;
    const float* gsm = tb + L.xc_off;  // grid block (global, L1-cached; read by the slot production)
    {
      const uint32_t t0 = (uint32_t)p.tex_base + (uint32_t)b * (uint32_t)(L.total_floats / 4) +
                          (uint32_t)(L.lut_off / 4);
      ad.texT = t0 - (((kMagic >> 2) * ad.tiles + (kMagic >> 2)) << 4);
      ad.texR = t0 - kMagic * (ad.cst + 1u);
    }
    asm volatile(
        "{\n.reg .pred p;\nWAITB_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAITB_%=;\n}\n" ::"r"(bar),
        "r"(phase)
        : "memory");
    phase ^= 1u;
    // slot row yr into ring buffer (yr - y_first) % 2
    auto produce_rows = [&](int yr) {
      float eyp;
      const int jyp = (int)(row_bracket(p.y0 + yr, p.rcp_h, sdm1, sdm2, eyp) - kMagic);
      float4* S = slots + ((yr - y_first) & 1) * nent;
      for (int e = threadIdx.x; e < nent; e += blockDim.x) {
        const int jx = e / (3 * (ds - 1)), rem = e - jx * 3 * (ds - 1);
        const int ch = rem / (ds - 1), jc = rem - ch * (ds - 1);
        SVDLUT_CHECK(jyp >= 0 && jyp <= ds - 2);
        const float4 v = bgrid_entry(gsm, L, ch, jx, jc, jyp, eyp);  // {M, M', N, N'}
        // the backward alone needs only d/dec = M' + N' ex: stored first, one LDS.64
        S[e] = L2 ? v : make_float4(v.y, v.w, v.x, v.z);
      }
    };
    produce_rows(y_first);
    __syncthreads();
    float gsum0 = 0.f, gsum1 = 0.f, gsum2 = 0.f;
    // brackets and gathers of the pixel at column xpix with samples (Xr, Xg, Xb)
    auto front = [&](PixFront& F, float Xr, float Xg, float Xb, int xpix, uint32_t slotK) {
      const float qr = __saturatef(Xr), qg = __saturatef(Xg), qb = __saturatef(Xb);
      F.br = bbracket(qr, tdm1, tdm2, F.dr);
      F.bg = bbracket(qg, tdm1, tdm2, F.dg);
      F.bb = bbracket(qb, tdm1, tdm2, F.db);
      F.jx = (int)(col_bracket(min(xpix, p.w - 1), p.rcp_w, sdm1, sdm2, F.ex) - kMagic);
      F.sr = bbracket(qr, sdm1, sdm2, F.er);
      F.sg = bbracket(qg, sdm1, sdm2, F.eg);
      F.sb = bbracket(qb, sdm1, sdm2, F.eb);
      SVDLUT_CHECK(F.br - kMagic <= (uint32_t)(dt - 2) && F.bg - kMagic <= (uint32_t)(dt - 2) &&
                   F.bb - kMagic <= (uint32_t)(dt - 2) && F.jx >= 0 && F.jx <= ds - 2 &&
                   F.sr - kMagic <= (uint32_t)(ds - 2) && F.sg - kMagic <= (uint32_t)(ds - 2) &&
                   F.sb - kMagic <= (uint32_t)(ds - 2));
      F.q[0] = bfetch<0>(ad, F.br, F.bg);
      F.q[1] = bfetch<1>(ad, F.br, F.bg);
      F.q[2] = bfetch<2>(ad, F.br, F.bg);
      F.q[3] = bfetch<3>(ad, F.br, F.bb);
      F.q[4] = bfetch<4>(ad, F.br, F.bb);
      F.q[5] = bfetch<5>(ad, F.br, F.bb);
      F.q[6] = bfetch<6>(ad, F.bg, F.bb);
      F.q[7] = bfetch<7>(ad, F.bg, F.bb);
      F.q[8] = bfetch<8>(ad, F.bg, F.bb);
      const uint32_t sa = slotK + (uint32_t)F.jx * jx_bytes;
      if (L2) {
        F.s[0] = blds4(sa + F.sr * 16u);
        F.s[1] = blds4(sa + chan_bytes + F.sg * 16u);
        F.s[2] = blds4(sa + 2u * chan_bytes + F.sb * 16u);
      } else {  // {M', N'} only
        const float2 t0 = blds2(sa + F.sr * 16u), t1 = blds2(sa + chan_bytes + F.sg * 16u),
                     t2 = blds2(sa + 2u * chan_bytes + F.sb * 16u);
        F.s[0] = make_float4(t0.x, t0.y, 0.f, 0.f);
        F.s[1] = make_float4(t1.x, t1.y, 0.f, 0.f);
        F.s[2] = make_float4(t2.x, t2.y, 0.f, 0.f);
      }
    };
    // Dynamic bound (DYN: the fused L2 step, or no caller statistics): the
    // fixed-point bound of this CTA's image segment comes from its first row
    // (a probe pass; in the L2 step forward-only), B = 1.5 min(max |gY|,
    // 6 rms gY) of that row; pixels above B take the f32 slow path.  When
    // more than 1/64 of a row's pixels did, B is raised to max(2 B, 1.5 x the
    // row's own min(max, 6 rms)) after the partials at the old scale are
    // flushed — sparse outliers never move it, growing residuals do.
    float loss_acc = 0.f;
    auto set_bound = [&](float bnd) {
      S = bnd > 0.f ? kFixedOne / bnd : 1.0f;
      bound = bnd > 0.f ? bnd : 0.f;
      invS = 1.0f / S;
    };
    auto warp_stats = [&](float m, float ss, int nbig, int slot) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        m = fmaxf(m, __shfl_xor_sync(full, m, off));
        ss += __shfl_xor_sync(full, ss, off);
        nbig += __shfl_xor_sync(full, nbig, off);
      }
      if (lane == 0) {
        atomicMax(reinterpret_cast<int*>(&s_max[slot]), __float_as_int(m));  // m >= 0
        atomicAdd(&s_ss[slot], ss);
        atomicAdd(&s_nbig[slot], nbig);
      }
    };
    auto row_bound = [&](int slot) {  // with headroom for the rows after it
      return kProbeHeadroom * fminf(s_max[slot], kOutlierSigmas * sqrtf(s_ss[slot] / (3.f * (float)p.w)));
    };
    if (DYN) {
      if (threadIdx.x == 0) {
        for (int i = 0; i < 3; ++i) {
          s_max[i] = s_ss[i] = 0.f;
          s_nbig[i] = 0;
        }
      }
      __syncthreads();
      float pm = 0.f, ps = 0.f;
      for (int x0 = warp * 128; x0 < p.w; x0 += kBwdWarps * 128) {
        const int xl = x0 + 4 * lane;
        BChunk cur;
        bload_chunk(X, GY, pl, y_first, x0, p.w, lane, vec, cur);
#pragma unroll
        for (int u = 0; u < kBPx; ++u) {
          const bool valid = xl + u < p.w;
          float g0 = valid ? cur.y0[u] : 0.f, g1 = valid ? cur.y1[u] : 0.f, g2 = valid ? cur.y2[u] : 0.f;
          if (L2) {  // the forward of the probe row
            PixFront F;
            front(F, cur.r[u], cur.g[u], cur.b[u], xl + u, slotK0);
            const float3 Y = pix_y(F);
            g0 = valid ? (Y.x - cur.y0[u]) * p.gscale : 0.f;
            g1 = valid ? (Y.y - cur.y1[u]) * p.gscale : 0.f;
            g2 = valid ? (Y.z - cur.y2[u]) * p.gscale : 0.f;
          }
          pm = fmaxf(pm, fmaxf(fabsf(g0), fmaxf(fabsf(g1), fabsf(g2))));
          ps = __fmaf_rn(g0, g0, __fmaf_rn(g1, g1, __fmaf_rn(g2, g2, ps)));
        }
      }
      warp_stats(pm, ps, 0, 2);
      __syncthreads();
      set_bound(row_bound(2));
    }
    // Rrow[par] = [Rx[c][vx] = sum g_c wx | Rc[c][vc] = sum g_c wc] of one row
    // into the xy / yc planes with that row's y weights, then zeroed
    auto fold_rows = [&](int par, int jyr, float eyr) {
      int* R = Rrow + par * 6 * ds;
      for (int i = threadIdx.x; i < 6 * ds; i += blockDim.x) {
        const int v = R[i];
        if (v != 0) {
          const bool isx = i < 3 * ds;
          const int c = (isx ? i : i - 3 * ds) / ds, t = (isx ? i : i - 3 * ds) - c * ds;
          int* e = isx ? E_xy + (c * ds + t) * ds + jyr : E_yc + (c * ds + jyr) * ds + t;
          const float fv = (float)v;
          atomicAdd(e, __float2int_rn(fv * (1.f - eyr)));
          atomicAdd(e + (isx ? 1 : ds), __float2int_rn(fv * eyr));
          R[i] = 0;
        }
      }
    };
    int jy_prev = 0;
    float ey_prev = 0.f;
    BChunk cur_out;     // backward: this warp's chunk of samples and gY, loaded ahead
    bool have = false;  // cur_out holds the chunk (loaded at the end of the previous one)

    for (int y = y_first; y <= y_last; ++y) {
      const int buf = (y - y_first) & 1;
      if (threadIdx.x == blockDim.x - 32) {
        for (int yy = (y == y_first ? y + 1 : y + kBwdL2Rows); yy <= y + kBwdL2Rows && yy <= y_last; ++yy) {
          bprefetch_row(X, pl, yy, p.w);
          bprefetch_row(GY, pl, yy, p.w);
        }
      }
      float ey;
      const int jy = (int)(row_bracket(p.y0 + y, p.rcp_h, sdm1, sdm2, ey) - kMagic);
      const uint32_t slotK = slotK0 + (uint32_t)buf * slot_row_bytes;
      // Lane mapping as in the forward: warp chunks of 128 consecutive
      // pixels, lane = 4 consecutive pixels.  Neighbouring lanes then share
      // cells, which keeps the table gathers cheap (4.5 instead of 8.7
      // cycles per LDS.128, tools/microbench/bwd_lds.txt); the atomics of
      // lanes that share a cell are spread over twelve words by the lane's
      // corner x channel rotation (3.6 cycles per ATOMS instead of 10).
      int* XR = XRrow + (y & 1) * kXRCopies * xr_size;
      const uint32_t sXRy = sXR + (uint32_t)((y & 1) * kXRCopies * xr_size) * 4u;
      float row_max = 0.f, row_ss = 0.f;  // fused L2 step: this thread's |gY| statistics of row y
      int row_big = 0;
      for (int x0 = warp * 128; x0 < p.w; x0 += kBwdWarps * 128) {
        // (backward: lanes past the row end run on clamped samples with gY = 0)
        const int xl = x0 + 4 * lane;
        if (L2 && xl >= p.w) continue;
        BChunk cur_in;
        BChunk& cur = L2 ? cur_in : cur_out;  // (the L2 step loads in place: less live state)
        if (L2 || !have) bload_chunk(X, GY, pl, y, x0, p.w, lane, vec, cur);
        float oxr[kBPx], oxg[kBPx], oxb[kBPx];
#pragma unroll
        for (int u = 0; u < kBPx; ++u) {
          const bool valid = xl + u < p.w;
          const float Xr = cur.r[u], Xg = cur.g[u], Xb = cur.b[u];
          PixFront F;
          front(F, Xr, Xg, Xb, xl + u, slotK);
          float g0, g1, g2;
          if (L2) {  // gY = gscale (Y - T); the loss sums (Y - T)^2
            const float3 Y = pix_y(F);
            const float r0 = valid ? Y.x - cur.y0[u] : 0.f, r1 = valid ? Y.y - cur.y1[u] : 0.f,
                        r2 = valid ? Y.z - cur.y2[u] : 0.f;
            loss_acc = __fmaf_rn(r0, r0, __fmaf_rn(r1, r1, __fmaf_rn(r2, r2, loss_acc)));
            g0 = r0 * p.gscale;
            g1 = r1 * p.gscale;
            g2 = r2 * p.gscale;
          } else {
            g0 = valid ? cur.y0[u] : 0.f;
            g1 = valid ? cur.y1[u] : 0.f;
            g2 = valid ? cur.y2[u] : 0.f;
          }
          if (DYN) {
            row_max = fmaxf(row_max, fmaxf(fabsf(g0), fmaxf(fabsf(g1), fabsf(g2))));
            row_ss = __fmaf_rn(g0, g0, __fmaf_rn(g1, g1, __fmaf_rn(g2, g2, row_ss)));
          }
          // outliers take the f32 slow path; the fixed-point path sees zeros
          const bool big = fmaxf(fabsf(g0), fmaxf(fabsf(g1), fabsf(g2))) > bound;
          const float f0 = big ? 0.f : g0, f1 = big ? 0.f : g1, f2 = big ? 0.f : g2;
          if (DYN) row_big += big ? 1 : 0;
          gsum0 += g0;
          gsum1 += g1;
          gsum2 += g2;
          const uint32_t br = F.br, bg = F.bg, bb = F.bb, sr = F.sr, sg = F.sg, sb = F.sb;
          const int jx = F.jx;
          const float dr = F.dr, dg = F.dg, db = F.db, er = F.er, eg = F.eg, eb = F.eb, ex = F.ex;
          SVDLUT_CHECK(jy >= 0 && jy <= ds - 2);
          // ---- input gradient from the coefficient cells ----
          // chunks {A0 A1 B0 B1} {C0 C1 D0 D1} {A2 C2 B2 D2} (svdlut_common.cuh):
          // d/da = B + D b, d/db = C + D a per channel
          float gar = 0.f, gag = 0.f, gab = 0.f;
          {
            const float4 c0 = F.q[0], c1 = F.q[1], c2 = F.q[2];  // rg
            gar += g0 * __fmaf_rn(c1.z, dg, c0.z) + g1 * __fmaf_rn(c1.w, dg, c0.w) + g2 * __fmaf_rn(c2.w, dg, c2.z);
            gag += g0 * __fmaf_rn(c1.z, dr, c1.x) + g1 * __fmaf_rn(c1.w, dr, c1.y) + g2 * __fmaf_rn(c2.w, dr, c2.y);
          }
          {
            const float4 c0 = F.q[3], c1 = F.q[4], c2 = F.q[5];  // rb
            gar += g0 * __fmaf_rn(c1.z, db, c0.z) + g1 * __fmaf_rn(c1.w, db, c0.w) + g2 * __fmaf_rn(c2.w, db, c2.z);
            gab += g0 * __fmaf_rn(c1.z, dr, c1.x) + g1 * __fmaf_rn(c1.w, dr, c1.y) + g2 * __fmaf_rn(c2.w, dr, c2.y);
          }
          {
            const float4 c0 = F.q[6], c1 = F.q[7], c2 = F.q[8];  // gb
            gag += g0 * __fmaf_rn(c1.z, db, c0.z) + g1 * __fmaf_rn(c1.w, db, c0.w) + g2 * __fmaf_rn(c2.w, db, c2.z);
            gab += g0 * __fmaf_rn(c1.z, dg, c1.x) + g1 * __fmaf_rn(c1.w, dg, c1.y) + g2 * __fmaf_rn(c2.w, dg, c2.y);
          }
          // d/dec = M' + N' ex
          const float gsr = g0 * (L2 ? __fmaf_rn(F.s[0].w, ex, F.s[0].y) : __fmaf_rn(F.s[0].y, ex, F.s[0].x));
          const float gsg = g1 * (L2 ? __fmaf_rn(F.s[1].w, ex, F.s[1].y) : __fmaf_rn(F.s[1].y, ex, F.s[1].x));
          const float gsb = g2 * (L2 ? __fmaf_rn(F.s[2].w, ex, F.s[2].y) : __fmaf_rn(F.s[2].y, ex, F.s[2].x));
          oxr[u] = (Xr < 0.f || Xr > 1.f) ? 0.f : __fmaf_rn(gar, tdm1, gsr * sdm1);
          oxg[u] = (Xg < 0.f || Xg > 1.f) ? 0.f : __fmaf_rn(gag, tdm1, gsg * sdm1);
          oxb[u] = (Xb < 0.f || Xb > 1.f) ? 0.f : __fmaf_rn(gab, tdm1, gsb * sdm1);

          // ---- scatter: LUT pairs, one fixed-point atomic per (corner, channel) ----
          // Lane l issues corner (k + l/3) % 4 at its k-th corner and channel
          // (j + l) % 3 at its j-th channel (lane-constant offsets kcoff /
          // kqa / kqb, rc*): up to twelve lanes that share a cell hit twelve
          // different words.
          const float fs[3] = {f0 * S, f1 * S, f2 * S};
          float s0v = fs[0], s1v = fs[1], s2v = fs[2];
          rot3(rot1, rot2, s0v, s1v, s2v);
          {  // pixels past the row end carry g = 0: their adds are zeros at clamped cells
#pragma unroll
            for (int pr = 0; pr < 3; ++pr) {
              const uint32_t ba = pr == 2 ? bg : br, bbq = pr == 0 ? bg : bb;
              const float da = pr == 2 ? dg : dr, dbb = pr == 0 ? dg : db;
              const uint32_t e = lutE[pr] + ba * rowB + bbq * 12u;
              SVDLUT_CHECK(((pr * dt + (int)(ba - kMagic) + 1) * (dt + kLutPad) + (int)(bbq - kMagic) + 1) * 3 + 2 <
                           A.grid_off);
              const float ea = 1.f - da, eb = 1.f - dbb;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float wk = (kqa[k] ? da : ea) * (kqb[k] ? dbb : eb);
                const float2 v01 = __ffma2_rn(make_float2(s0v, s1v), make_float2(wk, wk),
                                              make_float2(12582912.0f, 12582912.0f));
                ared(e + kcoff[k] + rcb0, __float_as_int(v01.x) - 0x4B400000);
                ared(e + kcoff[k] + rcb1, __float_as_int(v01.y) - 0x4B400000);
                ared(e + kcoff[k] + rcb2, __float_as_int(__fmaf_rn(s2v, wk, 12582912.0f)) - 0x4B400000);
              }
            }
          }
          if (big) {  // every scatter of this pixel straight to the global f32 sums
            const float gg[3] = {g0, g1, g2};
            const int ii[3] = {(int)(br - kMagic), (int)(bg - kMagic), (int)(bb - kMagic)};
            const float dd[3] = {dr, dg, db};
#pragma unroll
            for (int pr = 0; pr < 3; ++pr) {
              const int a = pr == 2 ? 1 : 0, bq = pr == 0 ? 1 : 2;
              float* e = Eg + A.lut_off + ((pr * dt + ii[a]) * (dt + kLutPad) + ii[bq]) * 3;
#pragma unroll
              for (int kc = 0; kc < 4; ++kc) {
                const float wgt = ((kc & 1) ? dd[a] : 1.f - dd[a]) * ((kc & 2) ? dd[bq] : 1.f - dd[bq]);
                float* ec = e + ((kc & 1) ? (dt + kLutPad) * 3 : 0) + ((kc & 2) ? 3 : 0);
#pragma unroll
                for (int c = 0; c < 3; ++c) atomicAdd(ec + c, gg[c] * wgt);
              }
            }
            const int jcs[3] = {(int)(sr - kMagic), (int)(sg - kMagic), (int)(sb - kMagic)};
            const float ecs[3] = {er, eg, eb};
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              float* xy = Eg + A.grid_off + c * ds * ds + jx * ds + jy;
              atomicAdd(xy, gg[c] * (1.f - ex) * (1.f - ey));
              atomicAdd(xy + ds, gg[c] * ex * (1.f - ey));
              atomicAdd(xy + 1, gg[c] * (1.f - ex) * ey);
              atomicAdd(xy + ds + 1, gg[c] * ex * ey);
              float* xc = Eg + A.grid_off + 3 * ds * ds + c * ds * ds + jx * ds + jcs[c];
              atomicAdd(xc, gg[c] * (1.f - ex) * (1.f - ecs[c]));
              atomicAdd(xc + ds, gg[c] * ex * (1.f - ecs[c]));
              atomicAdd(xc + 1, gg[c] * (1.f - ex) * ecs[c]);
              atomicAdd(xc + ds + 1, gg[c] * ex * ecs[c]);
              float* yc = Eg + A.grid_off + 6 * ds * ds + c * ds * ds + jy * ds + jcs[c];
              atomicAdd(yc, gg[c] * (1.f - ey) * (1.f - ecs[c]));
              atomicAdd(yc + ds, gg[c] * ey * (1.f - ecs[c]));
              atomicAdd(yc + 1, gg[c] * (1.f - ey) * ecs[c]);
              atomicAdd(yc + ds + 1, gg[c] * ey * ecs[c]);
            }
          }
          // ---- grid xc plane of this row: XR[c][vx][vc] += g_c wx wc, with the
          // same corner x channel rotation ----
          {
            const uint32_t jcr = sr - kMagic, jcg = sg - kMagic, jcb = sb - kMagic;
            uint32_t j0 = jcr, j1 = jcg, j2 = jcb;
            rot3(rot1, rot2, j0, j1, j2);
            float c0e = er, c1e = eg, c2e = eb;
            rot3(rot1, rot2, c0e, c1e, c2e);
            const uint32_t xb = sXRy + (uint32_t)(jx * ds) * 4u;
            const uint32_t x0p = xb + ((uint32_t)(rc0 * ds * ds) + j0) * 4u;
            const uint32_t x1p = xb + ((uint32_t)(rc1 * ds * ds) + j1) * 4u;
            const uint32_t x2p = xb + ((uint32_t)(rc2 * ds * ds) + j2) * 4u;
            const float wx0 = 1.f - ex;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float wx = kqa[k] ? ex : wx0;
              const float w0 = kqb[k] ? c0e : 1.f - c0e, w1 = kqb[k] ? c1e : 1.f - c1e,
                          w2 = kqb[k] ? c2e : 1.f - c2e;
              ared(x0p + kxoff[k], __float_as_int(__fmaf_rn(s0v * wx, w0, 12582912.0f)) - 0x4B400000);
              ared(x1p + kxoff[k], __float_as_int(__fmaf_rn(s1v * wx, w1, 12582912.0f)) - 0x4B400000);
              ared(x2p + kxoff[k], __float_as_int(__fmaf_rn(s2v * wx, w2, 12582912.0f)) - 0x4B400000);
            }
          }
        }
        if (GX) {
          const long long ro = (long long)y * p.w;
          if (vec && xl + 4 <= p.w) {
            __stcs(reinterpret_cast<float4*>(GX + ro + xl), make_float4(oxr[0], oxr[1], oxr[2], oxr[3]));
            __stcs(reinterpret_cast<float4*>(GX + pl + ro + xl), make_float4(oxg[0], oxg[1], oxg[2], oxg[3]));
            __stcs(reinterpret_cast<float4*>(GX + 2 * pl + ro + xl), make_float4(oxb[0], oxb[1], oxb[2], oxb[3]));
          } else {
#pragma unroll
            for (int u = 0; u < kBPx; ++u)
              if (xl + u < p.w) {
                GX[ro + xl + u] = oxr[u];
                GX[pl + ro + xl + u] = oxg[u];
                GX[2 * pl + ro + xl + u] = oxb[u];
              }
          }
        }
        // the warp's next chunk (this row or the next), loaded while this one
        // ends: its latency hides behind the row's end and barrier (not in
        // the L2 step, whose larger live state would spill)
        if (!L2) {
          int nx0 = x0 + kBwdWarps * 128, ny = y;
          if (nx0 >= p.w) {
            nx0 = warp * 128;
            ++ny;
          }
          have = ny <= y_last && nx0 < p.w;
          if (have) bload_chunk(X, GY, pl, ny, nx0, p.w, lane, vec, cur);
        }
      }
      px_since_flush += p.w;
      if (DYN) warp_stats(row_max, row_ss, row_big, y & 1);
      if (y < y_last) produce_rows(y + 1);  // the other half of the ring
      __syncthreads();
      if (DYN && threadIdx.x == 0) {  // row y + 1's statistics slot (row y - 1's was read last row)
        s_max[(y + 1) & 1] = 0.f;
        s_ss[(y + 1) & 1] = 0.f;
        s_nbig[(y + 1) & 1] = 0;
      }
      // the previous row's x-vertex / guide-vertex sums (complete since the
      // barrier) into the xy / yc planes with that row's y weights
      if (y > y_first) fold_rows((y - 1) & 1, jy_prev, ey_prev);
      // this row's xc sums into E_xc and its x-vertex / guide-vertex sums;
      // the buffer is zeroed for row y + 2 (rows y + 1 use the other one)
      for (int i = threadIdx.x; i < xr_size; i += blockDim.x) {
        int v = 0;
#pragma unroll
        for (int cp = 0; cp < kXRCopies; ++cp) {
          v += XR[i + cp * xr_size];
          XR[i + cp * xr_size] = 0;
        }
        if (v != 0) {
          const int c = i / (ds * ds), r2 = i - c * ds * ds, vx = r2 / ds, vc = r2 - vx * ds;
          E_xc[i] += v;  // one writer per entry in this phase
          int* R = Rrow + (y & 1) * 6 * ds;
          atomicAdd(R + c * ds + vx, v);
          atomicAdd(R + 3 * ds + c * ds + vc, v);
        }
      }
      jy_prev = jy;
      ey_prev = ey;
      if (DYN && y < y_last && s_nbig[y & 1] * 64 > p.w) {
        // every thread reads the same row statistics: raise the bound after
        // moving every partial at the old scale to the global f32 sums
        const float bnd = fmaxf(2.f * bound, row_bound(y & 1));
        {
          __syncthreads();                 // the xc fold of row y has landed
          fold_rows(y & 1, jy, ey);        // row y's x / guide vertex sums, old scale
          __syncthreads();
          for (int i = threadIdx.x; i < A.gsum_off; i += blockDim.x) {
            const int v = Ei[i];
            if (v != 0) {
              atomicAdd(Eg + i, (float)v * invS);
              Ei[i] = 0;
            }
          }
          __syncthreads();
          set_bound(bnd);
          px_since_flush = 0;
        }
      }
      if (px_since_flush + p.w > kMaxFlushPx && y < y_last) {  // keep shared partials < 2^31
        __syncthreads();  // the fold has landed
        for (int i = threadIdx.x; i < A.gsum_off; i += blockDim.x) {
          const int v = Ei[i];
          if (v != 0) {
            atomicAdd(Eg + i, (float)v * invS);
            Ei[i] = 0;
          }
        }
        px_since_flush = p.w;  // row y's xy / yc sums are still pending
        __syncthreads();
      }
    }
    __syncthreads();
    fold_rows(y_last & 1, jy_prev, ey_prev);
    // ---- per-image gY sums and flush of the shared accumulators ----
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      gsum0 += __shfl_xor_sync(full, gsum0, off);
      gsum1 += __shfl_xor_sync(full, gsum1, off);
      gsum2 += __shfl_xor_sync(full, gsum2, off);
    }
    if (lane == 0) {
      atomicAdd(Eg + A.gsum_off + 0, gsum0);
      atomicAdd(Eg + A.gsum_off + 1, gsum1);
      atomicAdd(Eg + A.gsum_off + 2, gsum2);
    }
    if (L2) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) loss_acc += __shfl_xor_sync(full, loss_acc, off);
      if (lane == 0) atomicAdd(p.loss + b, (double)loss_acc);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < A.gsum_off; i += blockDim.x) {
      const int v = Ei[i];
      if (v != 0) atomicAdd(Eg + i, (float)v * invS);
    }
    r += y_last - y_first + 1;
  }
}

// Converts the unweighted accumulators into parameter gradients.  grid.y = image.
__global__ void finalize_kernel(const float* __restrict__ lp, const float* __restrict__ lw,
                                const float* __restrict__ gp, const float* __restrict__ gw, int k,
                                AccLayout A, const float* __restrict__ E, float* dlp, float* dlw,
                                float* dlb, float* dgp, float* dgw, float* dgb) {
  const long long b = blockIdx.y;
  const int dt = A.dt, ds = A.ds;
  const float* Eb = E + b * (long long)A.total;
  const int task = blockIdx.x;  // 0..8: LUT planes (c,p); 9..: grid planes (kk, q)
  __shared__ double red[32];
  double acc = 0.0;
  if (task < 9) {
    const int c = task / 3, pr = task - c * 3;
    const float* T = lp + (b * 9 + task) * (long long)dt * dt;
    const float w = lw[b * 9 + task];
    float* D = dlp + (b * 9 + task) * (long long)dt * dt;
    for (int ij = threadIdx.x; ij < dt * dt; ij += blockDim.x) {
      const int i = ij / dt, j = ij - i * dt;
      const float e = Eb[A.lut_off + ((pr * dt + i) * (dt + kLutPad) + j) * 3 + c];
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
      const float e = Eb[A.grid_off + (q * 3 + c) * ds * ds + ab];
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
      if (task % 3 == 0) dlb[b * 3 + task / 3] = Eb[A.gsum_off + task / 3];
    } else {
      const int kq = task - 9;
      dgw[b * k * 3 + kq] = (float)s;
      if (kq % 3 == 0) dgb[b * k + kq / 3] = Eb[A.gsum_off + (kq / 3) % 3];
    }
  }
}

// The backward (target == NULL: gy given) or the fused L2 training step
// (target != NULL: gy = gscale (Y - target) formed per pixel from
// `tables_in`, which must be the forward's packed tables; loss[b] += sum
// (Y - target)^2, zeroed here).
static cudaError_t bwd_impl(const float* rgb, const float* gy, int batch, int h, int w, int y0,
                            int h_total, const float* lp, const float* lw, int dt, const float* gp,
                            const float* gw, int k, int ds, float* gx, float* dlp, float* dlw, float* dlb,
                            float* dgp, float* dgw, float* dgb, void* ws, cudaStream_t st,
                            const float* tables_in, const float* gmax_in, const double* gss_in,
                            const float* target, float gscale, double* loss) {
  const bool l2 = target != nullptr;
  const bool dyn = l2 || !gmax_in;  // no precomputed statistics: per-CTA probe bound
  if (l2 && (!tables_in || !loss)) return cudaErrorInvalidValue;
  const TableLayout L = TableLayout::make(dt, ds);
  const AccLayout A = AccLayout::make(dt, ds);
  const int nent = (ds - 1) * 3 * (ds - 1);
  const size_t staged = (size_t)kBwdStaged * L.plane_floats * 4;
  const size_t smem = staged + 2 * (size_t)nent * 16 + ((size_t)A.total + 12 * ds + 6 * kXRCopies * ds * ds) * 4;
  if (smem > (size_t)fwd_max_smem_bytes()) return cudaErrorInvalidValue;
  char* wp = (char*)ws;
  float* tables = (float*)wp;
  wp += rup((size_t)batch * L.bytes());
  float* E = (float*)wp;
  wp += rup((size_t)batch * A.total * 4);
  float* zb = (float*)wp;  // zero biases (biases do not enter any derivative)
  wp += rup((size_t)batch * (3 + k) * 4);
  // caller-provided max |gY| and sum gY^2 per image (gss may be NULL: bound
  // = max); without them (and in the L2 step) the kernel's per-CTA probe
  const float* gmax = dyn ? nullptr : gmax_in;
  const double* gss = dyn ? nullptr : gss_in;
  cudaError_t e;
  if ((e = cudaMemsetAsync(zb, 0, (size_t)batch * (3 + k) * 4, st)) != cudaSuccess) return e;
  if (l2 && (e = cudaMemsetAsync(loss, 0, (size_t)batch * 8, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(E, 0, (size_t)batch * A.total * 4, st)) != cudaSuccess) return e;
  if (tables_in) {
    tables = const_cast<float*>(tables_in);  // forward tables: biases do not enter the backward
  } else if ((e = launch_pack(lp, nullptr, nullptr, nullptr, 0, lw, zb, gp, gw, zb + 3 * batch, k, L,
                              batch, tables, st)) != cudaSuccess) {
    return e;
  }
  BwdParams p;
  p.rgb = rgb;
  p.gy = l2 ? target : gy;
  p.gscale = gscale;
  p.loss = loss;
  p.gx = gx;
  p.batch = batch;
  p.h = h;
  p.w = w;
  p.y0 = y0;
  p.tables = tables;
  p.L = L;
  p.A = A;
  p.rcp_w = 1.0 / (double)(w - 1);
  p.rcp_h = 1.0 / (double)(h_total - 1);
  p.E = E;
  p.gmax = gmax;
  p.gss = gss;
  if ((e = table_texture(tables, (size_t)batch * L.bytes(), st, &p.tex, &p.tex_base)) != cudaSuccess) return e;
  const long long rows = (long long)batch * h;
  if (rows > 0 && w > 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    long long grid = sms < rows ? sms : rows;
    const bool spec = dt == 33 && ds == 17;
    auto kern = l2    ? (spec ? fused_bwd_kernel<33, 17, true, true> : fused_bwd_kernel<0, 0, true, true>)
                : dyn ? (spec ? fused_bwd_kernel<33, 17, false, true> : fused_bwd_kernel<0, 0, false, true>)
                      : (spec ? fused_bwd_kernel<33, 17, false, false> : fused_bwd_kernel<0, 0, false, false>);
    const int inst = (spec ? 1 : 0) + (l2 ? 4 : dyn ? 2 : 0);
    // Attributes set once per (instantiation, device) to the largest request
    // any launch may make, so concurrent launches never see the limit lowered
    // under them (as for the forward kernel).
    constexpr int kMaxDev = 64;
    static std::atomic<int> configured[kMaxDev][6];
    if (dev >= kMaxDev || configured[dev][inst].load(std::memory_order_acquire) == 0) {
      if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    fwd_max_smem_bytes())) != cudaSuccess)
        return e;
      // smallest carve-out that fits the specialised layout: the rest of the
      // 256 KB array is L1 for the texture-path planes
      const int pct = (int)((smem + 2048 + (228 * 1024 - 1)) * 100 / (228 * 1024)) + 1;
      if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    pct > 100 ? 100 : pct)) != cudaSuccess)
        return e;
      if (dev < kMaxDev) configured[dev][inst].store(1, std::memory_order_release);
    }
    kern<<<(int)grid, kBwdWarps * 32, smem, st>>>(p);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = table_texture_used(p.tex, st)) != cudaSuccess) return e;
  }
  dim3 fg(9 + 3 * k, batch);
  finalize_kernel<<<fg, 256, 0, st>>>(lp, lw, gp, gw, k, A, E, dlp, dlw, dlb, dgp, dgw, dgb);
  return cudaGetLastError();
}

cudaError_t launch_fused_bwd(const float* rgb, const float* gy, int batch, int h, int w, int y0,
                             int h_total, const float* lp, const float* lw, int dt,
                             const float* gp, const float* gw, int k, int ds, float* gx,
                             float* dlp, float* dlw, float* dlb, float* dgp, float* dgw,
                             float* dgb, void* ws, size_t ws_bytes, cudaStream_t st,
                             const float* tables_in, const float* gmax_in, const double* gss_in) {
  (void)ws_bytes;
  return bwd_impl(rgb, gy, batch, h, w, y0, h_total, lp, lw, dt, gp, gw, k, ds, gx, dlp, dlw, dlb, dgp, dgw,
                  dgb, ws, st, tables_in, gmax_in, gss_in, nullptr, 0.f, nullptr);
}

cudaError_t launch_fused_l2_step(const float* rgb, const float* target, int batch, int h, int w, int y0,
                                 int h_total, const float* tables, float gscale, const float* lp,
                                 const float* lw, int dt, const float* gp, const float* gw, int k, int ds,
                                 float* gx, float* dlp, float* dlw, float* dlb, float* dgp, float* dgw,
                                 float* dgb, double* loss, void* ws, cudaStream_t st) {
  return bwd_impl(rgb, nullptr, batch, h, w, y0, h_total, lp, lw, dt, gp, gw, k, ds, gx, dlp, dlw, dlb, dgp,
                  dgw, dgb, ws, st, tables, nullptr, nullptr, target, gscale, loss);
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
