// svdlut_fwd.cu — K2: the fused slice + 2D-LUT apply forward (fast fp32 path).
//
// Replaces transform._fused_impl (reference transform.py:215-300).
//
// Design:
//   * One persistent CTA per SM.  The LUT chunk planes named by kSmemPlanes
//     and the grid block of one image are staged into shared memory by TMA
//     bulk copies (`cp.async.bulk`, mbarrier completion); the remaining LUT
//     chunk planes are gathered through the texture path, a second pipe beside
//     the shared-memory (LSU) pipe: an LDS.128 delivers 128 B of lane data
//     per clock, a TLD.128 64 B (tools/microbench/{ldsclean,texphase}.cu), so
//     the split balances the two (default: pair rg and chunk 0 of rb staged;
//     rb chunks 1-2 and pair gb, stored in 4x4-tiled cell order, gathered
//     through the texture path one pixel ahead of their use).
//   * A CTA owns a contiguous range of 128-pixel chunks over (image, row,
//     chunk) — balanced to one chunk — and its warps take the range's chunks
//     round robin (lane = 4 consecutive pixels, 128-bit streaming loads and
//     stores).  One thread bulk-prefetches input rows one row ahead into L2.
//   * Brackets are evaluated for two pixels at a time on the FP32x2 pipe
//     (__fmul2_rz / __fadd2_rz / __ffma2_rn); the merged grid slots carry a
//     padding guide cell so a guide of exactly 1.0 needs no min().
//   * Grid terms: per row, the CTA interpolates xy + xc + yc along y into
//     merged slots {M, M', N, N'} per (x-cell, channel, guide cell) in a ring
//     of kRing row buffers (mbarrier handshakes, warps may drift kRing-2 rows).
//   * Streaming I/O: 24 B/pixel of HBM traffic (3 f32 in, 3 f32 out).
#include <atomic>
#include <cstdint>

#include "svdlut_common.cuh"
#include "svdlut_io.cuh"
#include "svdlut_internal.h"

namespace svdlut {

#ifndef FWD_NW
#define FWD_NW 16
#endif
#ifndef FWD_PLANES
// LUT chunk planes staged in shared memory (bit 3*pair + chunk; pairs rg, rb,
// gb); the others (chunks 1-2 of rb, pair gb) go through the texture path
#define FWD_PLANES 0x0F
#endif
constexpr int kFwdWarps = FWD_NW;
constexpr int kPx = 4;                 // consecutive pixels per lane
constexpr int kChunk = 32 * kPx;       // pixels per warp chunk
#ifndef FWD_RING
#define FWD_RING 3
#endif
constexpr int kRing = FWD_RING;        // per-row grid slot buffers
constexpr int kAhead = kRing - 1;      // rows of slots produced ahead of the one consumed
#ifndef FWD_L2ROWS
#define FWD_L2ROWS 1
#endif
constexpr int kL2Rows = FWD_L2ROWS;    // rows of L2 prefetch distance for the input
constexpr uint32_t kSmemPlanes = FWD_PLANES;
constexpr uint32_t kMagicBits = 0x4B000000u;  // bits of 2^23
constexpr float kMagic = 8388608.0f;

__host__ __device__ constexpr int popcount9(uint32_t m) {
  return (int)((m & 1u) + ((m >> 1) & 1u) + ((m >> 2) & 1u) + ((m >> 3) & 1u) + ((m >> 4) & 1u) +
               ((m >> 5) & 1u) + ((m >> 6) & 1u) + ((m >> 7) & 1u) + ((m >> 8) & 1u));
}
__host__ __device__ constexpr bool plane_in_smem(int idx) { return (kSmemPlanes >> idx) & 1u; }
__host__ __device__ constexpr int smem_plane_slot(int idx) { return popcount9(kSmemPlanes & ((1u << idx) - 1u)); }
constexpr int kSmemPlaneCount = popcount9(kSmemPlanes);

struct FwdParams {
  const void* in;           // input samples (format IN of the kernel)
  void* out;                // output samples (format OUT)
  int batch, h, w;
  long long pl_in, pl_out;  // f32 plane strides in floats (h*w for packed images)
  int y0;                   // first row of this strip in an image of h_total rows
  const float* tables;
  TableLayout L;
  cudaTextureObject_t tex;  // float4 texels over the packed tables
  int tex_base;             // texel index of image 0's table start
  double rcp_w;             // RN64(1 / (W - 1)) for the exact column brackets
  double rcp_h;             // RN64(1 / (h_total - 1)) for the row brackets
  int* nonfinite;
  // OUT == kL2Grad (fused L2 loss): target image (f32 planar, like the input),
  // per-image sum of squared residuals (f64) and max |gY| (f32 bits), and the
  // gradient scale 2 / N of mean((Y - T)^2)
  const float* target;
  double* loss;
  float* gmax;
  float gscale;
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ float4 lds4(uint32_t a) {
  return *reinterpret_cast<const float4*>(__cvta_shared_to_generic(a));
}
// Texture gather as volatile PTX: keeps the one-pixel-ahead issue order (the
// compiler otherwise hoists a chunk's texture gathers to its top and runs
// out of registers for the shared-memory gathers).
__device__ __forceinline__ float4 texv4(cudaTextureObject_t t, int i) {
  float4 v;
  asm volatile("tex.1d.v4.f32.s32 {%0,%1,%2,%3}, [%4, {%5}];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(t), "r"(i));
  return v;
}

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

// Colour / guide brackets of two pixels (interp.py:35-45, exact floor; see
// svdlut_common.cuh): biased index bits m (2^23 + i as float) and delta.
// CAP: i = min(floor(t), d-2); without it a value of exactly 1.0 lands on
// index d-1 (the padding guide slot stands for (d-2, delta 1)).
template <bool CAP>
__device__ __forceinline__ void bracket2(float2 q, float dm1, float2& m, float2& delta) {
  float2 t = __fmul2_rz(q, f2(dm1));
  if (CAP) t = f2(fminf(t.x, dm1 - 1.0f), fminf(t.y, dm1 - 1.0f));
  m = __fadd2_rz(t, f2(kMagic));
  const float2 nf = __ffma2_rn(m, f2(-1.0f), f2(kMagic));  // -floor(t), exact
  delta = __ffma2_rn(q, f2(dm1), nf);
}

// Merged grid coefficients of channel c at (row bracket jy/ey, x-cell jx, guide cell jc):
//   {M, M', N, N'} with term = M + N*ex + (M' + N'*ex)*ec  (biases included);
// jc == ds-1 is the padding slot: cell ds-2 at ec = 1.  `gb` is the image's
// grid block (shared-memory copy).
__device__ __forceinline__ float4 grid_slot(const float* gb, const TableLayout& L, int ds, int c,
                                            int jx, int jc, int jy, float ey) {
  const int jcc = min(jc, ds - 2);
  const float4 x = reinterpret_cast<const float4*>(gb)[(c * (ds - 1) + jx) * (ds - 1) + jcc];
  const float* Y = gb + (L.gyc_off - L.xc_off) + c * ds * ds;
  const float y00 = Y[jy * ds + jcc], y01 = Y[jy * ds + jcc + 1];
  const float y10 = Y[(jy + 1) * ds + jcc], y11 = Y[(jy + 1) * ds + jcc + 1];
  const float q0 = __fmaf_rn(ey, y10 - y00, y00), q1 = __fmaf_rn(ey, y11 - y01, y01);
  const float* X = gb + (L.gxy_off - L.xc_off);
  const float v00 = X[(jx * ds + jy) * 3 + c], v01 = X[(jx * ds + jy + 1) * 3 + c];
  const float v10 = X[((jx + 1) * ds + jy) * 3 + c], v11 = X[((jx + 1) * ds + jy + 1) * 3 + c];
  const float r0 = __fmaf_rn(ey, v01 - v00, v00), r1 = __fmaf_rn(ey, v11 - v10, v10);
  float4 s = make_float4(x.x + q0 + r0, x.z + (q1 - q0), x.y + (r1 - r0), x.w);
  if (jc != jcc) {  // at ec = 1: {M + M', M', N + N', N'}
    s.x += s.y;
    s.z += s.w;
  }
  return s;
}

template <int PX>
struct ChunkIn {
  float r[PX], g[PX], b[PX];
};

// Shared-memory bytes of the staged tables (LUT chunk planes + grid block).
__host__ __device__ inline uint32_t staged_bytes(const TableLayout& L) {
  return (uint32_t)kSmemPlaneCount * (uint32_t)L.plane_floats * 4u + (uint32_t)L.grid_floats() * 4u;
}

template <int DT, int DS, bool CHECK, int IN, int OUT>
__global__ void __launch_bounds__(kFwdWarps * 32, 1) fused_fwd_kernel(FwdParams p) {
  constexpr int NW = kFwdWarps;
  constexpr bool LOSS = OUT == kL2Grad;
  constexpr int OUTF = LOSS ? (int)kF32 : OUT;  // storage format of the output
  float loss_acc = 0.f, gmax_acc = 0.f;         // LOSS: this thread's partials
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t bar_storage;
  __shared__ __align__(8) uint64_t ring_bar[2 * kRing];
  const int dt = DT ? DT : p.L.dt;
  const int ds = DS ? DS : p.L.ds;
  const TableLayout L = TableLayout::make(dt, ds);
  const uint32_t bar = smem_addr(&bar_storage);
  const uint32_t sbase = smem_addr(smem);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;

  // slot ring: full[i] completes when every warp wrote its share of the row
  // in buffer i, empty[i] when every warp finished reading it
  const uint32_t full0 = smem_addr(&ring_bar[0]), empty0 = smem_addr(&ring_bar[kRing]);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    for (int i = 0; i < 2 * kRing; ++i) mbar_init(smem_addr(&ring_bar[i]), NW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const uint32_t plane_bytes = (uint32_t)L.plane_floats * 4u;
  const uint32_t tables_bytes = staged_bytes(L);
  const int nent = L.slot_entries();
  float4* slots = reinterpret_cast<float4*>(reinterpret_cast<char*>(smem) + tables_bytes);
  const float tdm1 = (float)(dt - 1);
  const float sdm1 = (float)(ds - 1), sdm2 = (float)(ds - 2);

  const uint32_t cst = (uint32_t)L.cst;
  const uint32_t cst16 = cst * 16u;
  // smem address of cell (bits_a, bits_b) of a staged plane of pair p:
  //   lutK + bits_a*cst16 + bits_b*16 + (plane slot)*plane_bytes
  const uint32_t lutK = sbase - kMagicBits * (cst16 + 16u);
  const uint32_t chan_bytes = (uint32_t)ds * 16u;      // one channel of a slot row
  const uint32_t jx_bytes = 3u * chan_bytes;          // one x-cell of a slot row
  const uint32_t slot_row_bytes = (uint32_t)nent * 16u;
  const uint32_t slotK0 = smem_addr(slots) - kMagicBits * (jx_bytes + 16u);

  // contiguous range of global chunks g = ((image b) * h + row y) * cpr + k
  const int cpr = (p.w + kChunk - 1) / kChunk;
  const long long chunks_total = (long long)p.batch * p.h * cpr;
  const long long g_begin = (long long)blockIdx.x * chunks_total / gridDim.x;
  const long long g_end = (long long)(blockIdx.x + 1) * chunks_total / gridDim.x;
  const long long pl = p.pl_in, opl = p.pl_out;  // plane strides (floats)
  const long long plane_len = (long long)p.h * p.w;
  // Programmatic dependent launch: the table-packing kernel before this one
  // releases it early.  The input image is not written by that kernel, so the
  // first rows of this CTA's range stream into L2 while the tables are
  // packed; every read of the tables comes after griddepcontrol.wait.
  if (threadIdx.x == blockDim.x - 32 && g_begin < g_end) {
    const long long r0 = g_begin / cpr;
    const int b0 = (int)(r0 / p.h), y0r = (int)(r0 - (long long)b0 * p.h);
    const int y_end = (int)min((long long)p.h, (long long)y0r + kL2Rows + 1);
    for (int yy = y0r; yy < y_end; ++yy) {
      Src<IN>::prefetch_row(Src<IN>::image(p.in, b0, pl), pl, plane_len, yy, p.w);
      if (LOSS) Src<kF32>::prefetch_row(Src<kF32>::image(p.target, b0, pl), pl, plane_len, yy, p.w);
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const bool vec_in = ((p.w & 3) == 0) && Src<IN>::aligned(p.in, pl);
  const bool vec_out = ((p.w & 3) == 0) && Dst<OUTF>::aligned(p.out, opl) &&
                       (!LOSS || Src<kF32>::aligned(p.target, pl));
  uint32_t phase = 0;
  uint32_t nrow = 0;  // CTA row ordinal (slot ring position)
  bool bad = false;

  long long g_seg = g_begin;
  while (g_seg < g_end) {
    const long long r_seg = g_seg / cpr;              // global row of the segment's first chunk
    const int b = (int)(r_seg / p.h);
    const long long g_img_end = min(g_end, (long long)(b + 1) * p.h * cpr);
    const int y_first = (int)(r_seg - (long long)b * p.h);
    const int y_last = (int)((g_img_end - 1) / cpr - (long long)b * p.h);
    const float* tb = p.tables + (long long)b * L.total_floats;
    // the image's grid block (shared-memory copy, read by the slot production)
    const float* gsm = reinterpret_cast<const float*>(reinterpret_cast<const char*>(smem) +
                                                      kSmemPlaneCount * plane_bytes);
    // ---- stage image b's tables into shared memory (TMA bulk copies) ----
    __syncthreads();  // every warp is done reading the previous image's tables
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_expect_tx(bar, tables_bytes);
#pragma unroll
      for (int idx = 0; idx < 9; ++idx)
        if (plane_in_smem(idx)) {
          const char* src = reinterpret_cast<const char*>(tb + L.plane_off(idx / 3, idx % 3));
          for (uint32_t off = 0; off < plane_bytes; off += 32768u)
            bulk_g2s(sbase + smem_plane_slot(idx) * plane_bytes + off, src + off, min(32768u, plane_bytes - off),
                     bar);
        }
      const char* gsrc = reinterpret_cast<const char*>(tb + L.xc_off);
      const uint32_t gbytes = (uint32_t)L.grid_floats() * 4u;
      for (uint32_t off = 0; off < gbytes; off += 32768u)
        bulk_g2s(sbase + kSmemPlaneCount * plane_bytes + off, gsrc + off, min(32768u, gbytes - off), bar);

    }
    const void* src = Src<IN>::image(p.in, b, pl);
    void* dst = Dst<OUTF>::image(p.out, b, opl);
    const void* tsrc = LOSS ? Src<kF32>::image(p.target, b, pl) : nullptr;
    // texel of cell (bits_a, bits_b) of plane idx: texK + bits_a*cst + bits_b + plane_off/4
    const uint32_t texK = (uint32_t)p.tex_base + (uint32_t)b * (uint32_t)(L.total_floats / 4) -
                          kMagicBits * (cst + 1u);
    const uint32_t ptex = (uint32_t)L.plane_floats / 4u;  // texels per plane
    const uint32_t tiles = (uint32_t)L.tiles();
    // tiled index of the biased bits minus the row-stride bias already in texK
    const uint32_t texT = kMagicBits * (cst + 1u) - (((kMagicBits >> 2) * tiles + (kMagicBits >> 2)) << 4);

    // this warp's chunks: global chunk g_seg + warp + NW*i (< g_img_end), as
    // (row cy, chunk ck) advanced in 32-bit
    int cy, ck;
    {
      const long long g0 = g_seg + warp;
      cy = (int)(g0 / cpr - (long long)b * p.h);
      ck = (int)(g0 % cpr);
    }
    const int k_end = (int)((g_img_end - 1) % cpr) + 1;  // chunks of row y_last in the segment
    auto in_seg = [&](int y, int k) { return y < y_last || (y == y_last && k < k_end); };
    ChunkIn<kPx> cur, tgt;
    auto load = [&](int y, int k) {
      Src<IN>::template load<kPx>(src, pl, y, k * kChunk + kPx * lane, p.w, vec_in, cur.r, cur.g, cur.b);
      if (LOSS) Src<kF32>::template load<kPx>(tsrc, pl, y, k * kChunk + kPx * lane, p.w, vec_out, tgt.r, tgt.g, tgt.b);
    };
    if (in_seg(cy, ck)) load(cy, ck);  // the first chunk's loads overlap the table copy
    mbar_wait(bar, phase);
    phase ^= 1u;

    // this warp's share of the slots of row y (CTA row ordinal n) into ring buffer n % kRing
    auto produce = [&](uint32_t n, int y) {
      float ey;
      const int jy = (int)(row_bracket(p.y0 + y, p.rcp_h, sdm1, sdm2, ey) - kMagicBits);
      float4* S = slots + (n % kRing) * nent;
      for (int e = warp * 32 + lane; e < nent; e += NW * 32) {
        const int jx = e / (3 * ds), rem = e - jx * 3 * ds;
        const int ch = rem / ds, jc = rem - ch * ds;
        SVDLUT_CHECK(jx >= 0 && jx <= ds - 2 && jy >= 0 && jy <= ds - 2 && (int)(n % kRing) < kRing);
        S[e] = grid_slot(gsm, L, ds, ch, jx, jc, jy, ey);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(full0 + 8u * (n % kRing));
    };
    const uint32_t n0 = nrow;
    const int cnt = y_last - y_first + 1;
    for (int i = 0; i < kAhead && i < cnt; ++i) produce(n0 + i, y_first + i);

    for (int y = y_first; y <= y_last; ++y) {
      const uint32_t n = n0 + (uint32_t)(y - y_first);
      if (threadIdx.x == blockDim.x - 32) {  // L2 prefetch of the input rows ahead
        for (int yy = (y == y_first ? y + 1 : y + kL2Rows); yy <= y + kL2Rows && yy <= y_last; ++yy) {
          Src<IN>::prefetch_row(src, pl, plane_len, yy, p.w);
          if (LOSS) Src<kF32>::prefetch_row(tsrc, pl, plane_len, yy, p.w);
        }
      }
      mbar_wait(full0 + 8u * (n % kRing), (n / kRing) & 1u);
      const uint32_t slotK = slotK0 + (n % kRing) * slot_row_bytes;
      // ---- this warp's chunks of row y ----
      while (cy == y && in_seg(cy, ck)) {
        const int xl = ck * kChunk + kPx * lane;
        SVDLUT_CHECK(cy >= 0 && cy < p.h && ck >= 0 && ck < cpr);
        int ny = cy, nk = ck + NW;  // this warp's next chunk
        while (nk >= cpr) {
          nk -= cpr;
          ++ny;
        }
        const bool has_next = in_seg(ny, nk);

        // column brackets (x-cell bits, ex) of the lane's 4 pixels: exact t(x)
        // (lanes past the row end use the last column; never stored)
        const float2 tx01 = f2(col_t_value(min(xl, p.w - 1), p.rcp_w, sdm1),
                               col_t_value(min(xl + 1, p.w - 1), p.rcp_w, sdm1));
        const float2 tx23 = f2(col_t_value(min(xl + 2, p.w - 1), p.rcp_w, sdm1),
                               col_t_value(min(xl + 3, p.w - 1), p.rcp_w, sdm1));
        // brackets of pixel pair h2 (two pixels at a time on the FP32x2 pipe):
        // x-cell bits / ex, colour bits / deltas vs d_t (mc*, d*) and guide
        // bits / deltas vs d_s (ms*, e*).  Pair 1's colour brackets are computed
        // while pixel 1 runs (its texture gathers are issued there).
        float2 mx[2], ex[2], mcr[2], mcg[2], mcb[2], dr[2], dg[2], db[2];
        float2 msr[2], msg[2], msb[2], er[2], eg[2], eb[2];
        auto q2 = [&](const float* v, int h2) { return f2(__saturatef(v[2 * h2]), __saturatef(v[2 * h2 + 1])); };
        auto colour_brackets = [&](int h2) {
          bracket2<true>(q2(cur.r, h2), tdm1, mcr[h2], dr[h2]);
          bracket2<true>(q2(cur.g, h2), tdm1, mcg[h2], dg[h2]);
          bracket2<true>(q2(cur.b, h2), tdm1, mcb[h2], db[h2]);
        };
        auto grid_brackets = [&](int h2) {
          const float2 t = h2 ? tx23 : tx01;
          mx[h2] = __fadd2_rz(f2(fminf(t.x, sdm2), fminf(t.y, sdm2)), f2(kMagic));
          ex[h2] = __fadd2_rn(t, __ffma2_rn(mx[h2], f2(-1.0f), f2(kMagic)));  // t - floor(min(t, ds-2)): exact
          bracket2<false>(q2(cur.r, h2), sdm1, msr[h2], er[h2]);
          bracket2<false>(q2(cur.g, h2), sdm1, msg[h2], eg[h2]);
          bracket2<false>(q2(cur.b, h2), sdm1, msb[h2], eb[h2]);
        };
        colour_brackets(0);
        auto lo = [](const float2& v, int u) { return (u & 1) ? v.y : v.x; };
        auto bits = [](const float2& v, int u) { return __float_as_uint((u & 1) ? v.y : v.x); };

        // texture-path planes of pixel u: issued one pixel ahead
        float4 tq[9];
        // cell index of (bits_a, bits_b) in plane idx (svdlut_common.cuh): row
        // stride or 4x4 tiles; the 2^23 biases of the index bits fold into
        // texK / lutK (texT moves a tiled index onto the row-stride bias)
        auto cell_of = [&](int idx, uint32_t ba, uint32_t bbv) -> uint32_t {
          return plane_tiled(idx) ? (((ba >> 2) * tiles + (bbv >> 2)) << 4) + ((ba & 3u) << 2) + (bbv & 3u) + texT
                                  : ba * cst + bbv;
        };
        auto tex_issue = [&](int u, float4 (&tq_)[9], uint32_t dep) {
          const uint32_t br = bits(mcr[u >> 1], u), bg = bits(mcg[u >> 1], u), bb = bits(mcb[u >> 1], u);
#pragma unroll
          for (int idx = 0; idx < 9; ++idx) {
            if (plane_in_smem(idx)) continue;
            const int pr = idx / 3;
            const uint32_t ba = pr == 2 ? bg : br, bbv = pr == 0 ? bg : bb;
            tq_[idx] = texv4(p.tex, (int)(cell_of(idx, ba, bbv) + texK + (uint32_t)(L.plane_off(pr, idx % 3) / 4) + dep));
          }
        };
        tex_issue(0, tq, 0u);
        float o0[kPx], o1[kPx], o2[kPx];
#pragma unroll
        for (int u = 0; u < kPx; ++u) {
          if ((u & 1) == 0) grid_brackets(u >> 1);
          if (u == 1) colour_brackets(1);  // pixel 2's texture gathers are issued during pixel 1
          const uint32_t br = bits(mcr[u >> 1], u), bg = bits(mcg[u >> 1], u), bb = bits(mcb[u >> 1], u);
          SVDLUT_CHECK(br - kMagicBits <= (uint32_t)(dt - 2) && bg - kMagicBits <= (uint32_t)(dt - 2) &&
                       bb - kMagicBits <= (uint32_t)(dt - 2));
          SVDLUT_CHECK(bits(mx[u >> 1], u) - kMagicBits <= (uint32_t)(ds - 2) &&
                       bits(msr[u >> 1], u) - kMagicBits <= (uint32_t)(ds - 1) &&
                       bits(msg[u >> 1], u) - kMagicBits <= (uint32_t)(ds - 1) &&
                       bits(msb[u >> 1], u) - kMagicBits <= (uint32_t)(ds - 1));
          const float a_r = lo(dr[u >> 1], u), a_g = lo(dg[u >> 1], u), a_b = lo(db[u >> 1], u);
          // shared-memory planes
          float4 c[9];
          const uint32_t ur = br * cst16 + lutK;
          const uint32_t row_a[3] = {ur + bg * 16u, ur + bb * 16u, bg * cst16 + bb * 16u + lutK};
#pragma unroll
          for (int idx = 0; idx < 9; ++idx) {
            if (!plane_in_smem(idx)) continue;
            const int pr = idx / 3;
            const uint32_t a = plane_tiled(idx)
                                   ? cell_of(idx, pr == 2 ? bg : br, pr == 0 ? bg : bb) * 16u + lutK
                                   : row_a[pr];
            c[idx] = lds4(a + (uint32_t)smem_plane_slot(idx) * plane_bytes);
          }
          const uint32_t sa = slotK + bits(mx[u >> 1], u) * jx_bytes;
          const float4 s0 = lds4(sa + bits(msr[u >> 1], u) * 16u);
          const float4 s1 = lds4(sa + chan_bytes + bits(msg[u >> 1], u) * 16u);
          const float4 s2 = lds4(sa + 2u * chan_bytes + bits(msb[u >> 1], u) * 16u);
#pragma unroll
          for (int idx = 0; idx < 9; ++idx)
            if (!plane_in_smem(idx)) c[idx] = tq[idx];
          if (u + 1 < kPx) {
            // next pixel's texture gathers, after this pixel's shared gathers;
            // the (never taken) dependency on the last LDS stops ptxas from
            // hoisting all of the chunk's TLDs to its top
            tex_issue(u + 1, tq, s2.w != s2.w ? 1u : 0u);
          }
          // LUT pairs: v = A + B a + (C + D a) b, channels 0/1 on FP32x2
          float2 acc01;
          float acc2;
#pragma unroll
          for (int pr = 0; pr < 3; ++pr) {
            const float da = pr == 2 ? a_g : a_r, dbv = pr == 0 ? a_g : a_b;
            const float4 k0 = c[3 * pr], k1 = c[3 * pr + 1], k2 = c[3 * pr + 2];
            const float2 s01 = __ffma2_rn(f2(k1.z, k1.w), f2(da), f2(k1.x, k1.y));  // C + D a
            const float2 ts2 = __ffma2_rn(f2(k2.z, k2.w), f2(da), f2(k2.x, k2.y));  // {A2 + B2 a, C2 + D2 a}
            if (pr == 0) {
              acc01 = __ffma2_rn(s01, f2(dbv), __ffma2_rn(f2(k0.z, k0.w), f2(da), f2(k0.x, k0.y)));
              acc2 = __fmaf_rn(ts2.y, dbv, ts2.x);
            } else {
              acc01 = __ffma2_rn(f2(k0.z, k0.w), f2(da), __fadd2_rn(acc01, f2(k0.x, k0.y)));
              acc01 = __ffma2_rn(s01, f2(dbv), acc01);
              acc2 = __fmaf_rn(ts2.y, dbv, acc2 + ts2.x);
            }
          }
          // grids: one merged (xy + xc + yc) slot per channel {M, M', N, N'}
          const float e_x = lo(ex[u >> 1], u);
          const float2 p0 = __ffma2_rn(f2(s0.z, s0.w), f2(e_x), f2(s0.x, s0.y));
          const float2 p1 = __ffma2_rn(f2(s1.z, s1.w), f2(e_x), f2(s1.x, s1.y));
          const float2 p2 = __ffma2_rn(f2(s2.z, s2.w), f2(e_x), f2(s2.x, s2.y));
          const float2 o01 = __fadd2_rn(acc01, f2(__fmaf_rn(p0.y, lo(er[u >> 1], u), p0.x),
                                                  __fmaf_rn(p1.y, lo(eg[u >> 1], u), p1.x)));
          o0[u] = o01.x;
          o1[u] = o01.y;
          o2[u] = acc2 + __fmaf_rn(p2.y, lo(eb[u >> 1], u), p2.x);
          if (CHECK) bad |= !(isfinite(o0[u]) && isfinite(o1[u]) && isfinite(o2[u]));
        }
        if (LOSS) {  // gY = (Y - T) * 2/N, loss partial, max |gY| (pixels past the row end excluded)
#pragma unroll
          for (int u = 0; u < kPx; ++u) {
            const bool in_row = xl + u < p.w;
            const float r0 = o0[u] - tgt.r[u], r1 = o1[u] - tgt.g[u], r2 = o2[u] - tgt.b[u];
            o0[u] = r0 * p.gscale;
            o1[u] = r1 * p.gscale;
            o2[u] = r2 * p.gscale;
            if (in_row) {
              loss_acc = __fmaf_rn(r0, r0, __fmaf_rn(r1, r1, __fmaf_rn(r2, r2, loss_acc)));
              gmax_acc = fmaxf(gmax_acc, fmaxf(fabsf(o0[u]), fmaxf(fabsf(o1[u]), fabsf(o2[u]))));
            }
          }
        }
        Dst<OUTF>::template store<kPx>(dst, opl, y, xl, p.w, vec_out, o0, o1, o2);
        if (has_next) load(ny, nk);
        cy = ny;
        ck = nk;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8u * (n % kRing));
      if (y + kAhead <= y_last) {
        // buffer (n+kAhead) % kRing last held row n-1 (of this image segment
        // when y > y_first; otherwise the segment-start barrier covers it)
        if (y > y_first) mbar_wait(empty0 + 8u * ((n - 1) % kRing), ((n - 1) / kRing) & 1u);
        produce(n + kAhead, y + kAhead);
      }
    }
    nrow = n0 + (uint32_t)cnt;
    g_seg = g_img_end;
    if (LOSS) {  // this image's partials: warp reduction, one atomic per warp
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        loss_acc += __shfl_xor_sync(0xffffffffu, loss_acc, off);
        gmax_acc = fmaxf(gmax_acc, __shfl_xor_sync(0xffffffffu, gmax_acc, off));
      }
      if (lane == 0) {
        atomicAdd(p.loss + b, (double)loss_acc);
        atomicMax(reinterpret_cast<int*>(p.gmax) + b, __float_as_int(gmax_acc));  // gmax >= 0
      }
      loss_acc = 0.f;
      gmax_acc = 0.f;
    }
  }
  if (CHECK) {
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(p.nonfinite, 1);
  }
}

// dynamic shared memory of the kernel: staged planes + the slot ring
size_t fwd_smem_bytes(int dt, int ds) {
  const TableLayout L = TableLayout::make(dt, ds);
  return (size_t)staged_bytes(L) + kRing * (size_t)L.slot_entries() * 16;
}

int fwd_max_smem_bytes() { return kMaxSmemBytes - kSmemReserve; }

// Shared-memory carve-out granularity of the 256 KB L1/shared array (KB)
// and the L1 the texture-path planes want to stay resident in.
static int carveout_kb(size_t smem) {
  static const int kOpts[] = {0, 8, 16, 32, 64, 100, 132, 164, 196, 228};
  for (int o : kOpts)
    if ((size_t)o * 1024 >= smem + 1024) return o;
  return 228;
}

static int g_num_sms = 0;

template <int DT, int DS, int IN, int OUT>
static cudaError_t launch_dims(const FwdParams& p, bool check, int grid, size_t smem, cudaStream_t st) {
  auto kern = check ? fused_fwd_kernel<DT, DS, true, IN, OUT> : fused_fwd_kernel<DT, DS, false, IN, OUT>;
  // Function attributes are set once per (instantiation, device): the largest
  // dynamic shared memory any launch may request (tables + slots + the widest
  // column table), so concurrent launches / captured graphs never see the
  // limit lowered under them.  Setting them is not a stream operation.
  constexpr int kMaxDev = 64;
  static std::atomic<int> configured[kMaxDev][2];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= kMaxDev || configured[dev][check].load(std::memory_order_acquire) == 0) {
    const int maxsm = fwd_max_smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm);
    if (e != cudaSuccess) return e;
    if (dev < kMaxDev) configured[dev][check].store(1, std::memory_order_release);
  }
  // smallest carve-out that fits (a hint, not a limit): the rest of the
  // 256 KB array stays L1 for the texture-path planes
  static std::atomic<int> carve[kMaxDev][2];
  const int kb = carveout_kb(smem);
  if (dev < kMaxDev && carve[dev][check].load(std::memory_order_relaxed) != kb) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, (kb * 100 + 227) / 228);
    if (e != cudaSuccess) return e;
    carve[dev][check].store(kb, std::memory_order_relaxed);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kFwdWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  // Programmatic dependent launch: the kernel's prologue (barriers, L2
  // prefetch of its first input rows) may overlap the table-packing kernel
  // before it; every table read comes after griddepcontrol.wait.
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

template <int IN, int OUT>
static cudaError_t launch_fmt(const FwdParams& p, const TableLayout& L, bool chk, int grid, size_t smem,
                              cudaStream_t st) {
  if (L.dt == 33 && L.ds == 17) return launch_dims<33, 17, IN, OUT>(p, chk, grid, smem, st);
  if (IN == kF32 && OUT == kF32 && L.dt == 17 && L.ds == 8)
    return launch_dims<17, 8, IN, OUT>(p, chk, grid, smem, st);
  return launch_dims<0, 0, IN, OUT>(p, chk, grid, smem, st);
}

bool fused_fwd_formats_supported(int in_fmt, int out_fmt) {
  return in_fmt >= kF32 && in_fmt <= kU16 && out_fmt >= kF32 && out_fmt <= kU16;
}

static cudaError_t launch_fwd_impl(const void* in, int in_fmt, void* out, int out_fmt, int batch, int h,
                                   int w, int y0, int h_total, const float* tables, const TableLayout& L,
                                   int* nonfinite, cudaStream_t st, long long pl_in, long long pl_out,
                                   const float* target, double* loss, float* gmax, float gscale) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (g_num_sms == 0) {
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  FwdParams p;
  p.in = in;
  p.out = out;
  p.batch = batch;
  p.h = h;
  p.w = w;
  p.pl_in = pl_in > 0 ? pl_in : (long long)h * w;
  p.pl_out = pl_out > 0 ? pl_out : (long long)h * w;
  p.y0 = y0;
  p.tables = tables;
  p.L = L;
  p.rcp_w = 1.0 / (double)(w - 1);
  p.rcp_h = 1.0 / (double)(h_total - 1);
  p.nonfinite = nonfinite;
  p.target = target;
  p.loss = loss;
  p.gmax = gmax;
  p.gscale = gscale;
  const long long rows = (long long)batch * h;
  if (rows == 0 || w == 0) return cudaSuccess;
  cudaError_t e = table_texture(tables, (size_t)batch * L.bytes(), st, &p.tex, &p.tex_base);
  if (e != cudaSuccess) return e;
  long long grid = g_num_sms;
  const long long chunks = rows * ((w + kChunk - 1) / kChunk);
  if (grid > chunks) grid = chunks;
  const size_t smem = fwd_smem_bytes(L.dt, L.ds);
  const bool chk = nonfinite != nullptr;
  const int g = (int)grid;
  const int fmt = in_fmt * 3 + out_fmt;
  if (out_fmt == kL2Grad) {
    e = launch_fmt<kF32, kL2Grad>(p, L, chk, g, smem, st);
  } else {
    switch (fmt) {
      case kF32 * 3 + kF32: e = launch_fmt<kF32, kF32>(p, L, chk, g, smem, st); break;
      case kU8 * 3 + kU8: e = launch_fmt<kU8, kU8>(p, L, chk, g, smem, st); break;
      case kU16 * 3 + kU16: e = launch_fmt<kU16, kU16>(p, L, chk, g, smem, st); break;
      case kU8 * 3 + kF32: e = launch_fmt<kU8, kF32>(p, L, chk, g, smem, st); break;
      case kU16 * 3 + kF32: e = launch_fmt<kU16, kF32>(p, L, chk, g, smem, st); break;
      case kF32 * 3 + kU8: e = launch_fmt<kF32, kU8>(p, L, chk, g, smem, st); break;
      case kF32 * 3 + kU16: e = launch_fmt<kF32, kU16>(p, L, chk, g, smem, st); break;
      case kU8 * 3 + kU16: e = launch_fmt<kU8, kU16>(p, L, chk, g, smem, st); break;
      default: e = launch_fmt<kU16, kU8>(p, L, chk, g, smem, st); break;
    }
  }
  if (e != cudaSuccess) return e;
  return table_texture_used(p.tex, st);
}

cudaError_t launch_fused_fwd(const float* rgb, float* out, int batch, int h, int w, int y0,
                             int h_total, const float* tables, const TableLayout& L,
                             int* nonfinite, cudaStream_t st, long long pl_in, long long pl_out) {
  return launch_fwd_impl(rgb, kF32, out, kF32, batch, h, w, y0, h_total, tables, L, nonfinite, st, pl_in,
                         pl_out, nullptr, nullptr, nullptr, 0.f);
}

cudaError_t launch_fused_fwd_l2(const float* rgb, const float* target, float* gy, int batch, int h, int w,
                                int y0, int h_total, const float* tables, const TableLayout& L,
                                double* loss, float* gmax, float gscale, cudaStream_t st) {
  return launch_fwd_impl(rgb, kF32, gy, kL2Grad, batch, h, w, y0, h_total, tables, L, nullptr, st, 0, 0,
                         target, loss, gmax, gscale);
}

cudaError_t launch_fused_fwd_io(const void* in, int in_fmt, void* out, int out_fmt, int batch, int h,
                                int w, int y0, int h_total, const float* tables, const TableLayout& L,
                                int* nonfinite, cudaStream_t st, long long pl_in, long long pl_out) {
  if (!fused_fwd_formats_supported(in_fmt, out_fmt)) return cudaErrorInvalidValue;
  return launch_fwd_impl(in, in_fmt, out, out_fmt, batch, h, w, y0, h_total, tables, L, nonfinite, st,
                         pl_in, pl_out, nullptr, nullptr, nullptr, 0.f);
}

}  // namespace svdlut
