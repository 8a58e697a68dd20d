// svdlut_fwd.cu — K2: the fused slice + 2D-LUT apply forward (fast fp32 path).
//
// Replaces transform._fused_impl (reference transform.py:215-300).
//
// Design:
//   * One persistent CTA per SM (15 warps); LUT pairs rg, rb and the grid
//     block of one image (≈180 KB at d_t=33 / d_s=17) live in shared memory,
//     staged by TMA bulk copies (`cp.async.bulk`, mbarrier completion); pair
//     gb is gathered through the texture path, which runs beside the
//     shared-memory pipe.  A CTA owns a contiguous range of rows over
//     (image, row) and re-stages only when the range crosses an image.
//   * Warps take 128-pixel chunks of a row (lane = 4 consecutive pixels,
//     128-bit streaming loads/stores).  One thread per CTA bulk-prefetches
//     the input rows two rows ahead into L2 (`cp.async.bulk.prefetch.L2`), so
//     the chunk loads issued at the top of each chunk hit L2 and no registers
//     are spent on a register-level prefetch (measured: 73 -> 67.6 µs).
//   * Per pixel, all nine shared-memory gathers (rg, rb cells: 3 × LDS.128
//     each; one merged grid slot per channel) are issued back to back, the
//     three texture gathers of pair gb one pixel ahead.  LUT cells hold
//     channel-packed coefficients with the weights folded in:
//     v = A + B·a + C·b + D·a·b (channels 0/1 on the FP32x2 pipe).
//   * Grid terms: per row, the CTA interpolates xy + xc + yc along y into
//     merged slots {M, M', N, N'} per (x-cell, channel, guide cell) in a ring
//     of three row buffers (mbarrier handshakes, warps may drift by a row).
//   * Integer work stays on 32-bit shared addresses; the colour floor is an
//     add of 2^23 (svdlut_common.cuh), so the index bits feed IMADs directly.
//   * Streaming I/O: 24 B/pixel of HBM traffic (3 f32 in, 3 f32 out).  The
//     kernel is bound by the shared-memory pipe (~87% of active cycles, 1.6
//     wavefronts per pixel), not by HBM — DESIGN.md §3 has the budget.
#include <atomic>
#include <cstdint>
#include <mutex>
#include <vector>

#include "svdlut_common.cuh"
#include "svdlut_io.cuh"
#include "svdlut_internal.h"

namespace svdlut {

// Kernel shape (pixels per lane PX, warps per CTA NW) is a template choice;
// the default below is what launch_fused_fwd uses (FWD_PX / FWD_NW override
// it at build time for experiments).
#ifndef FWD_PX
#define FWD_PX 4
#endif
#ifndef FWD_NW
#define FWD_NW 15  // 15 x 128 px = 1920: divides 1080p / 4K / 8K rows exactly
#endif
#ifndef FWD_L2PF
#define FWD_L2PF 2  // rows of L2 prefetch distance for the input planes (0: off)
#endif
#ifndef FWD_REGPF
#define FWD_REGPF 0  // next chunk's pixels prefetched into registers under this chunk's math
#endif
#ifndef FWD_CHUNKSPLIT
#define FWD_CHUNKSPLIT 0  // 1: CTA ranges in 128-px chunks (balanced ends, but ~4% slower per CTA); 0: whole rows
#endif
constexpr int kPx = FWD_PX;
constexpr int kFwdWarps = FWD_NW;
constexpr int kChunk = 32 * kPx;
#ifndef FWD_RING
#define FWD_RING 4  // per-row grid slot buffers (warps may drift FWD_RING - 2 rows apart); 3: -2%, 5: +1% smooth but -1% noise
#endif
constexpr int kRing = FWD_RING;
constexpr int kAhead = kRing - 1;  // rows of slots produced ahead of the one being consumed
constexpr uint32_t kMagicBits = 0x4B000000u;  // bits of 2^23

struct FwdParams {
  const void* in;           // input samples (format IN of the kernel)
  void* out;                // output samples (format OUT)
  int batch, h, w;
  long long pl_in, pl_out;  // f32 plane strides in floats (h*w for packed images)
  int y0;                   // first row of this strip in an image of h_total rows
  const float* tables;
  TableLayout L;
  cudaTextureObject_t tex;  // float4 texels over the packed tables (pair gb reads)
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
  int col_smem;             // 1: column brackets come from a per-CTA smem table of t values
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
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
#ifndef FWD_GRID_SMEM
// 1: the grid block (xc, gxy, gyc; ~19 KB) is staged in shared memory with
// the LUT pairs; 0: the once-per-row slot production reads it from global
// memory through L1, which lowers the smem carve-out to 164 KB and leaves
// ~92 KB of L1 for the texture-path LUT pair
#define FWD_GRID_SMEM 1  // 0 measured slower (73.9 vs 70.1 us smooth, 153 vs 149 uniform)
#endif
#ifndef FWD_ILV
// 1 (f32 in/out): a lane's four pixels are x0 + lane + 32u (u = 0..3) instead
// of four consecutive ones, so the eight lanes of an LDS.128 phase hold eight
// neighbouring pixels (fewer distinct LUT cells per phase, fewer bank
// conflicts); loads / stores become coalesced 32-bit accesses.  Measured 4K:
// smooth 66.8 -> 73.2 us (32 B of spills), uniform noise 140.4 -> 128.9 us
#define FWD_ILV 0
#endif
#ifndef FWD_COLTAB_MAXW
// column brackets from a per-CTA shared-memory table for rows narrower than
// this, computed inline per pixel (one f64 multiply) for wider rows: the
// table's LDS costs shared-pipe wavefronts, the inline path ALU work; measured
// 4K smooth 67.6 -> 66.9 us inline, 8 x 1080p 155.1 -> 156.4 us inline
#define FWD_COLTAB_MAXW 2560
#endif
#ifndef FWD_BREUSE
// 1: the colour brackets of pair gb's axes (g, b), computed one pixel ahead
// for the texture gathers, are reused for pairs rg / rb instead of being
// recomputed (same cbracket, same values)
#define FWD_BREUSE 1
#endif
#ifndef FWD_TGT_LATE
// L2-loss epilogue: 1 loads the target chunk right before the epilogue (its
// 12 registers are not live across the pixel math, but the load latency is
// exposed: 8 x 1080p 214 vs 203 us, more spills); 0 loads it with the input
// chunk
#define FWD_TGT_LATE 0
#endif
#ifndef FWD_TEXDEP
#define FWD_TEXDEP 1  // next pixel's TLD index depends on this pixel's last LDS (see below)
#endif
#ifndef FWD_LDS_PLAIN
#define FWD_LDS_PLAIN 1
#endif
__device__ __forceinline__ float4 lds4(uint32_t a) {
#if FWD_LDS_PLAIN
  // an ordinary shared load (the scheduler may move it; still ordered
  // against the mbarrier waits, which clobber memory)
  return *reinterpret_cast<const float4*>(__cvta_shared_to_generic(a));
#else
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a));
  return v;
#endif
}
// Texture gather as volatile PTX: keeps the one-pixel-ahead issue order of the
// source (the compiler otherwise hoists all of a chunk's TLDs to its top and
// runs out of registers for the shared-memory gathers).
__device__ __forceinline__ float4 texv4(cudaTextureObject_t t, int i) {
  float4 v;
  asm volatile("tex.1d.v4.f32.s32 {%0,%1,%2,%3}, [%4, {%5}];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(t), "r"(i));
  return v;
}

// Colour bracket returning the 2^23-biased index bits (see svdlut_common.cuh).
__device__ __forceinline__ uint32_t cbracket(float q, float dm1, float dm2, float& delta) {
  const float t = fminf(__fmul_rz(q, dm1), dm2);
  const float m = __fadd_rz(t, 8388608.0f);
  delta = __fmaf_rn(q, dm1, -(m - 8388608.0f));
  return __float_as_uint(m);
}

// One LUT pair's contribution A + B a + (C + D a) b for the three channels;
// cell = {A0 A1 B0 B1 | C0 C1 D0 D1 | A2 B2 C2 D2} (cell_index in
// svdlut_common.cuh): channels 0/1 on the FP32x2 pipe.
template <bool FIRST>
__device__ __forceinline__ void cell_term(const float4& c0, const float4& c1, const float4& c2,
                                          float da, float db, float2& acc01, float& acc2) {
  const float2 a2 = make_float2(da, da);
  const float2 t = __ffma2_rn(make_float2(c0.z, c0.w), a2, make_float2(c0.x, c0.y));
  const float2 s = __ffma2_rn(make_float2(c1.z, c1.w), a2, make_float2(c1.x, c1.y));
  const float v2 = __fmaf_rn(db, __fmaf_rn(c2.w, da, c2.z), __fmaf_rn(c2.y, da, c2.x));
  if (FIRST) {
    acc01 = __ffma2_rn(s, make_float2(db, db), t);
    acc2 = v2;
  } else {
    acc01 = __ffma2_rn(s, make_float2(db, db), __fadd2_rn(t, acc01));
    acc2 += v2;
  }
}

// Merged grid slot {M, M', N, N'}: M + N ex + (M' + N' ex) ec.
__device__ __forceinline__ float slot_term(const float4& g, float ex, float ec) {
  const float2 pq = __ffma2_rn(make_float2(g.z, g.w), make_float2(ex, ex), make_float2(g.x, g.y));
  return __fmaf_rn(ec, pq.y, pq.x);
}

template <int PX>
struct ChunkIn {
  float r[PX], g[PX], b[PX];  // PX consecutive pixels per lane
};

// Grid part of one image's tables (shared memory copy; slot builds / wide path).
struct GridG {
  const float4* xc;   // [c][jx][jc] {A,B,C,D}
  const float* gxy;   // [a][b][3]
  const float* gyc;   // [c][a][b]
};

// Merged grid coefficients of channel c at (row bracket jy/ey, x-cell jx, guide cell jc):
//   {M, M', N, N'} with term = M + N*ex + (M' + N'*ex)*ec  (biases included)
__device__ __forceinline__ float4 grid_entry(const GridG& G, int ds, int c, int jx, int jc, int jy,
                                             float ey) {
  const float4 x = G.xc[(c * (ds - 1) + jx) * (ds - 1) + jc];
  const float* Y = G.gyc + c * ds * ds;
  const float y00 = Y[jy * ds + jc], y01 = Y[jy * ds + jc + 1];
  const float y10 = Y[(jy + 1) * ds + jc], y11 = Y[(jy + 1) * ds + jc + 1];
  const float q0 = __fmaf_rn(ey, y10 - y00, y00), q1 = __fmaf_rn(ey, y11 - y01, y01);
  const float* X = G.gxy;
  const float v00 = X[(jx * ds + jy) * 3 + c], v01 = X[(jx * ds + jy + 1) * 3 + c];
  const float v10 = X[((jx + 1) * ds + jy) * 3 + c];
  const float v11 = X[((jx + 1) * ds + jy + 1) * 3 + c];
  const float r0 = __fmaf_rn(ey, v01 - v00, v00), r1 = __fmaf_rn(ey, v11 - v10, v10);
  return make_float4(x.x + q0 + r0, x.z + (q1 - q0), x.y + (r1 - r0), x.w);
}

#ifndef FWD_TEX_RB
// 1: pair rb also through the texture path (not staged).  Measured 4K:
// smooth 66.8 -> 73.0 us, uniform noise 140 -> 314 us (the texture pipe and
// its L1 become the bound)
#define FWD_TEX_RB 0
#endif
// Shared-memory image of the tables: LUT pairs rg, rb then the grid block
// (xc, gxy, gyc); pair gb is read through the texture path.
__host__ __device__ inline uint32_t smem_grid_off(const TableLayout& L) {
  return (FWD_TEX_RB ? 1u : 2u) * (uint32_t)L.pair_floats * 4u;
}
__host__ __device__ inline uint32_t smem_tables_bytes(const TableLayout& L) {
  return smem_grid_off(L) + (FWD_GRID_SMEM ? (uint32_t)(L.lut2_off - L.xc_off) * 4u : 0u);
}

template <int DT, int DS, bool CHECK, int PX, int NW, int IN, int OUT>
__global__ void __launch_bounds__(NW * 32, 1) fused_fwd_kernel(FwdParams p) {
  static_assert(PX == 4 || (IN == kF32 && (OUT == kF32 || OUT == kL2Grad)),
                "integer formats use 4-pixel lanes");
  constexpr bool LOSS = OUT == kL2Grad;
  constexpr int OUTF = LOSS ? (int)kF32 : OUT;  // storage format of the output
  float loss_acc = 0.f, gmax_acc = 0.f;         // LOSS: this thread's partials
  constexpr int CH = 32 * PX;  // pixels per warp chunk
  constexpr bool ILV = FWD_ILV && PX == 4 && IN == kF32 && (OUT == kF32 || OUT == kL2Grad);
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t bar_storage;
  const int dt = DT ? DT : p.L.dt;
  const int ds = DS ? DS : p.L.ds;
  const TableLayout L = TableLayout::make(dt, ds);
  const uint32_t bar = smem_addr(&bar_storage);
  const uint32_t sbase = smem_addr(smem);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;

  // slot ring: full[i] completes when every warp wrote its share of the row in
  // buffer i, empty[i] when every warp finished reading it
  __shared__ __align__(8) uint64_t ring_bar[2 * kRing];
  const uint32_t full0 = smem_addr(&ring_bar[0]), empty0 = smem_addr(&ring_bar[kRing]);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    for (int i = 0; i < 2 * kRing; ++i) mbar_init(smem_addr(&ring_bar[i]), NW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const uint32_t lut_smem_bytes = smem_grid_off(L);
  const uint32_t table_bytes = smem_tables_bytes(L);
  const int nent = (ds - 1) * 3 * (ds - 1);                  // slot entries per row
  float4* slots = reinterpret_cast<float4*>(reinterpret_cast<char*>(smem) + table_bytes);
  // column table: t(x) = RN32(RN32(x/(W-1)) * (d_s-1)) for every column, built once
  float* col_t = reinterpret_cast<float*>(slots + kRing * nent);
  const uint32_t col_addr = smem_addr(col_t);
  if (p.col_smem) {
    const int wpad = (p.w + 3) & ~3;
    for (int x = threadIdx.x; x < wpad; x += blockDim.x) {
      const int xc = min(x, p.w - 1);
      col_t[x] = __fmul_rn(__double2float_rn(__dmul_rn((double)xc, p.rcp_w)), (float)(ds - 1));
    }
  }

  // inputs and tables may come from the previous kernel in the stream (PDL)
  asm volatile("griddepcontrol.wait;" ::: "memory");

  GridG G;
  auto set_grid = [&](const float* gsm) {  // gsm + table offset = grid block
    G.xc = reinterpret_cast<const float4*>(gsm + L.xc_off);
    G.gxy = gsm + L.gxy_off;
    G.gyc = gsm + L.gyc_off;
  };
  if (FWD_GRID_SMEM) set_grid(smem + lut_smem_bytes / 4 - L.xc_off);  // global offset -> smem

  const float tdm1 = (float)(dt - 1), tdm2 = (float)(dt - 2);
  const float sdm1 = (float)(ds - 1), sdm2 = (float)(ds - 2);
  const uint32_t cst48 = (uint32_t)L.cst * 48u;
  const uint32_t pair_bytes = (uint32_t)(dt - 1) * cst48;
  const uint32_t cst3 = (uint32_t)L.cst * 3u;
  // address = base + bits_a*cst48 + bits_b*48 with the 2^23 bias folded in
  const uint32_t lutK = sbase + (uint32_t)L.lut_off * 4u - kMagicBits * (cst48 + 48u);
  const uint32_t chan_bytes = (uint32_t)(ds - 1) * 16u;  // one channel of a slot row
  const uint32_t jx_bytes = 3u * chan_bytes;             // one x-cell of a slot row
  const uint32_t slot_row_bytes = (uint32_t)nent * 16u;
  const uint32_t slotK0 = smem_addr(slots) - kMagicBits * 16u;

  // contiguous range of global chunks g = (image b, row y) * cpr + k for this
  // CTA: rows r_begin .. r_end-1, the first and last possibly partial (whole
  // rows unless FWD_CHUNKSPLIT)
  const int cpr = (p.w + CH - 1) / CH;
#if FWD_CHUNKSPLIT
  const long long chunks_total = (long long)p.batch * p.h * cpr;
  const long long g_begin = (long long)blockIdx.x * chunks_total / gridDim.x;
  const long long g_end = (long long)(blockIdx.x + 1) * chunks_total / gridDim.x;
#else
  const long long rows_total = (long long)p.batch * p.h;
  const long long g_begin = (long long)blockIdx.x * rows_total / gridDim.x * cpr;
  const long long g_end = (long long)(blockIdx.x + 1) * rows_total / gridDim.x * cpr;
#endif
  const long long r_begin = g_begin / cpr;
  const long long r_end = (g_end + cpr - 1) / cpr;
  const int k_first = (int)(g_begin - r_begin * cpr);
  const int k_last = (int)(g_end - (r_end - 1) * cpr);  // exclusive, in the last row
  const long long pl = p.pl_in, opl = p.pl_out;  // plane strides (floats)
  const long long plane_len = (long long)p.h * p.w;
  const bool vec_in = ((p.w & 3) == 0) && Src<IN>::aligned(p.in, pl);
  const bool vec_out = ((p.w & 3) == 0) && Dst<OUTF>::aligned(p.out, opl) &&
                       (!LOSS || Src<kF32>::aligned(p.target, pl));
  uint32_t phase = 0;
  uint32_t nrow = 0;  // CTA row ordinal (slot ring position)
  bool bad = false;

  long long r = r_begin;
  while (r < r_end) {
    const int b = (int)(r / p.h);
    const int y_first = (int)(r - (long long)b * p.h);
    const int y_last = (int)(min(r_end, (long long)(b + 1) * p.h) - 1 - (long long)b * p.h);
    const float* tb = p.tables + (long long)b * L.total_floats;
    if (!FWD_GRID_SMEM) set_grid(tb);
    // ---- stage image b's tables into shared memory (TMA bulk copy) ----
    __syncthreads();  // every warp is done reading the previous image's tables
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_expect_tx(bar, table_bytes);
      const char* src = reinterpret_cast<const char*>(tb);
      for (uint32_t off = 0; off < lut_smem_bytes; off += 32768u)  // LUT pairs kept in smem
        bulk_g2s(sbase + off, src + off, min(32768u, lut_smem_bytes - off), bar);
      const char* gsrc = src + (size_t)L.xc_off * 4;
      const uint32_t gbytes = table_bytes - lut_smem_bytes;
      for (uint32_t off = 0; off < gbytes; off += 32768u)       // grid block
        bulk_g2s(sbase + lut_smem_bytes + off, gsrc + off, min(32768u, gbytes - off), bar);
    }
    const void* src = Src<IN>::image(p.in, b, pl);
    void* dst = Dst<OUTF>::image(p.out, b, opl);
    const void* tsrc = LOSS ? Src<kF32>::image(p.target, b, pl) : nullptr;
    // texel index of pair rb's cell (ir, ib) (FWD_TEX_RB) = texKrb + bits_r*cst3 + bits_b*3
    [[maybe_unused]] const uint32_t texKrb = (uint32_t)p.tex_base + (uint32_t)b * (uint32_t)(L.total_floats / 4) +
                                             (uint32_t)((L.lut_off + L.pair_floats) / 4) - kMagicBits * (cst3 + 3u);
    // texel index of pair gb's cell (ig, ib) = texK + bits_g*cst3 + bits_b*3
    const uint32_t texK = (uint32_t)p.tex_base + (uint32_t)b * (uint32_t)(L.total_floats / 4) +
                          (uint32_t)(L.lut2_off / 4) - kMagicBits * (cst3 + 3u);

    // chunk range [klo, khi) of row y of this segment; the warp takes
    // klo + warp, klo + warp + NW, ...
    // in 32-bit: the only rows with a partial chunk range are the CTA's first
    // (row yf of this segment, or none: -1) and last (yl, or beyond y_last)
    const long long rb0 = (long long)b * p.h;
    const int yf = r_begin - rb0 < 0 ? -1 : (int)(r_begin - rb0);
    const int yl = (int)min(r_end - 1 - rb0, (long long)p.h);
    auto klo = [&](int y) { return y == yf ? k_first : 0; };
    auto khi = [&](int y) { return y == yl ? k_last : cpr; };
    // move (y, k) forward to this warp's next chunk (y > y_last: none left)
    auto settle = [&](int& y, int& k) {
      while (y <= y_last && k >= khi(y)) {
        ++y;
        k = y <= y_last ? klo(y) + warp : 0;
      }
    };
    // the first chunk's loads overlap the table copy
    // chunk k of row y: the input, and the f32 target of the loss epilogue
    auto load_ilv = [&](const void* img, int y, int k, ChunkIn<PX>& c) {
      const float* pp = static_cast<const float*>(img) + (long long)y * p.w;
#pragma unroll
      for (int u = 0; u < PX; ++u) {
        const int xx = min(k * CH + lane + 32 * u, p.w - 1);
        c.r[u] = io_ld_f(pp + xx);
        c.g[u] = io_ld_f(pp + pl + xx);
        c.b[u] = io_ld_f(pp + 2 * pl + xx);
      }
    };
    auto load_chunk = [&](const void* img, int y, int k, bool vec, ChunkIn<PX>& c) {
      if constexpr (ILV) load_ilv(img, y, k, c);
      else Src<IN>::template load<PX>(img, pl, y, k * CH + PX * lane, p.w, vec, c.r, c.g, c.b);
    };
    auto load_target = [&](const void* img, int y, int k, bool vec, ChunkIn<PX>& c) {
      if constexpr (ILV) load_ilv(img, y, k, c);
      else Src<kF32>::template load<PX>(img, pl, y, k * CH + PX * lane, p.w, vec, c.r, c.g, c.b);
    };
    ChunkIn<PX> cur, tgt;
    int cur_y = y_first, cur_k = klo(y_first) + warp;
    settle(cur_y, cur_k);
    if (cur_y <= y_last) {
      load_chunk(src, cur_y, cur_k, vec_in, cur);
      if (LOSS && !FWD_TGT_LATE)
        load_target(tsrc, cur_y, cur_k, vec_out, tgt);
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
#ifdef FWD_DBG_TIMES
    if (CHECK && threadIdx.x == 0 && r == r_begin) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      reinterpret_cast<unsigned long long*>(p.nonfinite + 2)[2 * blockIdx.x] = t;
    }
#endif
    // This warp's share of the slots of row y (CTA row ordinal n) into ring
    // buffer n % kRing.  Row n+kAhead is produced once row n is done, so warps
    // may drift apart instead of meeting at a CTA barrier every row.
    // x-cell of column x (the per-pixel rule: floor(min(t, d_s - 2)))
    auto jx_of = [&](int x) -> int {
      if (p.col_smem) return (int)floorf(fminf(col_t[x], sdm2));
      float e;
      return (int)(col_bracket(x, p.rcp_w, sdm1, sdm2, e) - kMagicBits);
    };
    auto produce = [&](uint32_t n, int y) {
      float ey;
      const int jy = (int)(row_bracket(p.y0 + y, p.rcp_h, sdm1, sdm2, ey) - kMagicBits);
      float4* S = slots + (n % kRing) * nent;
      // only the x-cells this CTA's chunks of row y touch (all of them for a
      // full row; a partial first / last row of a chunk range needs fewer)
      int e_lo = 0, e_hi = nent;  // a full row touches every x-cell
      if (y == yf || y == yl) {
        const int x_lo = klo(y) * CH, x_hi = min(khi(y) * CH, p.w) - 1;
        e_lo = x_hi >= x_lo ? jx_of(x_lo) * 3 * (ds - 1) : 0;
        e_hi = x_hi >= x_lo ? (jx_of(x_hi) + 1) * 3 * (ds - 1) : 0;
      }
      for (int e = e_lo + warp * 32 + lane; e < e_hi; e += NW * 32) {
        const int jx = e / (3 * (ds - 1)), rem = e - jx * 3 * (ds - 1);
        const int ch = rem / (ds - 1), jc = rem - ch * (ds - 1);
        S[e] = grid_entry(G, ds, ch, jx, jc, jy, ey);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(full0 + 8u * (n % kRing));
    };
    const uint32_t n0 = nrow;
    const int cnt = y_last - y_first + 1;
    for (int i = 0; i < kAhead && i < cnt; ++i) produce(n0 + i, y_first + i);

    for (int y = y_first; y <= y_last; ++y) {
      const uint32_t n = n0 + (uint32_t)(y - y_first);
      if (FWD_L2PF > 0 && threadIdx.x == blockDim.x - 32) {
        if (y == y_first)
          for (int yy = y + 1; yy < y + FWD_L2PF && yy <= y_last; ++yy) {
            Src<IN>::prefetch_row(src, pl, plane_len, yy, p.w);
            if (LOSS) Src<kF32>::prefetch_row(tsrc, pl, plane_len, yy, p.w);
          }
        if (y + FWD_L2PF <= y_last) {
          Src<IN>::prefetch_row(src, pl, plane_len, y + FWD_L2PF, p.w);
          if (LOSS) Src<kF32>::prefetch_row(tsrc, pl, plane_len, y + FWD_L2PF, p.w);
        }
      }
      mbar_wait(full0 + 8u * (n % kRing), (n / kRing) & 1u);
      const uint32_t slotK = slotK0 + (n % kRing) * slot_row_bytes;
      // ---- this warp's chunks of row y: k = warp, warp + W, ... ----
      for (; cur_y == y;) {
        ChunkIn<PX> nxt;
        int nxt_y = cur_y, nxt_k = cur_k + NW;
        settle(nxt_y, nxt_k);
#if FWD_REGPF
        if (nxt_y <= y_last)
          load_chunk(src, nxt_y, nxt_k, vec_in, nxt);
#endif

        const int xl = cur_k * CH + PX * lane;
        // x of this lane's pixel u
        auto xof = [&](int u) { return ILV ? cur_k * CH + lane + 32 * u : xl + u; };
        int jxs[PX];
        float exs[PX];
        if (p.col_smem) {
          float ts[PX];
          if (ILV) {
#pragma unroll
            for (int u = 0; u < PX; ++u) ts[u] = col_t[min(xof(u), p.w - 1)];
          } else if (PX == 4) {
            // lanes past the row end read the last (in-bounds) group; their
            // pixels are never stored
            const int xt = min(xl, ((p.w + 3) & ~3) - 4);
            const float4 t4 = lds4(col_addr + (uint32_t)xt * 4u);
            ts[0] = t4.x; ts[PX > 1 ? 1 : 0] = t4.y; ts[PX > 2 ? 2 : 0] = t4.z; ts[PX > 3 ? 3 : 0] = t4.w;
          } else {
#pragma unroll
            for (int u = 0; u < PX; ++u) ts[u] = col_t[min(xl + u, p.w - 1)];
          }
#pragma unroll
          for (int u = 0; u < PX; ++u) {
            const float m = __fadd_rz(fminf(ts[u], sdm2), 8388608.0f);
            exs[u] = ts[u] - (m - 8388608.0f);
            jxs[u] = (int)(__float_as_uint(m) - kMagicBits);
          }
        } else {
#pragma unroll
          for (int u = 0; u < PX; ++u)
            jxs[u] = (int)(col_bracket(min(xof(u), p.w - 1), p.rcp_w, sdm1, sdm2, exs[u]) - kMagicBits);
        }

        // Pair gb is gathered through the texture path one pixel ahead of its
        // use (software pipeline depth 1), hiding the texture latency behind
        // the shared-memory work of the previous pixel.
        float o0[PX], o1[PX], o2[PX];
        float4 tx0, tx1, tx2;  // in-flight texture cells of the next pixel
        float tdg, tdb;        // its deltas
        uint32_t nbg, nbb;     // and its colour brackets (g, b)
        {
          nbg = cbracket(__saturatef(cur.g[0]), tdm1, tdm2, tdg);
          nbb = cbracket(__saturatef(cur.b[0]), tdm1, tdm2, tdb);
          const int ti = (int)(nbg * cst3 + nbb * 3u + texK);
          tx0 = texv4(p.tex, ti);
          tx1 = texv4(p.tex, ti + 1);
          tx2 = texv4(p.tex, ti + 2);
        }
#pragma unroll
        for (int u = 0; u < PX; ++u) {
          const float4 c0 = tx0, c1 = tx1, c2 = tx2;
          const float dg = tdg, db = tdb;
          const float qr = __saturatef(cur.r[u]), qg = __saturatef(cur.g[u]),
                      qb = __saturatef(cur.b[u]);
          float dr, dg_, db_;
          const uint32_t br = cbracket(qr, tdm1, tdm2, dr);
#if FWD_BREUSE
          const uint32_t bg = nbg, bb = nbb;
          dg_ = dg;
          db_ = db;
#else
          const uint32_t bg = cbracket(qg, tdm1, tdm2, dg_);
          const uint32_t bb = cbracket(qb, tdm1, tdm2, db_);
#endif
          float er, eg, eb;
          const uint32_t sr = cbracket(qr, sdm1, sdm2, er);
          const uint32_t sg = cbracket(qg, sdm1, sdm2, eg);
          const uint32_t sb = cbracket(qb, sdm1, sdm2, eb);
          const uint32_t ur = br * cst48 + lutK;
          const uint32_t ag = ur + bg * 48u, ab = ur + bb * 48u + pair_bytes;
          const uint32_t sa = slotK + (uint32_t)jxs[u] * jx_bytes;
          // every shared-memory gather of the pixel back to back (lds4 is
          // volatile, so program order is issue order): nine LDS.128 in
          // flight per warp instead of one cell's three at a time
          const float4 rg0 = lds4(ag), rg1 = lds4(ag + 16), rg2 = lds4(ag + 32);
#if FWD_TEX_RB
          const int tr = (int)(br * cst3 + bb * 3u + texKrb);
          const float4 rb0 = texv4(p.tex, tr), rb1 = texv4(p.tex, tr + 1), rb2 = texv4(p.tex, tr + 2);
          (void)ab;
#else
          const float4 rb0 = lds4(ab), rb1 = lds4(ab + 16), rb2 = lds4(ab + 32);
#endif
          const float4 s0 = lds4(sa + sr * 16u);
          const float4 s1 = lds4(sa + chan_bytes + sg * 16u);
          const float4 s2 = lds4(sa + 2u * chan_bytes + sb * 16u);
          if (u + 1 < PX) {
            // next pixel's texture gathers, issued after this pixel's shared
            // gathers: the index carries a (never taken) dependency on the
            // last LDS so ptxas cannot hoist every TLD of the chunk to its top
            // (which starves the LDS of registers)
            nbg = cbracket(__saturatef(cur.g[u + 1]), tdm1, tdm2, tdg);
            nbb = cbracket(__saturatef(cur.b[u + 1]), tdm1, tdm2, tdb);
            const int ti = (int)(nbg * cst3 + nbb * 3u + texK) + (FWD_TEXDEP && s2.w != s2.w ? 1 : 0);
            tx0 = texv4(p.tex, ti);
            tx1 = texv4(p.tex, ti + 1);
            tx2 = texv4(p.tex, ti + 2);
          }
          float2 acc01;
          float acc2;
          cell_term<true>(rg0, rg1, rg2, dr, dg_, acc01, acc2);    // pair rg (shared memory)
          cell_term<false>(rb0, rb1, rb2, dr, db_, acc01, acc2);   // pair rb (shared memory)
          cell_term<false>(c0, c1, c2, dg, db, acc01, acc2);       // pair gb (texture path)
          // grids: one merged (xy + xc + yc) coefficient cell per channel
          const float ex = exs[u];
          o0[u] = acc01.x + slot_term(s0, ex, er);
          o1[u] = acc01.y + slot_term(s1, ex, eg);
          o2[u] = acc2 + slot_term(s2, ex, eb);
          if (CHECK) bad |= !(isfinite(o0[u]) && isfinite(o1[u]) && isfinite(o2[u]));
        }
        if (LOSS) {  // gY = (Y - T) * 2/N, loss partial, max |gY| (pixels past the row end excluded)
          if (FWD_TGT_LATE)
            Src<kF32>::template load<PX>(tsrc, pl, cur_y, xl, p.w, vec_out, tgt.r, tgt.g, tgt.b);
#pragma unroll
          for (int u = 0; u < PX; ++u) {
            const bool in_row = xof(u) < p.w;
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
        if constexpr (ILV) {
          float* pp = static_cast<float*>(dst) + (long long)cur_y * p.w;
#pragma unroll
          for (int u = 0; u < PX; ++u)
            if (xof(u) < p.w) {
              __stcs(pp + xof(u), o0[u]);
              __stcs(pp + opl + xof(u), o1[u]);
              __stcs(pp + 2 * opl + xof(u), o2[u]);
            }
        } else {
          Dst<OUTF>::template store<PX>(dst, opl, cur_y, xl, p.w, vec_out, o0, o1, o2);
        }
#if FWD_REGPF
        cur = nxt;
#else
        if (nxt_y <= y_last) {
          load_chunk(src, nxt_y, nxt_k, vec_in, cur);
          if (LOSS && !FWD_TGT_LATE)
            load_target(tsrc, nxt_y, nxt_k, vec_out, tgt);
        }
#endif
        cur_y = nxt_y;
        cur_k = nxt_k;
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
    r += y_last - y_first + 1;
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
#ifdef FWD_DBG_TIMES
  __syncthreads();
  if (CHECK && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    reinterpret_cast<unsigned long long*>(p.nonfinite + 2)[2 * blockIdx.x + 1] = t;
  }
#endif
}

size_t fwd_smem_bytes(int dt, int ds) {
  const TableLayout L = TableLayout::make(dt, ds);
  // staged tables + double-buffered per-row grid slots [jx][c][jc] (float4)
  return (size_t)smem_tables_bytes(L) + kRing * (size_t)(ds - 1) * 3 * (ds - 1) * 16;
}

// Keep at least this much of the 256 KB L1/shared array as L1 so the
// texture-path LUT pair stays resident; the column table is added only if it
// fits under the limit.
constexpr size_t kSmemForL1Tex = 196 * 1024 - 2048;

int fwd_max_smem_bytes() { return kMaxSmemBytes - kSmemReserve; }

static int g_num_sms = 0;

// ---- texture objects over packed-table buffers --------------------------------
// One linear float4 texture per (device, buffer, size), cached; evicted
// objects are destroyed only after an event recorded behind their last use
// has completed, so kernels still in flight never lose their texture.
namespace {
struct TexEntry {
  int dev;
  const void* base;
  size_t bytes;
  cudaTextureObject_t tex;
  cudaEvent_t last_use;
  unsigned long long stamp;
  bool pinned;  // referenced by a captured CUDA graph: never retired
};
struct TexRetired {
  cudaTextureObject_t tex;
  cudaEvent_t ev;
};
std::mutex g_tex_mu;
std::vector<TexEntry> g_tex;
std::vector<TexRetired> g_tex_retired;
unsigned long long g_tex_clock = 0;
constexpr size_t kTexCache = 32;

void reap_retired() {
  for (size_t i = 0; i < g_tex_retired.size();) {
    if (cudaEventQuery(g_tex_retired[i].ev) == cudaSuccess) {
      cudaDestroyTextureObject(g_tex_retired[i].tex);
      cudaEventDestroy(g_tex_retired[i].ev);
      g_tex_retired[i] = g_tex_retired.back();
      g_tex_retired.pop_back();
    } else {
      cudaGetLastError();  // clear cudaErrorNotReady
      ++i;
    }
  }
}

bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cs != cudaStreamCaptureStatusNone;
}

// Texture over [base, base + bytes); base must be textureAlignment-aligned.
// During stream capture no events are queried or recorded and the entry is
// pinned, since the graph keeps using the texture object on every replay.
cudaError_t tex_for(int dev, const void* base, size_t bytes, cudaStream_t st, cudaTextureObject_t* out) {
  std::lock_guard<std::mutex> lock(g_tex_mu);
  const bool cap = capturing(st);
  if (!cap) reap_retired();
  TexEntry* hit = nullptr;
  for (auto& e : g_tex)
    if (e.dev == dev && e.base == base && e.bytes == bytes) hit = &e;
  if (!hit) {
    if (g_tex.size() >= kTexCache) {  // retire the least recently used unpinned entry
      long lru = -1;
      for (size_t i = 0; i < g_tex.size(); ++i)
        if (!g_tex[i].pinned && (lru < 0 || g_tex[i].stamp < g_tex[lru].stamp)) lru = (long)i;
      if (lru >= 0) {
        g_tex_retired.push_back({g_tex[lru].tex, g_tex[lru].last_use});
        g_tex[lru] = g_tex.back();
        g_tex.pop_back();
      }
    }
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = const_cast<void*>(base);
    rd.res.linear.desc = cudaCreateChannelDesc<float4>();
    rd.res.linear.sizeInBytes = bytes;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    TexEntry e{dev, base, bytes, 0, nullptr, 0, false};
    cudaError_t err = cudaCreateTextureObject(&e.tex, &rd, &td, nullptr);
    if (err != cudaSuccess) return err;
    err = cudaEventCreateWithFlags(&e.last_use, cudaEventDisableTiming);
    if (err != cudaSuccess) return err;
    g_tex.push_back(e);
    hit = &g_tex.back();
  }
  hit->stamp = ++g_tex_clock;
  hit->pinned |= cap;
  *out = hit->tex;
  return cudaSuccess;
}

// Marks the texture's last use after the launch just issued on `st`.
cudaError_t tex_mark_used(cudaTextureObject_t tex, cudaStream_t st) {
  if (capturing(st)) return cudaSuccess;
  std::lock_guard<std::mutex> lock(g_tex_mu);
  for (auto& t : g_tex)
    if (t.tex == tex) return cudaEventRecord(t.last_use, st);
  return cudaSuccess;
}
}  // namespace

// Texture object over a batch of packed tables (also used by the backward).
cudaError_t fwd_texture(const float* tables, int batch, const TableLayout& L, cudaStream_t st,
                        cudaTextureObject_t* tex, int* tex_base) {
  int dev = 0;
  cudaGetDevice(&dev);
  int talign = 512;
  cudaDeviceGetAttribute(&talign, cudaDevAttrTextureAlignment, dev);
  const uintptr_t tb = reinterpret_cast<uintptr_t>(tables);
  const uintptr_t base = tb / (uintptr_t)talign * (uintptr_t)talign;
  const size_t bytes = (size_t)(tb - base) + (size_t)batch * L.bytes();
  *tex_base = (int)((tb - base) / 16);
  return tex_for(dev, reinterpret_cast<const void*>(base), bytes, st, tex);
}

cudaError_t fwd_texture_used(cudaTextureObject_t tex, cudaStream_t st) { return tex_mark_used(tex, st); }

template <int DT, int DS, int IN, int OUT>
static cudaError_t launch_dims(const FwdParams& p, bool check, int grid, size_t smem,
                               cudaStream_t st) {
  auto kern = check ? fused_fwd_kernel<DT, DS, true, kPx, kFwdWarps, IN, OUT>
                    : fused_fwd_kernel<DT, DS, false, kPx, kFwdWarps, IN, OUT>;
  // function attributes are set once per (instantiation, device, smem size);
  // setting them is not a stream operation, so graph capture does not see it
  constexpr int kMaxDev = 64;
  static std::atomic<size_t> configured[kMaxDev][2];
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<size_t>* seen = dev < kMaxDev ? &configured[dev][check] : nullptr;
  cudaError_t e = cudaSuccess;
  if (!seen || seen->load(std::memory_order_relaxed) != smem) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // smallest shared-memory carve-out that fits: the rest of the 256 KB stays
    // L1 for the texture-path LUT pair
    const int pct = (int)((smem + 2048 + (228 * 1024 - 1)) * 100 / (228 * 1024)) + 1;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct > 100 ? 100 : pct);
    if (e != cudaSuccess) return e;
    if (seen) seen->store(smem, std::memory_order_relaxed);
  }
  // Programmatic dependent launch: the kernel's prologue (barriers, column
  // table) may overlap the tail of the table-packing kernel before it; every
  // global access comes after griddepcontrol.wait.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kFwdWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
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
  if (in_fmt < kF32 || in_fmt > kU16 || out_fmt < kF32 || out_fmt > kU16) return false;
  if (in_fmt == kF32 && out_fmt == kF32) return true;
  return kPx == 4;
}

cudaError_t launch_fused_fwd(const float* rgb, float* out, int batch, int h, int w, int y0,
                             int h_total, const float* tables, const TableLayout& L,
                             int* nonfinite, cudaStream_t st, long long pl_in, long long pl_out) {
  return launch_fused_fwd_io(rgb, kF32, out, kF32, batch, h, w, y0, h_total, tables, L, nonfinite,
                             st, pl_in, pl_out);
}

static cudaError_t launch_fwd_impl(const void* in, int in_fmt, void* out, int out_fmt, int batch, int h,
                                   int w, int y0, int h_total, const float* tables, const TableLayout& L,
                                   int* nonfinite, cudaStream_t st, long long pl_in, long long pl_out,
                                   const float* target, double* loss, float* gmax, float gscale);

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
  // texture over the whole batch of tables, base aligned down to textureAlignment
  int talign = 512;
  cudaDeviceGetAttribute(&talign, cudaDevAttrTextureAlignment, dev);
  const uintptr_t tb = reinterpret_cast<uintptr_t>(tables);
  const uintptr_t base = tb / (uintptr_t)talign * (uintptr_t)talign;
  const size_t bytes = (size_t)(tb - base) + (size_t)batch * L.bytes();
  p.tex_base = (int)((tb - base) / 16);
  cudaError_t e = tex_for(dev, reinterpret_cast<const void*>(base), bytes, st, &p.tex);
  if (e != cudaSuccess) return e;
  long long grid = g_num_sms;
  const long long chunks = rows * ((w + kChunk - 1) / kChunk);
  if (grid > chunks) grid = chunks;
  size_t smem = fwd_smem_bytes(L.dt, L.ds);
  const size_t col_bytes = (size_t)((w + 3) & ~3) * 4;
  p.col_smem = w < FWD_COLTAB_MAXW && smem + col_bytes <= kSmemForL1Tex ? 1 : 0;
  if (p.col_smem) smem += col_bytes;
  const bool chk = nonfinite != nullptr;
  const int g = (int)grid;
  const int fmt = in_fmt * 3 + out_fmt;
  if (out_fmt == kL2Grad) {
    e = launch_fmt<kF32, kL2Grad>(p, L, chk, g, smem, st);
  } else if (fmt == kF32 * 3 + kF32) {
    e = launch_fmt<kF32, kF32>(p, L, chk, g, smem, st);
  } else {
#if FWD_PX == 4
    switch (fmt) {
      case kU8 * 3 + kU8: e = launch_fmt<kU8, kU8>(p, L, chk, g, smem, st); break;
      case kU16 * 3 + kU16: e = launch_fmt<kU16, kU16>(p, L, chk, g, smem, st); break;
      case kU8 * 3 + kF32: e = launch_fmt<kU8, kF32>(p, L, chk, g, smem, st); break;
      case kU16 * 3 + kF32: e = launch_fmt<kU16, kF32>(p, L, chk, g, smem, st); break;
      case kF32 * 3 + kU8: e = launch_fmt<kF32, kU8>(p, L, chk, g, smem, st); break;
      case kF32 * 3 + kU16: e = launch_fmt<kF32, kU16>(p, L, chk, g, smem, st); break;
      case kU8 * 3 + kU16: e = launch_fmt<kU8, kU16>(p, L, chk, g, smem, st); break;
      default: e = launch_fmt<kU16, kU8>(p, L, chk, g, smem, st); break;
    }
#else
    e = cudaErrorInvalidValue;
#endif
  }
  if (e != cudaSuccess) return e;
  return tex_mark_used(p.tex, st);
}

}  // namespace svdlut
