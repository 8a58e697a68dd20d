// svdlut_fwd.cu — K2: the fused slice + 2D-LUT apply forward (fast fp32 path).
//
// Replaces transform._fused_impl (reference transform.py:215-300).
//
// Design:
//   * One persistent CTA per SM (the packed tables of one image, ≈187 KB at
//     d_t=33 / d_s=17, live in shared memory; staged by a TMA bulk copy
//     `cp.async.bulk` completing on an mbarrier).
//   * Work = 128-pixel row chunks over (image, row, chunk), split into one
//     contiguous range per CTA; a CTA re-stages tables only when its range
//     crosses into the next image.  Warps take chunks round-robin and
//     software-pipeline the next chunk's global loads under the current
//     chunk's math.
//   * Per pixel: 6 brackets, 9 LUT terms as 3 channel-packed coefficient
//     cells (3×LDS.128 each), 1 channel-packed xy cell (3×LDS.128) and one
//     xc + one yc cell per output channel (LDS.128 each); every term is
//     v = A + B·a + C·b + D·a·b with weights folded in by the prologue.
//   * Streaming I/O: 24 B/pixel of HBM traffic (3 f32 in, 3 f32 out).
#include <cstdint>
#include "svdlut_common.cuh"
#include "svdlut_internal.h"

namespace svdlut {

constexpr int kFwdWarps = 16;
constexpr int kPx = 4;              // pixels per lane per chunk
constexpr int kChunk = 32 * kPx;    // pixels per warp chunk

struct FwdParams {
  const float* rgb;
  float* out;
  int h, w;
  const float* tables;
  TableLayout L;
  const SpatialBr* col;
  const SpatialBr* row;
  int cpr;             // chunks per row
  long long per_img;   // h * cpr
  long long total;     // batch * h * cpr
  int* nonfinite;
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

// v += A + B*a + C*b + D*a*b for 3 packed channels: cell = {A0 A1 A2 B0|B1 B2 C0 C1|C2 D0 D1 D2}
__device__ __forceinline__ void cell3(const float* cellp, float a, float b, float& o0, float& o1,
                                      float& o2) {
  const float4* q = reinterpret_cast<const float4*>(cellp);
  const float4 c0 = q[0], c1 = q[1], c2 = q[2];
  o0 += __fmaf_rn(b, __fmaf_rn(c2.y, a, c1.z), __fmaf_rn(c0.w, a, c0.x));
  o1 += __fmaf_rn(b, __fmaf_rn(c2.z, a, c1.w), __fmaf_rn(c1.x, a, c0.y));
  o2 += __fmaf_rn(b, __fmaf_rn(c2.w, a, c2.x), __fmaf_rn(c1.y, a, c0.z));
}
// v = A + B*a + C*b + D*a*b for one channel cell {A,B,C,D}
__device__ __forceinline__ float cell1(const float* cellp, float a, float b) {
  const float4 c = *reinterpret_cast<const float4*>(cellp);
  return __fmaf_rn(b, __fmaf_rn(c.w, a, c.z), __fmaf_rn(c.y, a, c.x));
}

struct PixCtx {
  const float* lut0;  // pair rg base
  const float* lut1;  // pair rb base
  const float* lut2;  // pair gb base
  const float* xy;
  const float* xc;    // channel 0 base; channel c at + c*xcs
  const float* yc;
  int cst, css, xcs;
  float tdm1, tdm2, sdm1, sdm2;
};

__device__ __forceinline__ void apply_pixel(const PixCtx& C, float r, float g, float bl, int jx,
                                            float ex, int jy, float ey, float& o0, float& o1,
                                            float& o2) {
  const float qr = clamp01(r), qg = clamp01(g), qb = clamp01(bl);
  int ir, ig, ib;
  float dr, dg, db;
  color_bracket(qr, C.tdm1, C.tdm2, ir, dr);
  color_bracket(qg, C.tdm1, C.tdm2, ig, dg);
  color_bracket(qb, C.tdm1, C.tdm2, ib, db);
  o0 = 0.f;
  o1 = 0.f;
  o2 = 0.f;
  cell3(C.lut0 + (ir * C.cst + ig) * 12, dr, dg, o0, o1, o2);
  cell3(C.lut1 + (ir * C.cst + ib) * 12, dr, db, o0, o1, o2);
  cell3(C.lut2 + (ig * C.cst + ib) * 12, dg, db, o0, o1, o2);
  cell3(C.xy + (jx * C.css + jy) * 12, ex, ey, o0, o1, o2);
  int jr, jg, jb;
  float er, eg, eb;
  color_bracket(qr, C.sdm1, C.sdm2, jr, er);
  color_bracket(qg, C.sdm1, C.sdm2, jg, eg);
  color_bracket(qb, C.sdm1, C.sdm2, jb, eb);
  o0 += cell1(C.xc + (jx * C.css + jr) * 4, ex, er);
  o1 += cell1(C.xc + C.xcs + (jx * C.css + jg) * 4, ex, eg);
  o2 += cell1(C.xc + 2 * C.xcs + (jx * C.css + jb) * 4, ex, eb);
  o0 += cell1(C.yc + (jy * C.css + jr) * 4, ey, er);
  o1 += cell1(C.yc + C.xcs + (jy * C.css + jg) * 4, ey, eg);
  o2 += cell1(C.yc + 2 * C.xcs + (jy * C.css + jb) * 4, ey, eb);
}

// Inputs of one 128-pixel chunk for one lane.
struct ChunkIn {
  float r[kPx], g[kPx], b[kPx];
  int jx[kPx];
  float ex[kPx];
};

// INTERLEAVE=false: lane owns 4 consecutive pixels (128-bit loads/stores).
// INTERLEAVE=true : lane owns pixels lane + 32u (32-bit loads, a warp
//                   instruction covers 32 consecutive pixels — better
//                   shared-memory locality on smooth images).
template <bool INTERLEAVE>
__device__ __forceinline__ void load_chunk(const FwdParams& p, const float* plane0, long long rowoff,
                                           int x0, int lane, bool vec_ok, ChunkIn& in) {
  const long long pl = (long long)p.h * p.w;
  if (!INTERLEAVE) {
    const int x = x0 + lane * kPx;
    if (vec_ok && x + kPx <= p.w) {
      const float4 r4 = __ldcs(reinterpret_cast<const float4*>(plane0 + rowoff + x));
      const float4 g4 = __ldcs(reinterpret_cast<const float4*>(plane0 + pl + rowoff + x));
      const float4 b4 = __ldcs(reinterpret_cast<const float4*>(plane0 + 2 * pl + rowoff + x));
      in.r[0] = r4.x; in.r[1] = r4.y; in.r[2] = r4.z; in.r[3] = r4.w;
      in.g[0] = g4.x; in.g[1] = g4.y; in.g[2] = g4.z; in.g[3] = g4.w;
      in.b[0] = b4.x; in.b[1] = b4.y; in.b[2] = b4.z; in.b[3] = b4.w;
      const int4 c01 = __ldg(reinterpret_cast<const int4*>(p.col + x));
      const int4 c23 = __ldg(reinterpret_cast<const int4*>(p.col + x + 2));
      in.jx[0] = c01.x; in.ex[0] = __int_as_float(c01.y);
      in.jx[1] = c01.z; in.ex[1] = __int_as_float(c01.w);
      in.jx[2] = c23.x; in.ex[2] = __int_as_float(c23.y);
      in.jx[3] = c23.z; in.ex[3] = __int_as_float(c23.w);
    } else {
#pragma unroll
      for (int u = 0; u < kPx; ++u) {
        const int xx = min(x + u, p.w - 1);
        in.r[u] = __ldcs(plane0 + rowoff + xx);
        in.g[u] = __ldcs(plane0 + pl + rowoff + xx);
        in.b[u] = __ldcs(plane0 + 2 * pl + rowoff + xx);
        const SpatialBr c = p.col[xx];
        in.jx[u] = c.i;
        in.ex[u] = c.d;
      }
    }
  } else {
#pragma unroll
    for (int u = 0; u < kPx; ++u) {
      const int xx = min(x0 + lane + 32 * u, p.w - 1);
      in.r[u] = __ldcs(plane0 + rowoff + xx);
      in.g[u] = __ldcs(plane0 + pl + rowoff + xx);
      in.b[u] = __ldcs(plane0 + 2 * pl + rowoff + xx);
      const SpatialBr c = p.col[xx];
      in.jx[u] = c.i;
      in.ex[u] = c.d;
    }
  }
}

template <bool INTERLEAVE, bool CHECK>
__global__ void __launch_bounds__(kFwdWarps * 32, 1) fused_fwd_kernel(FwdParams p) {
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t bar_storage;
  const uint32_t bar = smem_addr(&bar_storage);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const TableLayout& L = p.L;

  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  PixCtx C;
  C.lut0 = smem + L.lut_off;
  C.lut1 = C.lut0 + (L.dt - 1) * L.cst * 12;
  C.lut2 = C.lut1 + (L.dt - 1) * L.cst * 12;
  C.xy = smem + L.xy_off;
  C.xc = smem + L.xc_off;
  C.yc = smem + L.yc_off;
  C.cst = L.cst;
  C.css = L.css;
  C.xcs = (L.ds - 1) * L.css * 4;
  C.tdm1 = (float)(L.dt - 1);
  C.tdm2 = (float)(L.dt - 2);
  C.sdm1 = (float)(L.ds - 1);
  C.sdm2 = (float)(L.ds - 2);

  const long long c_begin = (long long)blockIdx.x * p.total / gridDim.x;
  const long long c_end = (long long)(blockIdx.x + 1) * p.total / gridDim.x;
  const bool vec_ok = (p.w % kPx) == 0;
  const uint32_t table_bytes = (uint32_t)L.bytes();
  uint32_t phase = 0;
  bool bad = false;

  long long c = c_begin;
  while (c < c_end) {
    const int b = (int)(c / p.per_img);
    const long long phase_end = min(c_end, (long long)(b + 1) * p.per_img);
    // ---- stage image b's tables into shared memory (TMA bulk copy) ----
    __syncthreads();  // every warp is done reading the previous image's tables
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_expect_tx(bar, table_bytes);
      const char* src = reinterpret_cast<const char*>(p.tables + (long long)b * L.total_floats);
      const uint32_t dst = smem_addr(smem);
      for (uint32_t off = 0; off < table_bytes; off += 32768u) {
        const uint32_t n = min(32768u, table_bytes - off);
        bulk_g2s(dst + off, src + off, n, bar);
      }
    }
    const float* plane0 = p.rgb + (long long)b * 3 * p.h * p.w;
    float* oplane0 = p.out + (long long)b * 3 * p.h * p.w;
    const long long pl = (long long)p.h * p.w;

    // first chunk's loads overlap the table copy
    long long t = c + warp;
    ChunkIn cur;
    int cur_y = 0, cur_x0 = 0;
    if (t < phase_end) {
      const long long rem = t - (long long)b * p.per_img;
      cur_y = (int)(rem / p.cpr);
      cur_x0 = (int)(rem - (long long)cur_y * p.cpr) * kChunk;
      load_chunk<INTERLEAVE>(p, plane0, (long long)cur_y * p.w, cur_x0, lane, vec_ok, cur);
    }
    mbar_wait(bar, phase);
    phase ^= 1u;

    for (; t < phase_end; t += kFwdWarps) {
      // prefetch the next chunk of this warp
      const long long tn = t + kFwdWarps;
      ChunkIn nxt;
      int nxt_y = 0, nxt_x0 = 0;
      if (tn < phase_end) {
        const long long rem = tn - (long long)b * p.per_img;
        nxt_y = (int)(rem / p.cpr);
        nxt_x0 = (int)(rem - (long long)nxt_y * p.cpr) * kChunk;
        load_chunk<INTERLEAVE>(p, plane0, (long long)nxt_y * p.w, nxt_x0, lane, vec_ok, nxt);
      }
      const SpatialBr rb = p.row[cur_y];
      float o0[kPx], o1[kPx], o2[kPx];
#pragma unroll
      for (int u = 0; u < kPx; ++u) {
        apply_pixel(C, cur.r[u], cur.g[u], cur.b[u], cur.jx[u], cur.ex[u], rb.i, rb.d, o0[u],
                    o1[u], o2[u]);
        if (CHECK) bad |= !(isfinite(o0[u]) && isfinite(o1[u]) && isfinite(o2[u]));
      }
      const long long rowoff = (long long)cur_y * p.w;
      if (!INTERLEAVE) {
        const int x = cur_x0 + lane * kPx;
        if (vec_ok && x + kPx <= p.w) {
          __stcs(reinterpret_cast<float4*>(oplane0 + rowoff + x), make_float4(o0[0], o0[1], o0[2], o0[3]));
          __stcs(reinterpret_cast<float4*>(oplane0 + pl + rowoff + x), make_float4(o1[0], o1[1], o1[2], o1[3]));
          __stcs(reinterpret_cast<float4*>(oplane0 + 2 * pl + rowoff + x), make_float4(o2[0], o2[1], o2[2], o2[3]));
        } else {
#pragma unroll
          for (int u = 0; u < kPx; ++u) {
            if (x + u < p.w) {
              __stcs(oplane0 + rowoff + x + u, o0[u]);
              __stcs(oplane0 + pl + rowoff + x + u, o1[u]);
              __stcs(oplane0 + 2 * pl + rowoff + x + u, o2[u]);
            }
          }
        }
      } else {
#pragma unroll
        for (int u = 0; u < kPx; ++u) {
          const int xx = cur_x0 + lane + 32 * u;
          if (xx < p.w) {
            __stcs(oplane0 + rowoff + xx, o0[u]);
            __stcs(oplane0 + pl + rowoff + xx, o1[u]);
            __stcs(oplane0 + 2 * pl + rowoff + xx, o2[u]);
          }
        }
      }
      cur = nxt;
      cur_y = nxt_y;
      cur_x0 = nxt_x0;
    }
    c = phase_end;
  }
  if (CHECK) {
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(p.nonfinite, 1);
  }
}

static int g_num_sms = 0;

int fwd_max_smem_bytes() { return kMaxSmemBytes - kSmemReserve; }

template <bool IL, bool CHK>
static cudaError_t launch_variant(const FwdParams& p, int grid, size_t smem, cudaStream_t st) {
  auto kern = fused_fwd_kernel<IL, CHK>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kFwdWarps * 32, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_fused_fwd(const float* rgb, float* out, int batch, int h, int w,
                             const float* tables, const TableLayout& L, const SpatialBr* col,
                             const SpatialBr* row, int* nonfinite, int variant, cudaStream_t st) {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  FwdParams p;
  p.rgb = rgb;
  p.out = out;
  p.h = h;
  p.w = w;
  p.tables = tables;
  p.L = L;
  p.col = col;
  p.row = row;
  p.cpr = (w + kChunk - 1) / kChunk;
  p.per_img = (long long)h * p.cpr;
  p.total = (long long)batch * p.per_img;
  p.nonfinite = nonfinite;
  if (p.total == 0) return cudaSuccess;
  long long grid = g_num_sms;
  if (grid > p.total) grid = p.total;
  const size_t smem = L.bytes();
  const bool il = variant == 1;
  if (nonfinite) {
    return il ? launch_variant<true, true>(p, (int)grid, smem, st)
              : launch_variant<false, true>(p, (int)grid, smem, st);
  }
  return il ? launch_variant<true, false>(p, (int)grid, smem, st)
            : launch_variant<false, false>(p, (int)grid, smem, st);
}

}  // namespace svdlut
