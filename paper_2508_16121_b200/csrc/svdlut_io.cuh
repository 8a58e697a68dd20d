// svdlut_io.cuh — sample formats of the fused forward's input and output.
//
//   kF32   planar float32 (B, 3, H, W): the reference's Image.data layout
//          (core_types.py:62-88), 24 B/pixel of HBM traffic in + out.
//   kU8    PNM P6 payload order (B, H, W, 3) uint8, maxval 255
//   kU16   PNM P6 payload order (B, H, W, 3) big-endian uint16, maxval 65535
//
// Decode (pnm.load, pnm.py:72-80): f = f32(f64(v) / maxval).  For integer
// v <= 65535 this is the correctly rounded f32 quotient RN32(v / maxval): v /
// maxval is never within 2^-40 (relative) of an f32 rounding midpoint (maxval
// is odd), so the intermediate f64 rounding cannot move it across one; the
// kernel computes it with a reciprocal and one FMA correction (io_decode).
//
// Encode (pnm.save, pnm.py:83-108): q = floor(clip(x, 0, 1) * maxval + 0.5)
// in f64.  With x in [0,1] as f32, p = RN32(x * maxval) and e = fma(x,
// maxval, -p) is the exact product error, so x * maxval = p + e exactly and
// q = floor(p) + (frac(p) + e >= 1/2), evaluated without rounding (see
// io_quantize).  Bit-identical to the f64 formula for every f32 x
// (tests/test_gpu_io.py checks every quantization boundary +- 3 ulps).
//
// A lane always handles 4 consecutive pixels: 12 bytes (u8) / 24 bytes (u16)
// in HWC order, i.e. 32-bit / 64-bit aligned vector accesses when the width
// is a multiple of 4.
#pragma once
#include <cstdint>

namespace svdlut {

enum SampleFmt { kF32 = 0, kU8 = 1, kU16 = 2, kL2Grad = 3 /* f32 planar gY of a fused L2 loss */ };

__host__ __device__ constexpr int fmt_bytes(int fmt) { return fmt == kF32 ? 4 : (fmt == kU8 ? 1 : 2); }

// ---- raw streaming accesses ---------------------------------------------------
__device__ __forceinline__ float4 io_ld_f4(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ float io_ld_f(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t io_ld_u32(const void* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint2 io_ld_u32x2(const void* p) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t io_ld_u8(const void* p) {
  uint16_t v;
  asm volatile("ld.global.nc.u8 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void io_st_u32(void* p, uint32_t v) {
  asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void io_st_u32x2(void* p, uint32_t a, uint32_t b) {
  asm volatile("st.global.cs.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void io_st_u8(void* p, uint32_t v) {
  asm volatile("st.global.cs.u8 [%0], %1;" ::"l"(p), "h"((uint16_t)v) : "memory");
}

__device__ __forceinline__ void io_prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
__device__ __forceinline__ void io_prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// Bulk L2 prefetch of the 16-byte aligned cover of [lo, hi) clipped to [.., end).
__device__ __forceinline__ void io_prefetch_range(const char* lo, const char* hi, const char* end) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(lo) & ~(uintptr_t)15;
  uintptr_t b = (reinterpret_cast<uintptr_t>(hi) + 15) & ~(uintptr_t)15;
  const uintptr_t e = reinterpret_cast<uintptr_t>(end) & ~(uintptr_t)15;
  if (b > e) b = e;
  if (b > a) io_prefetch_l2(reinterpret_cast<const void*>(a), (uint32_t)(b - a));
}

// ---- integer samples <-> float ------------------------------------------------
// PRMT builds 0x4B00hhll (= 2^23 + v as a float) from the sample's bytes; one
// FADD removes the bias exactly.
__device__ __forceinline__ float io_biased(uint32_t w, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(w), "r"(0x4B000000u), "r"(sel));
  return __uint_as_float(r) - 8388608.0f;
}
// v / maxval correctly rounded from the reciprocal and one FMA correction
// step (q0 = v*r, rem = v - q0*m exact, q = q0 + rem*r); verified against
// f32(f64(v) / maxval) for every v (exhaustive, tests/test_gpu_io.py).
template <int FMT>
__device__ __forceinline__ float io_decode(float v) {
  const float m = FMT == kU8 ? 255.0f : 65535.0f;
  const float r = FMT == kU8 ? (1.0f / 255.0f) : (1.0f / 65535.0f);
  const float q0 = __fmul_rn(v, r);
  const float rem = __fmaf_rn(-q0, m, v);
  return __fmaf_rn(rem, r, q0);
}
template <int FMT>
__device__ __forceinline__ uint32_t io_quantize(float x) {
  const float m = FMT == kU8 ? 255.0f : 65535.0f;
  x = __saturatef(x);                       // clip to [0, 1] (NaN -> 0; flagged separately)
  const float p = __fmul_rn(x, m);          // v = x*m = p + e exactly
  const float e = __fmaf_rn(x, m, -p);
  const float kb = __fadd_rz(p, 8388608.0f);  // 2^23 + floor(p)
  const float f = __fsub_rn(p, __fsub_rn(kb, 8388608.0f));  // frac(p), exact
  // floor(v + 1/2) = floor(p) + (frac(p) + e >= 1/2); f - 1/2 is exact
  // whenever it can matter (f >= 1/4, Sterbenz), and |e| <= ulp(p)/2
  const uint32_t up = __fsub_rn(f, 0.5f) >= -e ? 1u : 0u;
  return __float_as_uint(kb) - 0x4B000000u + up;
}

// ---- source formats -----------------------------------------------------------
// `img` points at the image's first sample; plane stride `pl` (in samples)
// only matters for kF32.
template <int FMT>
struct Src;

template <>
struct Src<kF32> {
  static __device__ __forceinline__ const void* image(const void* base, long long b, long long pl) {
    return static_cast<const float*>(base) + b * 3 * pl;
  }
  template <int PX>
  static __device__ __forceinline__ void load(const void* img, long long pl, int y, int x, int w,
                                              bool vec, float* r, float* g, float* b) {
    const float* p = static_cast<const float*>(img) + (long long)y * w;
    if (vec && x + PX <= w) {
      if (PX == 4) {
        const float4 a = io_ld_f4(p + x), c = io_ld_f4(p + pl + x), d = io_ld_f4(p + 2 * pl + x);
        r[0] = a.x; r[PX > 1 ? 1 : 0] = a.y; r[PX > 2 ? 2 : 0] = a.z; r[PX > 3 ? 3 : 0] = a.w;
        g[0] = c.x; g[PX > 1 ? 1 : 0] = c.y; g[PX > 2 ? 2 : 0] = c.z; g[PX > 3 ? 3 : 0] = c.w;
        b[0] = d.x; b[PX > 1 ? 1 : 0] = d.y; b[PX > 2 ? 2 : 0] = d.z; b[PX > 3 ? 3 : 0] = d.w;
        return;
      }
    }
#pragma unroll
    for (int u = 0; u < PX; ++u) {
      const int xx = min(x + u, w - 1);
      r[u] = io_ld_f(p + xx);
      g[u] = io_ld_f(p + pl + xx);
      b[u] = io_ld_f(p + 2 * pl + xx);
    }
  }
  // L1 prefetch of a lane's PX samples per channel (issued a chunk ahead)
  static __device__ __forceinline__ void prefetch_l1(const void* img, long long pl, int y, int x, int w) {
    const float* p = static_cast<const float*>(img) + (long long)y * w + min(x, w - 1);
    io_prefetch_l1(p);
    io_prefetch_l1(p + pl);
    io_prefetch_l1(p + 2 * pl);
  }
  static __device__ __forceinline__ void prefetch_row(const void* img, long long pl, long long plane_len,
                                                      int y, int w) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float* pc = static_cast<const float*>(img) + c * pl;
      io_prefetch_range(reinterpret_cast<const char*>(pc + (long long)y * w),
                        reinterpret_cast<const char*>(pc + (long long)(y + 1) * w),
                        reinterpret_cast<const char*>(pc + plane_len));
    }
  }
  static __device__ __forceinline__ bool aligned(const void* p, long long pl) {
    return ((reinterpret_cast<uintptr_t>(p) & 15) == 0) && ((pl & 3) == 0);
  }
};

template <int FMT>
struct SrcHwc {
  static constexpr int kB = fmt_bytes(FMT);
  static __device__ __forceinline__ const void* image(const void* base, long long b, long long hw) {
    return static_cast<const char*>(base) + b * 3 * hw * kB;
  }
  template <int PX>
  static __device__ __forceinline__ void load(const void* img, long long, int y, int x, int w, bool vec,
                                              float* r, float* g, float* b) {
    static_assert(PX == 4, "integer sample formats use 4-pixel lanes");
    const char* p = static_cast<const char*>(img) + ((long long)y * w + x) * 3 * kB;
    float v[12];
    if (vec && x + 4 <= w) {
      if (FMT == kU8) {  // [r0 g0 b0 r1 | g1 b1 r2 g2 | b2 r3 g3 b3]
        const uint32_t w0 = io_ld_u32(p), w1 = io_ld_u32(p + 4), w2 = io_ld_u32(p + 8);
        const uint32_t ws[3] = {w0, w1, w2};
#pragma unroll
        for (int i = 0; i < 12; ++i) v[i] = io_biased(ws[i >> 2], 0x7550u | (uint32_t)(i & 3));
      } else {  // 12 big-endian samples in 6 words: [hi lo hi lo]
        const uint2 a = io_ld_u32x2(p), c = io_ld_u32x2(p + 8), d = io_ld_u32x2(p + 16);
        const uint32_t ws[6] = {a.x, a.y, c.x, c.y, d.x, d.y};
#pragma unroll
        for (int i = 0; i < 12; ++i) v[i] = io_biased(ws[i >> 1], (i & 1) ? 0x7523u : 0x7501u);
      }
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const char* q = static_cast<const char*>(img) + ((long long)y * w + min(x + u, w - 1)) * 3 * kB;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          if (FMT == kU8) {
            v[3 * u + c] = (float)io_ld_u8(q + c);
          } else {
            v[3 * u + c] = (float)((io_ld_u8(q + 2 * c) << 8) | io_ld_u8(q + 2 * c + 1));
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      r[u] = io_decode<FMT>(v[3 * u]);
      g[u] = io_decode<FMT>(v[3 * u + 1]);
      b[u] = io_decode<FMT>(v[3 * u + 2]);
    }
  }
  static __device__ __forceinline__ void prefetch_l1(const void* img, long long, int y, int x, int w) {
    io_prefetch_l1(static_cast<const char*>(img) + ((long long)y * w + min(x, w - 1)) * 3 * kB);
  }
  static __device__ __forceinline__ void prefetch_row(const void* img, long long, long long plane_len,
                                                      int y, int w) {
    const char* p = static_cast<const char*>(img);
    const long long row = (long long)w * 3 * kB;
    io_prefetch_range(p + y * row, p + (y + 1) * row, p + plane_len * 3 * kB);
  }
  static __device__ __forceinline__ bool aligned(const void* p, long long) {
    return (reinterpret_cast<uintptr_t>(p) & (FMT == kU8 ? 3 : 7)) == 0;
  }
};
template <>
struct Src<kU8> : SrcHwc<kU8> {};
template <>
struct Src<kU16> : SrcHwc<kU16> {};

// ---- destination formats ------------------------------------------------------
template <int FMT>
struct Dst;

template <>
struct Dst<kF32> {
  static __device__ __forceinline__ void* image(void* base, long long b, long long pl) {
    return static_cast<float*>(base) + b * 3 * pl;
  }
  template <int PX>
  static __device__ __forceinline__ void store(void* img, long long pl, int y, int x, int w, bool vec,
                                               const float* o0, const float* o1, const float* o2) {
    float* p = static_cast<float*>(img) + (long long)y * w;
    if (vec && x + PX <= w && PX == 4) {
      __stcs(reinterpret_cast<float4*>(p + x), make_float4(o0[0], o0[PX > 1 ? 1 : 0], o0[PX > 2 ? 2 : 0], o0[PX > 3 ? 3 : 0]));
      __stcs(reinterpret_cast<float4*>(p + pl + x), make_float4(o1[0], o1[PX > 1 ? 1 : 0], o1[PX > 2 ? 2 : 0], o1[PX > 3 ? 3 : 0]));
      __stcs(reinterpret_cast<float4*>(p + 2 * pl + x), make_float4(o2[0], o2[PX > 1 ? 1 : 0], o2[PX > 2 ? 2 : 0], o2[PX > 3 ? 3 : 0]));
      return;
    }
#pragma unroll
    for (int u = 0; u < PX; ++u) {
      if (x + u < w) {
        __stcs(p + x + u, o0[u]);
        __stcs(p + pl + x + u, o1[u]);
        __stcs(p + 2 * pl + x + u, o2[u]);
      }
    }
  }
  static __device__ __forceinline__ bool aligned(const void* p, long long pl) {
    return ((reinterpret_cast<uintptr_t>(p) & 15) == 0) && ((pl & 3) == 0);
  }
};

template <int FMT>
struct DstHwc {
  static constexpr int kB = fmt_bytes(FMT);
  static __device__ __forceinline__ void* image(void* base, long long b, long long hw) {
    return static_cast<char*>(base) + b * 3 * hw * kB;
  }
  template <int PX>
  static __device__ __forceinline__ void store(void* img, long long, int y, int x, int w, bool vec,
                                               const float* o0, const float* o1, const float* o2) {
    static_assert(PX == 4, "integer sample formats use 4-pixel lanes");
    uint32_t q[12];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      q[3 * u] = io_quantize<FMT>(o0[u]);
      q[3 * u + 1] = io_quantize<FMT>(o1[u]);
      q[3 * u + 2] = io_quantize<FMT>(o2[u]);
    }
    char* p = static_cast<char*>(img) + ((long long)y * w + x) * 3 * kB;
    if (vec && x + 4 <= w) {
      if (FMT == kU8) {
#pragma unroll
        for (int i = 0; i < 3; ++i)
          io_st_u32(p + 4 * i, q[4 * i] | (q[4 * i + 1] << 8) | (q[4 * i + 2] << 16) | (q[4 * i + 3] << 24));
      } else {  // big-endian samples: bytes [hi lo] per sample
        uint32_t wd[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          uint32_t r;
          asm("prmt.b32 %0, %1, %2, 0x4501;" : "=r"(r) : "r"(q[2 * i]), "r"(q[2 * i + 1]));
          wd[i] = r;
        }
        io_st_u32x2(p, wd[0], wd[1]);
        io_st_u32x2(p + 8, wd[2], wd[3]);
        io_st_u32x2(p + 16, wd[4], wd[5]);
      }
      return;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (x + u < w) {
        char* s = p + u * 3 * kB;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          if (FMT == kU8) {
            io_st_u8(s + c, q[3 * u + c]);
          } else {
            io_st_u8(s + 2 * c, q[3 * u + c] >> 8);
            io_st_u8(s + 2 * c + 1, q[3 * u + c] & 0xffu);
          }
        }
      }
    }
  }
  static __device__ __forceinline__ bool aligned(const void* p, long long) {
    return (reinterpret_cast<uintptr_t>(p) & (FMT == kU8 ? 3 : 7)) == 0;
  }
};
template <>
struct Dst<kU8> : DstHwc<kU8> {};
template <>
struct Dst<kU16> : DstHwc<kU16> {};

}  // namespace svdlut
