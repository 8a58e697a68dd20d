// svdlut_common.cuh — shared device helpers and the packed-table layout.
//
// Index semantics (reference /root/reference/pkg/src/svdlut):
//   colour axes   interp._bracket (interp.py:35-45): clamp to [0,1] with strict
//                 compares, t = p*(d-1) EXACT (f64 in the reference), i = trunc(t)
//                 capped at d-2, delta = t - i.
//   spatial axes  transform._spatial_brackets (transform.py:144-149) +
//                 interp.bracket_array (interp.py:114-123): pos = f32(x)/f32(W-1)
//                 (IEEE f32 division), t = f32(pos*(d-1)) (round-to-nearest),
//                 i = min(floor(t), d-2), delta = t - i (exact).
// The fp32 colour bracket uses a round-toward-zero product: for t >= 0,
// floor(rz(q*(d-1))) == floor(q*(d-1)) because every integer below 2^24 is
// representable, so cell selection is bit-exact with the f64 reference for
// every d; delta = fma(q, d-1, -i) rounds the exact product once.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace svdlut {

constexpr int kMaxSmemBytes = 232448;       // sharedMemPerBlockOptin on B200 (measured)
constexpr int kSmemReserve = 1024;           // mbarrier + scratch

// ---- packed per-image table layout (floats; every block 16 B aligned) ------
//
//   lut  [pair 3][i  d_t-1][j  cst][12]   coefficient cells, 3 channels packed:
//        {A0 A1 A2 B0 | B1 B2 C0 C1 | C2 D0 D1 D2} with
//        v_c(a,b) = A_c + B_c*da + C_c*db + D_c*da*db   (weights lw folded in)
//   xy   [jx d_s-1][jy css][12]           merged xy grid, channels packed likewise
//   xc   [c 3][jx d_s-1][jc css][4]        merged xc grid of output channel c: {A,B,C,D}
//   yc   [c 3][jy d_s-1][jc css][4]        merged yc grid (+ the summed biases in A)
//
// Row strides cst = (d_t-1)|1 and css = (d_s-1)|1 are odd so that vertically
// adjacent cells fall in different shared-memory bank groups.
struct TableLayout {
  int dt, ds, cst, css;
  int lut_off, xy_off, xc_off, yc_off;  // in floats
  int total_floats;                      // rounded up to 32 floats (128 B)
  __host__ __device__ static TableLayout make(int dt, int ds) {
    TableLayout L;
    L.dt = dt;
    L.ds = ds;
    L.cst = (dt - 1) | 1;
    L.css = (ds - 1) | 1;
    L.lut_off = 0;
    L.xy_off = L.lut_off + 3 * (dt - 1) * L.cst * 12;
    L.xc_off = L.xy_off + (ds - 1) * L.css * 12;
    L.yc_off = L.xc_off + 3 * (ds - 1) * L.css * 4;
    int end = L.yc_off + 3 * (ds - 1) * L.css * 4;
    L.total_floats = (end + 31) & ~31;
    return L;
  }
  __host__ __device__ size_t bytes() const { return (size_t)total_floats * 4; }
};

// Spatial bracket entry (per column / per row): cell index and f32 delta.
struct SpatialBr {
  int32_t i;
  float d;
};

// transform.py:144-149 / interp.py:114-123, exact f32 semantics.
__device__ __forceinline__ SpatialBr spatial_bracket(int n, int size, int d) {
  float pos = __fdiv_rn((float)n, (float)(size - 1));
  pos = fminf(fmaxf(pos, 0.0f), 1.0f);
  float t = __fmul_rn(pos, (float)(d - 1));
  float f = fminf(floorf(t), (float)(d - 2));
  SpatialBr b;
  b.i = (int32_t)f;
  b.d = t - f;  // exact (Sterbenz / f == 0)
  return b;
}

// interp.py:35-45 in fp32 with exact cell selection (see header comment).
// q must already be clamped to [0,1] (clamp01).  The floor is taken with a
// round-toward-zero add of 2^23 (t < 2^22), which keeps the whole bracket on
// the full-rate FMA/ALU pipes instead of the conversion pipe:
//   m = rz(t + 2^23) = 2^23 + floor(t)   ->  i = bits(m) - bits(2^23)
__device__ __forceinline__ void color_bracket(float q, float dm1, float dm2, int& i,
                                              float& delta) {
  const float t = fminf(__fmul_rz(q, dm1), dm2);
  const float m = __fadd_rz(t, 8388608.0f);
  i = __float_as_int(m) - 0x4B000000;
  delta = __fmaf_rn(q, dm1, -(m - 8388608.0f));
}

// clamp to [0,1] with the strict-compare semantics of interp.py:37-40;
// NaN -> 0 so indices always stay in range.
__device__ __forceinline__ float clamp01(float p) { return __saturatef(p); }

}  // namespace svdlut
