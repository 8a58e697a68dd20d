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
//   lut01 [pair rg|rb][i d_t-1][j cst][12]  LUT coefficient cells, 3 channels
//         packed {A0 A1 B0 B1 | C0 C1 D0 D1 | A2 B2 C2 D2} (cell_index):
//         channels 0/1 as float2 pairs for the packed FP32x2 pipe,
//         v_c(a,b) = A_c + B_c*da + C_c*db + D_c*da*db   (weights lw folded in)
//   xc    [c 3][jx d_s-1][jc d_s-1][4]   merged xc grid of output channel c,
//         {A,B,C,D} over (ex, ec)        (sum over k%3==c of gw[k,1]*G[k,1])
//   gxy   [a d_s][b d_s][3]              merged xy grid vertices, channels packed
//   gyc   [c 3][a d_s][b d_s]            merged yc grid vertices + the channel's
//                                        total bias lb[c] + sum gb[k]
//   lut2  [i d_t-1][j cst][12]           pair gb, same cell format
//
// The fused kernel stages everything before lut2 in shared memory (one TMA
// bulk copy of a contiguous prefix) and gathers lut2 through the texture
// path, which runs beside the shared-memory pipe.
// gxy / gyc are vertex planes: the fused kernel interpolates them along y once
// per row (per warp) into per-(row, x-cell) coefficient slots.
// The LUT cell row stride cst is the smallest value >= d_t-1 with
// cst % 8 == 3: a 16-byte chunk of cell n sits in bank group (3n + k) % 8, so
// the 3x3 cell neighbourhood a noisy pixel run touches maps to distinct bank
// groups (offsets {0, +-1, +-cst, +-cst+-1} mod 8 collide only for the two
// opposite diagonals).
// Position of coefficient k (0 A, 1 B, 2 C, 3 D) of output channel c in a cell.
__host__ __device__ constexpr int cell_index(int c, int k) { return c < 2 ? 2 * k + c : 8 + k; }

struct TableLayout {
  int dt, ds, cst;
  int pair_floats;                               // one LUT pair
  int lut_off, xc_off, gxy_off, gyc_off, lut2_off;  // in floats
  int total_floats;                              // rounded up to 32 floats (128 B)
  __host__ __device__ static TableLayout make(int dt, int ds) {
    TableLayout L;
    L.dt = dt;
    L.ds = ds;
    L.cst = (dt - 1) + ((3 - (dt - 1)) & 7);
    L.pair_floats = (dt - 1) * L.cst * 12;
    L.lut_off = 0;
    L.xc_off = L.lut_off + 2 * L.pair_floats;
    L.gxy_off = L.xc_off + 3 * (ds - 1) * (ds - 1) * 4;
    L.gyc_off = L.gxy_off + ((ds * ds * 3 + 3) & ~3);
    L.lut2_off = (L.gyc_off + 3 * ds * ds + 31) & ~31;
    L.total_floats = (L.lut2_off + L.pair_floats + 31) & ~31;
    return L;
  }
  __host__ __device__ int pair_off(int p) const { return p < 2 ? lut_off + p * pair_floats : lut2_off; }
  __host__ __device__ size_t bytes() const { return (size_t)total_floats * 4; }
  // bytes of the shared-memory prefix (everything but lut2)
  __host__ __device__ int staged_bytes() const { return lut2_off * 4; }
  // one per-warp grid slot of the fused kernel: for a (row y, x-cell jx) the
  // merged xy + xc + yc grid term of channel c over guide cell jc is
  //   M + N*ex + (M' + N'*ex)*ec   stored as float4 [c 3][jc d_s-1]
  __host__ __device__ int slot_bytes() const { return 3 * (ds - 1) * 16; }
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

// Column bracket of transform._spatial_brackets (transform.py:144-149) without
// a table: pos = RN32(x / (W-1)) equals RN32(RN64(x * RN64(1/(W-1)))) for
// integers 0 <= x <= W-1 < 2^24 (the f64 product is within 2^-52 relative of
// x/(W-1), which is never closer than 2^-49 relative to an f32 rounding
// boundary), then t = RN32(pos*(d_s-1)), j = min(floor(t), d_s-2), e = t - j.
// Returns the 2^23-biased index bits.
__device__ __forceinline__ uint32_t col_bracket(int x, double rcp, float sdm1, float sdm2,
                                                float& e) {
  const float pos = __double2float_rn(__dmul_rn((double)x, rcp));
  const float t = __fmul_rn(pos, sdm1);
  const float m = __fadd_rz(fminf(t, sdm2), 8388608.0f);
  e = t - (m - 8388608.0f);
  return __float_as_uint(m);
}
// Row bracket: same rule over the global row index of an image of h_total rows.
__device__ __forceinline__ uint32_t row_bracket(int y, double rcp, float sdm1, float sdm2,
                                                float& e) {
  return col_bracket(y, rcp, sdm1, sdm2, e);
}

}  // namespace svdlut
