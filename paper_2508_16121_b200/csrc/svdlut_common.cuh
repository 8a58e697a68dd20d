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

// Debug builds (-DSVDLUT_BOUNDS_CHECK, tests/test_gpu_bounds.py) check every
// table / slot / accumulator index the kernels form and trap on a violation;
// release builds compile the checks away.  (compute-sanitizer is not
// available on the GPU pool.)
#ifdef SVDLUT_BOUNDS_CHECK
#define SVDLUT_CHECK(cond)   \
  do {                       \
    if (!(cond)) __trap();   \
  } while (0)
#else
#define SVDLUT_CHECK(cond) \
  do {                     \
  } while (0)
#endif

constexpr int kMaxSmemBytes = 232448;       // sharedMemPerBlockOptin on B200 (measured)
constexpr int kSmemReserve = 1024;           // mbarrier + scratch

// ---- packed per-image table layout (floats; every block 16 B aligned) ------
//
// LUT pairs rg, rb, gb (pair p = 0, 1, 2; first cell axis = first named
// channel) as coefficient cells v_c(a, b) = A_c + B_c a + C_c b + D_c a b with
// the mixing weights lw folded in, stored as nine float4 PLANES [p][k]
// (structure of arrays), plane k of pair p holding chunk k of every cell:
//     k = 0  {A0 A1 B0 B1}     channels 0/1 as float2 pairs for FFMA2
//     k = 1  {C0 C1 D0 D1}
//     k = 2  {A2 C2 B2 D2}     so {A2 + B2 a, C2 + D2 a} is one FFMA2
// Planes gathered from shared memory store cell (i, j) at index i*cst + j,
// cst >= dt-1 with cst % 8 == 3: the 3x3 cell neighbourhood a run of pixels
// touches maps to distinct 16-byte bank groups except the two opposite
// diagonals.  Planes gathered through the texture path (kTiledPlanes: pair
// gb and chunks 1-2 of pair rb) store their cells in 4x4 tiles, index
// ((i/4)*T + j/4)*16 + (i%4)*4 + j%4 with T = ceil((dt-1)/4): the cells a
// warp's pixels touch then share a few 128-byte cache lines (a texture gather
// costs a cycle per distinct line beyond four).
//
// Grid block (K grids merged per output channel c: grid k feeds output and
// guide channel k%3, transform.py:269-297):
//   xc   [c 3][jx ds-1][jc ds-1] float4 {A,B,C,D} over (ex, ec) (sum over
//        k%3==c of gw[k,1]*G[k,1])
//   gxy  [a ds][b ds][3]   merged xy vertices, channels packed
//   gyc  [c 3][a ds][b ds] merged yc vertices + the channel's total bias
//        lb[c] + sum gb[k]
// The fused kernel interpolates xy / yc along y once per row into merged
// per-(row, jx, c, jc) slots {M, M', N, N'} (term M + N ex + (M' + N' ex) ec).
__host__ __device__ constexpr int cst_for(int dt) { return (dt - 1) + ((3 - (dt - 1)) & 7); }
// chunk planes (bit 3*pair + chunk) stored in the 4x4-tiled cell order
#ifndef SVDLUT_TILED_PLANES
#define SVDLUT_TILED_PLANES 0x1F0u
#endif
constexpr unsigned kTiledPlanes = SVDLUT_TILED_PLANES;  // rb chunks 1-2, gb chunks 0-2
__host__ __device__ constexpr bool plane_tiled(int idx) { return (kTiledPlanes >> idx) & 1u; }

struct TableLayout {
  int dt, ds, cst;
  int plane_floats;                  // one LUT float4 plane (the larger of the two cell orders)
  int lut_off;                       // 9 planes [pair][chunk]
  int xc_off, gxy_off, gyc_off;      // grid block
  int total_floats;                  // rounded up to 32 floats (128 B)
  __host__ __device__ static TableLayout make(int dt, int ds) {
    TableLayout L;
    L.dt = dt;
    L.ds = ds;
    L.cst = cst_for(dt);
    const int T = (dt + 2) / 4;  // ceil((dt-1)/4) tiles per side
    L.plane_floats = ((dt - 1) * L.cst > T * T * 16 ? (dt - 1) * L.cst : T * T * 16) * 4;
    L.lut_off = 0;
    L.xc_off = L.lut_off + 9 * L.plane_floats;
    L.gxy_off = L.xc_off + 3 * (ds - 1) * (ds - 1) * 4;
    L.gyc_off = L.gxy_off + ((ds * ds * 3 + 3) & ~3);
    L.total_floats = (L.gyc_off + 3 * ds * ds + 31) & ~31;
    return L;
  }
  __host__ __device__ int plane_off(int p, int k) const { return lut_off + (3 * p + k) * plane_floats; }
  __host__ __device__ int tiles() const { return (dt + 2) / 4; }
  // cell (i, j) within chunk plane idx = 3*pair + chunk (in float4 units)
  __host__ __device__ int cell_index(int idx, int i, int j) const {
    return !plane_tiled(idx) ? i * cst + j : ((i >> 2) * tiles() + (j >> 2)) * 16 + ((i & 3) << 2) + (j & 3);
  }
  __host__ __device__ size_t bytes() const { return (size_t)total_floats * 4; }
  __host__ __device__ int grid_floats() const { return total_floats - xc_off; }
  // merged grid slots of one row: [jx ds-1][c 3][jc ds] float4, the last jc
  // being the padding slot for a guide value of exactly 1.0
  __host__ __device__ int slot_entries() const { return (ds - 1) * 3 * ds; }
};

// Position of coefficient q (0 A, 1 B, 2 C, 3 D) of output channel c within
// the 12 floats {chunk0, chunk1, chunk2} of a cell: slot / 4 = plane (chunk),
// slot % 4 = float in the float4.
__host__ __device__ constexpr int coef_slot(int c, int q) {
  return c < 2 ? (q == 0 ? c : q == 1 ? 2 + c : q == 2 ? 4 + c : 6 + c)
               : (q == 0 ? 8 : q == 1 ? 10 : q == 2 ? 9 : 11);
}

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
// t = RN32(RN32(x / (W-1)) * (d_s-1)) of a column (uncapped), as col_bracket.
__device__ __forceinline__ float col_t_value(int x, double rcp, float sdm1) {
  return __fmul_rn(__double2float_rn(__dmul_rn((double)x, rcp)), sdm1);
}

}  // namespace svdlut
