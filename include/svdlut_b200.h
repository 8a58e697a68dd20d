/*
 * svdlut_b200.h — C ABI of the B200-native SVDLUT apply path (sm_100a).
 *
 * Drop-in boundary for the reference operator surface
 * (/root/reference/pkg/src/svdlut):
 *
 *   svdlut_fused_fwd          replaces transform.fused_enhance / _fused_impl
 *                             (transform.py:308-353, kernel transform.py:215-300)
 *   svdlut_fused_fwd_exact    same, f64 op-for-op (bit-identical to the reference)
 *   svdlut_reconstruct        replaces svd.reconstruct_lut (svd.py:210-220)
 *   svdlut_pack_tables        the on-device table prologue the fused kernel reads
 *   svdlut_fused_bwd /        backward of the apply and of the reconstruction
 *   svdlut_reconstruct_bwd    (no reference counterpart)
 *   svdlut_indices            per-pixel cell selection (interp.py:35-45,
 *                             transform.py:144-149) for the bit-exact index test
 *   svdlut_enhance_host       host-buffer entry (H2D + apply + D2H pipelined)
 *   svdlut_reconstruct_host   host-buffer svd.reconstruct_lut (svd.py:210-220)
 *   svdlut_fused_fwd_io       fused apply with PNM sample formats in/out:
 *                             decode of pnm.load (pnm.py:72-80) and the
 *                             quantization of pnm.save (pnm.py:83-108) fused
 *   svdlut_enhance_host_io    host-buffer entry with the same formats
 *   svdlut_slice_grids        transform.slice_grid2d   (transform.py:152-178)
 *   svdlut_apply_lut2d        transform.apply_lut2d    (transform.py:123-141)
 *   svdlut_combine_slices     transform.combine_slices (transform.py:181-193)
 *   svdlut_apply_lut3d        transform.apply_lut3d    (transform.py:93-120)
 *                             (the multi-pass "original structure" and the 3D-LUT
 *                             baseline, bitwise equal to the reference)
 *   svdlut_fused_fwd_l2       forward + L2 loss epilogue (training step, config 5)
 *   svdlut_fused_bwd_packed   svdlut_fused_bwd reusing the forward's tables / max|gY|
 *   svdlut_fused_l2_step      forward + L2 loss + backward in one pass (training step)
 *   svdlut_occurrence         analysis.occurrence_stats (analysis.py:109-122), the
 *                             source of utilization_rate (analysis.py:74-106)
 *
 * Conventions
 *   - Plain pointers and sizes; no framework types.  `stream` is a
 *     cudaStream_t passed as void* (NULL = legacy default stream).
 *   - All device buffers are caller-owned (no allocation inside a call except
 *     in svdlut_ctx_*, which owns its own staging buffers).
 *   - Images are planar float32 (B, 3, H, W) C-contiguous; channel order r,g,b.
 *   - LUT planes (B, 3, 3, d_t, d_t): [out channel][pair rg|rb|gb][a][b],
 *     first plane axis = first named channel (core_types.py:119-125).
 *   - Grid planes (B, K, 3, d_s, d_s): [grid][xy|xc|yc][a][b]; grid k reads
 *     guide channel k%3 and adds into output channel k%3 (transform.py:269-297).
 *   - (y0, h_total): the call covers rows y0..y0+H-1 of an image with h_total
 *     rows; positions are normalised by the global h_total-1 (row strips).
 *   - Return value is an svdlut_status; svdlut_last_error() gives the message
 *     (thread-local).  Status codes map 1:1 onto the reference exception
 *     classes (errors.py:4-31), see INTEGRATION.md.
 *   - Stream-ordered and thread-safe across streams.
 */
#ifndef SVDLUT_B200_H
#define SVDLUT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SVDLUT_OK = 0,
  SVDLUT_ERR_DIMENSION_MISMATCH = 1, /* errors.DimensionMismatch */
  SVDLUT_ERR_DEGENERATE_IMAGE = 2,   /* errors.DegenerateImage (W or H_total < 2) */
  SVDLUT_ERR_BAD_GRID_COUNT = 3,     /* errors.BadGridCount (K % 3 != 0) */
  SVDLUT_ERR_BAD_VERTEX_COUNT = 4,   /* errors.BadVertexCount (d < 2) */
  SVDLUT_ERR_NON_FINITE = 5,         /* errors.NonFiniteValue */
  SVDLUT_ERR_INVALID_ARGUMENT = 6,   /* NULL pointer, misaligned buffer, bad size */
  SVDLUT_ERR_UNSUPPORTED = 7,        /* dims beyond the fast kernel (use _exact) */
  SVDLUT_ERR_CUDA = 8                /* CUDA runtime error (message has details) */
} svdlut_status;

int svdlut_version(void);
const char* svdlut_last_error(void);
const char* svdlut_status_name(int status);

/* ---- table prologue ---------------------------------------------------- */

/* Bytes of one image's packed tables (LUT coefficient cells + merged grid
 * cells), or 0 if (d_t, d_s) are invalid. */
size_t svdlut_table_bytes(int d_t, int d_s);

/* 1 if the fast fused kernel supports (d_t, d_s) (tables fit in shared
 * memory), else 0. */
int svdlut_fast_supported(int d_t, int d_s);

/* Bytes of workspace svdlut_fused_fwd needs (the packed tables of the batch). */
size_t svdlut_workspace_bytes(int batch, int h, int w, int d_t, int d_s);

/* svd.reconstruct_lut, batched: planes[b,c,p] = f32((f64 u * f64 s) @ f64 vt).
 * u (B,3,3,d_t,n_s), s (B,3,3,n_s), vt (B,3,3,n_s,d_t) -> planes (B,3,3,d_t,d_t). */
int svdlut_reconstruct(const float* u, const float* s, const float* vt, int batch, int d_t,
                       int n_s, float* planes, void* stream);

/* Fold weights into the LUT planes, merge the K grids per output channel and
 * write each image's coefficient tables (svdlut_table_bytes each, 16 B
 * aligned) into `tables`. */
int svdlut_pack_tables(const float* lut_planes, const float* lw, const float* lb, int d_t,
                       const float* grid_planes, const float* gw, const float* gb, int k,
                       int d_s, int batch, void* tables, void* stream);

/* Same tables straight from the SVD factors (svdlut_reconstruct fused into
 * the packing; the planes are never materialised).  u (B,3,3,d_t,n_s),
 * s (B,3,3,n_s), vt (B,3,3,n_s,d_t); LUT entries are bit-identical to
 * svdlut_reconstruct's. */
int svdlut_pack_tables_factors(const float* u, const float* s, const float* vt, int n_s,
                               const float* lw, const float* lb, int d_t,
                               const float* grid_planes, const float* gw, const float* gb, int k,
                               int d_s, int batch, void* tables, void* stream);

/* ---- forward ------------------------------------------------------------ */

/* Fused slice + 2D-LUT apply from packed tables (fast fp32 kernel, within
 * 1e-5 of the reference; cell selection bit-exact).  Spatial brackets are
 * computed in the kernel; `workspace` is unused (may be NULL) and kept for
 * ABI stability. */
int svdlut_fused_fwd_packed(const float* rgb, int batch, int h, int w, int y0, int h_total,
                            const void* tables, int d_t, int d_s, float* out, void* workspace,
                            size_t workspace_bytes, void* stream);

/* As svdlut_fused_fwd_packed, plus: `nonfinite` (device int, may be NULL) is
 * OR-ed with 1 if any output sample is NaN/Inf (the check core_types.py:55-59
 * does on the host). */
int svdlut_fused_fwd_packed_ex(const float* rgb, int batch, int h, int w, int y0, int h_total,
                               const void* tables, int d_t, int d_s, float* out, void* workspace,
                               size_t workspace_bytes, int* nonfinite, void* stream);

/* Reference-shaped entry: pack + apply.  `workspace` >= svdlut_workspace_bytes. */
/* Sample formats of the _io entry points.  F32: planar float32 (B,3,H,W).
 * U8 / U16BE: PNM P6 payload order (B,H,W,3), uint8 (maxval 255) or
 * big-endian uint16 (maxval 65535).  Integer input decodes as
 * f32(f64(v) / maxval) (pnm.py:79); integer output quantizes as
 * floor(clip(y, 0, 1) * maxval + 0.5) in exact arithmetic (pnm.py:83-86). */
enum { SVDLUT_FMT_F32 = 0, SVDLUT_FMT_U8 = 1, SVDLUT_FMT_U16BE = 2 };

/* As svdlut_fused_fwd_packed_ex with explicit sample formats (any pair).  Integer images need 4-byte (U8) / 8-byte
 * (U16BE) aligned buffers for the vector path (any alignment works). */
int svdlut_fused_fwd_io(const void* in, int in_fmt, int batch, int h, int w, int y0, int h_total,
                        const void* tables, int d_t, int d_s, void* out, int out_fmt, int* nonfinite,
                        void* stream);

int svdlut_fused_fwd(const float* rgb, int batch, int h, int w, int y0, int h_total,
                     const float* lut_planes, const float* lw, const float* lb, int d_t,
                     const float* grid_planes, const float* gw, const float* gb, int k, int d_s,
                     float* out, void* workspace, size_t workspace_bytes, void* stream);

/* f64 op-for-op restatement of transform.py:215-300: output is bitwise equal
 * to the reference fused_enhance.  Any d_t, d_s >= 2, any K % 3 == 0. */
int svdlut_fused_fwd_exact(const float* rgb, int batch, int h, int w, int y0, int h_total,
                           const float* lut_planes, const float* lw, const float* lb, int d_t,
                           const float* grid_planes, const float* gw, const float* gb, int k,
                           int d_s, float* out, void* stream);

/* Cell selection exactly as the fast kernel computes it:
 * idx (B, 8, H, W) int32 = ir, ig, ib (vs d_t), jr, jg, jb (vs d_s), jx, jy. */
int svdlut_indices(const float* rgb, int batch, int h, int w, int y0, int h_total, int d_t,
                   int d_s, int32_t* idx, void* stream);

/* ---- backward ----------------------------------------------------------- */

/* Bytes of scratch svdlut_fused_bwd needs. */
size_t svdlut_bwd_workspace_bytes(int batch, int h, int w, int d_t, int d_s, int k);

/* Gradients of the fused apply given gy (B,3,H,W).  Outputs are OVERWRITTEN:
 * gx (B,3,H,W) (may be NULL), dlut_planes (B,3,3,d_t,d_t), dlw (B,3,3),
 * dlb (B,3), dgrid_planes (B,K,3,d_s,d_s), dgw (B,K,3), dgb (B,K). */
int svdlut_fused_bwd(const float* rgb, const float* gy, int batch, int h, int w, int y0,
                     int h_total, const float* lut_planes, const float* lw, int d_t,
                     const float* grid_planes, const float* gw, int k, int d_s, float* gx,
                     float* dlut_planes, float* dlw, float* dlb, float* dgrid_planes,
                     float* dgw, float* dgb, void* workspace, size_t workspace_bytes,
                     void* stream);

/* Backward of svdlut_reconstruct: du, ds, dvt (overwritten) from dplanes. */
int svdlut_reconstruct_bwd(const float* u, const float* s, const float* vt,
                           const float* dplanes, int batch, int d_t, int n_s, float* du,
                           float* ds, float* dvt, void* stream);

/* ---- host-buffer entry (end-to-end) ------------------------------------ */

typedef struct svdlut_ctx svdlut_ctx;

/* A context owns streams, device scratch and pinned staging on `device`. */
svdlut_ctx* svdlut_ctx_create(int device);
void svdlut_ctx_destroy(svdlut_ctx* ctx);

/* One image from HOST memory to HOST memory: H2D of rgb + tables, pack,
 * apply, D2H of out, pipelined over row strips on three streams (copy-in,
 * compute, copy-out).  Host buffers
 * may be pinned (DMA directly) or pageable (staged).  Blocks until `out` is
 * written.  exact != 0 selects the f64 kernel.  *nonfinite (optional) is set
 * to 1 if any output sample is NaN/Inf. */
int svdlut_enhance_host(svdlut_ctx* ctx, const float* rgb, int h, int w,
                        const float* lut_planes, const float* lw, const float* lb, int d_t,
                        const float* grid_planes, const float* gw, const float* gb, int k,
                        int d_s, float* out, int exact, int* nonfinite);

/* ---- multi-pass "original structure" + 3D LUT (f64, bitwise equal to the
 * reference's numpy stages; f32 rasters between stages) ------------------ */
/* fs (B, K, H, W): per-grid slicing maps of rows y0.. of an h_total-row image. */
int svdlut_slice_grids(const float* rgb, int batch, int h, int w, int y0, int h_total,
                       const float* grid_planes, const float* gw, const float* gb, int k, int d_s,
                       float* fs, void* stream);
/* out (B, 3, H, W): weighted 2D-LUT transform + per-channel bias. */
int svdlut_apply_lut2d(const float* rgb, int batch, int h, int w, const float* lut_planes,
                       const float* lw, const float* lb, int d_t, float* out, void* stream);
/* out = base + sum of maps j = c, c+3, ... (f32, map order). */
int svdlut_combine_slices(const float* base, const float* fs, int batch, int h, int w, int k,
                          float* out, void* stream);
/* out (B, 3, H, W): trilinear 3D LUT, cubes (B, 3, d, d, d) [c][r][g][b]. */
int svdlut_apply_lut3d(const float* rgb, int batch, int h, int w, const float* cubes, int d,
                       float* out, void* stream);

/* Training step, forward half: gy = (Y - target) * gscale (f32 planar, as
 * rgb), loss_sum[b] = sum over image b of (Y - target)^2 (f64), gmax[b] =
 * max |gy| of image b — the scale the backward's fixed-point scatter needs.
 * With gscale = 2 / (B*3*H*W), gy is d mean((Y - T)^2) / dY. */
int svdlut_fused_fwd_l2(const float* rgb, const float* target, int batch, int h, int w, int y0,
                        int h_total, const void* tables, int d_t, int d_s, float* gy, double* loss_sum,
                        float* gmax, float gscale, void* stream);

/* svdlut_fused_bwd with optional packed `tables` (from svdlut_pack_tables*,
 * biases are irrelevant to the backward) and optional per-image statistics
 * of gy: `gmax` (>= max |gy|, e.g. from svdlut_fused_fwd_l2) and `gsumsq`
 * (sum of gy^2, f64, may be NULL).  The vertex scatter is 32-bit fixed point
 * scaled by B = min(gmax, 6 rms(gy)); pixels with |gy| > B scatter through
 * f32 atomics instead.  With NULL gmax each CTA sets its own bound from a
 * probe of its first row, B = 1.5 min(max |gy|, 6 rms gy) of that row, and
 * raises it (flushing its partials) when more than 1/64 of a row's pixels
 * exceed it. */
int svdlut_fused_bwd_packed(const float* rgb, const float* gy, int batch, int h, int w, int y0,
                            int h_total, const void* tables, const float* gmax, const double* gsumsq,
                            const float* lut_planes, const float* lw, int d_t,
                            const float* grid_planes, const float* gw, int k, int d_s, float* gx,
                            float* dlut_planes, float* dlw, float* dlb, float* dgrid_planes,
                            float* dgw, float* dgb, void* workspace, size_t workspace_bytes,
                            void* stream);

/* One training step of mean((Y - target)^2) in a single pass over the pixels:
 * Y from the forward's packed `tables` (svdlut_pack_tables, biases included),
 * gy = gscale (Y - target) per pixel, then the backward of svdlut_fused_bwd
 * (gx may be NULL).  loss_sum[b] = sum (Y - target)^2 over image b (f64,
 * written).  The fixed-point bound of each CTA's rows comes from a probe of
 * its first row and grows with the running min(max |gy|, 6 rms gy); pixels
 * above it scatter through f32 atomics.  Workspace: svdlut_bwd_workspace_bytes. */
int svdlut_fused_l2_step(const float* rgb, const float* target, int batch, int h, int w, int y0,
                         int h_total, const void* tables, float gscale, const float* lut_planes,
                         const float* lw, int d_t, const float* grid_planes, const float* gw, int k,
                         int d_s, float* gx, float* dlut_planes, float* dlw, float* dlb,
                         float* dgrid_planes, float* dgw, float* dgb, double* loss_sum, void* workspace,
                         size_t workspace_bytes, void* stream);

/* cube (d, d, d) u64, zeroed then filled: how often each cube vertex is a
 * corner of some pixel's bracketing cell, over a batch of (B, 3, H, W) images
 * (exact counts). */
int svdlut_occurrence(const float* rgb, int batch, int h, int w, int d, unsigned long long* cube,
                      void* stream);

/* svdlut_enhance_host with sample formats (fast kernel only): e.g. a PNM
 * payload in, a PNM payload out — 6 B/pixel over PCIe instead of 24 (U8). */
int svdlut_enhance_host_io(svdlut_ctx* ctx, const void* in, int in_fmt, int h, int w,
                           const float* lut_planes, const float* lw, const float* lb, int d_t,
                           const float* grid_planes, const float* gw, const float* gb, int k, int d_s,
                           void* out, int out_fmt, int* nonfinite);

/* reconstruct_lut (svd.py:210-220) from HOST factors to HOST planes: one H2D
 * of (u, s, vt) through the context's pinned staging, svdlut_reconstruct,
 * one D2H.  Shapes as svdlut_reconstruct with B = batch.  Blocks until
 * `planes` is written. */
int svdlut_reconstruct_host(svdlut_ctx* ctx, const float* u, const float* s, const float* vt,
                            int batch, int d_t, int n_s, float* planes);

#ifdef __cplusplus
}
#endif

#endif /* SVDLUT_B200_H */
