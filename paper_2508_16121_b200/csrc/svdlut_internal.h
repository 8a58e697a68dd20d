// svdlut_internal.h — launchers shared between the .cu translation units.
#pragma once
#include <cuda_runtime.h>
#include "svdlut_common.cuh"

namespace svdlut {

cudaError_t launch_reconstruct(const float* u, const float* s, const float* vt, int batch, int dt,
                               int ns, float* planes, cudaStream_t st);
// LUT planes from `lp`, or (lp == NULL) reconstructed on the fly from (fu, fs, fvt, ns).
cudaError_t launch_pack(const float* lp, const float* fu, const float* fs, const float* fvt, int ns,
                        const float* lw, const float* lb, const float* gp, const float* gw,
                        const float* gb, int k, const TableLayout& L, int batch, float* tables,
                        cudaStream_t st);

// Fast fused forward from packed tables; spatial brackets are computed in the
// kernel (rows of a strip y0.. of an image with h_total rows).
cudaError_t launch_fused_fwd(const float* rgb, float* out, int batch, int h, int w, int y0,
                             int h_total, const float* tables, const TableLayout& L,
                             int* nonfinite, cudaStream_t st, long long pl_in = 0,
                             long long pl_out = 0);

// Same with explicit sample formats (SampleFmt in svdlut_io.cuh: 0 f32 planar,
// 1 u8 HWC, 2 big-endian u16 HWC); plane strides apply to f32 only.
cudaError_t launch_fused_fwd_io(const void* in, int in_fmt, void* out, int out_fmt, int batch, int h,
                                int w, int y0, int h_total, const float* tables, const TableLayout& L,
                                int* nonfinite, cudaStream_t st, long long pl_in = 0,
                                long long pl_out = 0);
bool fused_fwd_formats_supported(int in_fmt, int out_fmt);
// Fused forward + L2 loss epilogue: gy = (Y - target) * gscale (f32 planar),
// loss[b] += sum (Y - T)^2 (f64), gmax[b] = max |gy| (both accumulated: zero them first).
cudaError_t launch_fused_fwd_l2(const float* rgb, const float* target, float* gy, int batch, int h, int w,
                                int y0, int h_total, const float* tables, const TableLayout& L,
                                double* loss, float* gmax, float gscale, cudaStream_t st);

cudaError_t launch_fused_exact(const float* rgb, float* out, int batch, int h, int w, int y0,
                               int h_total, const float* lp, const float* lw, const float* lb,
                               int dt, const float* gp, const float* gw, const float* gb, int k,
                               int ds, cudaStream_t st);

// Multi-pass "original structure" (svdlut_naive.cu), f64, bitwise equal to the
// reference's slice_grid2d / apply_lut2d / combine_slices / apply_lut3d.
cudaError_t launch_slice(const float* rgb, float* fs, int batch, int h, int w, int y0, int h_total,
                         const float* gp, const float* gw, const float* gb, int k, int ds,
                         cudaStream_t st);
cudaError_t launch_lut2d(const float* rgb, float* out, int batch, int h, int w, const float* lp,
                         const float* lw, const float* lb, int dt, cudaStream_t st);
cudaError_t launch_combine(const float* base, const float* fs, float* out, int batch, int h, int w,
                           int k, cudaStream_t st);
cudaError_t launch_lut3d(const float* rgb, float* out, int batch, int h, int w, const float* cubes,
                         int d, cudaStream_t st);

// analysis.occurrence_stats: u64 corner-touch counts of a d^3 cube (zeroed first)
cudaError_t launch_occurrence(const float* rgb, int batch, int h, int w, int d, unsigned long long* cube,
                              cudaStream_t st);

cudaError_t launch_indices(const float* rgb, int batch, int h, int w, int y0, int h_total,
                           int dt, int ds, int32_t* idx, cudaStream_t st);

cudaError_t launch_fused_bwd(const float* rgb, const float* gy, int batch, int h, int w, int y0,
                             int h_total, const float* lp, const float* lw, int dt,
                             const float* gp, const float* gw, int k, int ds, float* gx,
                             float* dlp, float* dlw, float* dlb, float* dgp, float* dgw,
                             float* dgb, void* ws, size_t ws_bytes, cudaStream_t st,
                             const float* tables_in = nullptr, const float* gmax_in = nullptr,
                             const double* gss_in = nullptr);
size_t bwd_workspace_bytes(int batch, int h, int w, int dt, int ds, int k);
cudaError_t launch_fused_l2_step(const float* rgb, const float* target, int batch, int h, int w, int y0,
                                 int h_total, const float* tables, float gscale, const float* lp,
                                 const float* lw, int dt, const float* gp, const float* gw, int k, int ds,
                                 float* gx, float* dlp, float* dlw, float* dlb, float* dgp, float* dgw,
                                 float* dgb, double* loss, void* ws, cudaStream_t st);

cudaError_t launch_reconstruct_bwd(const float* u, const float* s, const float* vt,
                                   const float* dplanes, int batch, int dt, int ns, float* du,
                                   float* ds, float* dvt, cudaStream_t st);

// texture object over a batch of packed tables (svdlut_tex.cu); *tex_base is
// the texel index of `tables`; mark the use after each launch on `st`
cudaError_t table_texture(const float* tables, size_t bytes, cudaStream_t st, cudaTextureObject_t* tex,
                          int* tex_base);
cudaError_t table_texture_used(cudaTextureObject_t tex, cudaStream_t st);

int fwd_max_smem_bytes();
// dynamic shared memory the fast kernel needs for (d_t, d_s): tables + per-warp row tables
size_t fwd_smem_bytes(int dt, int ds);

}  // namespace svdlut
