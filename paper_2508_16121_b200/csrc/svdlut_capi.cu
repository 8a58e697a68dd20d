// svdlut_capi.cu — the extern "C" boundary (include/svdlut_b200.h).
//
// Validation mirrors the reference operator's error behaviour before any
// compute (transform.py:321-326, core_types.py:62-213):
//   K % 3 != 0                       -> SVDLUT_ERR_BAD_GRID_COUNT   (BadGridCount)
//   W < 2 or H_total < 2             -> SVDLUT_ERR_DEGENERATE_IMAGE (DegenerateImage)
//   d_t < 2 or d_s < 2               -> SVDLUT_ERR_BAD_VERTEX_COUNT (BadVertexCount)
//   inconsistent shapes / strip      -> SVDLUT_ERR_DIMENSION_MISMATCH
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/svdlut_b200.h"
#include "svdlut_common.cuh"
#include "svdlut_internal.h"

using namespace svdlut;

namespace {

thread_local char g_err[512] = "";

int fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return status;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(SVDLUT_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define CUDA_TRY(expr, where)                      \
  do {                                             \
    cudaError_t _e = (expr);                       \
    if (_e != cudaSuccess) return cuda_fail(_e, where); \
  } while (0)

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int check_image(int batch, int h, int w, int y0, int h_total) {
  if (batch < 0 || h < 0 || w < 0) return fail(SVDLUT_ERR_DIMENSION_MISMATCH, "negative size");
  if (w < 2 || h_total < 2)
    return fail(SVDLUT_ERR_DEGENERATE_IMAGE, "slicing needs at least 2 px in each direction");
  if (y0 < 0 || y0 + h > h_total)
    return fail(SVDLUT_ERR_DIMENSION_MISMATCH, "row strip [%d, %d) outside image of %d rows", y0,
                y0 + h, h_total);
  return SVDLUT_OK;
}

int check_dims(int dt, int ds) {
  if (dt < 2 || ds < 2) return fail(SVDLUT_ERR_BAD_VERTEX_COUNT, "need at least 2 vertices per axis");
  if (dt > 4096 || ds > 4096) return fail(SVDLUT_ERR_UNSUPPORTED, "vertex count too large");
  return SVDLUT_OK;
}

int check_k(int k) {
  if (k < 1) return fail(SVDLUT_ERR_DIMENSION_MISMATCH, "need at least one grid");
  if (k % 3 != 0) return fail(SVDLUT_ERR_BAD_GRID_COUNT, "grid count %d is not a multiple of 3", k);
  return SVDLUT_OK;
}



}  // namespace

extern "C" {

int svdlut_version(void) { return 10000; }

const char* svdlut_last_error(void) { return g_err; }

const char* svdlut_status_name(int s) {
  switch (s) {
    case SVDLUT_OK: return "OK";
    case SVDLUT_ERR_DIMENSION_MISMATCH: return "DimensionMismatch";
    case SVDLUT_ERR_DEGENERATE_IMAGE: return "DegenerateImage";
    case SVDLUT_ERR_BAD_GRID_COUNT: return "BadGridCount";
    case SVDLUT_ERR_BAD_VERTEX_COUNT: return "BadVertexCount";
    case SVDLUT_ERR_NON_FINITE: return "NonFiniteValue";
    case SVDLUT_ERR_INVALID_ARGUMENT: return "InvalidArgument";
    case SVDLUT_ERR_UNSUPPORTED: return "Unsupported";
    case SVDLUT_ERR_CUDA: return "CudaError";
    default: return "Unknown";
  }
}

size_t svdlut_table_bytes(int d_t, int d_s) {
  if (d_t < 2 || d_s < 2 || d_t > 4096 || d_s > 4096) return 0;
  return TableLayout::make(d_t, d_s).bytes();
}

int svdlut_fast_supported(int d_t, int d_s) {
  if (d_t < 2 || d_s < 2) return 0;
  return fwd_smem_bytes(d_t, d_s) <= (size_t)fwd_max_smem_bytes() ? 1 : 0;
}

size_t svdlut_workspace_bytes(int batch, int h, int w, int d_t, int d_s) {
  (void)h;
  (void)w;
  if (batch < 0) return 0;
  return (size_t)batch * svdlut_table_bytes(d_t, d_s) + 256;  // packed tables only
}

int svdlut_reconstruct(const float* u, const float* s, const float* vt, int batch, int d_t,
                       int n_s, float* planes, void* stream) {
  if (batch < 0) return fail(SVDLUT_ERR_DIMENSION_MISMATCH, "negative batch");
  if (d_t < 2) return fail(SVDLUT_ERR_BAD_VERTEX_COUNT, "factored LUT needs at least 2 vertices per axis");
  if (n_s < 1 || n_s > d_t) return fail(SVDLUT_ERR_DIMENSION_MISMATCH, "rank %d outside 1..%d", n_s, d_t);
  if (batch == 0) return SVDLUT_OK;
  if (!u || !s || !vt || !planes) return fail(SVDLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  CUDA_TRY(launch_reconstruct(u, s, vt, batch, d_t, n_s, planes, (cudaStream_t)stream),
           "svdlut_reconstruct");
  return SVDLUT_OK;
}

int svdlut_pack_tables(const float* lut_planes, const float* lw, const float* lb, int d_t,
                       const float* grid_planes, const float* gw, const float* gb, int k,
                       int d_s, int batch, void* tables, void* stream) {
  int rc;
  if ((rc = check_k(k)) != SVDLUT_OK) return rc;
  if ((rc = check_dims(d_t, d_s)) != SVDLUT_OK) return rc;
  if (batch == 0) return SVDLUT_OK;
  if (!lut_planes || !lw || !lb || !grid_planes || !gw || !gb || !tables)
    return fail(SVDLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (!aligned16(tables)) return fail(SVDLUT_ERR_INVALID_ARGUMENT, "tables must be 16-byte aligned");
  if (!svdlut_fast_supported(d_t, d_s))
    return fail(SVDLUT_ERR_UNSUPPORTED, "packed tables serve the fast kernel only (d_t=%d d_s=%d)", d_t, d_s);
  const TableLayout L = TableLayout::make(d_t, d_s);
  CUDA_TRY(launch_pack(lut_planes, nullptr, nullptr, nullptr, 0, lw, lb, grid_planes, gw, gb, k, L,
                       batch, (float*)tables, (cudaStream_t)stream),
           "svdlut_pack_tables");
  return SVDLUT_OK;
}

int svdlut_pack_tables_factors(const float* u, const float* s, const float* vt, int n_s,
                               const float* lw, const float* lb, int d_t,
                               const float* grid_planes, const float* gw, const float* gb, int k,
                               int d_s, int batch, void* tables, void* stream) {
  int rc;
  if ((rc = check_k(k)) != SVDLUT_OK) return rc;
  if ((rc = check_dims(d_t, d_s)) != SVDLUT_OK) return rc;
  if (n_s < 1 || n_s > d_t) return fail(SVDLUT_ERR_DIMENSION_MISMATCH, "rank %d outside 1..%d", n_s, d_t);
  if (batch == 0) return SVDLUT_OK;
  if (!u || !s || !vt || !lw || !lb || !grid_planes || !gw || !gb || !tables)
    return fail(SVDLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (!aligned16(tables)) return fail(SVDLUT_ERR_INVALID_ARGUMENT, "tables must be 16-byte aligned");
  if (!svdlut_fast_supported(d_t, d_s))
    return fail(SVDLUT_ERR_UNSUPPORTED, "packed tables serve the fast kernel only (d_t=%d d_s=%d)", d_t, d_s);
  const TableLayout L = TableLayout::make(d_t, d_s);
  CUDA_TRY(launch_pack(nullptr, u, s, vt, n_s, lw, lb, grid_planes, gw, gb, k, L, batch,
                       (float*)tables, (cudaStream_t)stream),
           "svdlut_pack_tables_factors");
  return SVDLUT_OK;
}

static int fused_fwd_packed_impl(const float* rgb, int batch, int h, int w, int y0, int h_total,
                                 const void* tables, int d_t, int d_s, float* out, void* ws,
                                 size_t ws_bytes, int* nonfinite, cudaStream_t st) {
  (void)ws;
  (void)ws_bytes;
  int rc;
  if ((rc = check_image(batch, h, w, y0, h_total)) != SVDLUT_OK) return rc;
  if ((rc = check_dims(d_t, d_s)) != SVDLUT_OK) return rc;
  if (!svdlut_fast_supported(d_t, d_s))
    return fail(SVDLUT_ERR_UNSUPPORTED,
                "tables for d_t=%d d_s=%d exceed shared memory; use svdlut_fused_fwd_exact", d_t, d_s);
  if ((long long)batch * h * w == 0) return SVDLUT_OK;
  if (!rgb || !tables || !out) return fail(SVDLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (!aligned16(tables)) return fail(SVDLUT_ERR_INVALID_ARGUMENT, "tables must be 16-byte aligned");
  const TableLayout L = TableLayout::make(d_t, d_s);
  CUDA_TRY(launch_fused_fwd(rgb, out, batch, h, w, y0, h_total, (const float*)tables, L, nonfinite, st),
           "fused forward");
  return SVDLUT_OK;
}

int svdlut_fused_fwd_packed(const float* rgb, int batch, int h, int w, int y0, int h_total,
                            const void* tables, int d_t, int d_s, float* out, void* workspace,
                            size_t workspace_bytes, void* stream) {
  return fused_fwd_packed_impl(rgb, batch, h, w, y0, h_total, tables, d_t, d_s, out, workspace,
                               workspace_bytes, nullptr, (cudaStream_t)stream);
}

// Extended entry used by the Python layer: optional device non-finite flag.
int svdlut_fused_fwd_packed_ex(const float* rgb, int batch, int h, int w, int y0, int h_total,
                               const void* tables, int d_t, int d_s, float* out, void* workspace,
                               size_t workspace_bytes, int* nonfinite, void* stream) {
  return fused_fwd_packed_impl(rgb, batch, h, w, y0, h_total, tables, d_t, d_s, out, workspace,
                               workspace_bytes, nonfinite, (cudaStream_t)stream);
}

int svdlut_fused_fwd_io(const void* in, int in_fmt, int batch, int h, int w, int y0, int h_total,
                        const void* tables, int d_t, int d_s, void* out, int out_fmt, int* nonfinite,
                        void* stream) {
  int rc;
  if ((rc = check_image(batch, h, w, y0, h_total)) != SVDLUT_OK) return rc;
  if ((rc = check_dims(d_t, d_s)) != SVDLUT_OK) return rc;
  if (!fused_fwd_formats_supported(in_fmt, out_fmt))
    return fail(SVDLUT_ERR_INVALID_ARGUMENT, "unsupported sample formats (in %d, out %d)", in_fmt, out_fmt);
  if (!svdlut_fast_supported(d_t, d_s))
    return fail(SVDLUT_ERR_UNSUPPORTED, "tables for d_t=%d d_s=%d exceed shared memory", d_t, d_s);
  if ((long long)batch * h * w == 0) return SVDLUT_OK;
  if (!in || !tables || !out) return fail(SVDLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (!aligned16(tables)) return fail(SVDLUT_ERR_INVALID_ARGUMENT, "tables must be 16-byte aligned");
  const TableLayout L = TableLayout::make(d_t, d_s);
  CUDA_TRY(launch_fused_fwd_io(in, in_fmt, out, out_fmt, batch, h, w, y0, h_total, (const float*)tables,
                               L, nonfinite, (cudaStream_t)stream),
           "fused forward (sample formats)");
  return SVDLUT_OK;
}

int svdlut_fused_fwd(const float* rgb, int batch, int h, int w, int y0, int h_total,
                     const float* lut_planes, const float* lw, const float* lb, int d_t,
                     const float* grid_planes, const float* gw, const float* gb, int k, int d_s,
                     float* out, void* workspace, size_t workspace_bytes, void* stream) {
  int rc;
  if ((rc = check_k(k)) != SVDLUT_OK) return rc;
  if ((rc = check_image(batch, h, w, y0, h_total)) != SVDLUT_OK) return rc;
  if ((rc = check_dims(d_t, d_s)) != SVDLUT_OK) return rc;
  if (!svdlut_fast_supported(d_t, d_s))
    return fail(SVDLUT_ERR_UNSUPPORTED,
                "tables for d_t=%d d_s=%d exceed shared memory; use svdlut_fused_fwd_exact", d_t, d_s);
  if (batch == 0) return SVDLUT_OK;
  const size_t need = svdlut_workspace_bytes(batch, h, w, d_t, d_s);
  if (!workspace || workspace_bytes < need)
    return fail(SVDLUT_ERR_INVALID_ARGUMENT, "workspace too small (%zu < %zu)", workspace_bytes, need);
  const size_t tb = (size_t)batch * svdlut_table_bytes(d_t, d_s);
  if ((rc = svdlut_pack_tables(lut_planes, lw, lb, d_t, grid_planes, gw, gb, k, d_s, batch,
                               workspace, stream)) != SVDLUT_OK)
    return rc;
  (void)tb;
  return fused_fwd_packed_impl(rgb, batch, h, w, y0, h_total, workspace, d_t, d_s, out, nullptr, 0,
                               nullptr, (cudaStream_t)stream);
}

int svdlut_fused_fwd_exact(const float* rgb, int batch, int h, int w, int y0, int h_total,
                           const float* lut_planes, const float* lw, const float* lb, int d_t,
                           const float* grid_planes, const float* gw, const float* gb, int k,
                           int d_s, float* out, void* stream) {
  int rc;
  if ((rc = check_k(k)) != SVDLUT_OK) return rc;
  if ((rc = check_image(batch, h, w, y0, h_total)) != SVDLUT_OK) return rc;
  if ((rc = check_dims(d_t, d_s)) != SVDLUT_OK) return rc;
  if ((long long)batch * h * w == 0) return SVDLUT_OK;
  if (!rgb || !lut_planes || !lw || !lb || !grid_planes || !gw || !gb || !out)
    return fail(SVDLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  CUDA_TRY(launch_fused_exact(rgb, out, batch, h, w, y0, h_total, lut_planes, lw, lb, d_t,
                              grid_planes, gw, gb, k, d_s, (cudaStream_t)stream),
           "exact forward");
  return SVDLUT_OK;
}

int svdlut_indices(const float* rgb, int batch, int h, int w, int y0, int h_total, int d_t,
                   int d_s, int32_t* idx, void* stream) {
  int rc;
  if ((rc = check_image(batch, h, w, y0, h_total)) != SVDLUT_OK) return rc;
  if ((rc = check_dims(d_t, d_s)) != SVDLUT_OK) return rc;
  if ((long long)batch * h * w == 0) return SVDLUT_OK;
  if (!rgb || !idx) return fail(SVDLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  CUDA_TRY(launch_indices(rgb, batch, h, w, y0, h_total, d_t, d_s, idx, (cudaStream_t)stream),
           "indices");
  return SVDLUT_OK;
}

size_t svdlut_bwd_workspace_bytes(int batch, int h, int w, int d_t, int d_s, int k) {
  if (batch < 0 || h < 0 || w < 0 || d_t < 2 || d_s < 2 || k < 1) return 0;
  return bwd_workspace_bytes(batch, h, w, d_t, d_s, k);
}

int svdlut_fused_bwd(const float* rgb, const float* gy, int batch, int h, int w, int y0,
                     int h_total, const float* lut_planes, const float* lw, int d_t,
                     const float* grid_planes, const float* gw, int k, int d_s, float* gx,
                     float* dlut_planes, float* dlw, float* dlb, float* dgrid_planes,
                     float* dgw, float* dgb, void* workspace, size_t workspace_bytes,
                     void* stream) {
  int rc;
  if ((rc = check_k(k)) != SVDLUT_OK) return rc;
  if ((rc = check_image(batch, h, w, y0, h_total)) != SVDLUT_OK) return rc;
  if ((rc = check_dims(d_t, d_s)) != SVDLUT_OK) return rc;
  if (w > 32767)
    return fail(SVDLUT_ERR_UNSUPPORTED, "backward rows are limited to 32767 pixels (got %d)", w);
  if (batch == 0) return SVDLUT_OK;
  if (!rgb || !gy || !lut_planes || !lw || !grid_planes || !gw || !dlut_planes || !dlw || !dlb ||
      !dgrid_planes || !dgw || !dgb)
    return fail(SVDLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  const size_t need = bwd_workspace_bytes(batch, h, w, d_t, d_s, k);
  if (!workspace || workspace_bytes < need)
    return fail(SVDLUT_ERR_INVALID_ARGUMENT, "workspace too small (%zu < %zu)", workspace_bytes, need);
  CUDA_TRY(launch_fused_bwd(rgb, gy, batch, h, w, y0, h_total, lut_planes, lw, d_t, grid_planes,
                            gw, k, d_s, gx, dlut_planes, dlw, dlb, dgrid_planes, dgw, dgb,
                            workspace, workspace_bytes, (cudaStream_t)stream),
           "fused backward");
  return SVDLUT_OK;
}

int svdlut_slice_grids(const float* rgb, int batch, int h, int w, int y0, int h_total,
                       const float* grid_planes, const float* gw, const float* gb, int k, int d_s,
                       float* fs, void* stream) {
  int rc;
  if ((rc = check_image(batch, h, w, y0, h_total)) != SVDLUT_OK) return rc;
  if (k < 1) return fail(SVDLUT_ERR_DIMENSION_MISMATCH, "need at least one grid");
  if (d_s < 2) return fail(SVDLUT_ERR_BAD_VERTEX_COUNT, "need at least 2 vertices per axis");
  if ((long long)batch * h * w == 0) return SVDLUT_OK;
  if (!rgb || !grid_planes || !gw || !gb || !fs) return fail(SVDLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  CUDA_TRY(launch_slice(rgb, fs, batch, h, w, y0, h_total, grid_planes, gw, gb, k, d_s,
                        (cudaStream_t)stream),
           "slice_grids");
  return SVDLUT_OK;
}

int svdlut_apply_lut2d(const float* rgb, int batch, int h, int w, const float* lut_planes,
                       const float* lw, const float* lb, int d_t, float* out, void* stream) {
  if (batch < 0 || h < 0 || w < 0) return fail(SVDLUT_ERR_DIMENSION_MISMATCH, "negative size");
  if (d_t < 2) return fail(SVDLUT_ERR_BAD_VERTEX_COUNT, "need at least 2 vertices per axis");
  if ((long long)batch * h * w == 0) return SVDLUT_OK;
  if (!rgb || !lut_planes || !lw || !lb || !out) return fail(SVDLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  CUDA_TRY(launch_lut2d(rgb, out, batch, h, w, lut_planes, lw, lb, d_t, (cudaStream_t)stream),
           "apply_lut2d");
  return SVDLUT_OK;
}

int svdlut_combine_slices(const float* base, const float* fs, int batch, int h, int w, int k,
                          float* out, void* stream) {
  int rc;
  if ((rc = check_k(k)) != SVDLUT_OK) return rc;
  if (batch < 0 || h < 0 || w < 0) return fail(SVDLUT_ERR_DIMENSION_MISMATCH, "negative size");
  if ((long long)batch * h * w == 0) return SVDLUT_OK;
  if (!base || !fs || !out) return fail(SVDLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  CUDA_TRY(launch_combine(base, fs, out, batch, h, w, k, (cudaStream_t)stream), "combine_slices");
  return SVDLUT_OK;
}

int svdlut_apply_lut3d(const float* rgb, int batch, int h, int w, const float* cubes, int d,
                       float* out, void* stream) {
  if (batch < 0 || h < 0 || w < 0) return fail(SVDLUT_ERR_DIMENSION_MISMATCH, "negative size");
  if (d < 2) return fail(SVDLUT_ERR_BAD_VERTEX_COUNT, "3D LUT needs at least 2 vertices per axis");
  if ((long long)batch * h * w == 0) return SVDLUT_OK;
  if (!rgb || !cubes || !out) return fail(SVDLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  CUDA_TRY(launch_lut3d(rgb, out, batch, h, w, cubes, d, (cudaStream_t)stream), "apply_lut3d");
  return SVDLUT_OK;
}

int svdlut_occurrence(const float* rgb, int batch, int h, int w, int d, unsigned long long* cube,
                      void* stream) {
  if (batch < 0 || h < 0 || w < 0) return fail(SVDLUT_ERR_DIMENSION_MISMATCH, "negative size");
  if (d < 2) return fail(SVDLUT_ERR_BAD_VERTEX_COUNT, "need at least 2 vertices, got %d", d);
  if (d > 1024) return fail(SVDLUT_ERR_UNSUPPORTED, "cube too large (d=%d)", d);
  if (!cube || (!rgb && (long long)batch * h * w > 0)) return fail(SVDLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  CUDA_TRY(launch_occurrence(rgb, batch, h, w, d, cube, (cudaStream_t)stream), "occurrence");
  return SVDLUT_OK;
}

int svdlut_fused_fwd_l2(const float* rgb, const float* target, int batch, int h, int w, int y0,
                        int h_total, const void* tables, int d_t, int d_s, float* gy, double* loss_sum,
                        float* gmax, float gscale, void* stream) {
  int rc;
  if ((rc = check_image(batch, h, w, y0, h_total)) != SVDLUT_OK) return rc;
  if ((rc = check_dims(d_t, d_s)) != SVDLUT_OK) return rc;
  if (!svdlut_fast_supported(d_t, d_s))
    return fail(SVDLUT_ERR_UNSUPPORTED, "tables for d_t=%d d_s=%d exceed shared memory", d_t, d_s);
  if (!loss_sum || !gmax) return fail(SVDLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(loss_sum, 0, sizeof(double) * (size_t)batch, st), "fused_fwd_l2");
  CUDA_TRY(cudaMemsetAsync(gmax, 0, sizeof(float) * (size_t)batch, st), "fused_fwd_l2");
  if ((long long)batch * h * w == 0) return SVDLUT_OK;
  if (!rgb || !target || !tables || !gy) return fail(SVDLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (!aligned16(tables)) return fail(SVDLUT_ERR_INVALID_ARGUMENT, "tables must be 16-byte aligned");
  const TableLayout L = TableLayout::make(d_t, d_s);
  CUDA_TRY(launch_fused_fwd_l2(rgb, target, gy, batch, h, w, y0, h_total, (const float*)tables, L,
                               loss_sum, gmax, gscale, st),
           "fused forward + L2 loss");
  return SVDLUT_OK;
}

int svdlut_fused_bwd_packed(const float* rgb, const float* gy, int batch, int h, int w, int y0,
                            int h_total, const void* tables, const float* gmax, const double* gsumsq,
                            const float* lut_planes, const float* lw, int d_t,
                            const float* grid_planes, const float* gw, int k, int d_s, float* gx,
                            float* dlut_planes, float* dlw, float* dlb, float* dgrid_planes,
                            float* dgw, float* dgb, void* workspace, size_t workspace_bytes,
                            void* stream) {
  int rc;
  if ((rc = check_k(k)) != SVDLUT_OK) return rc;
  if ((rc = check_image(batch, h, w, y0, h_total)) != SVDLUT_OK) return rc;
  if ((rc = check_dims(d_t, d_s)) != SVDLUT_OK) return rc;
  if (w > 32767)
    return fail(SVDLUT_ERR_UNSUPPORTED, "backward rows are limited to 32767 pixels (got %d)", w);
  if (batch == 0) return SVDLUT_OK;
  if (!rgb || !gy || !lut_planes || !lw || !grid_planes || !gw || !dlut_planes || !dlw || !dlb ||
      !dgrid_planes || !dgw || !dgb)
    return fail(SVDLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (tables && !aligned16(tables)) return fail(SVDLUT_ERR_INVALID_ARGUMENT, "tables must be 16-byte aligned");
  const size_t need = bwd_workspace_bytes(batch, h, w, d_t, d_s, k);
  if (!workspace || workspace_bytes < need)
    return fail(SVDLUT_ERR_INVALID_ARGUMENT, "workspace too small (%zu < %zu)", workspace_bytes, need);
  CUDA_TRY(launch_fused_bwd(rgb, gy, batch, h, w, y0, h_total, lut_planes, lw, d_t, grid_planes, gw, k,
                            d_s, gx, dlut_planes, dlw, dlb, dgrid_planes, dgw, dgb, workspace,
                            workspace_bytes, (cudaStream_t)stream, (const float*)tables, gmax, gsumsq),
           "fused backward");
  return SVDLUT_OK;
}

int svdlut_fused_l2_step(const float* rgb, const float* target, int batch, int h, int w, int y0,
                         int h_total, const void* tables, float gscale, const float* lut_planes,
                         const float* lw, int d_t, const float* grid_planes, const float* gw, int k,
                         int d_s, float* gx, float* dlut_planes, float* dlw, float* dlb,
                         float* dgrid_planes, float* dgw, float* dgb, double* loss_sum, void* workspace,
                         size_t workspace_bytes, void* stream) {
  int rc;
  if ((rc = check_k(k)) != SVDLUT_OK) return rc;
  if ((rc = check_image(batch, h, w, y0, h_total)) != SVDLUT_OK) return rc;
  if ((rc = check_dims(d_t, d_s)) != SVDLUT_OK) return rc;
  if (!svdlut_fast_supported(d_t, d_s))
    return fail(SVDLUT_ERR_UNSUPPORTED, "tables for d_t=%d d_s=%d exceed shared memory", d_t, d_s);
  if (w > 32767)
    return fail(SVDLUT_ERR_UNSUPPORTED, "backward rows are limited to 32767 pixels (got %d)", w);
  if (batch == 0) return SVDLUT_OK;
  if (!rgb || !target || !tables || !lut_planes || !lw || !grid_planes || !gw || !dlut_planes || !dlw ||
      !dlb || !dgrid_planes || !dgw || !dgb || !loss_sum)
    return fail(SVDLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (!aligned16(tables)) return fail(SVDLUT_ERR_INVALID_ARGUMENT, "tables must be 16-byte aligned");
  const size_t need = bwd_workspace_bytes(batch, h, w, d_t, d_s, k);
  if (!workspace || workspace_bytes < need)
    return fail(SVDLUT_ERR_INVALID_ARGUMENT, "workspace too small (%zu < %zu)", workspace_bytes, need);
  CUDA_TRY(launch_fused_l2_step(rgb, target, batch, h, w, y0, h_total, (const float*)tables, gscale, lut_planes,
                                lw, d_t, grid_planes, gw, k, d_s, gx, dlut_planes, dlw, dlb, dgrid_planes, dgw,
                                dgb, loss_sum, workspace, (cudaStream_t)stream),
           "fused L2 step");
  return SVDLUT_OK;
}

int svdlut_reconstruct_bwd(const float* u, const float* s, const float* vt,
                           const float* dplanes, int batch, int d_t, int n_s, float* du,
                           float* ds, float* dvt, void* stream) {
  if (batch < 0) return fail(SVDLUT_ERR_DIMENSION_MISMATCH, "negative batch");
  if (d_t < 2) return fail(SVDLUT_ERR_BAD_VERTEX_COUNT, "factored LUT needs at least 2 vertices per axis");
  if (n_s < 1 || n_s > d_t) return fail(SVDLUT_ERR_DIMENSION_MISMATCH, "rank %d outside 1..%d", n_s, d_t);
  if (batch == 0) return SVDLUT_OK;
  if (!u || !s || !vt || !dplanes || !du || !ds || !dvt)
    return fail(SVDLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  CUDA_TRY(launch_reconstruct_bwd(u, s, vt, dplanes, batch, d_t, n_s, du, ds, dvt,
                                  (cudaStream_t)stream),
           "reconstruct backward");
  return SVDLUT_OK;
}

}  // extern "C"
