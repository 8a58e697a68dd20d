// svdlut_host.cu — host-buffer entry point (svdlut_enhance_host) and its
// context: the end-to-end path a host caller (the reference's numpy Image)
// goes through.  H2D of the image, table prologue, fused apply and D2H of the
// result run as a pipeline over row strips on three streams (copy-in,
// compute, copy-out) chained by per-strip events, so the H2D engine streams
// strip after strip, the D2H engine follows one strip behind and the kernels
// run in between (strips are independent thanks to the (y0, h_total)
// contract).  The step is then bound by the PCIe copies alone.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/svdlut_b200.h"
#include "svdlut_common.cuh"
#include "svdlut_io.cuh"
#include "svdlut_internal.h"

using namespace svdlut;


constexpr int kMaxStrips = 32;

// Host copy pool: a few threads that copy a strip between pageable user
// memory and page-locked staging in parallel (one thread moves ~10 GB/s, the
// PCIe link ~50 GB/s per direction).
class CopyPool {
 public:
  explicit CopyPool(int n) {
    for (int i = 0; i < n; ++i) th_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  // runs f(0..n-1) on the pool and the calling thread; returns when all are done
  void run(int n, const std::function<void(int)>& f) {
    {
      std::lock_guard<std::mutex> g(m_);
      job_ = &f;
      n_ = n;
      next_ = 0;
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> g(m_);
    done_cv_.wait(g, [this] { return done_ == n_; });
    job_ = nullptr;
  }

 private:
  void work() {
    for (;;) {
      int i;
      const std::function<void(int)>* f;
      {
        std::lock_guard<std::mutex> g(m_);
        if (!job_ || next_ >= n_) return;
        i = next_++;
        f = job_;
      }
      (*f)(i);
      std::lock_guard<std::mutex> g(m_);
      if (++done_ == n_) done_cv_.notify_all();
    }
  }
  void loop() {
    unsigned long long seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      work();
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* job_ = nullptr;
  int n_ = 0, next_ = 0, done_ = 0;
  unsigned long long gen_ = 0;
  bool stop_ = false;
};

struct svdlut_ctx {
  int device = 0;
  cudaStream_t st[3] = {nullptr, nullptr, nullptr};  // copy-in, compute, copy-out
  cudaEvent_t ev_in[kMaxStrips] = {};
  cudaEvent_t ev_k[kMaxStrips] = {};
  cudaEvent_t ev_out[kMaxStrips] = {};
  cudaEvent_t ev_par = nullptr;  // parameters on the device
  void* d_img = nullptr;  // input strips followed by output strips
  size_t d_img_bytes = 0;
  void* d_par = nullptr;  // parameters + packed tables + workspaces
  size_t d_par_bytes = 0;
  int* h_flag = nullptr;  // pinned flag readback
  float* h_stage = nullptr;  // pinned staging for small host transfers
  size_t h_stage_bytes = 0;
  // pageable images: two page-locked strip slots per direction + copy pool
  char* h_strip = nullptr;
  size_t h_strip_bytes = 0;
  CopyPool* pool = nullptr;
  std::mutex mu;
};

namespace {

cudaError_t ensure(void** buf, size_t* have, size_t need) {
  if (*have >= need) return cudaSuccess;
  if (*buf) cudaFree(*buf);
  *buf = nullptr;
  *have = 0;
  cudaError_t e = cudaMalloc(buf, need);
  if (e == cudaSuccess) *have = need;
  return e;
}

size_t rup(size_t v) { return (v + 255) / 256 * 256; }

// On a failed call, wait for whatever was already queued on the context's
// streams before its lock is released, so the next call cannot reuse device or
// staging buffers that copies or kernels of this one still touch.
struct DrainOnFailure {
  svdlut_ctx* ctx;
  bool ok = false;
  ~DrainOnFailure();
};

}  // namespace

DrainOnFailure::~DrainOnFailure() {
  if (ok) return;
  for (cudaStream_t st : ctx->st)
    if (st) cudaStreamSynchronize(st);
}

extern "C" {

svdlut_ctx* svdlut_ctx_create(int device) {
  svdlut_ctx* c = new svdlut_ctx();
  c->device = device;
  if (cudaSetDevice(device) != cudaSuccess) {
    delete c;
    return nullptr;
  }
  bool ok = true;
  for (int i = 0; i < 3; ++i)
    ok &= cudaStreamCreateWithFlags(&c->st[i], cudaStreamNonBlocking) == cudaSuccess;
  for (int i = 0; i < kMaxStrips; ++i) {
    ok &= cudaEventCreateWithFlags(&c->ev_in[i], cudaEventDisableTiming) == cudaSuccess;
    ok &= cudaEventCreateWithFlags(&c->ev_k[i], cudaEventDisableTiming) == cudaSuccess;
    ok &= cudaEventCreateWithFlags(&c->ev_out[i], cudaEventDisableTiming) == cudaSuccess;
  }
  ok &= cudaEventCreateWithFlags(&c->ev_par, cudaEventDisableTiming) == cudaSuccess;
  ok &= cudaHostAlloc((void**)&c->h_flag, sizeof(int), cudaHostAllocDefault) == cudaSuccess;
  if (!ok) {
    svdlut_ctx_destroy(c);
    return nullptr;
  }
  return c;
}

void svdlut_ctx_destroy(svdlut_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  for (int i = 0; i < 3; ++i) {
    if (c->st[i]) cudaStreamSynchronize(c->st[i]);
  }
  if (c->d_img) cudaFree(c->d_img);
  if (c->d_par) cudaFree(c->d_par);
  if (c->h_flag) cudaFreeHost(c->h_flag);
  if (c->h_stage) cudaFreeHost(c->h_stage);
  if (c->h_strip) cudaFreeHost(c->h_strip);
  delete c->pool;
  for (int i = 0; i < 3; ++i)
    if (c->st[i]) cudaStreamDestroy(c->st[i]);
  if (c->ev_par) cudaEventDestroy(c->ev_par);
  for (int i = 0; i < kMaxStrips; ++i) {
    if (c->ev_in[i]) cudaEventDestroy(c->ev_in[i]);
    if (c->ev_k[i]) cudaEventDestroy(c->ev_k[i]);
    if (c->ev_out[i]) cudaEventDestroy(c->ev_out[i]);
  }
  delete c;
}

}  // extern "C"

// Host-buffer pipeline for every sample format (svdlut_io.cuh): f32 planar
// images move as strip-major (3, hs, w) slabs (one 2D copy per strip), HWC
// integer images as contiguous row ranges.
static int enhance_host_impl(svdlut_ctx* ctx, const void* rgb, int in_fmt, int h, int w,
                             const float* lut_planes, const float* lw, const float* lb, int d_t,
                             const float* grid_planes, const float* gw, const float* gb, int k,
                             int d_s, void* out, int out_fmt, int exact, int* nonfinite) {
  if (!ctx) return SVDLUT_ERR_INVALID_ARGUMENT;
  if (!fused_fwd_formats_supported(in_fmt, out_fmt)) return SVDLUT_ERR_INVALID_ARGUMENT;
  if ((in_fmt != kF32 || out_fmt != kF32) && (exact || !svdlut_fast_supported(d_t, d_s)))
    return SVDLUT_ERR_UNSUPPORTED;  // integer formats: fast kernel only
  if (!rgb || !out || !lut_planes || !lw || !lb || !grid_planes || !gw || !gb)
    return SVDLUT_ERR_INVALID_ARGUMENT;
  if (k % 3 != 0 || k < 1) return k < 1 ? SVDLUT_ERR_DIMENSION_MISMATCH : SVDLUT_ERR_BAD_GRID_COUNT;
  if (w < 2 || h < 2) return SVDLUT_ERR_DEGENERATE_IMAGE;
  if (d_t < 2 || d_s < 2) return SVDLUT_ERR_BAD_VERTEX_COUNT;
  std::lock_guard<std::mutex> lock(ctx->mu);
  DrainOnFailure drain{ctx};
  const auto host_t0 = std::chrono::steady_clock::now();
  if (cudaSetDevice(ctx->device) != cudaSuccess) return SVDLUT_ERR_CUDA;
  const bool fast = !exact && svdlut_fast_supported(d_t, d_s);

  // ---- device buffers -------------------------------------------------------
  const size_t n_lut = 9ull * d_t * d_t, n_grid = (size_t)k * 3 * d_s * d_s;
  const size_t par_floats = n_lut + 9 + 3 + n_grid + 3ull * k + k;
  const size_t tb = fast ? svdlut_table_bytes(d_t, d_s) : 0;
  const size_t par_bytes = rup(par_floats * 4) + rup(tb) + 256;
  const size_t ib = fmt_bytes(in_fmt), ob = fmt_bytes(out_fmt);
  const size_t in_bytes = (size_t)3 * h * w * ib, out_bytes = (size_t)3 * h * w * ob;
  const size_t img_bytes = rup(in_bytes) + rup(out_bytes);
  if (ensure(&ctx->d_img, &ctx->d_img_bytes, img_bytes) != cudaSuccess) return SVDLUT_ERR_CUDA;
  if (ensure(&ctx->d_par, &ctx->d_par_bytes, par_bytes) != cudaSuccess) return SVDLUT_ERR_CUDA;
  char* d_in = (char*)ctx->d_img;
  char* d_out = (char*)ctx->d_img + rup(in_bytes);
  float* d_lut = (float*)ctx->d_par;
  float* d_lw = d_lut + n_lut;
  float* d_lb = d_lw + 9;
  float* d_grid = d_lb + 3;
  float* d_gw = d_grid + n_grid;
  float* d_gb = d_gw + 3ull * k;
  char* d_tables = (char*)ctx->d_par + rup(par_floats * 4);
  int* d_flag = (int*)(d_tables + rup(tb));

  cudaStream_t s_in = ctx->st[0], s_k = ctx->st[1], s_out = ctx->st[2];
  // ---- strip pipeline: H2D (s_in) -> kernel (s_k) -> D2H (s_out) ------------
  // ~12 MB strips at 4K: every copy has a fixed setup cost of several
  // microseconds, so fewer, larger copies win; the first strip is a quarter
  // of that and the last ones halve (see below), because the pipeline fill
  // (first H2D) and drain (last D2H) run one PCIe direction alone.
  const size_t plane = (size_t)h * w;
  const TableLayout L = TableLayout::make(d_t, d_s);
  static const size_t strip_env = [] {
    const char* e = getenv("SVDLUT_STRIP_KB");  // development knob: fixed strip size
    const long v = e ? atol(e) : 0;
    return v > 0 ? (size_t)v << 10 : (size_t)0;
  }();
  int bounds[kMaxStrips + 1];
  int n_strips = 0;
  {
    // about 4 strips per image (plus the edges), 2..12 MB each (measured best
    // for 4K f32, u16 and u8 payloads), sized by the larger direction
    const size_t row_b = (size_t)3 * w * std::max(ib, ob);
    const size_t target =
        strip_env ? strip_env : std::min((size_t)12 << 20, std::max((size_t)2 << 20, row_b * h / 4));
    const int unit = (int)std::max<size_t>(1, target / row_b);  // rows per strip
    // head: a quarter strip (the D2H engine idles until the first strip is
    // through); tail: halving strips (unit/2, unit/4, ...), because the copy-out
    // stream runs one strip behind, so the last full strip's D2H would
    // otherwise be paid after the input has finished arriving
    static const int tail_n = [] {
      const char* e = getenv("SVDLUT_TAIL");  // development knob: number of halving tail strips
      return e ? std::max(0, std::min(6, atoi(e))) : 3;
    }();
    const int head = std::max(1, unit / 4);
    int tail[8], nt = 0, tail_sum = 0;
    for (int k = 1; k <= tail_n; ++k) {
      tail[nt] = std::max(1, unit >> k);
      tail_sum += tail[nt++];
    }
    bounds[0] = 0;
    if (h <= head + tail_sum + unit) {
      bounds[n_strips = 1] = h;
    } else {
      const int mid = h - head - tail_sum;
      const int n_mid = std::min(kMaxStrips - 1 - nt, (mid + unit - 1) / unit);
      bounds[++n_strips] = head;
      for (int i = 1; i <= n_mid; ++i) bounds[++n_strips] = head + (int)((long long)mid * i / n_mid);
      for (int k = 0; k < nt; ++k) {
        bounds[n_strips + 1] = bounds[n_strips] + tail[k];
        ++n_strips;
      }
      bounds[n_strips] = h;  // (already equal)
    }
  }
  // SVDLUT_TRACE=1 (development): per-strip H2D / kernel / D2H completion
  // times relative to the start of the call, printed to stderr
  static const bool trace = getenv("SVDLUT_TRACE") != nullptr;
  cudaEvent_t tev[3 * kMaxStrips + 1], tks[kMaxStrips];
  if (trace) {
    for (auto& e : tev) cudaEventCreate(&e);
    for (auto& e : tks) cudaEventCreate(&e);
    cudaEventRecord(tev[3 * kMaxStrips], s_k);
    cudaPointerAttributes ai, ao;
    const bool oki = cudaPointerGetAttributes(&ai, rgb) == cudaSuccess;
    const bool oko = cudaPointerGetAttributes(&ao, out) == cudaSuccess;
    cudaGetLastError();
    fprintf(stderr, "host in %p type %d, out %p type %d (1 = page-locked), %d strips\n", rgb,
            oki ? (int)ai.type : -1, out, oko ? (int)ao.type : -1, n_strips);
  }
  // Pageable user buffers (plain numpy arrays) go through two page-locked
  // strip slots per direction, filled / drained by the copy pool, so the
  // copy engines still see page-locked strips (a pageable cudaMemcpy is staged
  // by the driver one piece at a time: 4K f32 8.9 ms instead of ~2.6).
  auto page_locked = [](const void* ptr) {
    cudaPointerAttributes a;
    const bool ok = cudaPointerGetAttributes(&a, ptr) == cudaSuccess && a.type == cudaMemoryTypeHost;
    cudaGetLastError();
    return ok;
  };
  const bool stage_in = !page_locked(rgb), stage_out = !page_locked(out);
  char* slot_in[2] = {nullptr, nullptr};
  char* slot_out[2] = {nullptr, nullptr};
  if (stage_in || stage_out) {
    size_t strip_max = 0;
    for (int s = 0; s < n_strips; ++s)
      strip_max = std::max(strip_max, (size_t)3 * (bounds[s + 1] - bounds[s]) * w * std::max(ib, ob));
    const size_t slot = rup(strip_max);
    if (ctx->h_strip_bytes < 4 * slot) {
      if (ctx->h_strip) cudaFreeHost(ctx->h_strip);
      ctx->h_strip = nullptr;
      ctx->h_strip_bytes = 0;
      if (cudaHostAlloc((void**)&ctx->h_strip, 4 * slot, cudaHostAllocDefault) != cudaSuccess)
        return SVDLUT_ERR_CUDA;
      ctx->h_strip_bytes = 4 * slot;
    }
    if (!ctx->pool) {
      static const int n_threads = [] {
        const char* e = getenv("SVDLUT_COPY_THREADS");  // pool size (the caller also copies)
        if (e && atoi(e) > 0) return atoi(e);
        // 4K f32 from pageable memory on a 16-core host: 3 threads 3.13 ms,
        // 7 threads 3.10 ms, 11 threads 5.3 ms (contention with the driver)
        const unsigned hc = std::thread::hardware_concurrency();
        return (int)std::max(1u, std::min(5u, hc / 2));
      }();
      ctx->pool = new CopyPool(n_threads);
    }
    for (int i = 0; i < 2; ++i) {
      slot_in[i] = ctx->h_strip + i * slot;
      slot_out[i] = ctx->h_strip + (2 + i) * slot;
    }
  }
  // copies strip rows [r0, r0 + hs) between the user image and a slot laid
  // out like the device strip ((3, hs, w) for f32, rows for HWC), in ~1 MB pieces
  auto strip_copy = [&](int r0, int hs, char* slotp, bool to_slot) {
    struct Part { const char* src; char* dst; size_t n; };
    Part parts[3];
    int np_ = 0;
    if ((to_slot ? in_fmt : out_fmt) == kF32) {
      for (int c = 0; c < 3; ++c) {
        const size_t user_off = ((size_t)c * plane + (size_t)r0 * w) * 4, slot_off = (size_t)c * hs * w * 4;
        const size_t n = (size_t)hs * w * 4;
        parts[np_++] = to_slot ? Part{(const char*)rgb + user_off, slotp + slot_off, n}
                               : Part{slotp + slot_off, (char*)out + user_off, n};
      }
    } else {
      const size_t eb = to_slot ? ib : ob;
      const size_t user_off = (size_t)3 * r0 * w * eb, n = (size_t)3 * hs * w * eb;
      parts[np_++] = to_slot ? Part{(const char*)rgb + user_off, slotp, n}
                             : Part{slotp, (char*)out + user_off, n};
    }
    constexpr size_t kPiece = 1 << 20;
    int pieces[3], total = 0;
    for (int i = 0; i < np_; ++i) total += (pieces[i] = (int)((parts[i].n + kPiece - 1) / kPiece));
    ctx->pool->run(total, [&](int t) {
      int i = 0;
      while (t >= pieces[i]) t -= pieces[i++];
      const size_t off = (size_t)t * kPiece, n = std::min(kPiece, parts[i].n - off);
      memcpy(parts[i].dst + off, parts[i].src + off, n);
    });
  };
  // H2D of strip s on the copy-in stream, then its ev_in event
  auto issue_h2d = [&](int s) -> int {
    const int r0 = bounds[s], hs = bounds[s + 1] - bounds[s];
    char* din = d_in + (size_t)3 * r0 * w * ib;
    if (stage_in) {  // slot s % 2 is free once the H2D of strip s - 2 is done
      if (s >= 2 && cudaEventSynchronize(ctx->ev_in[s - 2]) != cudaSuccess) return SVDLUT_ERR_CUDA;
      strip_copy(r0, hs, slot_in[s & 1], true);
      if (cudaMemcpyAsync(din, slot_in[s & 1], (size_t)3 * hs * w * ib, cudaMemcpyHostToDevice, s_in) !=
          cudaSuccess)
        return SVDLUT_ERR_CUDA;
    } else if (in_fmt == kF32) {  // the strip's 3 channel slabs: one 2D copy (host pitch = plane)
      if (cudaMemcpy2DAsync(din, (size_t)hs * w * 4, (const float*)rgb + (size_t)r0 * w, plane * 4,
                            (size_t)hs * w * 4, 3, cudaMemcpyHostToDevice, s_in) != cudaSuccess)
        return SVDLUT_ERR_CUDA;
    } else if (cudaMemcpyAsync(din, (const char*)rgb + (size_t)3 * r0 * w * ib, (size_t)3 * hs * w * ib,
                               cudaMemcpyHostToDevice, s_in) != cudaSuccess) {
      return SVDLUT_ERR_CUDA;
    }
    if (trace) cudaEventRecord(tev[3 * s], s_in);
    if (cudaEventRecord(ctx->ev_in[s], s_in) != cudaSuccess) return SVDLUT_ERR_CUDA;
    return SVDLUT_OK;
  };
  // ---- parameters + table prologue --------------------------------------------
  // One async copy from the context's page-locked staging (a cudaMemcpyAsync
  // from pageable memory blocks the host while the driver stages it), queued
  // on the copy-in stream ahead of the first strip: copies share the H2D
  // engine, and one queued on another stream behind the strips would hold the
  // first kernel back until all of the input has arrived.
  {
    const size_t need = par_floats * 4;
    if (ctx->h_stage_bytes < need) {
      if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
      ctx->h_stage = nullptr;
      ctx->h_stage_bytes = 0;
      if (cudaHostAlloc((void**)&ctx->h_stage, need, cudaHostAllocDefault) != cudaSuccess)
        return SVDLUT_ERR_CUDA;
      ctx->h_stage_bytes = need;
    }
    const float* src[6] = {lut_planes, lw, lb, grid_planes, gw, gb};
    const size_t cnt[6] = {n_lut, 9, 3, n_grid, 3ull * k, (size_t)k};
    float* hp = ctx->h_stage;
    for (int i = 0; i < 6; ++i) {
      memcpy(hp, src[i], cnt[i] * 4);
      hp += cnt[i];
    }
    if (cudaMemcpyAsync(d_lut, ctx->h_stage, need, cudaMemcpyHostToDevice, s_in) != cudaSuccess ||
        cudaEventRecord(ctx->ev_par, s_in) != cudaSuccess || cudaStreamWaitEvent(s_k, ctx->ev_par, 0) != cudaSuccess)
      return SVDLUT_ERR_CUDA;
  }
  if (!stage_in) {  // a page-locked input starts streaming right behind the parameters
    const int rc = issue_h2d(0);
    if (rc != SVDLUT_OK) return rc;
  }
  if (cudaMemsetAsync(d_flag, 0, sizeof(int), s_k) != cudaSuccess) return SVDLUT_ERR_CUDA;
  if (fast) {
    int rc = svdlut_pack_tables(d_lut, d_lw, d_lb, d_t, d_grid, d_gw, d_gb, k, d_s, 1, d_tables, s_k);
    if (rc != SVDLUT_OK) return rc;
  }
  for (int s = 0; s < n_strips; ++s) {
    const int r0 = bounds[s], r1 = bounds[s + 1];
    const int hs = r1 - r0;
    // device layout: f32 strip-major (3, hs, w) at the strip's offset; HWC
    // rows [r0, r1) contiguous, as on the host
    char* din = d_in + (size_t)3 * r0 * w * ib;
    char* dout = d_out + (size_t)3 * r0 * w * ob;
    if (s > 0 || stage_in) {
      const int rc = issue_h2d(s);
      if (rc != SVDLUT_OK) return rc;
    }
    if (cudaStreamWaitEvent(s_k, ctx->ev_in[s], 0) != cudaSuccess) return SVDLUT_ERR_CUDA;
    if (trace) cudaEventRecord(tks[s], s_k);
    if (fast) {
      if (launch_fused_fwd_io(din, in_fmt, dout, out_fmt, 1, hs, w, r0, h, (const float*)d_tables, L,
                              d_flag, s_k) != cudaSuccess)
        return SVDLUT_ERR_CUDA;
    } else {
      const int rc = svdlut_fused_fwd_exact((const float*)din, 1, hs, w, r0, h, d_lut, d_lw, d_lb, d_t,
                                            d_grid, d_gw, d_gb, k, d_s, (float*)dout, s_k);
      if (rc != SVDLUT_OK) return rc;
    }
    if (trace) cudaEventRecord(tev[3 * s + 1], s_k);
    if (cudaEventRecord(ctx->ev_k[s], s_k) != cudaSuccess) return SVDLUT_ERR_CUDA;
    if (cudaStreamWaitEvent(s_out, ctx->ev_k[s], 0) != cudaSuccess) return SVDLUT_ERR_CUDA;
    if (stage_out) {  // slot s % 2 still holds strip s - 2: drain it to the user buffer first
      if (s >= 2) {
        if (cudaEventSynchronize(ctx->ev_out[s - 2]) != cudaSuccess) return SVDLUT_ERR_CUDA;
        strip_copy(bounds[s - 2], bounds[s - 1] - bounds[s - 2], slot_out[s & 1], false);
      }
      if (cudaMemcpyAsync(slot_out[s & 1], dout, (size_t)3 * hs * w * ob, cudaMemcpyDeviceToHost, s_out) !=
              cudaSuccess ||
          cudaEventRecord(ctx->ev_out[s], s_out) != cudaSuccess)
        return SVDLUT_ERR_CUDA;
    } else if (out_fmt == kF32) {
      if (cudaMemcpy2DAsync((float*)out + (size_t)r0 * w, plane * 4, dout, (size_t)hs * w * 4,
                            (size_t)hs * w * 4, 3, cudaMemcpyDeviceToHost, s_out) != cudaSuccess)
        return SVDLUT_ERR_CUDA;
    } else if (cudaMemcpyAsync((char*)out + (size_t)3 * r0 * w * ob, dout, (size_t)3 * hs * w * ob,
                               cudaMemcpyDeviceToHost, s_out) != cudaSuccess) {
      return SVDLUT_ERR_CUDA;
    }
    if (trace) cudaEventRecord(tev[3 * s + 2], s_out);
  }
  if (trace) {
    const double enq_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0).count();
    cudaStreamSynchronize(s_out);
    fprintf(stderr, "host enqueue %.3f ms\n", enq_ms);
    for (int s = 0; s < n_strips; ++s) {
      float t[4];
      for (int i = 0; i < 3; ++i) cudaEventElapsedTime(&t[i], tev[3 * kMaxStrips], tev[3 * s + i]);
      cudaEventElapsedTime(&t[3], tev[3 * kMaxStrips], tks[s]);
      fprintf(stderr, "strip %2d  h2d done %7.3f  kernel start %7.3f done %7.3f  d2h done %7.3f ms\n", s, t[0],
              t[3], t[1], t[2]);
    }
    for (auto& e : tev) cudaEventDestroy(e);
    for (auto& e : tks) cudaEventDestroy(e);
  }
  if (stage_out) {
    for (int s = std::max(0, n_strips - 2); s < n_strips; ++s) {
      if (cudaEventSynchronize(ctx->ev_out[s]) != cudaSuccess) return SVDLUT_ERR_CUDA;
      strip_copy(bounds[s], bounds[s + 1] - bounds[s], slot_out[s & 1], false);
    }
  }
  // the last kernel's event already orders every flag write before s_out
  if (cudaMemcpyAsync(ctx->h_flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, s_out) != cudaSuccess)
    return SVDLUT_ERR_CUDA;
  if (cudaStreamSynchronize(s_out) != cudaSuccess) return SVDLUT_ERR_CUDA;
  if (nonfinite) *nonfinite = fast ? *ctx->h_flag : 0;
  drain.ok = true;
  return SVDLUT_OK;
}

extern "C" {

int svdlut_enhance_host(svdlut_ctx* ctx, const float* rgb, int h, int w,
                        const float* lut_planes, const float* lw, const float* lb, int d_t,
                        const float* grid_planes, const float* gw, const float* gb, int k,
                        int d_s, float* out, int exact, int* nonfinite) {
  return enhance_host_impl(ctx, rgb, kF32, h, w, lut_planes, lw, lb, d_t, grid_planes, gw, gb, k, d_s,
                           out, kF32, exact, nonfinite);
}

int svdlut_enhance_host_io(svdlut_ctx* ctx, const void* in, int in_fmt, int h, int w,
                           const float* lut_planes, const float* lw, const float* lb, int d_t,
                           const float* grid_planes, const float* gw, const float* gb, int k, int d_s,
                           void* out, int out_fmt, int* nonfinite) {
  return enhance_host_impl(ctx, in, in_fmt, h, w, lut_planes, lw, lb, d_t, grid_planes, gw, gb, k, d_s,
                           out, out_fmt, 0, nonfinite);
}

int svdlut_reconstruct_host(svdlut_ctx* ctx, const float* u, const float* s, const float* vt,
                            int batch, int d_t, int n_s, float* planes) {
  if (!ctx || !u || !s || !vt || !planes) return SVDLUT_ERR_INVALID_ARGUMENT;
  if (batch < 0) return SVDLUT_ERR_DIMENSION_MISMATCH;
  if (d_t < 2) return SVDLUT_ERR_BAD_VERTEX_COUNT;
  if (n_s < 1 || n_s > d_t) return SVDLUT_ERR_DIMENSION_MISMATCH;
  if (batch == 0) return SVDLUT_OK;
  std::lock_guard<std::mutex> lock(ctx->mu);
  DrainOnFailure drain{ctx};
  if (cudaSetDevice(ctx->device) != cudaSuccess) return SVDLUT_ERR_CUDA;
  const size_t nu = (size_t)batch * 9 * d_t * n_s, ns = (size_t)batch * 9 * n_s;
  const size_t np = (size_t)batch * 9 * d_t * d_t;
  const size_t in_f = 2 * nu + ns, stage_f = in_f > np ? in_f : np;
  if (ctx->h_stage_bytes < stage_f * 4) {
    if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
    ctx->h_stage = nullptr;
    ctx->h_stage_bytes = 0;
    if (cudaHostAlloc((void**)&ctx->h_stage, stage_f * 4, cudaHostAllocDefault) != cudaSuccess)
      return SVDLUT_ERR_CUDA;
    ctx->h_stage_bytes = stage_f * 4;
  }
  if (ensure(&ctx->d_par, &ctx->d_par_bytes, rup(in_f * 4) + rup(np * 4)) != cudaSuccess)
    return SVDLUT_ERR_CUDA;
  float* st = ctx->h_stage;
  memcpy(st, u, nu * 4);
  memcpy(st + nu, s, ns * 4);
  memcpy(st + nu + ns, vt, nu * 4);
  float* d_in = (float*)ctx->d_par;
  float* d_planes = (float*)((char*)ctx->d_par + rup(in_f * 4));
  cudaStream_t sk = ctx->st[1];
  if (cudaMemcpyAsync(d_in, st, in_f * 4, cudaMemcpyHostToDevice, sk) != cudaSuccess)
    return SVDLUT_ERR_CUDA;
  const int rc = svdlut_reconstruct(d_in, d_in + nu, d_in + nu + ns, batch, d_t, n_s, d_planes, sk);
  if (rc != SVDLUT_OK) return rc;
  if (cudaMemcpyAsync(st, d_planes, np * 4, cudaMemcpyDeviceToHost, sk) != cudaSuccess)
    return SVDLUT_ERR_CUDA;
  if (cudaStreamSynchronize(sk) != cudaSuccess) return SVDLUT_ERR_CUDA;
  memcpy(planes, st, np * 4);
  drain.ok = true;
  return SVDLUT_OK;
}

}  // extern "C"
