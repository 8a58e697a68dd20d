/*
 * svdlut_oracle.c — CPU restatement of the SVDLUT per-pixel apply path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker (or as the timed CPU baseline).  The product path in
 * paper_2508_16121_b200/ never links, imports or calls it.
 *
 * What it restates (reference = /root/reference/pkg/src/svdlut):
 *   oracle_bracket_f64    interp._bracket                  interp.py:35-45
 *   oracle_bracket_f32    interp.bracket_array             interp.py:114-123
 *   oracle_spatial        transform._spatial_brackets      transform.py:144-149
 *   oracle_fused_fwd      transform._fused_impl            transform.py:215-300
 *   oracle_reconstruct    svd.reconstruct_lut              svd.py:210-220
 *   oracle_fused_bwd      (no reference: SURVEY.md Appendix B, analytic f64)
 *
 * Numerics: all arithmetic in IEEE binary64 with no contraction (build with
 * -ffp-contract=off), in exactly the operation order of the numba kernel, so
 * oracle_fused_fwd is bit-identical to reference fused_enhance.  That claim is
 * pinned by tests/test_oracle.py against golden vectors produced by the real
 * reference (tests/golden/make_golden.py).
 *
 * Extension over the reference: (y0, h_total) lets a row strip of a taller
 * image be evaluated with the global normalisation y/(h_total-1), the
 * row-strip sharding contract of SURVEY.md §8(e).  y0=0, h_total=h is the
 * reference behaviour.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>
#include <pthread.h>

/* interp.py:35-45 — clamp (strict compares), exact f64 product, trunc, cap. */
static inline void bracket_f64(double p, int64_t d, int64_t* i_out, double* delta) {
  if (p < 0.0) {
    p = 0.0;
  } else if (p > 1.0) {
    p = 1.0;
  }
  double t = p * (double)(d - 1);
  int64_t i = (int64_t)t; /* int(t): truncation == floor for t >= 0 */
  if (i > d - 2) i = d - 2;
  *i_out = i;
  *delta = t - (double)i;
}

void oracle_bracket_f64(const float* p, int64_t n, int64_t d, int32_t* idx, double* delta) {
  for (int64_t k = 0; k < n; ++k) {
    int64_t i;
    double e;
    bracket_f64((double)p[k], d, &i, &e);
    idx[k] = (int32_t)i;
    delta[k] = e;
  }
}

/* interp.py:114-123 — f32 clip, f32 product, floor, min(d-2), f64 delta. */
void oracle_bracket_f32(const float* p, int64_t n, int64_t d, int32_t* idx, double* delta) {
  const float dm1 = (float)(d - 1);
  for (int64_t k = 0; k < n; ++k) {
    float v = p[k];
    /* np.clip(p, 0.0, 1.0) on float32 */
    if (v < 0.0f) v = 0.0f;
    if (v > 1.0f) v = 1.0f;
    float t = v * dm1;
    float f = floorf(t);
    if (f > (float)(d - 2)) f = (float)(d - 2);
    int32_t i = (int32_t)f;
    idx[k] = i;
    delta[k] = (double)t - (double)i;
  }
}

/* transform.py:144-149 — positions n/(size-1) in float32, then bracket_array. */
void oracle_spatial(int64_t size, int64_t d, int32_t* idx, double* delta) {
  const float den = (float)(size - 1);
  for (int64_t k = 0; k < size; ++k) {
    float pos = (float)k / den;
    oracle_bracket_f32(&pos, 1, d, idx + k, delta + k);
  }
}

/* Same, for a row strip: global row index y0+k over h_total rows. */
static void spatial_rows(int64_t y0, int64_t h, int64_t h_total, int64_t d, int32_t* idx,
                         double* delta) {
  const float den = (float)(h_total - 1);
  for (int64_t k = 0; k < h; ++k) {
    float pos = (float)(y0 + k) / den;
    oracle_bracket_f32(&pos, 1, d, idx + k, delta + k);
  }
}

#define LP(c, p, a, b) lp[(((c) * 3 + (p)) * dt + (a)) * dt + (b)]
#define GP(k, q, a, b) gp[(((k) * 3 + (q)) * ds + (a)) * ds + (b)]

/*
 * transform.py:215-300, op for op.  rgb/out are (3, h, w) planar f32.
 * lp (3,3,dt,dt), lw (3,3), lb (3), gp (k,3,ds,ds), gw (k,3), gb (k).
 * Returns 0, or -1 if scratch allocation failed.
 */
typedef struct {
  const float *rgb, *lp, *lw, *lb, *gp, *gw, *gb;
  int64_t h, w, dt, k, ds, r0, r1;
  const int32_t *ix, *iy;
  const double *dx, *dy;
  float* out;
} fwd_job;

/* Rows [r0, r1) of _fused_impl; rows are independent (prange contract). */
static void* fused_rows(void* arg) {
  const fwd_job* J = (const fwd_job*)arg;
  const float *rgb = J->rgb, *lp = J->lp, *lw = J->lw, *lb = J->lb, *gp = J->gp, *gw = J->gw,
              *gb = J->gb;
  const int64_t h = J->h, w = J->w, dt = J->dt, k = J->k, ds = J->ds;
  const int32_t *ix = J->ix, *iy = J->iy;
  const double *dx = J->dx, *dy = J->dy;
  float* out = J->out;
  const int64_t plane = h * w;
  for (int64_t y = J->r0; y < J->r1; ++y) {
    const int64_t jy = iy[y];
    const double ey = dy[y];
    for (int64_t x = 0; x < w; ++x) {
      const double r = (double)rgb[y * w + x];
      const double g = (double)rgb[plane + y * w + x];
      const double b = (double)rgb[2 * plane + y * w + x];
      int64_t ir, ig, ib;
      double dr, dg, db;
      bracket_f64(r, dt, &ir, &dr);
      bracket_f64(g, dt, &ig, &dg);
      bracket_f64(b, dt, &ib, &db);
      double w00 = (1.0 - dr) * (1.0 - dg);
      double w10 = dr * (1.0 - dg);
      double w01 = (1.0 - dr) * dg;
      double w11 = dr * dg;
      double a[3];
      for (int c = 0; c < 3; ++c) {
        a[c] = (double)lw[c * 3 + 0] *
               (((w00 * (double)LP(c, 0, ir, ig) + w10 * (double)LP(c, 0, ir + 1, ig)) +
                 w01 * (double)LP(c, 0, ir, ig + 1)) +
                w11 * (double)LP(c, 0, ir + 1, ig + 1));
      }
      w00 = (1.0 - dr) * (1.0 - db);
      w10 = dr * (1.0 - db);
      w01 = (1.0 - dr) * db;
      w11 = dr * db;
      for (int c = 0; c < 3; ++c) {
        a[c] += (double)lw[c * 3 + 1] *
                (((w00 * (double)LP(c, 1, ir, ib) + w10 * (double)LP(c, 1, ir + 1, ib)) +
                  w01 * (double)LP(c, 1, ir, ib + 1)) +
                 w11 * (double)LP(c, 1, ir + 1, ib + 1));
      }
      w00 = (1.0 - dg) * (1.0 - db);
      w10 = dg * (1.0 - db);
      w01 = (1.0 - dg) * db;
      w11 = dg * db;
      for (int c = 0; c < 3; ++c) {
        a[c] += (double)lw[c * 3 + 2] *
                (((w00 * (double)LP(c, 2, ig, ib) + w10 * (double)LP(c, 2, ig + 1, ib)) +
                  w01 * (double)LP(c, 2, ig, ib + 1)) +
                 w11 * (double)LP(c, 2, ig + 1, ib + 1));
      }
      for (int c = 0; c < 3; ++c) a[c] += (double)lb[c];
      int64_t jc3[3];
      double ec3[3];
      bracket_f64(r, ds, &jc3[0], &ec3[0]);
      bracket_f64(g, ds, &jc3[1], &ec3[1]);
      bracket_f64(b, ds, &jc3[2], &ec3[2]);
      const int64_t jx = ix[x];
      const double ex = dx[x];
      const double q00 = (1.0 - ex) * (1.0 - ey);
      const double q10 = ex * (1.0 - ey);
      const double q01 = (1.0 - ex) * ey;
      const double q11 = ex * ey;
      for (int64_t kk = 0; kk < k; ++kk) {
        const int ch = (int)(kk % 3);
        const int64_t jc = jc3[ch];
        const double ec = ec3[ch];
        double s = (double)gw[kk * 3 + 0] *
                   (((q00 * (double)GP(kk, 0, jx, jy) + q10 * (double)GP(kk, 0, jx + 1, jy)) +
                     q01 * (double)GP(kk, 0, jx, jy + 1)) +
                    q11 * (double)GP(kk, 0, jx + 1, jy + 1));
        double u0 = (1.0 - ex) * (1.0 - ec);
        double u1 = ex * (1.0 - ec);
        double u2 = (1.0 - ex) * ec;
        double u3 = ex * ec;
        s += (double)gw[kk * 3 + 1] *
             (((u0 * (double)GP(kk, 1, jx, jc) + u1 * (double)GP(kk, 1, jx + 1, jc)) +
               u2 * (double)GP(kk, 1, jx, jc + 1)) +
              u3 * (double)GP(kk, 1, jx + 1, jc + 1));
        u0 = (1.0 - ey) * (1.0 - ec);
        u1 = ey * (1.0 - ec);
        u2 = (1.0 - ey) * ec;
        u3 = ey * ec;
        s += (double)gw[kk * 3 + 2] *
             (((u0 * (double)GP(kk, 2, jy, jc) + u1 * (double)GP(kk, 2, jy + 1, jc)) +
               u2 * (double)GP(kk, 2, jy, jc + 1)) +
              u3 * (double)GP(kk, 2, jy + 1, jc + 1));
        s += (double)gb[kk];
        a[ch] += s;
      }
      out[y * w + x] = (float)a[0];
      out[plane + y * w + x] = (float)a[1];
      out[2 * plane + y * w + x] = (float)a[2];
    }
  }
  return NULL;
}

/*
 * transform.py:215-353 (fused_enhance minus validation): rows are split into
 * `threads` contiguous bands run on pthreads; every pixel is computed
 * independently, so the result is bitwise independent of `threads`.
 * Returns 0, or -1 on allocation / thread-creation failure.
 */
int oracle_fused_fwd(const float* rgb, int64_t h, int64_t w, int64_t y0, int64_t h_total,
                     const float* lp, int64_t dt, const float* lw, const float* lb,
                     const float* gp, int64_t k, int64_t ds, const float* gw, const float* gb,
                     float* out, int threads) {
  int32_t* ix = (int32_t*)malloc(sizeof(int32_t) * (size_t)w);
  int32_t* iy = (int32_t*)malloc(sizeof(int32_t) * (size_t)h);
  double* dx = (double*)malloc(sizeof(double) * (size_t)w);
  double* dy = (double*)malloc(sizeof(double) * (size_t)h);
  if (!ix || !iy || !dx || !dy) {
    free(ix); free(iy); free(dx); free(dy);
    return -1;
  }
  oracle_spatial(w, ds, ix, dx);
  spatial_rows(y0, h, h_total, ds, iy, dy);
  if (threads < 1) threads = 1;
  if (threads > h) threads = (int)h;
  if (threads > 256) threads = 256;
  fwd_job jobs[256];
  pthread_t tid[256];
  int rc = 0;
  for (int t = 0; t < threads; ++t) {
    fwd_job J = {rgb, lp, lw, lb, gp, gw, gb, h, w, dt, k, ds,
                 h * t / threads, h * (t + 1) / threads, ix, iy, dx, dy, out};
    jobs[t] = J;
  }
  int started = 0;
  for (int t = 1; t < threads; ++t) {
    if (pthread_create(&tid[t], NULL, fused_rows, &jobs[t]) != 0) { rc = -1; break; }
    started = t;
  }
  fused_rows(&jobs[0]);
  for (int t = 1; t <= started; ++t) pthread_join(tid[t], NULL);
  if (rc != 0) { /* finish any band whose thread failed to start */
    for (int t = started + 1; t < threads; ++t) fused_rows(&jobs[t]);
    rc = 0;
  }
  free(ix); free(iy); free(dx); free(dy);
  return rc;
}

/*
 * Per-pixel cell selection, for the bit-exact index test: idx is (8, h, w)
 * int32 = (ir, ig, ib) vs d_t, (jr, jg, jb) vs d_s, jx, jy.
 */
void oracle_indices(const float* rgb, int64_t h, int64_t w, int64_t y0, int64_t h_total,
                    int64_t dt, int64_t ds, int32_t* idx) {
  int32_t* ix = (int32_t*)malloc(sizeof(int32_t) * (size_t)w);
  int32_t* iy = (int32_t*)malloc(sizeof(int32_t) * (size_t)h);
  double* dx = (double*)malloc(sizeof(double) * (size_t)w);
  double* dy = (double*)malloc(sizeof(double) * (size_t)h);
  oracle_spatial(w, ds, ix, dx);
  spatial_rows(y0, h, h_total, ds, iy, dy);
  const int64_t plane = h * w;
  for (int64_t y = 0; y < h; ++y) {
    for (int64_t x = 0; x < w; ++x) {
      const int64_t o = y * w + x;
      for (int c = 0; c < 3; ++c) {
        int64_t i;
        double e;
        bracket_f64((double)rgb[c * plane + o], dt, &i, &e);
        idx[c * plane + o] = (int32_t)i;
        bracket_f64((double)rgb[c * plane + o], ds, &i, &e);
        idx[(3 + c) * plane + o] = (int32_t)i;
      }
      idx[6 * plane + o] = ix[x];
      idx[7 * plane + o] = iy[y];
    }
  }
  free(ix); free(iy); free(dx); free(dy);
}

/*
 * svd.py:210-220: planes[c,p] = f32((f64(u) * f64(s)) @ f64(vt)).
 * u (3,3,d,n), s (3,3,n), vt (3,3,n,d) -> planes (3,3,d,d).
 * The reference's matmul is BLAS dgemm; sums here run n = 0..n-1 in order.
 * f64 summation-order differences vanish in the final f32 rounding except at
 * exact ties (tests allow 1 ulp of f32 for that reason).
 */
void oracle_reconstruct(const float* u, const float* s, const float* vt, int64_t d, int64_t n,
                        float* planes) {
  for (int64_t cp = 0; cp < 9; ++cp) {
    const float* U = u + cp * d * n;
    const float* S = s + cp * n;
    const float* V = vt + cp * n * d;
    float* P = planes + cp * d * d;
    for (int64_t i = 0; i < d; ++i) {
      for (int64_t j = 0; j < d; ++j) {
        double acc = 0.0;
        for (int64_t m = 0; m < n; ++m) {
          acc += ((double)U[i * n + m] * (double)S[m]) * (double)V[m * d + j];
        }
        P[i * d + j] = (float)acc;
      }
    }
  }
}

/*
 * Backward of the fused apply (no reference exists).
 * f64 analytic gradients of
 *   Y_c = sum_p lw[c,p] B(T[c,p]) + lb[c]
 *         + sum_{k%3==c} (gw[k,0] B(G[k,0];x,y) + gw[k,1] B(G[k,1];x,X_c)
 *                         + gw[k,2] B(G[k,2];y,X_c) + gb[k])
 * given gy (3,h,w).  Cell choice follows the forward bracket (right cell at an
 * interior vertex, last cell at 1.0); d(delta)/dX = d-1 for 0 <= X <= 1 and 0
 * where the strict clamp is active.  All outputs are accumulated (+=) in f64.
 *   gx (3,h,w), dlp (3,3,dt,dt), dlw (3,3), dlb (3), dgp (k,3,ds,ds), dgw (k,3), dgb (k)
 */
int oracle_fused_bwd(const float* rgb, const float* gy, int64_t h, int64_t w, int64_t y0,
                     int64_t h_total, const float* lp, int64_t dt, const float* lw,
                     const float* gp, int64_t k, int64_t ds, const float* gw, double* gx,
                     double* dlp, double* dlw, double* dlb, double* dgp, double* dgw,
                     double* dgb) {
  int32_t* ix = (int32_t*)malloc(sizeof(int32_t) * (size_t)w);
  int32_t* iy = (int32_t*)malloc(sizeof(int32_t) * (size_t)h);
  double* dx = (double*)malloc(sizeof(double) * (size_t)w);
  double* dy = (double*)malloc(sizeof(double) * (size_t)h);
  if (!ix || !iy || !dx || !dy) {
    free(ix); free(iy); free(dx); free(dy);
    return -1;
  }
  oracle_spatial(w, ds, ix, dx);
  spatial_rows(y0, h, h_total, ds, iy, dy);
  const int64_t plane = h * w;
  static const int pa[3] = {0, 0, 1}; /* first axis channel of rg, rb, gb */
  static const int pb[3] = {1, 2, 2}; /* second axis channel */
  for (int64_t y = 0; y < h; ++y) {
    const int64_t jy = iy[y];
    const double ey = dy[y];
    for (int64_t x = 0; x < w; ++x) {
      const int64_t o = y * w + x;
      double X[3], g[3], e_t[3], e_s[3], m[3];
      int64_t i_t[3], i_s[3];
      for (int c = 0; c < 3; ++c) {
        X[c] = (double)rgb[c * plane + o];
        g[c] = (double)gy[c * plane + o];
        bracket_f64(X[c], dt, &i_t[c], &e_t[c]);
        bracket_f64(X[c], ds, &i_s[c], &e_s[c]);
        m[c] = (X[c] < 0.0 || X[c] > 1.0) ? 0.0 : 1.0;
      }
      double gxa[3] = {0.0, 0.0, 0.0}; /* d/d(delta_t) per input channel */
      double gxs[3] = {0.0, 0.0, 0.0}; /* d/d(delta_s) per input channel */
      for (int p = 0; p < 3; ++p) {
        const int A = pa[p], Bc = pb[p];
        const int64_t ia = i_t[A], ib = i_t[Bc];
        const double da = e_t[A], db = e_t[Bc];
        const double wv[4] = {(1 - da) * (1 - db), da * (1 - db), (1 - da) * db, da * db};
        for (int c = 0; c < 3; ++c) {
          const double P00 = LP(c, p, ia, ib), P10 = LP(c, p, ia + 1, ib);
          const double P01 = LP(c, p, ia, ib + 1), P11 = LP(c, p, ia + 1, ib + 1);
          const double lwv = lw[c * 3 + p];
          const double Bv = wv[0] * P00 + wv[1] * P10 + wv[2] * P01 + wv[3] * P11;
          dlw[c * 3 + p] += g[c] * Bv;
          const double s = g[c] * lwv;
          double* D = dlp + ((c * 3 + p) * dt) * dt;
          D[ia * dt + ib] += s * wv[0];
          D[(ia + 1) * dt + ib] += s * wv[1];
          D[ia * dt + ib + 1] += s * wv[2];
          D[(ia + 1) * dt + ib + 1] += s * wv[3];
          gxa[A] += s * ((1 - db) * (P10 - P00) + db * (P11 - P01));
          gxa[Bc] += s * ((1 - da) * (P01 - P00) + da * (P11 - P10));
        }
      }
      for (int c = 0; c < 3; ++c) dlb[c] += g[c];
      const int64_t jx = ix[x];
      const double ex = dx[x];
      for (int64_t kk = 0; kk < k; ++kk) {
        const int ch = (int)(kk % 3);
        const double gc = g[ch];
        const int64_t jc = i_s[ch];
        const double ec = e_s[ch];
        dgb[kk] += gc;
        /* q = 0: xy plane at (x, y) */
        {
          const double wv[4] = {(1 - ex) * (1 - ey), ex * (1 - ey), (1 - ex) * ey, ex * ey};
          const double P00 = GP(kk, 0, jx, jy), P10 = GP(kk, 0, jx + 1, jy);
          const double P01 = GP(kk, 0, jx, jy + 1), P11 = GP(kk, 0, jx + 1, jy + 1);
          dgw[kk * 3 + 0] += gc * (wv[0] * P00 + wv[1] * P10 + wv[2] * P01 + wv[3] * P11);
          const double s = gc * gw[kk * 3 + 0];
          double* D = dgp + ((kk * 3 + 0) * ds) * ds;
          D[jx * ds + jy] += s * wv[0];
          D[(jx + 1) * ds + jy] += s * wv[1];
          D[jx * ds + jy + 1] += s * wv[2];
          D[(jx + 1) * ds + jy + 1] += s * wv[3];
        }
        /* q = 1: xc plane at (x, X_ch); q = 2: yc plane at (y, X_ch) */
        for (int q = 1; q < 3; ++q) {
          const int64_t ja = q == 1 ? jx : jy;
          const double ea = q == 1 ? ex : ey;
          const double wv[4] = {(1 - ea) * (1 - ec), ea * (1 - ec), (1 - ea) * ec, ea * ec};
          const double P00 = GP(kk, q, ja, jc), P10 = GP(kk, q, ja + 1, jc);
          const double P01 = GP(kk, q, ja, jc + 1), P11 = GP(kk, q, ja + 1, jc + 1);
          dgw[kk * 3 + q] += gc * (wv[0] * P00 + wv[1] * P10 + wv[2] * P01 + wv[3] * P11);
          const double s = gc * gw[kk * 3 + q];
          double* D = dgp + ((kk * 3 + q) * ds) * ds;
          D[ja * ds + jc] += s * wv[0];
          D[(ja + 1) * ds + jc] += s * wv[1];
          D[ja * ds + jc + 1] += s * wv[2];
          D[(ja + 1) * ds + jc + 1] += s * wv[3];
          gxs[ch] += s * ((1 - ea) * (P01 - P00) + ea * (P11 - P10));
        }
      }
      for (int c = 0; c < 3; ++c) {
        gx[c * plane + o] += m[c] * (gxa[c] * (double)(dt - 1) + gxs[c] * (double)(ds - 1));
      }
    }
  }
  free(ix); free(iy); free(dx); free(dy);
  return 0;
}

/*
 * Backward of T = (U diag S) Vt for all nine planes, f64:
 *   dU = dT Vt^T diag S,  dS_n = sum_ij dT_ij U_in Vt_nj,  dVt = diag S U^T dT.
 */
void oracle_reconstruct_bwd(const float* u, const float* s, const float* vt, const double* dT,
                            int64_t d, int64_t n, double* du, double* ds_, double* dvt) {
  for (int64_t cp = 0; cp < 9; ++cp) {
    const float* U = u + cp * d * n;
    const float* S = s + cp * n;
    const float* V = vt + cp * n * d;
    const double* G = dT + cp * d * d;
    for (int64_t i = 0; i < d; ++i)
      for (int64_t m = 0; m < n; ++m) {
        double acc = 0.0;
        for (int64_t j = 0; j < d; ++j) acc += G[i * d + j] * (double)V[m * d + j];
        du[cp * d * n + i * n + m] = acc * (double)S[m];
      }
    for (int64_t m = 0; m < n; ++m) {
      double acc = 0.0;
      for (int64_t i = 0; i < d; ++i)
        for (int64_t j = 0; j < d; ++j)
          acc += G[i * d + j] * (double)U[i * n + m] * (double)V[m * d + j];
      ds_[cp * n + m] = acc;
    }
    for (int64_t m = 0; m < n; ++m)
      for (int64_t j = 0; j < d; ++j) {
        double acc = 0.0;
        for (int64_t i = 0; i < d; ++i) acc += (double)U[i * n + m] * G[i * d + j];
        dvt[cp * n * d + m * d + j] = acc * (double)S[m];
      }
  }
}

int oracle_max_threads(void) { return (int)sysconf(_SC_NPROCESSORS_ONLN); }
