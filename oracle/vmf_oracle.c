/*
 * vmf_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product in paper_1912_07133_b200/csrc and the CPU baseline leg of bench.py.
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
 * --impl reference) may load it.  The product path never links it.
 *
 * Every function restates one piece of the reference package `vmfilt`
 * (paths relative to /root/reference/pkg/src/vmfilt/):
 *
 *   orc_iir_rows   engine.py:65-102  (_iir_rows_kernel; validation 137-153)
 *   orc_iir_cols   engine.py:156-158 (iir_rows on x.T; same per-column
 *                  arithmetic, swept row-major instead of transposing)
 *   orc_conv_rows  engine.py:35-62   (_conv_rows_kernel; validation 112-121)
 *   orc_conv_cols  engine.py:124-126
 *   orc_laplacian  engine.py:205-228 D20 = conv_rows(B,(1,-2,1)),
 *                  D02 = conv_cols(B,(1,-2,1)); trace D20+D02 (blob.py:161)
 *   orc_detect3x3  stage-4 rule of SURVEY.md §8(d) (no reference function;
 *                  conventions from blob.py:162-168): strict 3x3 extremum
 *                  with edge-replicated neighbours, |L| >= thr
 *   orc_detect3x3x3 scale-space variant (config 3)
 *
 * Arithmetic is IEEE double with the reference's operation order and no FMA
 * contraction (built with -ffp-contract=off), so results are bit-identical to
 * numba's non-fastmath build of the reference kernels (pinned by
 * tests/test_oracle.py against tests/golden/).
 *
 * Row/column parallelism is a pthread parallel-for over independent lines,
 * the analogue of numba prange (engine.py:39,69).  Output does not depend on
 * the thread count (each line is computed by exactly one thread).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define ORC_KMAX 16
#define ORC_COLBLOCK 64

static int g_threads = 0;

int orc_max_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

void orc_set_threads(int n) { g_threads = n; }

static int nthreads(void) { return g_threads > 0 ? g_threads : orc_max_threads(); }

typedef void (*range_fn)(void *ctx, int64_t lo, int64_t hi);
typedef struct { range_fn fn; void *ctx; int64_t lo, hi; } par_job;

static void *par_run(void *p) {
  par_job *j = (par_job *)p;
  if (j->lo < j->hi) j->fn(j->ctx, j->lo, j->hi);
  return NULL;
}

/* Static split of [0, n) into contiguous ranges, one per thread. */
static void par_for(int64_t n, range_fn fn, void *ctx) {
  int t = nthreads();
  if (t > 256) t = 256;
  if (t <= 1 || n <= 1) { fn(ctx, 0, n); return; }
  if (t > n) t = (int)n;
  pthread_t th[256];
  par_job jobs[256];
  for (int i = 0; i < t; ++i) {
    jobs[i].fn = fn; jobs[i].ctx = ctx;
    jobs[i].lo = n * i / t; jobs[i].hi = n * (i + 1) / t;
  }
  for (int i = 1; i < t; ++i) pthread_create(&th[i], NULL, par_run, &jobs[i]);
  par_run(&jobs[0]);
  for (int i = 1; i < t; ++i) pthread_join(th[i], NULL);
}

/* engine.py:65-102, one row at a time. */
static void iir_line(const double *x, double *out, int64_t w, const double *bp,
                     const double *ap, int k, double b0, double sign) {
  double s[ORC_KMAX];
  double asum = 1.0;
  for (int m = 0; m < k; ++m) asum += ap[m];
  double w0 = x[0] / asum;
  for (int m = 0; m < k; ++m) s[m] = w0;
  for (int64_t n = 0; n < w; ++n) {
    double wn = x[n];
    double acc = b0 * x[n];
    for (int m = 0; m < k; ++m) {
      wn -= ap[m] * s[m];
      acc += bp[m] * s[m];
    }
    out[n] = acc;
    for (int m = k - 1; m > 0; --m) s[m] = s[m - 1];
    s[0] = wn;
  }
  w0 = x[w - 1] / asum;
  for (int m = 0; m < k; ++m) s[m] = w0;
  for (int64_t n = w - 1; n >= 0; --n) {
    double wn = x[n];
    double acc = 0.0;
    for (int m = 0; m < k; ++m) {
      wn -= ap[m] * s[m];
      acc += bp[m] * s[m];
    }
    out[n] += sign * acc;
    for (int m = k - 1; m > 0; --m) s[m] = s[m - 1];
    s[0] = wn;
  }
}

typedef struct {
  const double *x; double *out; int64_t h, w;
  const double *bp, *ap; int k; double b0, sign;
  const double *taps; int ntaps;
} line_ctx;

static void iir_rows_rng(void *c, int64_t lo, int64_t hi) {
  line_ctx *a = (line_ctx *)c;
  for (int64_t i = lo; i < hi; ++i)
    iir_line(a->x + i * a->w, a->out + i * a->w, a->w, a->bp, a->ap, a->k,
             a->b0, a->sign);
}

void orc_iir_rows(const double *x, double *out, int64_t h, int64_t w,
                  const double *bp, const double *ap, int k, double b0,
                  double sign) {
  line_ctx c = {x, out, h, w, bp, ap, k, b0, sign, NULL, 0};
  par_for(h, iir_rows_rng, &c);
}

/* iir_rows(x.T).T with the per-column arithmetic of engine.py:65-102,
 * swept row-major over blocks of columns (cache friendly; same results). */
static void iir_cols_rng(void *c, int64_t blo, int64_t bhi) {
  line_ctx *a = (line_ctx *)c;
  const double *x = a->x, *bp = a->bp, *ap = a->ap;
  double *out = a->out;
  int64_t h = a->h, w = a->w;
  int k = a->k;
  double b0 = a->b0, sign = a->sign;
  double asum = 1.0;
  for (int m = 0; m < k; ++m) asum += ap[m];
  for (int64_t bi = blo; bi < bhi; ++bi) {
    int64_t j0 = bi * ORC_COLBLOCK;
    int64_t nb = w - j0 < ORC_COLBLOCK ? w - j0 : ORC_COLBLOCK;
    double s[ORC_KMAX][ORC_COLBLOCK];
    for (int64_t j = 0; j < nb; ++j) {
      double w0 = x[j0 + j] / asum;
      for (int m = 0; m < k; ++m) s[m][j] = w0;
    }
    for (int64_t n = 0; n < h; ++n) {
      const double *xr = x + n * w + j0;
      double *orow = out + n * w + j0;
      for (int64_t j = 0; j < nb; ++j) {
        double wn = xr[j];
        double acc = b0 * xr[j];
        for (int m = 0; m < k; ++m) {
          wn -= ap[m] * s[m][j];
          acc += bp[m] * s[m][j];
        }
        orow[j] = acc;
        for (int m = k - 1; m > 0; --m) s[m][j] = s[m - 1][j];
        s[0][j] = wn;
      }
    }
    for (int64_t j = 0; j < nb; ++j) {
      double w0 = x[(h - 1) * w + j0 + j] / asum;
      for (int m = 0; m < k; ++m) s[m][j] = w0;
    }
    for (int64_t n = h - 1; n >= 0; --n) {
      const double *xr = x + n * w + j0;
      double *orow = out + n * w + j0;
      for (int64_t j = 0; j < nb; ++j) {
        double wn = xr[j];
        double acc = 0.0;
        for (int m = 0; m < k; ++m) {
          wn -= ap[m] * s[m][j];
          acc += bp[m] * s[m][j];
        }
        orow[j] += sign * acc;
        for (int m = k - 1; m > 0; --m) s[m][j] = s[m - 1][j];
        s[0][j] = wn;
      }
    }
  }
}

void orc_iir_cols(const double *x, double *out, int64_t h, int64_t w,
                  const double *bp, const double *ap, int k, double b0,
                  double sign) {
  line_ctx c = {x, out, h, w, bp, ap, k, b0, sign, NULL, 0};
  par_for((w + ORC_COLBLOCK - 1) / ORC_COLBLOCK, iir_cols_rng, &c);
}

/* engine.py:35-62: out[n] = sum_{m=-k..k} taps[k+m] x[clamp(n-m)], m ascending. */
static void conv_line(const double *x, double *out, int64_t w,
                      const double *taps, int k) {
  for (int64_t n = k; n < w - k; ++n) {
    double acc = 0.0;
    for (int m = -k; m <= k; ++m) acc += taps[k + m] * x[n - m];
    out[n] = acc;
  }
  for (int64_t n = 0; n < k && n < w; ++n) {
    double acc = 0.0;
    for (int m = -k; m <= k; ++m) {
      int64_t j = n - m;
      if (j < 0) j = 0;
      acc += taps[k + m] * x[j];
    }
    out[n] = acc;
  }
  for (int64_t n = (w - k > 0 ? w - k : 0); n < w; ++n) {
    double acc = 0.0;
    for (int m = -k; m <= k; ++m) {
      int64_t j = n - m;
      if (j < 0) j = 0;
      else if (j >= w) j = w - 1;
      acc += taps[k + m] * x[j];
    }
    out[n] = acc;
  }
}

static void conv_rows_rng(void *c, int64_t lo, int64_t hi) {
  line_ctx *a = (line_ctx *)c;
  int k = (a->ntaps - 1) / 2;
  for (int64_t i = lo; i < hi; ++i)
    conv_line(a->x + i * a->w, a->out + i * a->w, a->w, a->taps, k);
}

void orc_conv_rows(const double *x, double *out, int64_t h, int64_t w,
                   const double *taps, int ntaps) {
  line_ctx c = {x, out, h, w, NULL, NULL, 0, 0.0, 0.0, taps, ntaps};
  par_for(h, conv_rows_rng, &c);
}

/* conv_rows(x.T).T, same per-output accumulation order, swept row-major. */
static void conv_cols_rng(void *c, int64_t lo, int64_t hi) {
  line_ctx *a = (line_ctx *)c;
  int k = (a->ntaps - 1) / 2;
  int64_t h = a->h, w = a->w;
  for (int64_t n = lo; n < hi; ++n) {
    double *orow = a->out + n * w;
    for (int64_t j = 0; j < w; ++j) orow[j] = 0.0;
    for (int m = -k; m <= k; ++m) {
      int64_t r = n - m;
      if (r < 0) r = 0;
      else if (r >= h) r = h - 1;
      const double *xr = a->x + r * w;
      double t = a->taps[k + m];
      for (int64_t j = 0; j < w; ++j) orow[j] += t * xr[j];
    }
  }
}

void orc_conv_cols(const double *x, double *out, int64_t h, int64_t w,
                   const double *taps, int ntaps) {
  line_ctx c = {x, out, h, w, NULL, NULL, 0, 0.0, 0.0, taps, ntaps};
  par_for(h, conv_cols_rng, &c);
}

/* D20 + D02 with taps (1,-2,1) and replicate edges (engine.py:218-227,
 * blob.py:161): acc = 0 + 1*x[n+1] + (-2)*x[n] + 1*x[n-1] per axis. */
static void lap_rng(void *c, int64_t lo, int64_t hi) {
  line_ctx *a = (line_ctx *)c;
  const double *B = a->x;
  double *L = a->out;
  int64_t h = a->h, w = a->w;
  for (int64_t i = lo; i < hi; ++i) {
    int64_t iu = i > 0 ? i - 1 : 0, id = i < h - 1 ? i + 1 : h - 1;
    for (int64_t j = 0; j < w; ++j) {
      int64_t jl = j > 0 ? j - 1 : 0, jr = j < w - 1 ? j + 1 : w - 1;
      double dx = 0.0;
      dx += 1.0 * B[i * w + jr];
      dx += -2.0 * B[i * w + j];
      dx += 1.0 * B[i * w + jl];
      double dy = 0.0;
      dy += 1.0 * B[id * w + j];
      dy += -2.0 * B[i * w + j];
      dy += 1.0 * B[iu * w + j];
      L[i * w + j] = dx + dy;
    }
  }
}

void orc_laplacian(const double *B, double *L, int64_t h, int64_t w) {
  line_ctx c = {B, L, h, w, NULL, NULL, 0, 0.0, 0.0, NULL, 0};
  par_for(h, lap_rng, &c);
}

double orc_absmax(const double *a, int64_t n) {
  double m = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double v = fabs(a[i]);
    if (v > m) m = v;
  }
  return m;
}

/* 1 = strict max, -1 = strict min, 0 = neither, over the 8 in-frame
 * neighbours.  With edge-replicated padding a border pixel is its own
 * neighbour, so it can never be strict: border pixels return 0. */
static int extremum8(const double *L, int64_t h, int64_t w, int64_t i, int64_t j) {
  if (i <= 0 || j <= 0 || i >= h - 1 || j >= w - 1) return 0;
  double v = L[i * w + j];
  int gt = 1, lt = 1;
  for (int di = -1; di <= 1; ++di)
    for (int dj = -1; dj <= 1; ++dj) {
      if (!di && !dj) continue;
      double u = L[(i + di) * w + j + dj];
      if (!(v > u)) gt = 0;
      if (!(v < u)) lt = 0;
    }
  return gt ? 1 : (lt ? -1 : 0);
}

/* Detections in row-major (y, x) order; returns the count (may exceed cap,
 * only the first cap are written). */
int64_t orc_detect3x3(const double *L, int64_t h, int64_t w, double thr,
                      int32_t *ys, int32_t *xs, double *vals, int64_t cap) {
  int64_t cnt = 0;
  for (int64_t i = 1; i < h - 1; ++i)
    for (int64_t j = 1; j < w - 1; ++j) {
      double v = L[i * w + j];
      if (fabs(v) < thr) continue;
      int e = extremum8(L, h, w, i, j);
      if ((e == 1 && v >= thr) || (e == -1 && -v >= thr)) {
        if (cnt < cap) {
          ys[cnt] = (int32_t)i;
          xs[cnt] = (int32_t)j;
          vals[cnt] = v;
        }
        ++cnt;
      }
    }
  return cnt;
}

/* Scale-space 3x3x3 NMS over a stack N[s][h][w] (already sigma^2
 * normalised): strict extremum against the 8 in-scale neighbours and the 9
 * pixels of each existing adjacent scale (one-sided at the ends). */
int64_t orc_detect3x3x3(const double *N, int64_t ns, int64_t h, int64_t w,
                        double thr, int32_t *ss, int32_t *ys, int32_t *xs,
                        double *vals, int64_t cap) {
  int64_t cnt = 0, plane = h * w;
  for (int64_t s = 0; s < ns; ++s)
    for (int64_t i = 1; i < h - 1; ++i)
      for (int64_t j = 1; j < w - 1; ++j) {
        const double *P = N + s * plane;
        double v = P[i * w + j];
        if (fabs(v) < thr) continue;
        int e = extremum8(P, h, w, i, j);
        if (!e) continue;
        for (int64_t t = s - 1; t <= s + 1 && e; t += 2) {
          if (t < 0 || t >= ns) continue;
          const double *Q = N + t * plane;
          for (int di = -1; di <= 1 && e; ++di)
            for (int dj = -1; dj <= 1; ++dj) {
              double u = Q[(i + di) * w + j + dj];
              if (e == 1 && !(v > u)) { e = 0; break; }
              if (e == -1 && !(v < u)) { e = 0; break; }
            }
        }
        if ((e == 1 && v >= thr) || (e == -1 && -v >= thr)) {
          if (cnt < cap) {
            ss[cnt] = (int32_t)s;
            ys[cnt] = (int32_t)i;
            xs[cnt] = (int32_t)j;
            vals[cnt] = v;
          }
          ++cnt;
        }
      }
  return cnt;
}
