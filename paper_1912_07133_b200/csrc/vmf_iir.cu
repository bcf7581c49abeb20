// vmf_iir.cu -- three-part (forward + central + backward) IIR passes along
// rows or columns, fp32/u16 in, fp32 out, fp64 recurrence state.
//
// Replaces _iir_rows_kernel (engine.py:65-102) and its wrappers iir_rows /
// iir_cols (engine.py:137-158).  Same mathematics:
//   y+(n) = sum_m b_m x(n-m) - sum_m a_m y+(n-m)          (polyz.py:350-358)
//   y-(n) = sum_m b_m x(n+m) - sum_m a_m y-(n+m)
//   out   = (b_zero x + y+) + sign * y-
// with both one-sided recursions started in the steady state of a step at the
// first-seen sample (engine.py:76-78, 90-92).
//
// GPU realisation: a line of N samples is cut into C chunks of L samples so
// that lines x chunks fills the 148 SMs (one line alone is a 4096-step
// dependent chain).  Three phases, all exact in exact arithmetic:
//   1. carry : per (chunk, line) zero-state run of each direction; exports the
//              chunk-end DF-I history (last K outputs, last K inputs).
//   2. scan  : per line, sequential over chunks in each direction:
//              Y(c) = Yzs(c) + T_L [Y(c-1); X(c-1)] with T_L the K x 2K
//              zero-input transfer of the DF-I history over L samples
//              (host-precomputed in long double).  The DF-I basis keeps the
//              carried values O(|x|) instead of the DF-II states' 1/(1+sum a)
//              gain (SURVEY.md §7.3 hard part 2).
//   3. apply : per (chunk, line) DF-I recursion from the true histories; the
//              forward part is parked in shared memory (fp64) and combined
//              with the backward part on the way back.
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "vmf_common.cuh"
#include "vmf_iir.cuh"
#include "plan_cache.hpp"
#include "vmf_prof.cuh"
#include "vmf_rowpass.cuh"
#include "vmf_colpass.cuh"

namespace vmf {

// ---------------------------------------------------------------------------
// host-side planning
// ---------------------------------------------------------------------------

// Schur-Cohn step-down: all roots of z^K + a1 z^(K-1) + ... + aK strictly
// inside the unit circle.  Same predicate as stability_margin(f) > 0
// (engine.py:129-134, which uses np.roots).
bool poles_inside_unit_circle(const double *a_plus, int k) {
  long double a[VMF_MAX_IIR_ORDER + 1], nxt[VMF_MAX_IIR_ORDER + 1];
  a[0] = 1.0L;
  for (int i = 1; i <= k; ++i) a[i] = a_plus[i - 1];
  for (int i = k; i >= 1; --i) {
    long double ki = a[i];
    if (!(fabsl(ki) < 1.0L)) return false;
    long double den = 1.0L - ki * ki;
    for (int j = 0; j < i; ++j) nxt[j] = (a[j] - ki * a[i - j]) / den;
    for (int j = 0; j < i; ++j) a[j] = nxt[j];
  }
  return true;
}

// T (K x 2K, row-major, stride 2K): zero-input response of the DF-I
// recursion after `len` samples, mapping the start history
// [y(-1..-K); x(-1..-K)] to the end history y(len-1 .. len-K).
static void transfer_matrix(const double *b, const double *a, int k, int64_t len,
                            double *T) {
  for (int j = 0; j < 2 * k; ++j) {
    long double Y[VMF_MAX_IIR_ORDER], X[VMF_MAX_IIR_ORDER];
    for (int m = 0; m < k; ++m) {
      Y[m] = (j == m) ? 1.0L : 0.0L;
      X[m] = (j == k + m) ? 1.0L : 0.0L;
    }
    for (int64_t n = 0; n < len; ++n) {
      long double y = 0.0L;
      for (int m = 0; m < k; ++m) y += (long double)b[m] * X[m] - (long double)a[m] * Y[m];
      for (int m = k - 1; m > 0; --m) {
        Y[m] = Y[m - 1];
        X[m] = X[m - 1];
      }
      Y[0] = y;
      X[0] = 0.0L;
    }
    for (int i = 0; i < k; ++i) T[i * 2 * k + j] = (double)Y[i];
  }
}

// Causal impulse response h(0..n-1) of sum b z^-m / (1 + sum a z^-m).
static void impulse(const double *b, const double *a, int k, int n, double *h) {
  long double Y[VMF_MAX_IIR_ORDER] = {0}, X[VMF_MAX_IIR_ORDER] = {0};
  for (int q = 0; q < n; ++q) {
    long double y = 0.0L;
    for (int m = 0; m < k; ++m) y += (long double)b[m] * X[m] - (long double)a[m] * Y[m];
    h[q] = (double)y;
    for (int m = k - 1; m > 0; --m) {
      Y[m] = Y[m - 1];
      X[m] = X[m - 1];
    }
    Y[0] = y;
    X[0] = q == 0 ? 1.0L : 0.0L;
  }
}

void iir_geometry(int64_t n, int k, int64_t *L, int64_t *C, int64_t *Llast) {
  int64_t l = kIirChunk;
  if (l < k) l = k;
  int64_t c = cdiv(n, l);
  int64_t rem = n - (c - 1) * l;
  if (c > 1 && rem < k) {  // fold a too-short tail into the previous chunk
    c -= 1;
    rem += l;
  }
  *L = l;
  *C = c;
  *Llast = rem;
}

size_t iir_workspace_bytes(int64_t lines, int64_t length, int k) {
  if (k <= 0) return 0;
  int64_t L, C, Ll;
  iir_geometry(length, k, &L, &C, &Ll);
  return (size_t)(C * 2 * 2 * k * lines) * sizeof(double) + 256;
}

// ---------------------------------------------------------------------------
// device kernels
// ---------------------------------------------------------------------------

// carry[((c*2 + dir)*2K + j)*M + line]: j < K the y history, j >= K the x
// history, most recent first.  After the scan, j < K hold the true start
// history of chunk c (forward: samples before the chunk; backward: after).
__device__ __forceinline__ int64_t cidx(int64_t c, int dir, int j, int k, int64_t M,
                                        int64_t line) {
  return ((c * 2 + dir) * (2 * k) + j) * M + line;
}

// Zero-state chunk-end histories as a linear functional of the chunk's
// samples (no dependency chain, one sweep for both directions):
//   forward  y+(e-1-i) = sum_t h(len-1-i-t) x(r0+t)
//   backward y-(r0+i)  = sum_t h(t-i)       x(r0+t)
// with h the causal impulse response of sum b z^-m / (1 + sum a z^-m)
// (h(0) = 0), host-computed in long double.  K fp64 FMAs per sample and
// direction -- the same count as running the DF-II state recursion, but
// with the rounding of a short dot product instead of a 1/(1+sum a)-gain
// recursion.
template <int K, int O, typename T>
__global__ void __launch_bounds__(128) iir_carry_kernel(const T *__restrict__ x, int64_t ldx,
                                                        IirParams p,
                                                        double *__restrict__ carry) {
  int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t line = tid % p.M, c = tid / p.M;
  if (c >= p.C) return;
  int64_t r0 = c * p.L;
  int len = (int)((c == p.C - 1) ? p.Llast : p.L);
  double f[K], bk[K];
#pragma unroll
  for (int i = 0; i < K; ++i) f[i] = bk[i] = 0.0;
  for (int t = 0; t < len; ++t) {
    double v = ld64(line_ptr<O>(x, ldx, line, r0 + t));
#pragma unroll
    for (int i = 0; i < K; ++i) {
      int qf = len - 1 - i - t, qb = t - i;
      if (qf > 0) f[i] = fma(p.h[qf], v, f[i]);
      if (qb > 0) bk[i] = fma(p.h[qb], v, bk[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < K; ++i) {
    carry[cidx(c, 0, i, K, p.M, line)] = f[i];
    carry[cidx(c, 0, K + i, K, p.M, line)] = ld64(line_ptr<O>(x, ldx, line, r0 + len - 1 - i));
    carry[cidx(c, 1, i, K, p.M, line)] = bk[i];
    carry[cidx(c, 1, K + i, K, p.M, line)] = ld64(line_ptr<O>(x, ldx, line, r0 + i));
  }
}

template <int K>
__device__ __forceinline__ void propagate(const double *Tm, double *Y, double *X,
                                          const double *Yzs, const double *Xl) {
  double Yn[K];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    double acc = Yzs[i];
#pragma unroll
    for (int j = 0; j < K; ++j) acc = fma(Tm[i * 2 * K + j], Y[j], acc);
#pragma unroll
    for (int j = 0; j < K; ++j) acc = fma(Tm[i * 2 * K + K + j], X[j], acc);
    Yn[i] = acc;
  }
#pragma unroll
  for (int i = 0; i < K; ++i) {
    Y[i] = Yn[i];
    X[i] = Xl[i];
  }
}

template <int K, int O, typename T>
__global__ void __launch_bounds__(128) iir_scan_kernel(const T *__restrict__ x, int64_t ldx,
                                                       IirParams p, double *__restrict__ carry) {
  int64_t line = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (line >= p.M) return;
  double Y[K], X[K], Yzs[K], Xl[K];
  // forward, steady state of a step of x(0)
  double x0 = ld64(line_ptr<O>(x, ldx, line, 0));
#pragma unroll
  for (int i = 0; i < K; ++i) {
    Y[i] = p.yss * x0;
    X[i] = x0;
  }
  for (int64_t c = 0; c < p.C; ++c) {
    bool more = c < p.C - 1;
    if (more) {
#pragma unroll
      for (int i = 0; i < K; ++i) {
        Yzs[i] = carry[cidx(c, 0, i, K, p.M, line)];
        Xl[i] = carry[cidx(c, 0, K + i, K, p.M, line)];
      }
    }
#pragma unroll
    for (int i = 0; i < K; ++i) carry[cidx(c, 0, i, K, p.M, line)] = Y[i];
    if (more) propagate<K>(&p.T[0][0], Y, X, Yzs, Xl);
  }
  // backward, steady state of a step of x(N-1)
  double xn = ld64(line_ptr<O>(x, ldx, line, p.N - 1));
#pragma unroll
  for (int i = 0; i < K; ++i) {
    Y[i] = p.yss * xn;
    X[i] = xn;
  }
  for (int64_t c = p.C - 1; c >= 0; --c) {
    bool more = c > 0;
    if (more) {
#pragma unroll
      for (int i = 0; i < K; ++i) {
        Yzs[i] = carry[cidx(c, 1, i, K, p.M, line)];
        Xl[i] = carry[cidx(c, 1, K + i, K, p.M, line)];
      }
    }
#pragma unroll
    for (int i = 0; i < K; ++i) carry[cidx(c, 1, i, K, p.M, line)] = Y[i];
    if (more) propagate<K>((c == p.C - 1) ? &p.T[1][0] : &p.T[0][0], Y, X, Yzs, Xl);
  }
}

// DF-I step: y = sum b_m X[m] - sum a_m Y[m], with the a_1 term last so the
// loop-carried dependency is a single FMA.
template <int K>
__device__ __forceinline__ double dfi_step(const double *b, const double *a, const double *X,
                                           const double *Y) {
  double s = 0.0;
#pragma unroll
  for (int m = 0; m < K; ++m) s = fma(b[m], X[m], s);
#pragma unroll
  for (int m = K - 1; m >= 1; --m) s = fma(-a[m], Y[m], s);
  return fma(-a[0], Y[0], s);
}

template <int K>
__device__ __forceinline__ void push(double *H, double v) {
#pragma unroll
  for (int m = K - 1; m > 0; --m) H[m] = H[m - 1];
  H[0] = v;
}

template <int K, int O, typename T>
__global__ void __launch_bounds__(kIirApplyThreads) iir_apply_kernel(
    const T *__restrict__ x, int64_t ldx, float *__restrict__ y, int64_t ldy, IirParams p,
    const double *__restrict__ carry) {
  extern __shared__ double park[];  // [Lmax][blockDim]
  int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t line = tid % p.M, c = tid / p.M;
  if (c >= p.C) return;
  int64_t r0 = c * p.L, len = (c == p.C - 1) ? p.Llast : p.L;
  double a[K], b[K];
#pragma unroll
  for (int m = 0; m < K; ++m) {
    a[m] = p.a[m];
    b[m] = p.b[m];
  }
  double Y[K], X[K];
  // forward
#pragma unroll
  for (int i = 0; i < K; ++i) {
    Y[i] = carry[cidx(c, 0, i, K, p.M, line)];
    int64_t q = r0 - 1 - i;
    X[i] = ld64(line_ptr<O>(x, ldx, line, q < 0 ? 0 : q));
  }
  for (int64_t n = 0; n < len; ++n) {
    double xn = ld64(line_ptr<O>(x, ldx, line, r0 + n));
    double yp = dfi_step<K>(b, a, X, Y);
    park[n * blockDim.x + threadIdx.x] = fma(p.b0, xn, yp);
    push<K>(Y, yp);
    push<K>(X, xn);
  }
  // backward, combining on the way
#pragma unroll
  for (int i = 0; i < K; ++i) {
    Y[i] = carry[cidx(c, 1, i, K, p.M, line)];
    int64_t q = r0 + len + i;
    X[i] = ld64(line_ptr<O>(x, ldx, line, q > p.N - 1 ? p.N - 1 : q));
  }
  for (int64_t n = len - 1; n >= 0; --n) {
    double xn = ld64(line_ptr<O>(x, ldx, line, r0 + n));
    double ym = dfi_step<K>(b, a, X, Y);
    double out = fma(p.sign, ym, park[n * blockDim.x + threadIdx.x]);
    *line_ptr_out<O>(y, ldy, line, r0 + n) = (float)out;
    push<K>(Y, ym);
    push<K>(X, xn);
  }
}

// K = 0: no recursion, out = b_zero * x (engine.py:79-102 with k = 0).
template <typename T>
__global__ void scale_kernel(const T *__restrict__ x, int64_t ldx, float *__restrict__ y,
                             int64_t ldy, int64_t h, int64_t w, double b0) {
  int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= h * w) return;
  int64_t i = tid / w, j = tid % w;
  y[i * ldy + j] = (float)(b0 * ld64(x + i * ldx + j));
}

// ---------------------------------------------------------------------------
// host launcher
// ---------------------------------------------------------------------------
template <int K, int O, typename T>
static int launch_iir(const T *x, int64_t ldx, float *y, int64_t ldy, const IirParams &p,
                      double *carry, cudaStream_t st) {
  int64_t work = p.C * p.M;
  int nb = (int)cdiv(work, 128);
  {
    Launch g(K_IIR_CARRY, st);
    iir_carry_kernel<K, O, T><<<nb, 128, 0, st>>>(x, ldx, p, carry);
  }
  {
    Launch g(K_IIR_SCAN, st);
    iir_scan_kernel<K, O, T><<<(int)cdiv(p.M, 128), 128, 0, st>>>(x, ldx, p, carry);
  }
  size_t smem = (size_t)(p.L + K) * kIirApplyThreads * sizeof(double);
  static PerDevice attr_set;
  if (attr_set.first()) {
    cudaFuncSetAttribute(iir_apply_kernel<K, O, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
  }
  {
    Launch g(K_IIR_APPLY, st);
    iir_apply_kernel<K, O, T><<<(int)cdiv(work, kIirApplyThreads), kIirApplyThreads, smem, st>>>(
        x, ldx, y, ldy, p, carry);
  }
  return cuda_status("iir pass");
}

template <int O, typename T>
static int dispatch_k(const T *x, int64_t ldx, float *y, int64_t ldy, const IirParams &p,
                      double *carry, cudaStream_t st) {
  switch (p.K) {
    case 1: return launch_iir<1, O, T>(x, ldx, y, ldy, p, carry, st);
    case 2: return launch_iir<2, O, T>(x, ldx, y, ldy, p, carry, st);
    case 3: return launch_iir<3, O, T>(x, ldx, y, ldy, p, carry, st);
    case 4: return launch_iir<4, O, T>(x, ldx, y, ldy, p, carry, st);
    case 5: return launch_iir<5, O, T>(x, ldx, y, ldy, p, carry, st);
    case 6: return launch_iir<6, O, T>(x, ldx, y, ldy, p, carry, st);
    case 7: return launch_iir<7, O, T>(x, ldx, y, ldy, p, carry, st);
    case 8: return launch_iir<8, O, T>(x, ldx, y, ldy, p, carry, st);
  }
  return fail(VMF_EVALUE, "IIR order %d outside 0..%d", p.K, VMF_MAX_IIR_ORDER);
}

int iir_plan(IirParams *p, int64_t lines, int64_t length, const double *b_plus,
             const double *a_plus, int k, double b_zero, int sign) {
  if (k < 0 || k > VMF_MAX_IIR_ORDER)
    return fail(VMF_EVALUE, "IIR order %d outside 0..%d", k, VMF_MAX_IIR_ORDER);
  if (length < 2 * k + 1)
    return fail(VMF_EVALUE, "row length %lld < 2K+1 = %d", (long long)length, 2 * k + 1);
  static PlanCache<IirParams> cache;
  std::vector<unsigned char> key;
  key_add(key, lines);
  key_add(key, length);
  key_add(key, k);
  key_add(key, b_zero);
  key_add(key, sign);
  key_add(key, b_plus, sizeof(double) * k);
  key_add(key, a_plus, sizeof(double) * k);
  if (cache.get(key, p)) return VMF_OK;  // validated when it was stored
  if (k > 0 && !poles_inside_unit_circle(a_plus, k))
    return fail(VMF_ESTABILITY, "recursion has a pole on or outside the unit circle");
  memset(p, 0, sizeof(*p));
  p->K = k;
  p->M = lines;
  p->N = length;
  p->b0 = b_zero;
  p->sign = sign >= 0 ? 1.0 : -1.0;
  double asum = 1.0, bsum = 0.0;
  for (int m = 0; m < k; ++m) {
    p->a[m] = a_plus[m];
    p->b[m] = b_plus[m];
    asum += a_plus[m];
    bsum += b_plus[m];
  }
  p->yss = k ? bsum / asum : 0.0;
  if (k == 0) return VMF_OK;
  iir_geometry(length, k, &p->L, &p->C, &p->Llast);
  transfer_matrix(p->b, p->a, k, p->L, &p->T[0][0]);
  transfer_matrix(p->b, p->a, k, p->Llast, &p->T[1][0]);
  impulse(p->b, p->a, k, kIirHmax, p->h);
  cache.put(key, *p);
  return VMF_OK;
}

template <int O>
int iir_pass(const void *x, int x_dtype, float *y, int64_t h, int64_t w, int64_t ldx,
             int64_t ldy, const double *b_plus, const double *a_plus, int k, double b_zero,
             int sign, void *ws, size_t ws_bytes, cudaStream_t st) {
  int64_t lines = O == ROWS ? h : w, length = O == ROWS ? w : h;
  if (h < 1 || w < 1) return fail(VMF_EVALUE, "image must be a 2-D array");
  if (ldx < w || ldy < w)
    return fail(VMF_EVALUE, "row pitch smaller than width (ldx=%lld ldy=%lld w=%lld)",
                (long long)ldx, (long long)ldy, (long long)w);
  if (x_dtype < VMF_F32 || x_dtype > VMF_U16BE) return fail(VMF_EVALUE, "unsupported dtype");
  IirParams p;
  int rc = iir_plan(&p, lines, length, b_plus, a_plus, k, b_zero, sign);
  if (rc) return rc;
  if (k == 0) {
    int64_t n = h * w;
    Launch g(K_IIR_SCALE, st);
    return with_sample_type(x_dtype, x, [&](auto xt) {
      scale_kernel<<<(int)cdiv(n, 256), 256, 0, st>>>(xt, ldx, y, ldy, h, w, b_zero);
      return cuda_status("iir scale");
    });
  }
  if (O == ROWS && rowpass_supported(w, k) && !getenv("VMF_FORCE_GENERIC"))
    return with_sample_type(x_dtype, x,
                            [&](auto xt) { return rowpass_run(xt, ldx, y, ldy, p, h, w, st); });
  // columns, fp32, K 2..4: the band-parallel column pass (carry, scan, walk)
  // writing the blur -- the fused pipeline's kernels without the Laplacian;
  // needs its larger workspace (vmf_iir_cols_workspace_bytes)
  if (O == COLS && x_dtype == VMF_F32 && colpass_supported(h, w, k) &&
      !getenv("VMF_FORCE_GENERIC") && ws && ws_bytes >= colpass_workspace_bytes(h, w, k, 0) + 256)
    return colpass_run((const float *)x, ldx, y, ldy, nullptr, p, h, w, 1.0f, 0.0f, nullptr,
                       nullptr, 0, nullptr, nullptr, ws, ws_bytes, st, true);
  size_t need = iir_workspace_bytes(lines, length, k);
  if (ws_bytes < need || !ws)
    return fail(VMF_EVALUE, "IIR workspace too small: %zu < %zu bytes", ws_bytes, need);
  double *carry = (double *)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  return with_sample_type(x_dtype, x,
                          [&](auto xt) { return dispatch_k<O>(xt, ldx, y, ldy, p, carry, st); });
}

template int iir_pass<ROWS>(const void *, int, float *, int64_t, int64_t, int64_t, int64_t,
                            const double *, const double *, int, double, int, void *, size_t,
                            cudaStream_t);
template int iir_pass<COLS>(const void *, int, float *, int64_t, int64_t, int64_t, int64_t,
                            const double *, const double *, int, double, int, void *, size_t,
                            cudaStream_t);

}  // namespace vmf
