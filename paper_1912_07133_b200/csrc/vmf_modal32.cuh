// vmf_modal32.cuh -- fp32 modal realisation of the three-part IIR's causal
// part, shared by the fp32 "Laplacian-first" row and column passes
// (vmf_rowlap.cu, vmf_colpass32.cu).
//
// The reference's causal recursion (engine.py:79-88, DF-II:
// w(n) = x(n) - sum a_m s_m, y+(n) = sum b_m s_m) has the impulse response
// h(m), m >= 1.  In fp32 its direct forms lose up to 1e-3 of max|L| at
// sigma = 32 (poles near 1: DF-II carries x / (1 + sum a) ~ 3.4e4 x, DF-I
// feeds rounding through 1 / A(z)); the modal state-space form
//     u(n) = A u(n-1) + b x(n),   y+(n) = c . u(n-1),
// with A a Jordan chain (repeated real pole p: u1 = p u1 + x,
// u2 = p u2 + u1, ...) or a 2x2 rotation (complex pair p +- i q), keeps the
// rounding of every state relative to that state.  c is fitted to h(1..K) and
// the whole response is checked against the reference recursion (long
// double) before a plan is used.
#pragma once
#include <cmath>
#include <cstring>

#include "vmf_common.cuh"

namespace vmf {

// modal realisation: JORDAN (repeated real pole, K = 2..4) or CPAIR (K = 2)
enum Modal32Kind { M32_JORDAN = 0, M32_CPAIR = 1 };

// ---------------------------------------------------------------------------
// the recursion: u <- A u + b x, y = c . u (before the update)
// ---------------------------------------------------------------------------
template <int K, int KIND>
struct Rec32 {
  float u[K];
  __device__ __forceinline__ float out(const float *c) const {
    float y = c[0] * u[0];
#pragma unroll
    for (int i = 1; i < K; ++i) y = fmaf(c[i], u[i], y);
    return y;
  }
  __device__ __forceinline__ float out_from(const float *c, float acc) const {
#pragma unroll
    for (int i = 0; i < K; ++i) acc = fmaf(c[i], u[i], acc);
    return acc;
  }
  template <class P_>
  __device__ __forceinline__ void step(const P_ &P, float x) {
    if (KIND == M32_JORDAN) {
      u[0] = fmaf(P.p, u[0], x);
#pragma unroll
      for (int i = 1; i < K; ++i) u[i] = fmaf(P.p, u[i], u[i - 1]);
    } else {
      const float ur = u[0], ui = u[1];
      u[0] = fmaf(P.p, ur, fmaf(-P.q, ui, x));
      u[1] = fmaf(P.q, ur, P.p * ui);
    }
  }
};

// U = ((l - c) + (r - c)) + ((u - c) + (d - c)): every term a difference of
// neighbouring T values (rounding relative to the difference); the same
// expression everywhere, so the carry and apply passes see bitwise-equal U.
__device__ __forceinline__ float lap5(float l, float c, float r, float u, float d) {
  return ((l - c) + (r - c)) + ((u - c) + (d - c));
}

// ---------------------------------------------------------------------------
// host: long-double linear algebra and the realisation
// ---------------------------------------------------------------------------
typedef long double ld;

inline void matmul(const ld *A, const ld *B, ld *C, int k) {
  ld t[16];
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) {
      ld s = 0;
      for (int m = 0; m < k; ++m) s += A[i * k + m] * B[m * k + j];
      t[i * k + j] = s;
    }
  memcpy(C, t, sizeof(ld) * k * k);
}

inline void matpow(const ld *A, int64_t n, ld *out, int k) {
  ld R[16], P[16];
  for (int i = 0; i < k * k; ++i) R[i] = (i % (k + 1) == 0) ? 1 : 0;
  memcpy(P, A, sizeof(ld) * k * k);
  while (n > 0) {
    if (n & 1) matmul(R, P, R, k);
    matmul(P, P, P, k);
    n >>= 1;
  }
  memcpy(out, R, sizeof(ld) * k * k);
}

// solve M x = y (k <= 4), partial pivoting; false if singular
inline bool solve(ld *M, ld *y, int k) {
  for (int c = 0; c < k; ++c) {
    int piv = c;
    for (int r = c + 1; r < k; ++r)
      if (fabsl(M[r * k + c]) > fabsl(M[piv * k + c])) piv = r;
    if (fabsl(M[piv * k + c]) < 1e-300L) return false;
    if (piv != c) {
      for (int m = 0; m < k; ++m) {
        ld t = M[c * k + m];
        M[c * k + m] = M[piv * k + m];
        M[piv * k + m] = t;
      }
      ld t = y[c];
      y[c] = y[piv];
      y[piv] = t;
    }
    for (int r = 0; r < k; ++r) {
      if (r == c) continue;
      const ld f = M[r * k + c] / M[c * k + c];
      for (int m = 0; m < k; ++m) M[r * k + m] -= f * M[c * k + m];
      y[r] -= f * y[c];
    }
  }
  for (int c = 0; c < k; ++c) y[c] /= M[c * k + c];
  return true;
}

// Causal impulse response of the reference's DF-II recursion (engine.py:79-88)
inline void impulse_ref(const double *b, const double *a, int k, int n, ld *h) {
  ld s[VMF_MAX_IIR_ORDER] = {0};
  for (int t = 0; t < n; ++t) {
    ld y = 0, w = (t == 0) ? 1 : 0;
    for (int m = 0; m < k; ++m) {
      y += (ld)b[m] * s[m];
      w -= (ld)a[m] * s[m];
    }
    h[t] = y;
    for (int m = k - 1; m > 0; --m) s[m] = s[m - 1];
    s[0] = w;
  }
}

struct Modal {
  int kind, k;
  ld p, q;
  ld A[16], bv[4], c[4];
};

// repeated real pole (a_plus = coefficients of (1 - p w)^k) or, for k = 2, a
// complex pair; the output vector c matches the first k impulse-response
// samples and the whole response is verified against the reference's
// recursion.
inline bool modal_realise(const double *b, const double *a, int k, Modal *M) {
  if (k < 2 || k > 4) return false;
  memset(M, 0, sizeof(*M));
  M->k = k;
  const ld p = -(ld)a[0] / k;
  ld binom = 1, maxdev = 0, scale = 0;
  for (int m = 1; m <= k; ++m) {
    binom = binom * (k - m + 1) / m;
    const ld coef = binom * powl(-p, m);
    maxdev = fmaxl(maxdev, fabsl(coef - (ld)a[m - 1]));
    scale = fmaxl(scale, fabsl((ld)a[m - 1]));
  }
  if (maxdev <= 1e-13L * scale && p > 0 && p < 1) {
    M->kind = M32_JORDAN;
    M->p = p;
    for (int i = 0; i < k; ++i) {
      M->bv[i] = 1;
      for (int j2 = 0; j2 < k; ++j2) M->A[i * k + j2] = j2 <= i ? p : 0;
    }
  } else if (k == 2 && a[0] * a[0] - 4 * a[1] < 0) {
    M->kind = M32_CPAIR;
    M->p = -(ld)a[0] / 2;
    M->q = sqrtl(4 * (ld)a[1] - (ld)a[0] * a[0]) / 2;
    M->A[0] = M->p;
    M->A[1] = -M->q;
    M->A[2] = M->q;
    M->A[3] = M->p;
    M->bv[0] = 1;
    M->bv[1] = 0;
  } else {
    return false;
  }
  ld h[256];
  impulse_ref(b, a, k, 256, h);
  ld Mx[16], y[4], v[4], t[4];
  for (int i = 0; i < k; ++i) v[i] = M->bv[i];
  for (int m = 0; m < k; ++m) {  // row m: (A^m b)^T, matched to h(m + 1)
    for (int i = 0; i < k; ++i) Mx[m * k + i] = v[i];
    y[m] = h[m + 1];
    for (int i = 0; i < k; ++i) {
      t[i] = 0;
      for (int jj = 0; jj < k; ++jj) t[i] += M->A[i * k + jj] * v[jj];
    }
    memcpy(v, t, sizeof(ld) * k);
  }
  if (!solve(Mx, y, k)) return false;
  for (int i = 0; i < k; ++i) M->c[i] = y[i];
  // verify h(m) = c A^(m-1) b over 255 samples.  The reference's double
  // coefficients split a repeated pole by ~(1e-16)^(1/K) -- the Jordan model
  // then differs by ~1e-14 of sum |h| at sigma = 32, far below fp32.
  ld hsum = 0, err = 0;
  for (int i = 0; i < k; ++i) v[i] = M->bv[i];
  for (int m = 1; m < 256; ++m) {
    ld hm = 0;
    for (int i = 0; i < k; ++i) hm += M->c[i] * v[i];
    hsum += fabsl(h[m]);
    err = fmaxl(err, fabsl(hm - h[m]));
    for (int i = 0; i < k; ++i) {
      t[i] = 0;
      for (int jj = 0; jj < k; ++jj) t[i] += M->A[i * k + jj] * v[jj];
    }
    memcpy(v, t, sizeof(ld) * k);
  }
  return err <= 1e-10L * hsum;
}

}  // namespace vmf
