// vmf_dfi.cuh -- latency-pipelined evaluation of one DF-I recursion run.
//
//   y_t = sum_{m<K} b[m] x_{t-1-m} - sum_{m<K} a[m] y_{t-1-m}
//
// Written as the plain DF-I sum, sample t+1's terms form a chain of 2K
// dependent FMAs that an in-order warp issues only after y_t -- about 2K x 8
// cycles per sample on the fp64 pipe.  Here the terms of every pending sample
// are accumulated as soon as their inputs exist:
//
//   P[j] = partial sum of sample t+j: every x term with index <= t-1 and
//          every y term with index <= t-2,
//
// so producing y_t is ONE fma on y_{t-1} (the loop-carried dependency), and
// the other 2K-1 fmas of the step depend only on values that are already
// there.  Same terms, same count (2K fma per sample) as the plain sum; only
// the association differs (fp64, far inside the parity tolerance).
#pragma once

namespace vmf {

// Coefficients of one recursion direction.  The backward run of the
// three-part filter uses b_minus = sign * b_plus: folding the sign into the
// coefficients (and the start history) gives sign * y- bit for bit (a
// negation is exact) without a multiply per sample.
struct DfiCoef {
  double b[VMF_MAX_IIR_ORDER], a[VMF_MAX_IIR_ORDER];
};

template <int K>
struct DfiRun {
  double P[K];
  double yp;  // y_{t-1}

  // from a DF-I history: Y[i] = y_{t-1-i}, X[i] = x_{t-1-i}
  template <class Par>
  __device__ __forceinline__ void init(const Par &p, const double *Y, const double *X) {
    yp = Y[0];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      double s = 0.0;
#pragma unroll
      for (int m = K - 1; m >= j; --m) s = fma(p.b[m], X[m - j], s);
#pragma unroll
      for (int m = K - 1; m >= j + 1; --m) s = fma(-p.a[m], Y[m - j], s);
      P[j] = s;
    }
  }

  // returns y_t and consumes the input x_t
  template <class Par>
  __device__ __forceinline__ double step(const Par &p, double xt) {
    const double y = fma(-p.a[0], yp, P[0]);
#pragma unroll
    for (int j = 0; j < K - 1; ++j) P[j] = fma(-p.a[j + 1], yp, fma(p.b[j], xt, P[j + 1]));
    P[K - 1] = p.b[K - 1] * xt;
    yp = y;
    return y;
  }
};

}  // namespace vmf
