// vmf_rowpass.cu -- single-kernel three-part IIR pass along rows with whole
// rows resident in shared memory (the B200 row pass).
//
// Same mathematics as _iir_rows_kernel (engine.py:65-102): forward DF-II
// from the steady state of x[0], backward from the steady state of x[W-1],
// out = (b_zero x + y+) + sign y-.  One CTA owns R full rows:
//
//   a. load    : the R rows are staged in shared memory with cp.async
//                (coalesced 16-byte copies; a 4-float pad after every 32
//                samples makes the per-thread chunk reads bank-conflict
//                free).  Each row is padded to a multiple of 32 samples with
//                copies of x[W-1]: a steady state fed a constant stays
//                steady, so the backward recursion may start at the padded
//                end in the steady state of x[W-1] -- identical results on
//                the real samples, and every chunk is exactly 32 long.
//   b. carry   : thread = 32-sample chunk; zero-state chunk-end DF-I
//                histories as dot products with the impulse response h.
//   c. scan    : per row and direction, sequential over the chunks:
//                E_c = Yzs_c + Ty E_{c-1} + Tx X_{c-1} (DF-I history).
//   d. apply   : backward DF-I recursion from the true history with the
//                result parked in 32 fp32 registers (its rounding is
//                smoothed away by the column pass, see
//                tools/experiments/park_precision.py), then the forward
//                recursion writes out(n) in place of x(n).
//   e. store   : coalesced copy of the R rows to the output.
// fp64 state and accumulation throughout; fp32 in and out.
#include <cstring>

#include "vmf_common.cuh"
#include "vmf_iir.cuh"
#include "vmf_prof.cuh"
#include "vmf_rowpass.cuh"

namespace vmf {

__device__ __forceinline__ int sidx(int n) { return n + 4 * (n >> 5); }

template <typename T>
__device__ __forceinline__ float ldf(const T *p) {
  return (float)__ldg(p);
}

template <int K, typename T>
__global__ void __launch_bounds__(kRowMaxThreads, kRowMinBlocks) rowpass_kernel(const T *__restrict__ x, int64_t ldx,
                                                              float *__restrict__ y, int64_t ldy,
                                                              RowParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int R = p.R, C = p.C, Wp = C * kChunk, W = (int)p.W;
  const int rowf = Wp + Wp / 8;  // floats per padded row (Wp + 4 per 32)
  float *xs = reinterpret_cast<float *>(smem_raw);
  double *cf = reinterpret_cast<double *>(smem_raw + (size_t)R * rowf * sizeof(float));
  double *cb = cf + (size_t)R * C * K;

  const int tid = threadIdx.x;
  const int rr = tid / C, c = tid % C;
  const int64_t row0 = (int64_t)blockIdx.x * R;
  const int nrows = (int)((p.H - row0) < R ? (p.H - row0) : R);

  // ---- a. load ------------------------------------------------------------
  if (sizeof(T) == 4 && p.vec4) {
    const uint64_t pol = l2_policy_evict_first();  // the frame is read once
    for (int r = 0; r < nrows; ++r)
      for (int n = 4 * tid; n < W; n += 4 * blockDim.x)
        cp_async16_hint(xs + r * rowf + sidx(n), x + (row0 + r) * ldx + n, pol);
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
  } else {
    for (int r = 0; r < nrows; ++r)
      for (int n = tid; n < W; n += blockDim.x)
        xs[r * rowf + sidx(n)] = ldf(x + (row0 + r) * ldx + n);
  }
  __syncthreads();
  for (int r = 0; r < nrows; ++r)  // replicate x[W-1] into the padding
    for (int n = W + tid; n < Wp; n += blockDim.x) xs[r * rowf + sidx(n)] = xs[r * rowf + sidx(W - 1)];
  __syncthreads();

  const bool active = rr < nrows;
  float *xr = xs + rr * rowf;
  const int n0 = c * kChunk;

  // ---- b. zero-state carries (folded sample pairs) -------------------------
  if (active) {
    double P[K], Q[K];
#pragma unroll
    for (int i = 0; i < K; ++i) P[i] = Q[i] = 0.0;
    const float4 *v4 = reinterpret_cast<const float4 *>(xr + sidx(n0));
    float xv[kChunk];  // fp32 copies; the pair sums are formed in fp64
#pragma unroll
    for (int q = 0; q < kChunk / 4; ++q) {
      float4 v = v4[q];
      xv[4 * q] = v.x;
      xv[4 * q + 1] = v.y;
      xv[4 * q + 2] = v.z;
      xv[4 * q + 3] = v.w;
    }
#pragma unroll
    for (int t = 0; t < kChunk / 2; ++t) {
      const double xa = xv[t], xb = xv[kChunk - 1 - t];
      const double u = xa + xb, v = xa - xb;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        P[i] = fma(p.SP32[i][t], u, P[i]);
        Q[i] = fma(p.SQ32[i][t], v, Q[i]);
      }
    }
    double f[K], g[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      f[i] = P[i] + Q[i];
      g[i] = P[i] - Q[i];
    }
    // scan inputs d_c = Yzs_c + Tx X_{c-1} (x history before the chunk in
    // scan order; the steady state of the end sample for the first chunk,
    // plus Ty E_{-1} with E_{-1} = yss * that sample)
    double Xf[K], Xb[K];
    const double x0 = (double)xr[sidx(0)], xl = (double)xr[sidx(Wp - 1)];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      Xf[i] = c > 0 ? (double)xr[sidx(n0 - 1 - i)] : x0;
      Xb[i] = c < C - 1 ? (double)xr[sidx(n0 + kChunk + i)] : xl;
    }
#pragma unroll
    for (int i = 0; i < K; ++i) {
      double df = f[i], db = g[i];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        df = fma(p.Tx[i * K + j], Xf[j], df);
        db = fma(p.Tx[i * K + j], Xb[j], db);
      }
      if (c == 0) {
#pragma unroll
        for (int j = 0; j < K; ++j) df = fma(p.Ty[i * K + j], p.yss * x0, df);
      }
      if (c == C - 1) {
#pragma unroll
        for (int j = 0; j < K; ++j) db = fma(p.Ty[i * K + j], p.yss * xl, db);
      }
      cf[(rr * C + c) * K + i] = df;
      cb[(rr * C + c) * K + i] = db;
    }
  }
  __syncthreads();

  // ---- c. scan: one warp per (row, direction) ------------------------------
  // E_c = d_c + Ty E_{c-1},  d_c = Yzs_c + Tx X_{c-1}  (c in scan order; the
  // backward direction scans chunks from the right end).  Lane l owns cpl
  // consecutive chunks: local sequential scan, Kogge-Stone across lanes
  // with Ty^(cpl*2^j), then a sequential re-scan from the carry-in.
  {
    const int lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int cpl = p.cpl;
    for (int task = warp; task < 2 * nrows; task += nwarps) {
      const int r = task >> 1, dir = task & 1;
      double *cc = (dir == 0 ? cf : cb) + r * C * K;
      const bool live = lane * cpl < C;
      auto dval = [&](int sp, double *d) {
        const int ch = dir == 0 ? sp : C - 1 - sp;
#pragma unroll
        for (int i = 0; i < K; ++i) d[i] = cc[ch * K + i];
      };
      double A[K];
#pragma unroll
      for (int i = 0; i < K; ++i) A[i] = 0.0;
      if (live) {
        for (int q = 0; q < cpl; ++q) {
          double d[K], An[K];
          dval(lane * cpl + q, d);
#pragma unroll
          for (int i = 0; i < K; ++i) {
            double acc = d[i];
#pragma unroll
            for (int j = 0; j < K; ++j) acc = fma(p.Ty[i * K + j], A[j], acc);
            An[i] = acc;
          }
#pragma unroll
          for (int i = 0; i < K; ++i) A[i] = An[i];
        }
      }
      // inclusive Kogge-Stone over lanes: A_l += Ty^(cpl*o) A_{l-o}
#pragma unroll
      for (int lv = 0; lv < 5; ++lv) {
        const int o = 1 << lv;
        double B[K];
#pragma unroll
        for (int i = 0; i < K; ++i) B[i] = __shfl_up_sync(0xffffffffu, A[i], o);
        if (lane >= o) {
          const double *M = p.Tpow[lv];
#pragma unroll
          for (int i = 0; i < K; ++i) {
            double acc = A[i];
#pragma unroll
            for (int j = 0; j < K; ++j) acc = fma(M[i * K + j], B[j], acc);
            A[i] = acc;
          }
        }
      }
      // carry-in = inclusive value of the previous lane
      double E[K];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        double v = __shfl_up_sync(0xffffffffu, A[i], 1);
        E[i] = lane ? v : 0.0;
      }
      if (live) {
        for (int q = 0; q < cpl; ++q) {
          const int sp = lane * cpl + q;
          const int ch = dir == 0 ? sp : C - 1 - sp;
          double d[K], En[K];
          dval(sp, d);
#pragma unroll
          for (int i = 0; i < K; ++i) {
            double acc = d[i];
#pragma unroll
            for (int j = 0; j < K; ++j) acc = fma(p.Ty[i * K + j], E[j], acc);
            En[i] = acc;
          }
#pragma unroll
          for (int i = 0; i < K; ++i) {
            E[i] = En[i];
            cc[ch * K + i] = En[i];  // END history of chunk ch (scan order)
          }
        }
      }
      __syncwarp();
    }
  }
  __syncthreads();

  // ---- d. apply -------------------------------------------------------------
  // Backward first (reads only x, parks sign*y- in registers), then a barrier,
  // then the forward recursion overwrites x(n) with out(n) in place.
  float park[kChunk];
  float4 *v4 = reinterpret_cast<float4 *>(xr + sidx(n0));
  if (active) {
    double Xb[K], Yb[K];
    const double xl = (double)xr[sidx(Wp - 1)];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      int qb = n0 + kChunk + i;
      Xb[i] = (double)xr[sidx(qb > Wp - 1 ? Wp - 1 : qb)];
      Yb[i] = c < C - 1 ? cb[(rr * C + c + 1) * K + i] : p.yss * xl;
    }
#pragma unroll
    for (int q = kChunk / 4 - 1; q >= 0; --q) {
      float4 v = v4[q];
      float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int u = 3; u >= 0; --u) {
        double xv = (double)e[u];
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < K; ++m) s = fma(p.b[m], Xb[m], s);
#pragma unroll
        for (int m = K - 1; m >= 1; --m) s = fma(-p.a[m], Yb[m], s);
        s = fma(-p.a[0], Yb[0], s);
        park[4 * q + u] = (float)(p.sign * s);
#pragma unroll
        for (int m = K - 1; m > 0; --m) {
          Yb[m] = Yb[m - 1];
          Xb[m] = Xb[m - 1];
        }
        Yb[0] = s;
        Xb[0] = xv;
      }
    }
  }
  double Xf[K], Yf[K];
  if (active) {
    const double x0 = (double)xr[sidx(0)];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      int qf = n0 - 1 - i;
      Xf[i] = (double)xr[sidx(qf < 0 ? 0 : qf)];
      Yf[i] = c > 0 ? cf[(rr * C + c - 1) * K + i] : p.yss * x0;
    }
  }
  __syncthreads();  // every halo read before any chunk is overwritten
  if (active) {
#pragma unroll
    for (int q = 0; q < kChunk / 4; ++q) {
      float4 v = v4[q];
      float e[4] = {v.x, v.y, v.z, v.w};
      float o[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        double xv = (double)e[u];
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < K; ++m) s = fma(p.b[m], Xf[m], s);
#pragma unroll
        for (int m = K - 1; m >= 1; --m) s = fma(-p.a[m], Yf[m], s);
        s = fma(-p.a[0], Yf[0], s);
        o[u] = (float)(fma(p.b0, xv, s) + (double)park[4 * q + u]);
#pragma unroll
        for (int m = K - 1; m > 0; --m) {
          Yf[m] = Yf[m - 1];
          Xf[m] = Xf[m - 1];
        }
        Yf[0] = s;
        Xf[0] = xv;
      }
      v4[q] = make_float4(o[0], o[1], o[2], o[3]);
    }
  }
  __syncthreads();

  // ---- e. store --------------------------------------------------------------
  if (p.vec4) {
    const uint64_t pol = l2_policy_evict_last();  // T is read again by the column pass
    for (int r = 0; r < nrows; ++r)
      for (int n = 4 * tid; n < W; n += 4 * blockDim.x)
        st_v4_hint(y + (row0 + r) * ldy + n, *reinterpret_cast<const float4 *>(xs + r * rowf + sidx(n)),
                   pol);
  } else {
    for (int r = 0; r < nrows; ++r)
      for (int n = tid; n < W; n += blockDim.x) y[(row0 + r) * ldy + n] = xs[r * rowf + sidx(n)];
  }
}

// ---------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------
static void dfi_transfer(const double *b, const double *a, int k, int len, double *Ty,
                         double *Tx) {
  for (int j = 0; j < 2 * k; ++j) {
    long double Y[VMF_MAX_IIR_ORDER], X[VMF_MAX_IIR_ORDER];
    for (int m = 0; m < k; ++m) {
      Y[m] = (j == m) ? 1.0L : 0.0L;
      X[m] = (j == k + m) ? 1.0L : 0.0L;
    }
    for (int n = 0; n < len; ++n) {
      long double v = 0.0L;
      for (int m = 0; m < k; ++m) v += (long double)b[m] * X[m] - (long double)a[m] * Y[m];
      for (int m = k - 1; m > 0; --m) {
        Y[m] = Y[m - 1];
        X[m] = X[m - 1];
      }
      Y[0] = v;
      X[0] = 0.0L;
    }
    for (int i = 0; i < k; ++i) {
      if (j < k)
        Ty[i * k + j] = (double)Y[i];
      else
        Tx[i * k + (j - k)] = (double)Y[i];
    }
  }
}

// Ty over len samples only (zero-input DF-I response to the y history).
static void dfi_transfer_y(const double *b, const double *a, int k, int len, double *Ty) {
  for (int j = 0; j < k; ++j) {
    long double Y[VMF_MAX_IIR_ORDER];
    for (int m = 0; m < k; ++m) Y[m] = (j == m) ? 1.0L : 0.0L;
    for (int n = 0; n < len; ++n) {
      long double v = 0.0L;
      for (int m = 0; m < k; ++m) v -= (long double)a[m] * Y[m];
      for (int m = k - 1; m > 0; --m) Y[m] = Y[m - 1];
      Y[0] = v;
    }
    for (int i = 0; i < k; ++i) Ty[i * k + j] = (double)Y[i];
  }
}

static void impulse_resp(const double *b, const double *a, int k, int n, double *h) {
  long double Y[VMF_MAX_IIR_ORDER] = {0}, X[VMF_MAX_IIR_ORDER] = {0};
  for (int q = 0; q < n; ++q) {
    long double v = 0.0L;
    for (int m = 0; m < k; ++m) v += (long double)b[m] * X[m] - (long double)a[m] * Y[m];
    h[q] = (double)v;
    for (int m = k - 1; m > 0; --m) {
      Y[m] = Y[m - 1];
      X[m] = X[m - 1];
    }
    Y[0] = v;
    X[0] = q == 0 ? 1.0L : 0.0L;
  }
}

bool rowpass_supported(int64_t w, int k) {
  int64_t C = cdiv(w, kChunk);
  return k >= 1 && k <= VMF_MAX_IIR_ORDER && C <= kRowMaxThreads;
}

void rowpass_plan(RowParams *p, const IirParams &ip, int64_t h, int64_t w) {
  memset(p, 0, sizeof(*p));
  int k = ip.K;
  for (int m = 0; m < k; ++m) {
    p->b[m] = ip.b[m];
    p->a[m] = ip.a[m];
  }
  p->b0 = ip.b0;
  p->sign = ip.sign;
  p->yss = ip.yss;
  impulse_resp(ip.b, ip.a, k, kChunk + 1, p->h);
  dfi_transfer(ip.b, ip.a, k, (int)kChunk, p->Ty, p->Tx);
  p->H = h;
  p->W = w;
  int C = (int)cdiv(w, kChunk);
  if (C <= 32) {  // a power of two, so rows tile warps evenly
    int c2 = 1;
    while (c2 < C) c2 <<= 1;
    C = c2;
  } else {
    C = (int)cdiv(C, 32) * 32;
  }
  p->C = C;
  p->cpl = C <= 32 ? 1 : C / 32;
  // Tpow[j] = Ty^(cpl * 2^j), j = 0..4 (long double products)
  // Ty^n is the zero-input map of the y history over n*32 samples, so the
  // powers are computed directly in long double (no repeated squaring).
  for (int j = 0; j < 5; ++j)
    dfi_transfer_y(ip.b, ip.a, k, (p->cpl << j) * (int)kChunk, p->Tpow[j]);
  for (int i = 0; i < k && i < VMF_MAX_IIR_ORDER; ++i)
    for (int t = 0; t < kChunk / 2; ++t) {
      int qa = kChunk - 1 - i - t, qb = t - i;
      double A = qa > 0 ? p->h[qa] : 0.0, B = qb > 0 ? p->h[qb] : 0.0;
      p->SP32[i][t] = 0.5 * (A + B);
      p->SQ32[i][t] = 0.5 * (A - B);
    }
  int r = kRowThreads / p->C;
  if (r < 1) r = 1;
  while (r > 1 && (int64_t)r * p->C * kChunk * 5 / 4 * 4 > kRowTileBytes) --r;
  p->R = r;
}

size_t rowpass_smem(const RowParams &p, int k) {
  int Wp = p.C * (int)kChunk;
  return (size_t)p.R * (Wp + Wp / 8) * sizeof(float) + (size_t)2 * p.R * p.C * k * sizeof(double);
}

template <int K, typename T>
static int launch_rowpass(const T *x, int64_t ldx, float *y, int64_t ldy, RowParams p,
                          cudaStream_t st) {
  size_t smem = rowpass_smem(p, K);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(rowpass_kernel<K, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  p.vec4 = (sizeof(T) == 4) && (p.W % 4 == 0) && (ldx % 4 == 0) && (ldy % 4 == 0) &&
           ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0);
  if (sizeof(T) != 4) p.vec4 = (p.W % 4 == 0) && (ldy % 4 == 0) && ((uintptr_t)y % 16 == 0);
  int grid = (int)cdiv(p.H, p.R);
  Launch g(K_IIR_ROWS_FUSED, st);
  rowpass_kernel<K, T><<<grid, p.R * p.C, smem, st>>>(x, ldx, y, ldy, p);
  return cuda_status("row pass");
}

template <typename T>
int rowpass_run(const T *x, int64_t ldx, float *y, int64_t ldy, const IirParams &ip, int64_t h,
                int64_t w, cudaStream_t st) {
  RowParams p;
  rowpass_plan(&p, ip, h, w);
  switch (ip.K) {
    case 1: return launch_rowpass<1, T>(x, ldx, y, ldy, p, st);
    case 2: return launch_rowpass<2, T>(x, ldx, y, ldy, p, st);
    case 3: return launch_rowpass<3, T>(x, ldx, y, ldy, p, st);
    case 4: return launch_rowpass<4, T>(x, ldx, y, ldy, p, st);
    case 5: return launch_rowpass<5, T>(x, ldx, y, ldy, p, st);
    case 6: return launch_rowpass<6, T>(x, ldx, y, ldy, p, st);
    case 7: return launch_rowpass<7, T>(x, ldx, y, ldy, p, st);
    case 8: return launch_rowpass<8, T>(x, ldx, y, ldy, p, st);
  }
  return fail(VMF_EVALUE, "IIR order %d unsupported by the row pass", ip.K);
}

template int rowpass_run<float>(const float *, int64_t, float *, int64_t, const IirParams &,
                                int64_t, int64_t, cudaStream_t);
template int rowpass_run<uint16_t>(const uint16_t *, int64_t, float *, int64_t,
                                   const IirParams &, int64_t, int64_t, cudaStream_t);

}  // namespace vmf
