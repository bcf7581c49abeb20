// vmf_colpass.cu -- the fused second pass of the hot path: column IIR
// (iir_cols, engine.py:156-158 / kernel 65-102) + Laplacian D20 + D02
// (engine.py:218-227, blob.py:161) + threshold / 3x3 NMS,
// reading the row-pass output T once more from L2/HBM and writing L plus a
// short candidate list.  fp64 state, fp64 blur B, L computed from un-rounded
// B (tools/experiments/park_precision.py: this is what keeps L within 1e-5 of
// the reference instead of 7e-5).
//
// Column chunking is two-level:
//   bands (256 rows)  : zero-state band carries (colcarry) -> sequential band
//                       scan per column (colscan) -> true DF-I histories at
//                       every band edge;
//   sub-chunks (32)   : inside colapply a CTA (128 columns x one band) gets the
//                       backward starts of its 8 sub-chunks from a local
//                       carry + scan, then walks the band top-down: per
//                       sub-chunk a backward run parked in 32 fp64 registers
//                       and a forward run producing B, so the forward
//                       recursion never needs a carry inside the band.
// Rows are padded to a multiple of 32 with copies of the last row (a steady
// state fed its own constant stays steady), so every sub-chunk is full.
//
// Laplacian/NMS: B rows of a sub-chunk go to shared memory; L lags B by one
// row and NMS lags L by one row, so only 2 rows of B and L carry over between
// sub-chunks.  At band edges the 2 rows outside the band are recomputed from
// the band-edge histories (2 extra recursion steps).  A CTA computes 128
// columns and owns the 124 inner ones (2-column halo for Lx and the 3x3 NMS).
//
// Threshold: t = frac * max|L| is known only at the end, so a CTA keeps the
// strict extrema with |L| >= frac * (its running max) in shared memory --
// a superset of the final detections -- and flushes them at the band end;
// colfinal sorts the survivors of the final threshold by (y, x).  If a buffer
// overflows, the ordered full-frame NMS of vmf_stage4.cu runs instead.
#include <cstdlib>
#include <cstring>

#include "vmf_colpass.cuh"
#include "plan_cache.hpp"
#include "vmf_common.cuh"
#include "vmf_prof.cuh"
#include "vmf_stage4.cuh"
#include "vmf_dfi.cuh"
#include "vmf_tma.cuh"

namespace vmf {

__device__ __forceinline__ double ldT(const float *T, int64_t ldt, int64_t r, int64_t H,
                                      int64_t c) {
  return (double)__ldg(T + (r < H ? r : H - 1) * ldt + c);
}

// ---------------------------------------------------------------------------
// 1. band carries: zero-state end histories of every (band, column)
// ---------------------------------------------------------------------------
// Band records, coalesced along columns:
//   Z[((dir * NB + b) * 2K + i) * W + col], i in [0, K): zero-state end history
//   of band b (replaced by its true START history by the scan); i in [K, 2K):
//   the band's edge samples in scan order (fwd: x(r1-1-i), bwd: x(r0+i)).
__device__ __forceinline__ int64_t zidx(int dir, int b, int i, int NB, int K, int64_t W,
                                        int64_t col) {
  return ((int64_t)(dir * NB + b) * 2 * K + i) * W + col;
}

// One CTA = 128 columns x one 64-row band (one TMA box), 256 threads:
// threads j and j + 128 take the two halves of the band's 32 sample pairs of
// column j; records are written coalesced along columns.
constexpr int kCarryCols = kColThreads;
constexpr int kCarryThreads = 2 * kCarryCols;

// Folded zero-state sums of one half of a full band (pairs t0 .. t0+15 of
// rows (t, 63-t)), from the staged tile or straight from global memory.
template <int K, int HALF>
__device__ __forceinline__ void carry_half(const ColParams &p, const float *tile, bool tma,
                                           const float *src, int64_t ldt, int j, double *P,
                                           double *Q) {
  constexpr int kHalf = kBand / 4;  // pairs per thread
  constexpr int t0 = HALF * kHalf;
  float xa[kHalf], xb[kHalf];
  if (tma) {
#pragma unroll
    for (int t = 0; t < kHalf; ++t) {
      xa[t] = tile[(t0 + t) * kCarryCols + j];
      xb[t] = tile[(kBand - 1 - t0 - t) * kCarryCols + j];
    }
  } else {
#pragma unroll
    for (int t = 0; t < kHalf; ++t) {
      xa[t] = __ldg(src + (t0 + t) * ldt);
      xb[t] = __ldg(src + (kBand - 1 - t0 - t) * ldt);
    }
  }
#pragma unroll
  for (int t = 0; t < kHalf; ++t) {
    // pair sums in fp64: an fp32 sum would inject an fp32 rounding of |2T|
    // into every band carry, i.e. B errors of fp32-ulp size, which the
    // Laplacian amplifies past the 1e-4 tolerance at large sigma
    const double xa64 = (double)xa[t], xb64 = (double)xb[t];
    const double u = xa64 + xb64, v = xa64 - xb64;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      P[i] = fma(p.SP[i][t0 + t], u, P[i]);
      Q[i] = fma(p.SQ[i][t0 + t], v, Q[i]);
    }
  }
}

template <int K>
__global__ void __launch_bounds__(kCarryThreads) colcarry_kernel(
    const float *__restrict__ T, int64_t ldt, ColParams p, double *__restrict__ Z,
    const __grid_constant__ CUtensorMap tmap, int use_tma, CandState *__restrict__ cs) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // 128-byte aligned TMA destination, derived from the shared array itself so
  // the reads stay LDS
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem_raw);
  float *tile = reinterpret_cast<float *>(smem_raw + ((128u - (sbase & 127u)) & 127u));
  __shared__ __align__(8) uint64_t tbar;
  __shared__ double part[2 * K][kCarryCols];
  const int j = threadIdx.x & (kCarryCols - 1), half = threadIdx.x >> 7;
  const int b = blockIdx.y;
  const int len = b == p.NB - 1 ? p.Blast : kBand;
  const int64_t c0 = (int64_t)blockIdx.x * kCarryCols;
  const int64_t col = c0 + j;
  const int64_t r0 = (int64_t)b * kBand;
  const bool full = len == kBand && r0 + kBand <= p.H;
  const bool tma = use_tma && full && c0 + kCarryCols <= p.W;
  pdl_wait();  // T comes from the row pass
  if (blockIdx.x == 0 && blockIdx.y == 0) cand_reset(cs);
  if (tma) {
    if (threadIdx.x == 0) {
      mbar_init(&tbar, 1);
      mbar_expect_tx(&tbar, (unsigned)(kBand * kCarryCols * sizeof(float)));
      tma_load_2d_hint(tile, &tmap, &tbar, (int)c0, (int)r0, l2_policy_evict_last());
    }
    __syncthreads();
    mbar_wait(&tbar, 0);
  }
  const bool live = col < p.W;
  double P[K], Q[K];
#pragma unroll
  for (int i = 0; i < K; ++i) P[i] = Q[i] = 0.0;
  if (live && full) {
    // warp-uniform split so the weight indices are compile-time (the
    // coefficients stay constant-bank operands of the DFMAs)
    if (half == 0)
      carry_half<K, 0>(p, tile, tma, T + r0 * ldt + col, ldt, j, P, Q);
    else
      carry_half<K, 1>(p, tile, tma, T + r0 * ldt + col, ldt, j, P, Q);
  } else if (live && half == 0) {  // last (short or padded) band: direct weights
    for (int t = 0; t < len; ++t) {
      double x = ldT(T, ldt, r0 + t, p.H, col);
#pragma unroll
      for (int i = 0; i < K; ++i) {
        int qa = len - 1 - i - t, qb = t - i;
        if (qa > 0) P[i] = fma(p.h[qa], x, P[i]);
        if (qb > 0) Q[i] = fma(p.h[qb], x, Q[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < K; ++i) {  // (f, g) -> (P, Q): f = P + Q, g = P - Q
      double f = P[i], g = Q[i];
      P[i] = 0.5 * (f + g);
      Q[i] = 0.5 * (f - g);
    }
  }
  pdl_trigger();
  if (half == 1) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
      part[i][j] = P[i];
      part[K + i][j] = Q[i];
    }
  }
  __syncthreads();
  if (half == 0 && live) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const double Pt = P[i] + part[i][j], Qt = Q[i] + part[K + i][j];
      Z[zidx(0, b, i, p.NB, K, p.W, col)] = Pt + Qt;
      Z[zidx(1, b, i, p.NB, K, p.W, col)] = Pt - Qt;
      double ef, eb;
      if (tma) {  // edge rows are in the staged tile
        ef = (double)tile[(kBand - 1 - i) * kCarryCols + j];
        eb = (double)tile[i * kCarryCols + j];
      } else {
        ef = ldT(T, ldt, r0 + len - 1 - i, p.H, col);
        eb = ldT(T, ldt, r0 + i, p.H, col);
      }
      Z[zidx(0, b, K + i, p.NB, K, p.W, col)] = ef;
      Z[zidx(1, b, K + i, p.NB, K, p.W, col)] = eb;
    }
  }
}

// ---------------------------------------------------------------------------
// 2. band scan.  CTA = one direction x 16 columns: the records of all bands
//    are staged in shared memory with coalesced loads, then warp w scans
//    column w with lanes over bands (cpl bands per lane, Kogge-Stone with
//    TyB^(cpl 2^j)), and the true START histories go back coalesced:
//    fwd = y+(r0-1 .. r0-K), bwd = y-(r1 .. r1+K-1).
// ---------------------------------------------------------------------------
constexpr int kScanCols = 8;

template <int K>
__global__ void __launch_bounds__(32 * kScanCols, 48 / kScanCols) colscan_kernel(const float *__restrict__ T,
                                                                 int64_t ldt, ColParams p,
                                                                 double *__restrict__ Z) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int NB = p.NB, cpl = p.cpl;
  const int stride = 2 * K * kScanCols + 2;  // doubles per band row (+2: 16-byte aligned rows)
  double *sz = reinterpret_cast<double *>(smem_raw);  // [NB][2K][kScanCols] (+pad)
  const int dir = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * kScanCols;
  const int lane = threadIdx.x & 31, c = threadIdx.x >> 5;
  const int64_t col = c0 + c < p.W ? c0 + c : p.W - 1;
  pdl_wait();  // records come from the band carries
  // the end sample (steady-state start of the first band) is loaded now, so
  // its latency hides under the staging
  const double xe = ldT(T, ldt, dir == 0 ? 0 : p.H - 1, p.H, col);
  // staging with asynchronous 16-byte copies (two columns each), all in
  // flight at once: element pair e = (record row bi = b * 2K + i, c/2)
  {
    constexpr int kPairs = kScanCols / 2;
    const bool full = c0 + kScanCols <= p.W && p.W % 2 == 0;
    const double *zdir = Z + (int64_t)dir * NB * 2 * K * p.W + c0;
    for (int e = threadIdx.x; e < NB * 2 * K * kPairs; e += blockDim.x) {
      const int c = 2 * (e % kPairs), bi = e / kPairs;
      const int b = bi / (2 * K);
      double *dst = sz + bi * kScanCols + 2 * b + c;  // = b * stride + i * kScanCols + c
      const double *src = zdir + (int64_t)bi * p.W + c;
      if (full) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src));
      } else {
        const int i = bi - b * 2 * K;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int64_t col = c0 + c + u < p.W ? c0 + c + u : p.W - 1;
          dst[u] = Z[zidx(dir, b, i, NB, K, p.W, col)];
        }
      }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
  }
  pdl_trigger();
  __syncthreads();
  auto rec = [&](int sp) { return sz + (dir == 0 ? sp : NB - 1 - sp) * stride + c; };
  double dl[kMaxCpl][K];
#pragma unroll
  for (int q = 0; q < kMaxCpl; ++q) {  // d_sp = Yzs + TxB X_prev (+ TyB E_init first)
    const int sp = lane * cpl + q;
    if (q < cpl && sp < NB) {
      const double *r = rec(sp);
      const int b = dir == 0 ? sp : NB - 1 - sp;
      const int tb = b == NB - 1 ? 1 : 0;
      double X[K];
      if (sp == 0) {
#pragma unroll
        for (int i = 0; i < K; ++i) X[i] = xe;
      } else {
        const double *pr = rec(sp - 1);
#pragma unroll
        for (int i = 0; i < K; ++i) X[i] = pr[(K + i) * kScanCols];
      }
#pragma unroll
      for (int i = 0; i < K; ++i) {
        double acc = r[i * kScanCols];
#pragma unroll
        for (int m = 0; m < K; ++m) acc = fma(p.TxB[tb][i * K + m], X[m], acc);
        if (sp == 0) {
#pragma unroll
          for (int m = 0; m < K; ++m) acc = fma(p.TyB[tb][i * K + m], p.yss * xe, acc);
        }
        dl[q][i] = acc;
      }
    }
  }
  double A[K];
#pragma unroll
  for (int i = 0; i < K; ++i) A[i] = 0.0;
#pragma unroll
  for (int q = 0; q < kMaxCpl; ++q) {
    if (q < cpl && lane * cpl + q < NB) {
      double An[K];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        double acc = dl[q][i];
#pragma unroll
        for (int m = 0; m < K; ++m) acc = fma(p.TyB[0][i * K + m], A[m], acc);
        An[i] = acc;
      }
#pragma unroll
      for (int i = 0; i < K; ++i) A[i] = An[i];
    }
  }
#pragma unroll
  for (int lv = 0; lv < 5; ++lv) {
    const int o = 1 << lv;
    double B[K];
#pragma unroll
    for (int i = 0; i < K; ++i) B[i] = __shfl_up_sync(0xffffffffu, A[i], o);
    if (lane >= o) {
#pragma unroll
      for (int i = 0; i < K; ++i) {
        double acc = A[i];
#pragma unroll
        for (int m = 0; m < K; ++m) acc = fma(p.TyBp[lv][i * K + m], B[m], acc);
        A[i] = acc;
      }
    }
  }
  double E[K];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    double v = __shfl_up_sync(0xffffffffu, A[i], 1);
    E[i] = lane ? v : p.yss * xe;
  }
  __syncthreads();  // every warp has read its inputs before results overwrite them
#pragma unroll
  for (int q = 0; q < kMaxCpl; ++q) {
    const int sp = lane * cpl + q;
    if (q < cpl && sp < NB) {
      double *r = rec(sp);
#pragma unroll
      for (int i = 0; i < K; ++i) r[i * kScanCols] = E[i];
      if (sp == 0) {
#pragma unroll
        for (int i = 0; i < K; ++i) E[i] = dl[q][i];
      } else {
        double En[K];
#pragma unroll
        for (int i = 0; i < K; ++i) {
          double acc = dl[q][i];
#pragma unroll
          for (int m = 0; m < K; ++m) acc = fma(p.TyB[0][i * K + m], E[m], acc);
          En[i] = acc;
        }
#pragma unroll
        for (int i = 0; i < K; ++i) E[i] = En[i];
      }
    }
  }
  __syncthreads();
  {
    double *zdir = Z + (int64_t)dir * NB * 2 * K * p.W + c0;
    for (int e = threadIdx.x; e < NB * K * kScanCols; e += blockDim.x) {
      const int cc = e % kScanCols, bi = e / kScanCols;
      const int b = bi / K, i = bi - b * K;
      if (c0 + cc < p.W) zdir[(int64_t)(b * 2 * K + i) * p.W + cc] = sz[b * stride + i * kScanCols + cc];
    }
  }
}

// ---------------------------------------------------------------------------
// 3. walk a band: column IIR + Laplacian + NMS candidates
// ---------------------------------------------------------------------------
template <int K>
__device__ __forceinline__ double dfi(const ColParams &p, const double *X, const double *Y) {
  double s = 0.0;
#pragma unroll
  for (int m = 0; m < K; ++m) s = fma(p.b[m], X[m], s);
#pragma unroll
  for (int m = K - 1; m >= 1; --m) s = fma(-p.a[m], Y[m], s);
  return fma(-p.a[0], Y[0], s);
}

template <int K>
__device__ __forceinline__ void push2(double *Y, double y, double *X, double x) {
#pragma unroll
  for (int m = K - 1; m > 0; --m) {
    Y[m] = Y[m - 1];
    X[m] = X[m - 1];
  }
  Y[0] = y;
  X[0] = x;
}

constexpr int kTileRows(int k) { return kBand + 2 * k; }
constexpr int kEbRows = kBand + 4;  // B of rows r0-2 .. r1+1
// The TMA box must start at a 16-byte aligned column, so the tile spans 4
// more columns than the CTA computes: tile column j + 2 <-> thread j.
constexpr int kTileStride = kColThreads + 4;

template <int K>
struct ColSmem {
  // T rows r0-K .. r1+K-1 (clamped).  Column j is private to thread j during
  // the walk, so L(r) overwrites x(r) in place once x(r) is consumed; after
  // the walk the tile holds L rows r0-1 .. r1 for the NMS.
  float tile[kTileRows(K)][kTileStride];
  double eb[kColThreads / 32][4][kEbRows];  // B of lanes 0,1,30,31 per warp
  int cy[kCandSmem], cx[kCandSmem];
  float cv[kCandSmem];
  int ccount;
  unsigned int cmax;  // max |L| of this CTA (float bits)
};

// MODE 0: L + NMS candidates; 1: the same with lap_scale == 1 (no scaling
// multiply); 2: the fp64 blur B of the owned pixels to b64 (pitch W), no L;
// 3: the blur B rounded to fp32 into Lout (the iir_cols leaf)
template <int K, int MODE>
__global__ void __launch_bounds__(kColThreads, 4) colapply_kernel(
    const float *__restrict__ T, int64_t ldt, float *__restrict__ Lout, int64_t ldl, ColParams p,
    const double *__restrict__ Z, CandState *__restrict__ st, int *__restrict__ gy,
    int *__restrict__ gx, float *__restrict__ gv, int gcap,
    const __grid_constant__ CUtensorMap tmap, int use_tma, int vec_out, double *__restrict__ b64) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // 128-byte aligned base (the tile is a TMA destination), derived from the
  // shared array itself so every access stays an LDS / STS
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem_raw);
  ColSmem<K> &S = *reinterpret_cast<ColSmem<K> *>(smem_raw + ((128u - (sbase & 127u)) & 127u));
  const int j = threadIdx.x, lane = j & 31, wid = j >> 5;
  const int64_t c0 = (int64_t)blockIdx.x * kColOut;
  const int64_t col = c0 - kColHalo + j;
  const int64_t colc = col < 0 ? 0 : (col >= p.W ? p.W - 1 : col);
  const int b = blockIdx.y;
  const int64_t r0 = (int64_t)b * kBand;
  const int len = b == p.NB - 1 ? p.Blast : kBand;
  const int64_t r1 = r0 + len;
  const int nsub = len / kSub;
  const int64_t H = p.H;
  const bool own_col = j >= kColHalo && j < kColThreads - kColHalo && col < p.W;
  const int eslot = lane == 0 ? 0 : (lane == 1 ? 1 : (lane == 30 ? 2 : (lane == 31 ? 3 : -1)));
  const int64_t rown_hi = r1 < H ? r1 : H;  // owned rows [r0, rown_hi)

  // ---- stage the band's column tile (async 4-byte copies: any alignment) ---
  float *tcol = &S.tile[0][j + 2];  // tile row tr of this thread's column: tcol[tr * kTileStride]
  __shared__ __align__(8) uint64_t tbar;
  const bool tma = use_tma && len == kBand && r0 >= K && r1 + K <= H && c0 >= 4 &&
                   c0 + kColThreads <= p.W;
  if (tma) {  // one TMA box: rows r0-K .. r1+K-1, columns c0-4 .. c0+127
    if (j == 0) {
      mbar_init(&tbar, 1);
      mbar_expect_tx(&tbar, (unsigned)(kTileRows(K) * kTileStride * sizeof(float)));
      tma_load_2d_hint(&S.tile[0][0], &tmap, &tbar, (int)(c0 - 4), (int)(r0 - K),
                       l2_policy_evict_first());  // last use of T
    }
  } else {
    const int rows = len + 2 * K;
    const float *src = T + colc;
    if (r0 >= K && r1 + K <= H) {  // no clamping needed
      const float *s0 = src + (r0 - K) * ldt;
      for (int tr = 0; tr < rows; ++tr) {
        unsigned sa = (unsigned)__cvta_generic_to_shared(tcol + tr * kTileStride);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(s0 + tr * ldt));
      }
    } else {
      for (int tr = 0; tr < rows; ++tr) {
        int64_t r = r0 - K + tr;
        r = r < 0 ? 0 : (r >= H ? H - 1 : r);
        unsigned sa = (unsigned)__cvta_generic_to_shared(tcol + tr * kTileStride);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(src + r * ldt));
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  }
  if (j == 0) {
    S.ccount = 0;
    S.cmax = 0u;
  }
  pdl_wait();  // band histories and the CandState come from earlier kernels
  const float gbound = __uint_as_float(st->absmax_bits);  // global max so far (lower bound)
  double Ybot[K], Yf[K];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    Ybot[i] = Z[zidx(1, b, i, p.NB, K, p.W, colc)];
    Yf[i] = Z[zidx(0, b, i, p.NB, K, p.W, colc)];
  }
  if (tma) {
    __syncthreads();  // barrier initialised before anyone waits on it
    mbar_wait(&tbar, 0);
  } else {
    asm volatile("cp.async.wait_group 0;\n" ::);
  }
  __syncthreads();
  // tile row of image row r is r - r0 + K
#define TX(tr) ((double)tcol[(tr) * kTileStride])

  // ---- backward start of sub-chunk 0 when the band has two ---------------
  double E0[K];
#pragma unroll
  for (int i = 0; i < K; ++i) E0[i] = Ybot[i];
  if (nsub == 2) {
    double zb[K], zo[K];  // even / odd samples: two independent FMA chains per i
#pragma unroll
    for (int i = 0; i < K; ++i) zb[i] = zo[i] = 0.0;
#pragma unroll
    for (int t = 0; t < kSub; ++t) {
      double v = TX(K + kSub + t);
#pragma unroll
      for (int i = 0; i < K; ++i)
        if (t - i > 0) {
          if (t & 1)
            zo[i] = fma(p.h[t - i], v, zo[i]);
          else
            zb[i] = fma(p.h[t - i], v, zb[i]);
        }
    }
#pragma unroll
    for (int i = 0; i < K; ++i) zb[i] += zo[i];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      double acc = zb[i];
#pragma unroll
      for (int q = 0; q < K; ++q) acc = fma(p.Tx[i * K + q], TX(K + kBand + q), acc);
#pragma unroll
      for (int q = 0; q < K; ++q) acc = fma(p.Ty[i * K + q], Ybot[q], acc);
      E0[i] = acc;
    }
  }

  double Xf[K];
#pragma unroll
  for (int i = 0; i < K; ++i) Xf[i] = TX(K - 1 - i);  // rows r0-1-i (clamped at the top)
  const double lsc = (double)p.lap_scale;
  // 5-point Laplacian as (left + right) + (up + down) - 4 centre: the
  // horizontal neighbour sum of row r-1 comes from lane shuffles when B(r-1)
  // is produced (warp-edge lanes are recomputed after the walk)
  //
  // Software-pipelined so that no long dependency chain sits inside one
  // row step: the lane shuffles of B(r) are consumed one step later, the
  // part of L(r-1) that does not involve B(r) is formed before B(r) exists,
  // and the recursion itself is the latency-pipelined DfiRun (one fma on the
  // loop-carried value per row).
  double Bm2 = 0.0, Bm1 = 0.0;  // B of rows r-2, r-1
  double blp = 0.0, brp = 0.0;  // shuffles of B(r-1) (left / right neighbour)
  auto shfl_lr = [&](double bc) {
    blp = __shfl_up_sync(0xffffffffu, bc, 1);
    brp = __shfl_down_sync(0xffffffffu, bc, 1);
  };
  auto lap = [&](double sx, double bu, double bc, double bd) {
    return (float)(lsc * fma(-4.0, bc, sx + (bu + bd)));
  };
  float tmax = 0.0f;  // running max |L| of this column (valid columns, non-edge lanes)
  // lanes 0, 1, 30, 31 keep B(r0-2 .. r1+1) for the warp-edge recomputation
  const bool keep_b = eslot >= 0;
  double *ebw = &S.eb[wid][keep_b ? eslot : 0][0];  // B(r0 - 2 + q) at ebw[q]

  // The walk leaves L(r0-1 .. r1) in the tile (in place of x); lanes 0 / 31
  // hold placeholders until the recomputation below.
  DfiRun<K> rf;
  rf.init(p, Yf, Xf);
  for (int s = 0; s < nsub; ++s) {
    const int64_t rb = r0 + (int64_t)s * kSub;
    const int trb = K + s * kSub;  // tile row of rb
    const bool last = s == nsub - 1;
    double park[kSub];
    {
      double Yb[K], Xb[K];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        Yb[i] = p.sign * (last ? Ybot[i] : E0[i]);  // history of sign * y-
        Xb[i] = TX(trb + kSub + i);
      }
      DfiRun<K> rb_;
      rb_.init(p.bwd, Yb, Xb);
#pragma unroll
      for (int t = kSub - 1; t >= 0; --t) park[t] = rb_.step(p.bwd, TX(trb + t));  // sign*y-
      if (s == 0 && r0 > 0) {  // B at rows r0-2, r0-1 from the band-edge histories
        double x1 = TX(K - 1), x2 = TX(K - 2);
        double ym1 = rb_.step(p.bwd, x1);
        double ym2 = rb_.step(p.bwd, x2);
        Bm1 = ym1 + fma(p.b0, x1, Yf[0]);
        Bm2 = ym2 + fma(p.b0, x2, Yf[1]);
        shfl_lr(Bm1);
        if (keep_b) {
          ebw[0] = Bm2;
          ebw[1] = Bm1;
        }
      }
    }
    float *lp = tcol + (trb - 1) * kTileStride;  // L(rb + t - 1) at lp[t * stride]
    double *ep = ebw + 2 + s * kSub;              // B(rb + t) at ep[t]
    // forward run: B(rb+t); L(rb+t-1) = Lx + Ly as soon as B(rb+t) exists
    if (rb >= 1 && rb + kSub < H) {  // no image edge in reach
      // row r = rb + t: the x sample and b0 x + sign y- of the NEXT row are
      // formed one step early, and q = B(r-2) - 4 B(r-1) at the end of the
      // previous step, so after B(r) only two additions remain before L(r-1)
      double xn = TX(trb);
      double cn = fma(p.b0, xn, park[0]);
      double q = fma(-4.0, Bm1, Bm2);
#pragma unroll
      for (int t = 0; t < kSub; ++t) {
        const double xv = xn, ct = cn;
        if (t + 1 < kSub) {
          xn = TX(trb + t + 1);
          cn = fma(p.b0, xn, park[t + 1]);
        }
        const double Bt = rf.step(p, xv) + ct;
        const double sx = blp + brp;  // shuffled when B(r-1) was produced
        shfl_lr(Bt);
        const double l = sx + (Bt + q);
        const float v = MODE == 1 ? (float)l : (float)(lsc * l);
        lp[t * kTileStride] = v;
        tmax = fmaxf(tmax, fabsf(v));
        if (keep_b) ep[t] = Bt;
        if (MODE == 2 && own_col) b64[(rb + t) * p.W + col] = Bt;
        if (MODE == 3 && own_col) Lout[(rb + t) * ldl + col] = (float)Bt;
        q = fma(-4.0, Bt, Bm1);
        Bm2 = Bm1;
        Bm1 = Bt;
      }
    } else {
#pragma unroll
      for (int t = 0; t < kSub; ++t) {
        const int64_t r = rb + t;
        const double xv = TX(trb + t);
        const double Bt = rf.step(p, xv) + fma(p.b0, xv, park[t]);
        if (r == 0) Bm1 = Bt;  // replicate top edge: B(-1) = B(0)
        const double sxm1 = blp + brp;
        shfl_lr(Bt);
        const double bnext = r >= H ? Bm1 : Bt;  // replicate bottom edge
        if (r >= 1) {
          const float v = (float)fma(lsc, bnext, lsc * fma(-4.0, Bm1, sxm1 + Bm2));
          lp[t * kTileStride] = v;
          if (r - 1 < H) tmax = fmaxf(tmax, fabsf(v));
        }
        if (keep_b) ep[t] = Bt;
        if (MODE == 2 && own_col && r < H) b64[r * p.W + col] = Bt;
        if (MODE == 3 && own_col && r < H) Lout[r * ldl + col] = (float)Bt;
        Bm2 = Bm1;
        Bm1 = Bt;
      }
    }
    if (last) {  // B at rows r1, r1+1 -> L(r1-1), L(r1)
      const int tr1 = K + len;
      double xr1 = TX(tr1), xr2 = TX(tr1 + 1);
      double y0 = rf.step(p, xr1);
      double y1 = rf.step(p, xr2);
      double B1 = fma(p.sign, Ybot[0], fma(p.b0, xr1, y0));
      double B2 = fma(p.sign, Ybot[1], fma(p.b0, xr2, y1));
      const double sxm1 = blp + brp;
      shfl_lr(B1);
      const double sx1 = blp + brp;
      if (r1 - 1 < H) {
        const float v = lap(sxm1, Bm2, Bm1, r1 >= H ? Bm1 : B1);
        tcol[(tr1 - 1) * kTileStride] = v;
        tmax = fmaxf(tmax, fabsf(v));
      }
      if (r1 < H) {
        const float v = lap(sx1, Bm1, B1, r1 + 1 >= H ? B1 : B2);
        tcol[tr1 * kTileStride] = v;
        tmax = fmaxf(tmax, fabsf(v));
      }
      if (keep_b) {
        ebw[len + 2] = B1;
        ebw[len + 3] = B2;
      }
    }
  }
#undef TX
  if (MODE >= 2) return;  // B only (fp64 to b64, or fp32 to Lout)
  pdl_trigger();
  __syncthreads();

  // ---- warp-edge columns (lanes 0 / 31): L recomputed from the kept B ------
  // The 2 x (rows) recomputations of a warp are spread over its 32 lanes; the
  // arithmetic is the walk's, so every column gets bit-identical formulas.
  {
    const int64_t rlo = r0 > 0 ? r0 - 1 : 0;
    const int64_t rhi = r1 < H ? r1 : H - 1;
    const int nr = (int)(rhi - rlo + 1);
    float pmax = 0.0f;
    for (int idx = lane; idx < 2 * nr; idx += 32) {
      const int side = idx & 1;
      const int64_t r = rlo + (idx >> 1);
      const int jj = wid * 32 + (side ? 31 : 0);
      if (jj == 0 || jj == kColThreads - 1) continue;  // CTA halo columns
      const int q = (int)(r - r0 + 2);
      const int qu = (int)((r > 0 ? r - 1 : 0) - r0 + 2);
      const int qd = (int)((r + 1 < H ? r + 1 : H - 1) - r0 + 2);
      const double *bcv = side ? S.eb[wid][3] : S.eb[wid][0];
      const double bl = side ? S.eb[wid][2][q] : S.eb[wid - 1][3][q];
      const double br = side ? S.eb[wid + 1][0][q] : S.eb[wid][1][q];
      const double bc = bcv[q];
      const float v = lap(bl + br, bcv[qu], bc, bcv[qd]);
      S.tile[r - r0 + K][jj + 2] = v;
      const int64_t cj = c0 - kColHalo + jj;
      if (cj >= 0 && cj < p.W) pmax = fmaxf(pmax, fabsf(v));
    }
    // the walk values of edge lanes were placeholders; columns outside the
    // image never count
    if (lane == 0 || lane == 31 || col < 0 || col >= p.W) tmax = 0.0f;
    tmax = fmaxf(tmax, pmax);
    tmax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(tmax)));
    if (lane == 0) atomicMax(&S.cmax, __float_as_uint(tmax));
  }
  __syncthreads();
  // publish this CTA's max now (later CTAs prune with it) and pick up what
  // earlier CTAs published since this one started
  if (j == 0) atomicMax(&st->absmax_bits, S.cmax);
  const float gnow = fmaxf(gbound, __uint_as_float(*(volatile unsigned *)&st->absmax_bits));

  // ---- store the owned L block (rows r0 .. r1-1, columns c0 .. c0+123) ----
  // fused with the strict 3x3 NMS over frac * max(this CTA's max |L|, the
  // global max published so far): a lower bound of the final threshold, so
  // the candidates are a superset that the flush and the finaliser filter.
  {
    const int nrow = (int)(rown_hi - r0);
    const int ncol = (int)(p.W - c0 < kColOut ? p.W - c0 : kColOut);
    // frac <= 0: L only (scale-space stacks), no candidates
    const float th = p.frac > 0.0f ? p.frac * fmaxf(__uint_as_float(S.cmax), gnow)
                                   : __int_as_float(0x7f800000);
    auto test = [&](int q, int c, float v) -> bool {  // tile row q + K, tile column 4 + c
      const int64_t r = r0 + q, cc = c0 + c;
      if (r < 1 || r > H - 2 || cc < 1 || cc > p.W - 2) return false;
      const int tr = q + K, tc = 4 + c;
      bool gt = true, lt = true;
#pragma unroll
      for (int di = -1; di <= 1; ++di)
#pragma unroll
        for (int dj = -1; dj <= 1; ++dj) {
          if (!di && !dj) continue;
          const float u = S.tile[tr + di][tc + dj];
          gt &= v > u;
          lt &= v < u;
        }
      // a maximum counts when L >= t, a minimum when -L >= t (|L| >= t alone
      // would admit a maximum of a negative region)
      return (gt && v >= th) || (lt && -v >= th);
    };
    if (vec_out && ncol == kColOut) {  // 31 float4 per row, one row per warp
      const bool act = lane < kColOut / 4;
      const uint64_t lpol = l2_policy_evict_first();  // L streams out
      float *dst = Lout + r0 * ldl + c0 + 4 * lane;
#pragma unroll 4
      for (int q = wid; q < nrow; q += kColThreads / 32) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (act) {
          v = *reinterpret_cast<const float4 *>(&S.tile[q + K][4 + 4 * lane]);
          st_v4_hint(dst + q * ldl, v, lpol);
        }
        const float m4 = fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
        if (__any_sync(0xffffffffu, act && m4 >= th)) {  // (warp-uniform) rare
          const float vv[4] = {v.x, v.y, v.z, v.w};
          unsigned m = 0u;
          if (act && m4 >= th) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (fabsf(vv[i]) >= th && test(q, 4 * lane + i, vv[i])) m |= 1u << i;
          }
          cand_push_warp(&S.ccount, S.cy, S.cx, S.cv, kCandSmem, st, gy, gx, gv, gcap, m, (int)(r0 + q), (int)(c0 + 4 * lane), vv);
        }
      }
    } else {
      for (int q = wid; q < nrow; q += kColThreads / 32)
        for (int cl = 0; cl < ncol; cl += 32) {
          const int c = cl + lane;
          float v = 0.0f;
          if (c < ncol) {
            v = S.tile[q + K][4 + c];
            Lout[(r0 + q) * ldl + c0 + c] = v;
          }
          const unsigned m = c < ncol && fabsf(v) >= th && test(q, c, v) ? 1u : 0u;
          const float vv[4] = {v, 0.f, 0.f, 0.f};
          cand_push_warp(&S.ccount, S.cy, S.cx, S.cv, kCandSmem, st, gy, gx, gv, gcap, m, (int)(r0 + q), (int)(c0 + c), vv);
        }
    }
  }
  __syncthreads();

  // ---- flush candidates that survive the best threshold known now ---------
  __shared__ float thr_end;
  if (j == 0) {
    unsigned old = atomicMax(&st->absmax_bits, S.cmax);
    float m = fmaxf(__uint_as_float(old), __uint_as_float(S.cmax));
    thr_end = p.frac * m;
  }
  __syncthreads();
  const int n = S.ccount < kCandSmem ? S.ccount : kCandSmem;
  for (int q = j; q < n; q += blockDim.x) {
    if (!(fabsf(S.cv[q]) >= thr_end)) continue;
    int k = atomicAdd(&st->count, 1);
    if (k < gcap) {
      gy[k] = S.cy[q];
      gx[k] = S.cx[q];
      gv[k] = S.cv[q];
    } else {
      st->overflow = 1;
    }
  }
}

// ---------------------------------------------------------------------------
// 4. final threshold + (y, x) order: one CTA, bitonic sort in shared memory
// ---------------------------------------------------------------------------
constexpr int kSortCap = 4096;
constexpr int kFinThreads = 1024;

// Ordered full-frame NMS by one CTA: the (rare) fallback when a candidate
// buffer overflowed.  Rows in order, each row compacted with a block scan, so
// the output is sorted by (y, x) like the fast path.
__device__ void final_fullscan(const float *__restrict__ L, int64_t ldl, int64_t H, int64_t W,
                               float thr, int32_t *det_yx, float *det_val, int64_t cap,
                               int64_t *n_det) {
  __shared__ int wsum[kFinThreads / 32];
  __shared__ long long base;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int64_t r = 1; r + 1 < H; ++r) {
    for (int64_t c0 = 0; c0 < W; c0 += kFinThreads) {
      const int64_t c = c0 + threadIdx.x;
      bool det = false;
      float v = 0.0f;
      if (c >= 1 && c + 1 < W) {
        v = L[r * ldl + c];
        if (fabsf(v) >= thr) {
          bool gt = true, lt = true;
          for (int di = -1; di <= 1; ++di)
            for (int dj = -1; dj <= 1; ++dj) {
              if (!di && !dj) continue;
              float u = L[(r + di) * ldl + c + dj];
              gt &= v > u;
              lt &= v < u;
            }
          det = (gt && v >= thr) || (lt && -v >= thr);
        }
      }
      unsigned bal = __ballot_sync(0xffffffffu, det);
      if (lane == 0) wsum[wid] = __popc(bal);
      __syncthreads();
      int before = 0, total = 0;
      for (int w = 0; w < kFinThreads / 32; ++w) {
        if (w < wid) before += wsum[w];
        total += wsum[w];
      }
      before += __popc(bal & ((1u << lane) - 1u));
      if (det) {
        long long pos = base + before;
        if (pos < cap) {
          det_yx[2 * pos] = (int32_t)r;
          det_yx[2 * pos + 1] = (int32_t)c;
          det_val[pos] = v;
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) base += total;
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) *n_det = base;
}

// In-place ascending bitonic sort of (key, val) pairs in shared memory; n keys
// padded with ~0 up to a power of two np (every thread of the CTA calls it).
__device__ void smem_bitonic(unsigned long long *key, float *val, int n, int np) {
  for (int q = n + threadIdx.x; q < np; q += blockDim.x) key[q] = ~0ull;
  __syncthreads();
  for (int kk = 2; kk <= np; kk <<= 1)
    for (int jj = kk >> 1; jj > 0; jj >>= 1) {
      for (int i = threadIdx.x; i < np; i += blockDim.x) {
        const int ix = i ^ jj;
        if (ix > i) {
          const bool up = (i & kk) == 0;
          const unsigned long long a = key[i], c = key[ix];
          if ((a > c) == up) {
            key[i] = c;
            key[ix] = a;
            const float t = val[i];
            val[i] = val[ix];
            val[ix] = t;
          }
        }
      }
      __syncthreads();
    }
}

__device__ __forceinline__ void write_dets(const unsigned long long *key, const float *val, int n,
                                           int64_t base, int64_t W, int32_t *det_yx,
                                           float *det_val, int64_t cap) {
  for (int q = threadIdx.x; q < n; q += blockDim.x) {
    const int64_t o = base + q;
    if (o < cap) {
      det_yx[2 * o] = (int32_t)(key[q] / (unsigned long long)W);
      det_yx[2 * o + 1] = (int32_t)(key[q] % (unsigned long long)W);
      det_val[o] = val[q];
    }
  }
}

constexpr int kBigCap = 6144;  // keys per CTA of the large-list path (72 KB)
constexpr unsigned long long kLookAgg = 1ull << 62, kLookPre = 2ull << 62;
constexpr unsigned long long kLookMask = (1ull << 62) - 1;

// Final threshold + (y, x) order.  Small lists (<= kSortCap candidates, the
// usual case) are sorted by CTA 0 alone; the other CTAs return at once.
// Larger lists use all kFinCtas CTAs: CTA b owns the rows [b H / G, (b+1) H / G),
// collects its survivors (the list is read from L2 by every CTA), learns how
// many the earlier row ranges hold by a decoupled look-back over the
// CandState's look[] words, and writes its sorted survivors at that offset --
// so the output never depends on how the candidates were appended, and the
// cost grows with the list instead of falling off a one-CTA cliff.  Only an
// overflow of the global list itself takes the ordered full-frame scan.
__global__ void __launch_bounds__(kFinThreads) colfinal_kernel(
    CandState *__restrict__ st, const int *__restrict__ gy, const int *__restrict__ gx,
    const float *__restrict__ gv, int gcap, const float *__restrict__ L, int64_t ldl, int64_t H,
    int64_t W, float frac, int32_t *det_yx, float *det_val, int64_t cap, int64_t *n_det,
    float *thr_out, int force_full) {
  extern __shared__ __align__(16) unsigned char fsm[];
  unsigned long long *key = reinterpret_cast<unsigned long long *>(fsm);
  __shared__ int m;
  __shared__ long long prefix;
  // let the next kernel (the next scale's row pass, which waits for this grid
  // before it overwrites anything this kernel reads) start now
  pdl_trigger();
  pdl_wait();
  const int count = st->count, overflow = st->overflow;
  const float thr = frac * __uint_as_float(st->absmax_bits);
  const int n = count < gcap ? count : gcap;
  const bool big = n > kSortCap;
  if (blockIdx.x == 0 && threadIdx.x == 0 && thr_out) *thr_out = thr;
  // global list overflow: exact, slow path over L (a pass that keeps L in
  // its tiles -- L null -- sizes its list for every possible candidate)
  if ((force_full || overflow) && L) {
    if (blockIdx.x == 0) final_fullscan(L, ldl, H, W, thr, det_yx, det_val, cap, n_det);
    return;
  }
  if (!big && blockIdx.x != 0) return;
  float *val = reinterpret_cast<float *>(fsm + (big ? kBigCap : kSortCap) * sizeof(unsigned long long));
  if (threadIdx.x == 0) m = 0;
  __syncthreads();
  if (!big) {
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
      const float v = gv[q];
      const int yy = gy[q], xx = gx[q];  // loaded together: one round trip
      if (!(fabsf(v) >= thr)) continue;
      const int k = atomicAdd(&m, 1);
      key[k] = (unsigned long long)yy * (unsigned long long)W + (unsigned long long)xx;
      val[k] = v;
    }
    __syncthreads();
    const int mm = m;
    if (mm <= kFinThreads) {
      // rank sort: keys are distinct (y, x) positions; broadcast smem reads
      if (threadIdx.x < mm) {
        const unsigned long long mine = key[threadIdx.x];
        int rank = 0;
        for (int q = 0; q < mm; ++q) rank += key[q] < mine;
        if (rank < cap) {
          det_yx[2 * rank] = (int32_t)(mine / (unsigned long long)W);
          det_yx[2 * rank + 1] = (int32_t)(mine % (unsigned long long)W);
          det_val[rank] = val[threadIdx.x];
        }
      }
    } else {
      int np = 1;
      while (np < mm) np <<= 1;
      smem_bitonic(key, val, mm, np);
      write_dets(key, val, mm, 0, W, det_yx, det_val, cap);
    }
    if (threadIdx.x == 0) *n_det = mm;
    return;
  }
  // ---- large list: row ranges over kFinCtas CTAs ---------------------------
  const int G = gridDim.x, b = blockIdx.x;
  const int64_t ylo = H * b / G, yhi = H * (b + 1) / G;
  for (int q = threadIdx.x; q < n; q += blockDim.x) {
    const int yy = gy[q];
    if (yy < ylo || yy >= yhi) continue;
    const float v = gv[q];
    if (!(fabsf(v) >= thr)) continue;
    const int k = atomicAdd(&m, 1);
    if (k < kBigCap) {
      key[k] = (unsigned long long)yy * (unsigned long long)W + (unsigned long long)gx[q];
      val[k] = v;
    }
  }
  __syncthreads();
  const int T = m;
  {
    // every CTA publishes its own count; CTA b then reads the counts of all
    // CTAs j < b at once (one thread each, spinning only on a CTA that has
    // not counted yet -- it was dispatched earlier) and sums them: no serial
    // chain of inclusive prefixes from CTA to CTA
    volatile unsigned long long *look = st->look;
    __shared__ long long wsum[kFinThreads / 32];
    if (threadIdx.x == 0) look[b] = kLookAgg | (unsigned long long)T;
    long long v = 0;
    for (int j = threadIdx.x; j < b; j += blockDim.x) {
      unsigned long long f;
      do {
        f = look[j];
      } while (!(f & kLookAgg));
      v += (long long)(f & kLookMask);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long acc = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) acc += wsum[w];
      prefix = acc;
      if (b == G - 1) *n_det = acc + T;
    }
  }
  __syncthreads();
  const long long base = prefix;
  if (T <= kBigCap) {
    int np = 1;
    while (np < T) np <<= 1;
    smem_bitonic(key, val, T, np);
    write_dets(key, val, T, base, W, det_yx, det_val, cap);
    return;
  }
  // more survivors in this row range than shared memory holds: one row at a
  // time (a row has at most W / 2 strict extrema <= kBigCap for W <= 12288)
  long long off = base;
  for (int64_t r = ylo; r < yhi; ++r) {
    __syncthreads();
    if (threadIdx.x == 0) m = 0;
    __syncthreads();
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
      if (gy[q] != r) continue;
      const float v = gv[q];
      if (!(fabsf(v) >= thr)) continue;
      const int k = atomicAdd(&m, 1);
      if (k < kBigCap) {
        key[k] = (unsigned long long)r * (unsigned long long)W + (unsigned long long)gx[q];
        val[k] = v;
      }
    }
    __syncthreads();
    const int mr = m < kBigCap ? m : kBigCap;
    int np = 1;
    while (np < mr) np <<= 1;
    smem_bitonic(key, val, mr, np);
    write_dets(key, val, mr, off, W, det_yx, det_val, cap);
    off += mr;
  }
}

// ---------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------
static void transfer_ld(const double *b, const double *a, int k, int len, double *Ty,
                        double *Tx) {
  for (int jj = 0; jj < 2 * k; ++jj) {
    long double Y[VMF_MAX_IIR_ORDER], X[VMF_MAX_IIR_ORDER];
    for (int m = 0; m < k; ++m) {
      Y[m] = (jj == m) ? 1.0L : 0.0L;
      X[m] = (jj == k + m) ? 1.0L : 0.0L;
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
      if (jj < k)
        Ty[i * k + jj] = (double)Y[i];
      else
        Tx[i * k + (jj - k)] = (double)Y[i];
    }
  }
}

static void impulse_ld(const double *b, const double *a, int k, int n, double *h) {
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

bool colpass_supported(int64_t h, int64_t w, int k) {
  return k >= 2 && k <= 4 && h >= 2 * kSub && w >= 1 &&
         cdiv(cdiv(h, kSub) * kSub, kBand) <= 32 * kMaxCpl;
}

static void col_geometry(int64_t h, int64_t *Hp, int *NB, int *Blast) {
  int64_t hp = cdiv(h, kSub) * kSub;
  int nb = (int)cdiv(hp, kBand);
  *Hp = hp;
  *NB = nb;
  *Blast = (int)(hp - (int64_t)(nb - 1) * kBand);
}

static int64_t cand_capacity(int64_t h, int64_t w) {
  int64_t c = h * w / 64;
  if (c < 65536) c = 65536;
  return c;
}

size_t colpass_workspace_bytes(int64_t h, int64_t w, int k, int64_t) {
  int64_t Hp;
  int NB, Bl;
  col_geometry(h, &Hp, &NB, &Bl);
  int64_t gcap = cand_capacity(h, w);
  size_t z = (size_t)NB * 2 * 2 * k * w * sizeof(double);
  return 4096 + ((z + 255) & ~(size_t)255) + (size_t)gcap * 12 + 1024 +
         detect_workspace_bytes(1, h, w);
}

int64_t colpass_cand_capacity(int64_t h, int64_t w) { return cand_capacity(h, w); }

int colfinal_launch(CandState *cs, const int *gy, const int *gx, const float *gv, int64_t gcap,
                    const float *L, int64_t ldl, int64_t H, int64_t W, float frac,
                    int32_t *det_yx, float *det_val, int64_t cap, int64_t *n_det_dev,
                    float *thr_dev, cudaStream_t st) {
  Launch g(K_FINALIZE, st);
  const int fsmem = kBigCap * (int)(sizeof(unsigned long long) + sizeof(float));
  static PerDevice fattr;
  if (fattr.first()) {
    cudaFuncSetAttribute(colfinal_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, fsmem);
  }
  launch_pdl(colfinal_kernel, dim3(kFinCtas), dim3(kFinThreads), fsmem, st, cs, gy, gx, gv, (int)gcap, L,
             ldl, H, W, frac, det_yx, det_val, cap, n_det_dev, thr_dev,
             getenv("VMF_FORCE_FULLSCAN") ? 1 : 0);
  return cuda_status("finaliser");
}

template <int K>
static int launch_colpass(const float *T, int64_t ldt, float *L, int64_t ldl, const ColParams &p,
                          double *b64, bool blur_only,
                          int32_t *det_yx, float *det_val, int64_t cap, int64_t *n_det_dev,
                          float *thr_dev, void *ws, size_t ws_bytes, cudaStream_t st) {
  char *base = (char *)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  CandState *cs = (CandState *)base;
  int *fallback = (int *)(base + 64);
  size_t z = (size_t)p.NB * 2 * 2 * K * p.W * sizeof(double);
  double *Z = (double *)(base + 4096);
  char *q = base + 4096 + ((z + 255) & ~(size_t)255);
  int64_t gcap = cand_capacity(p.H, p.W);
  int *gy = (int *)q;
  int *gx = gy + gcap;
  float *gv = (float *)(gx + gcap);
  void *dws = (void *)(((uintptr_t)(gv + gcap) + 255) & ~(uintptr_t)255);
  size_t dws_b = detect_workspace_bytes(1, p.H, p.W);
  {
    Launch g(K_COL_CARRY, st);
    dim3 grid((unsigned)cdiv(p.W, kCarryCols), (unsigned)p.NB);
    CUtensorMap cmap;
    memset(&cmap, 0, sizeof(cmap));
    int ctma = make_tmap_2d_f32(&cmap, T, p.H, p.W, ldt, kCarryCols, kBand) &&
               !getenv("VMF_NO_TMA");
    cudaGetLastError();
    const int csm = kBand * kCarryCols * (int)sizeof(float) + 128;
    static PerDevice cattr;
    if (cattr.first()) {
      cudaFuncSetAttribute(colcarry_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, csm);
    }
    launch_pdl(colcarry_kernel<K>, grid, dim3(kCarryThreads), csm, st, T, ldt, p, Z, cmap, ctma,
               cs);
  }
  {
    Launch g(K_COL_SCAN, st);
    const int ssm = (int)((size_t)p.NB * (2 * K * kScanCols + 2) * sizeof(double));
    static PerDevice sattr;
    if (sattr.first()) {
      cudaFuncSetAttribute(colscan_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024);
    }
    launch_pdl(colscan_kernel<K>, dim3((unsigned)cdiv(p.W, kScanCols), 2), dim3(32 * kScanCols),
               ssm, st, T, ldt, p, Z);
  }

  {
    Launch g(K_IIR_COLS_FUSED, st);
    static PerDevice attr;
    if (attr.first()) {
      cudaFuncSetAttribute(colapply_kernel<K, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(ColSmem<K>) + 128);
      cudaFuncSetAttribute(colapply_kernel<K, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(ColSmem<K>) + 128);
      cudaFuncSetAttribute(colapply_kernel<K, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(ColSmem<K>) + 128);
      cudaFuncSetAttribute(colapply_kernel<K, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(ColSmem<K>) + 128);
    }
    dim3 grid((unsigned)cdiv(p.W, kColOut), (unsigned)p.NB);
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    int use_tma = make_tmap_2d_f32(&tmap, T, p.H, p.W, ldt, kTileStride, kTileRows(K)) &&
                  !getenv("VMF_NO_TMA");
    cudaGetLastError();
    auto kern = blur_only ? colapply_kernel<K, 3>
                : b64   ? colapply_kernel<K, 2>
                        : (p.lap_scale == 1.0f ? colapply_kernel<K, 1> : colapply_kernel<K, 0>);
    launch_pdl(kern, grid, dim3(kColThreads), sizeof(ColSmem<K>) + 128, st, T, ldt, L, ldl, p,
               (const double *)Z, cs, gy, gx, gv, (int)gcap, tmap, use_tma,
               (int)(ldl % 4 == 0 && (uintptr_t)L % 16 == 0), b64);
  }
  if (p.frac > 0.0f && !b64 && !blur_only)
    colfinal_launch(cs, gy, gx, gv, gcap, L, ldl, p.H, p.W, p.frac, det_yx, det_val, cap,
                    n_det_dev, thr_dev, st);
  return cuda_status("column pass");
}

int colpass_run(const float *T, int64_t ldt, float *L, int64_t ldl, double *b64,
                const IirParams &ip,
                int64_t h, int64_t w, float lap_scale, float frac, int32_t *det_yx,
                float *det_val, int64_t cap, int64_t *n_det_dev, float *thr_dev, void *ws,
                size_t ws_bytes, cudaStream_t st, bool blur_only) {
  size_t need = colpass_workspace_bytes(h, w, ip.K, cap);
  if (!ws || ws_bytes < need)
    return fail(VMF_EVALUE, "column-pass workspace too small: %zu < %zu bytes", ws_bytes, need);
  ColParams p;
  static PlanCache<ColParams> cache;
  std::vector<unsigned char> key;
  key_add(key, h);
  key_add(key, w);
  key_add(key, ip.K);
  key_add(key, ip.b0);
  key_add(key, ip.sign);
  key_add(key, ip.b, sizeof(double) * ip.K);
  key_add(key, ip.a, sizeof(double) * ip.K);
  if (!cache.get(key, &p)) {
    memset(&p, 0, sizeof(p));
    const int k = ip.K;
    for (int m = 0; m < k; ++m) {
      p.b[m] = ip.b[m];
      p.a[m] = ip.a[m];
    }
    p.b0 = ip.b0;
    p.sign = ip.sign;
    for (int m = 0; m < k; ++m) {
      p.bwd.b[m] = ip.sign * ip.b[m];
      p.bwd.a[m] = ip.a[m];
    }
    p.yss = ip.yss;
    impulse_ld(ip.b, ip.a, k, kHMax, p.h);
    transfer_ld(ip.b, ip.a, k, kSub, p.Ty, p.Tx);
    p.H = h;
    p.W = w;
    col_geometry(h, &p.Hp, &p.NB, &p.Blast);
    transfer_ld(ip.b, ip.a, k, kBand, p.TyB[0], p.TxB[0]);
    transfer_ld(ip.b, ip.a, k, p.Blast, p.TyB[1], p.TxB[1]);
    for (int i = 0; i < k; ++i)
      for (int t = 0; t < kBand / 2; ++t) {
        int qa = kBand - 1 - i - t, qb = t - i;
        double A = qa > 0 ? p.h[qa] : 0.0, B = qb > 0 ? p.h[qb] : 0.0;
        p.SP[i][t] = 0.5 * (A + B);
        p.SQ[i][t] = 0.5 * (A - B);
      }
    p.cpl = (p.NB + 31) / 32;

    if (p.cpl > kMaxCpl) return fail(VMF_EVALUE, "image too tall for the fused column pass");
    for (int l = 0; l < 5; ++l) {
      double tx[VMF_MAX_IIR_ORDER * VMF_MAX_IIR_ORDER];
      transfer_ld(ip.b, ip.a, k, (p.cpl << l) * kBand, p.TyBp[l], tx);
    }
    cache.put(key, p);
  }
  p.lap_scale = lap_scale;
  p.frac = frac;
  switch (ip.K) {
    case 2: return launch_colpass<2>(T, ldt, L, ldl, p, b64, blur_only, det_yx, det_val, cap, n_det_dev, thr_dev,
                                     ws, ws_bytes, st);
    case 3: return launch_colpass<3>(T, ldt, L, ldl, p, b64, blur_only, det_yx, det_val, cap, n_det_dev, thr_dev,
                                     ws, ws_bytes, st);
    case 4: return launch_colpass<4>(T, ldt, L, ldl, p, b64, blur_only, det_yx, det_val, cap, n_det_dev, thr_dev,
                                     ws, ws_bytes, st);
  }
  return fail(VMF_EVALUE, "fused column pass supports K = 2..4, got %d", ip.K);
}

}  // namespace vmf
