// vmf_colpass32.cu -- the fused second pass in fp32, "Laplacian first":
// column IIR (iir_cols, engine.py:156-158 / kernel 65-102) + Laplacian
// D20 + D02 (engine.py:218-227, blob.py:161) + threshold / 3x3 NMS
// (SURVEY.md §8(d)), reading the row-pass output T and writing L plus a short
// candidate list.
//
// Why fp32 is enough here.  The reference forms B = C(T) (column filter with
// steady-state starts) and then L = D20(B) + D02(B) with replicate edges; L is
// ~1e-3 of B at sigma = 32, so any fp32 rounding of B costs ~1e-4 of max|L|.
// By linearity and shift invariance on the replicate-extended column the
// same L is
//     L = C(U) + corrections at rows 0 and H-1,
//     U = 5-point Laplacian of T (replicate edges; rows past the bottom are
//         clamped copies, so there U = D20 T(H-1)), steady-state starts from
//         D20 T of rows 0 / H-1,
//     L(0)   += sign * sum_{m>=1} h(m) G(m),   G(m) = T(m) - T(m-1),
//     L(H-1) -=        sum_{m>=1} h(m) G(H-m),
// and every quantity in it is a difference of T, so fp32 rounding is relative
// to |L|, not |B|.  The recursion itself must be well conditioned in fp32: the
// causal part B(z)/A(z) is realised in modal form (a Jordan chain
// u1 = p u1 + x, u2 = p u2 + u1, ... for the repeated real pole of the
// repeated-pole blurs; a rotation for the complex pair of the Butterworth
// blur), y+(n) = c . u(n-1) -- DF-I in fp32 misses the tolerance by 16x at
// sigma = 32.  tools/experiments/col_lapfirst_chunked.py is the numpy
// prototype of exactly this chunking (fp32 throughout): its error equals the
// fp64 column pass's on the same fp32 T at every config scale.
//
// Chunking (as the fp64 pass): bands of 64 rows; colcarry32 computes the
// zero-state end states of both directions of every (band, column) by folded
// sample pairs, and band partials of the two boundary corrections; colscan32
// turns them into the true start state of every band (fp64 arithmetic over
// fp32 records, sequential over the bands per column and direction) and
// sums the corrections; colapply32 (128 columns x one band per CTA) walks up (the
// backward part parked in registers) and down (L produced directly), then
// stores the owned 124 x 64 block fused with the 3x3 NMS, exactly like the
// fp64 pass.  L of the halo rows r0-1 / r1 (for the NMS) comes from the band
// start states through c A^-1.
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <vector>

#include "plan_cache.hpp"
#include "vmf_colpass.cuh"
#include "vmf_common.cuh"
#include "vmf_prof.cuh"
#include "vmf_tma.cuh"
#include "vmf_modal32.cuh"
#include "vmf_rowlap.cuh"

namespace vmf {

constexpr int kB32 = 64;                 // rows per band
constexpr int kC32 = 128;                // columns per CTA (carry and apply)
constexpr int kC32Out = kC32 - 4;        // owned columns per apply CTA
constexpr int kT32Stride = kC32 + 4;     // apply tile stride: tile col j+2 <-> thread j
constexpr int kT32Rows = kB32 + 4;       // T rows r0-2 .. r1+1
constexpr int kL32Rows = kB32 + 2;       // U / L rows r0-1 .. r1
constexpr int kCarryStride = kC32 + 8;   // carry tile: cols c0-4 .. c0+131
constexpr int kCarryRows = kB32 + 2;     // T rows r0-1 .. r1
constexpr int kCand32 = 256;             // per-CTA candidate buffer
constexpr int kMaxNB32 = 128;            // bands (H <= 8192: the scan's shared staging)
constexpr int kScan32Cols = 32;
constexpr int kHm32Max = 2048;           // boundary-correction weights h(1..Mh)

struct Col32Params {
  float p, q;               // JORDAN: pole p; CPAIR: p + i q
  float c[4];               // y+(n) = c . u(n-1)
  float ci[4];              // c A^-1 (halo rows)
  float e1;                 // c A^-1 b
  float b0, sign, lsc, frac;
  float SP[4][kB32 / 2], SQ[4][kB32 / 2];  // folded band-carry weights
  float Wh[kB32 / 2][4];    // A^t b, t < 32: the half-band carry (V-mode apply)
  float A32[16];            // A^32 (fp32)
  float cs[4];              // sign * c
  double AL[16];            // A^64, row-major K x K
  double Iss[4];            // (I - A)^-1 b: steady state per unit input
  int64_t H, W;
  int NB, K, Mh;            // bands; order; boundary-correction length
};

// h(m) = c A^(m-1) b, m = 0..Mh (h(0) = 0): the boundary-correction weights,
// a kernel parameter of the carry pass only
struct Hm32 {
  float h[kHm32Max + 1];
};

// Band records, coalesced along columns: R[(b * (2K + 2) + q) * W + col]
//   q < K: forward zero-state end state (-> forward start state uf(r0-1)),
//   K <= q < 2K: backward (-> ub(r1)), 2K / 2K+1: the band's partials of the
//   top / bottom boundary corrections.
__device__ __forceinline__ int64_t ridx(int b, int q, int K, int64_t W, int64_t col) {
  return ((int64_t)b * (2 * K + 2) + q) * W + col;
}

// ---------------------------------------------------------------------------
// 1. band carries
// ---------------------------------------------------------------------------
// One CTA = 128 columns x one band, 256 threads: threads j and j + 128 take the
// two halves of the band's 32 sample pairs (t, 63 - t) of column j.  The tile
// holds T rows r0-1 .. r1 (clamped), columns c0-4 .. c0+131 (clamped).
// VM: the input is V = R(Lap5 X) of the fp32 row pass (U = V itself, no
// horizontal neighbours); the border partials then come from the row pass.
template <int K, bool VM>
__global__ void __launch_bounds__(2 * kC32) colcarry32_kernel(
    const float *__restrict__ T, int64_t ldt, Col32Params p, float *__restrict__ R,
    const __grid_constant__ Hm32 hm, const __grid_constant__ CUtensorMap tmap, int use_tma,
    CandState *__restrict__ cs, const float *__restrict__ Vb) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem_raw);
  float *tile = reinterpret_cast<float *>(smem_raw + ((128u - (sbase & 127u)) & 127u));
  __shared__ __align__(8) uint64_t tbar;
  __shared__ float part[2 * K + 2][kC32];
  const int j = threadIdx.x & (kC32 - 1), half = threadIdx.x >> 7;
  const int b = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * kC32;
  const int64_t col = c0 + j;
  const int64_t r0 = (int64_t)b * kB32;
  const int64_t H = p.H, W = p.W;
  const bool tma = use_tma && r0 >= 1 && r0 + kB32 + 1 <= H && c0 >= 4 && c0 + kC32 + 4 <= W;
  pdl_wait();  // T comes from the row pass
  if (blockIdx.x == 0 && blockIdx.y == 0) cand_reset(cs);
  // tile <- rows r0-1 .. r1, columns c0-4 .. c0+131 of src (TMA box, or
  // clamped loads: replicate edges, rows past H repeat H-1)
  auto stage = [&](const CUtensorMap *map, const float *src, int64_t ld, unsigned phase) {
    (void)phase;
    if (tma) {
      if (threadIdx.x == 0) {
        if (phase == 0) mbar_init(&tbar, 1);
        mbar_expect_tx(&tbar, (unsigned)(kCarryRows * kCarryStride * sizeof(float)));
        tma_load_2d_hint(tile, map, &tbar, (int)(c0 - 4), (int)(r0 - 1), l2_policy_evict_last());
      }
      __syncthreads();
      mbar_wait(&tbar, phase);
    } else {
      for (int e = threadIdx.x; e < kCarryRows * kCarryStride; e += blockDim.x) {
        const int tr = e / kCarryStride, tc = e - tr * kCarryStride;
        int64_t r = r0 - 1 + tr, c = c0 - 4 + tc;
        c = c < 0 ? 0 : (c >= W ? W - 1 : c);
        if (VM && r >= H) {  // below the image the column input is the virtual row Vb
          tile[e] = __ldg(Vb + c);
          continue;
        }
        r = r < 0 ? 0 : (r >= H ? H - 1 : r);
        tile[e] = __ldg(src + r * ld + c);
      }
      __syncthreads();
    }
  };
  stage(&tmap, T, ldt, 0);
  // tile row of image row r: r - r0 + 1; tile column of column c0 + j: j + 4
  const float *tc = tile + j + 4;
#define TT(tr, dc) tc[(tr) * kCarryStride + (dc)]
  auto U = [&](int tr) {
    return VM ? TT(tr, 0) : lap5(TT(tr, -1), TT(tr, 0), TT(tr, 1), TT(tr - 1, 0), TT(tr + 1, 0));
  };
  float P[K], Q[K];
#pragma unroll
  for (int i = 0; i < K; ++i) P[i] = Q[i] = 0.0f;
  // warp-uniform halves, so the weight indices are compile-time constants
  // (the weights stay constant-bank operands of the FFMAs)
  auto run = [&](auto HALF) {
    constexpr int t0 = decltype(HALF)::value * (kB32 / 4);
#pragma unroll
    for (int t = 0; t < kB32 / 4; ++t) {
      const float ua = U(1 + t0 + t), ub = U(kB32 - t0 - t);
      const float s = ua + ub, d = ua - ub;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        P[i] = fmaf(p.SP[i][t0 + t], s, P[i]);
        Q[i] = fmaf(p.SQ[i][t0 + t], d, Q[i]);
      }
    }
  };
  if (half == 0)
    run(std::integral_constant<int, 0>());
  else
    run(std::integral_constant<int, 1>());
  // boundary-correction partials (bands within Mh rows of the top / bottom):
  // top = sum h(r) G(r), bottom = sum h(H - r) G(r) over this band's rows
  // 1 <= r < H, G(r) = T(r) - T(r-1); each half takes 32 rows
  // (V mode: the row pass accumulates the border partials of the frame)
  float pt = 0.0f, pb = 0.0f;
  const bool top = !VM && r0 < p.Mh + 1, bot = !VM && r0 + kB32 > H - 1 - p.Mh;
  if (top || bot) {  // (CTA-uniform)
    for (int t = half * (kB32 / 2); t < (half + 1) * (kB32 / 2); ++t) {
      const int64_t r = r0 + t;
      if (r < 1 || r >= H) continue;
      const float g = TT(t + 1, 0) - TT(t, 0);
      if (top && r <= p.Mh) pt = fmaf(hm.h[r], g, pt);
      if (bot && H - r <= p.Mh) pb = fmaf(hm.h[H - r], g, pb);
    }
  }
#undef TT
  pdl_trigger();
  if (half == 1) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
      part[i][j] = P[i];
      part[K + i][j] = Q[i];
    }
    part[2 * K][j] = pt;
    part[2 * K + 1][j] = pb;
  }
  __syncthreads();
  if (half == 0 && col < W) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const float Pt = P[i] + part[i][j], Qt = Q[i] + part[K + i][j];
      R[ridx(b, i, K, W, col)] = Pt + Qt;       // forward
      R[ridx(b, K + i, K, W, col)] = Pt - Qt;   // backward
    }
    R[ridx(b, 2 * K, K, W, col)] = pt + part[2 * K][j];
    R[ridx(b, 2 * K + 1, K, W, col)] = pb + part[2 * K + 1][j];
  }
}

// ---------------------------------------------------------------------------
// 2. band scan.  CTA = 32 columns, both directions.  The records of its
//    columns are staged in shared memory with coalesced 16-byte copies; then
//    one thread per (column, direction) runs the band recursion
//    u <- A^64 u + z sequentially in fp64 (64 bands: ~1.5k cycles of DFMA
//    latency), writing each band's start state over its zero-state carry, and
//    one thread per (column, correction) sums the boundary partials in band
//    order; the start states go back with coalesced stores.
// ---------------------------------------------------------------------------
template <int K, bool VM>
__global__ void __launch_bounds__(256) colscan32_kernel(const float *__restrict__ T, int64_t ldt,
                                                       Col32Params p, float *__restrict__ R,
                                                       float *__restrict__ Cc,
                                                       const float *__restrict__ Vt,
                                                       const float *__restrict__ Vb,
                                                       CandState *__restrict__ cst) {
  extern __shared__ __align__(16) float ss[];  // [NB][2K+2][32]
  constexpr int Q = 2 * K + 2;
  const int NB = p.NB;
  const int64_t W = p.W, H = p.H;
  const int64_t c0 = (int64_t)blockIdx.x * kScan32Cols;
  const int tid = threadIdx.x;
  __shared__ float es[2][kScan32Cols];
  // V on the band-boundary rows (the bound below): the row pass wrote it long
  // before, so the loads go out ahead of the wait for the carries
  constexpr int kBnd = 16;  // boundary values per thread ((NB - 1) x 32 <= 16 x 256)
  float vb[kBnd];
  if (VM && p.frac > 0.0f) {
#pragma unroll
    for (int k = 0; k < kBnd; ++k) {
      const int e = tid + k * (int)blockDim.x;
      const int b = 1 + e / kScan32Cols, c = e - (b - 1) * kScan32Cols;
      const int64_t r1 = (int64_t)b * kB32, col = c0 + c;
      vb[k] = (b < NB && r1 < H - 1 && col < W) ? __ldg(T + r1 * ldt + col) : 0.0f;
    }
  }
  pdl_wait();  // records come from the band carries
  const bool full = c0 + kScan32Cols <= W && (W & 3) == 0;
  if (full) {
    for (int e = tid; e < NB * Q * (kScan32Cols / 4); e += blockDim.x) {
      const int row = e / (kScan32Cols / 4), v = e - row * (kScan32Cols / 4);  // row = b Q + q
      const unsigned sa = (unsigned)__cvta_generic_to_shared(ss + row * kScan32Cols + 4 * v);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa),
                   "l"(R + (int64_t)row * W + c0 + 4 * v));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  } else {
    for (int e = tid; e < NB * Q * kScan32Cols; e += blockDim.x) {
      const int row = e / kScan32Cols, c = e - row * kScan32Cols;
      const int64_t col = c0 + c < W ? c0 + c : W - 1;
      ss[e] = R[(int64_t)row * W + col];
    }
  }
  if (tid < 2 * kScan32Cols && VM) {  // steady-state inputs: the row pass's virtual rows
    const int dir = tid / kScan32Cols, c = tid - dir * kScan32Cols;
    const int64_t cc = c0 + c < W ? c0 + c : W - 1;
    es[dir][c] = dir == 0 ? Vt[cc] : Vb[cc];
  } else if (tid < 2 * kScan32Cols) {  // steady-state inputs: D20 T of row 0 / H-1
    const int dir = tid / kScan32Cols, c = tid - dir * kScan32Cols;
    const int64_t cc = c0 + c < W ? c0 + c : W - 1;
    const int64_t er = dir == 0 ? 0 : H - 1;
    const int64_t cl = cc > 0 ? cc - 1 : 0, cr = cc + 1 < W ? cc + 1 : W - 1;
    const float tl = __ldg(T + er * ldt + cl), tcv = __ldg(T + er * ldt + cc),
                tr = __ldg(T + er * ldt + cr);
    es[dir][c] = (tl - tcv) + (tr - tcv);
  }
  if (full) asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  pdl_trigger();
  if (tid < 2 * kScan32Cols) {
    const int dir = tid / kScan32Cols, c = tid - dir * kScan32Cols;
    const double e = (double)es[dir][c];
    double u[K];
#pragma unroll
    for (int i = 0; i < K; ++i) u[i] = p.Iss[i] * e;
    for (int s = 0; s < NB; ++s) {
      const int b = dir == 0 ? s : NB - 1 - s;
      float *rec = ss + (b * Q + dir * K) * kScan32Cols + c;
      double z[K];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        z[i] = (double)rec[i * kScan32Cols];
        rec[i * kScan32Cols] = (float)u[i];  // start state of band b
      }
      double un[K];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        double a = z[i];
#pragma unroll
        for (int m = 0; m < K; ++m) a = fma(p.AL[i * K + m], u[m], a);
        un[i] = a;
      }
#pragma unroll
      for (int i = 0; i < K; ++i) u[i] = un[i];
    }
  } else if (!VM && tid < 4 * kScan32Cols) {  // boundary corrections, band order
    // (V mode: the row pass computes the column direction's border rows)
    const int which = (tid - 2 * kScan32Cols) / kScan32Cols;
    const int c = tid - (2 + which) * kScan32Cols;
    double a = 0.0;
    for (int b = 0; b < NB; ++b) a += (double)ss[(b * Q + 2 * K + which) * kScan32Cols + c];
    if (c0 + c < W) Cc[(int64_t)which * W + c0 + c] = (float)a;
  }
  __syncthreads();
  // V mode: L on the band-boundary rows r1 = 64 b (b >= 1, r1 < H - 1) from the
  // start states just formed -- the apply's bottom-halo formula,
  //   L(r1) = c uf(b) + b0 V(r1) + s (c A^-1 ub(b-1) - e1 V(r1)),
  // exact L values, so their max (a hair below, for the rounding differences
  // to the apply's own walk) is a lower bound of max |L| that the apply's
  // candidate threshold can use from its first CTA on
  if (VM && p.frac > 0.0f) {
    float bmax = 0.0f;
#pragma unroll
    for (int k = 0; k < kBnd; ++k) {
      const int e = tid + k * (int)blockDim.x;
      const int b = 1 + e / kScan32Cols, c = e - (b - 1) * kScan32Cols;
      const int64_t r1 = (int64_t)b * kB32, col = c0 + c;
      if (b >= NB || r1 >= H - 1 || col >= W) continue;
      const float v = vb[k];
      float yp = 0.0f, ym = 0.0f;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        yp = fmaf(p.c[i], ss[(b * Q + i) * kScan32Cols + c], yp);
        ym = fmaf(p.ci[i], ss[((b - 1) * Q + K + i) * kScan32Cols + c], ym);
      }
      const float l = (yp + p.b0 * v + p.sign * fmaf(-p.e1, v, ym)) * p.lsc;
      bmax = fmaxf(bmax, fabsf(l));
    }
    bmax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(bmax)));
    if ((tid & 31) == 0) atomicMax(&cst->bound_bits, __float_as_uint(bmax * 0.999f));
  }
  // start states back over the carries (q < 2K), coalesced
  if (full) {
    for (int e = tid; e < NB * 2 * K * (kScan32Cols / 4); e += blockDim.x) {
      const int r2 = e / (kScan32Cols / 4), v = e - r2 * (kScan32Cols / 4);
      const int b = r2 / (2 * K), q = r2 - b * 2 * K;
      const float4 val = *reinterpret_cast<const float4 *>(ss + (b * Q + q) * kScan32Cols + 4 * v);
      *reinterpret_cast<float4 *>(R + (int64_t)(b * Q + q) * W + c0 + 4 * v) = val;
    }
  } else {
    for (int e = tid; e < NB * 2 * K * kScan32Cols; e += blockDim.x) {
      const int r2 = e / kScan32Cols, c = e - r2 * kScan32Cols;
      const int b = r2 / (2 * K), q = r2 - b * 2 * K;
      if (c0 + c < W) R[(int64_t)(b * Q + q) * W + c0 + c] = ss[(b * Q + q) * kScan32Cols + c];
    }
  }

}

// ---------------------------------------------------------------------------
// 3. walk a band: U, the column recursion in both directions, L, NMS
// ---------------------------------------------------------------------------
struct Col32Smem {
  float tile[kT32Rows][kT32Stride];  // T rows r0-2 .. r1+1, cols c0-4 .. c0+127
  float lt[kL32Rows][kT32Stride];    // U, then L, rows r0-1 .. r1 (same columns)
  int cy[kCand32], cx[kCand32];
  float cv[kCand32];
  int ccount;
  unsigned int cmax;
};

// LSC: multiply by lap_scale (sigma^2 normalisation of the scale-space stack)
template <int K, int KIND, bool LSC, bool VM>
__global__ void __launch_bounds__(kC32, 3) colapply32_kernel(
    const float *__restrict__ T, int64_t ldt, float *__restrict__ Lout, int64_t ldl,
    Col32Params p, const float *__restrict__ R, const float *__restrict__ Cc, float ctop_mul,
    CandState *__restrict__ st, int *__restrict__ gy, int *__restrict__ gx,
    float *__restrict__ gv, int gcap, const __grid_constant__ CUtensorMap tmap, int use_tma,
    int vec_out, const float *__restrict__ Vb) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem_raw);
  Col32Smem &S = *reinterpret_cast<Col32Smem *>(smem_raw + ((128u - (sbase & 127u)) & 127u));
  __shared__ __align__(8) uint64_t tbar;
  const int j = threadIdx.x, lane = j & 31, wid = j >> 5;
  const int64_t H = p.H, W = p.W;
  const int64_t c0 = (int64_t)blockIdx.x * kC32Out;
  const int64_t col = c0 - 2 + j;
  const int64_t colc = col < 0 ? 0 : (col >= W ? W - 1 : col);
  const int b = blockIdx.y;
  const int64_t r0 = (int64_t)b * kB32, r1 = r0 + kB32;
  const bool tma = use_tma && r0 >= 2 && r1 + 2 <= H && c0 >= 4 && c0 + kC32 <= W;
  if (tma) {  // one box: rows r0-2 .. r1+1, columns c0-4 .. c0+127
    if (j == 0) {
      mbar_init(&tbar, 1);
      mbar_expect_tx(&tbar, (unsigned)(kT32Rows * kT32Stride * sizeof(float)));
      tma_load_2d_hint(&S.tile[0][0], &tmap, &tbar, (int)(c0 - 4), (int)(r0 - 2),
                       l2_policy_evict_first());  // last use of T
    }
  } else {  // clamped 4-byte async copies (replicate edges)
    for (int e = j; e < kT32Rows * kT32Stride; e += kC32) {
      const int tr = e / kT32Stride, tcn = e - tr * kT32Stride;
      int64_t r = r0 - 2 + tr, c = c0 - 4 + tcn;
      c = c < 0 ? 0 : (c >= W ? W - 1 : c);
      const float *src = T + (r < 0 ? 0 : (r >= H ? H - 1 : r)) * ldt + c;
      if (VM && r >= H) src = Vb + c;  // below the image: the virtual row Vb
      const unsigned sa = (unsigned)__cvta_generic_to_shared(&S.tile[tr][tcn]);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(src));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  }
  if (j == 0) {
    S.ccount = 0;
    S.cmax = 0u;
  }
  pdl_wait();  // band start states, corrections and the CandState come from earlier kernels
  const float gbound = __uint_as_float(st->absmax_bits);  // global max so far (lower bound)
  Rec32<K, KIND> rb, rf;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    rf.u[i] = R[ridx(b, i, K, W, colc)];
    rb.u[i] = R[ridx(b, K + i, K, W, colc)];
  }
  // boundary corrections of rows 0 and H-1 where this band computes them
  const float ctop = r0 == 0 ? ctop_mul * Cc[colc] : 0.0f;
  const float cbot = (H - 1 >= r0 - 1 && H - 1 <= r1) ? Cc[W + colc] : 0.0f;
  if (tma) {
    __syncthreads();  // barrier initialised before anyone waits on it
    mbar_wait(&tbar, 0);
  } else {
    asm volatile("cp.async.wait_group 0;\n" ::);
  }
  __syncthreads();

  // ---- up: U of rows r1 .. r0-1 into lt, the backward recursion parked ----
  // T tile row of image row r: r - r0 + 2; lt row: r - r0 + 1
  const float *tcol = &S.tile[0][j + 2];
  float *lcol = &S.lt[0][j + 2];
  float park[kB32];
  float ym_below, ym_above;
  {
    float td = tcol[(kB32 + 3) * kT32Stride];  // T(r1+1)
    float tcv = tcol[(kB32 + 2) * kT32Stride]; // T(r1)
    // r = r1 (halo): y-(r1) = c A^-1 ub(r1) - e1 U(r1)
    {
      const float tu = tcol[(kB32 + 1) * kT32Stride];
      const float u = VM ? tcv
                         : lap5(tcol[(kB32 + 2) * kT32Stride - 1], tcv,
                                tcol[(kB32 + 2) * kT32Stride + 1], tu, td);
      if (!VM) lcol[(kB32 + 1) * kT32Stride] = u;
      ym_below = fmaf(-p.e1, u, rb.out(p.ci));
      td = tcv;
      tcv = tu;
    }
#pragma unroll
    for (int t = kB32 - 1; t >= 0; --t) {  // rows r0 + t
      const float tu = tcol[(t + 1) * kT32Stride];
      const float u = VM ? tcv
                         : lap5(tcol[(t + 2) * kT32Stride - 1], tcv, tcol[(t + 2) * kT32Stride + 1],
                                tu, td);
      if (!VM) lcol[(t + 1) * kT32Stride] = u;
      park[t] = rb.out(p.c);  // y-(r0 + t)
      rb.step(p, u);
      td = tcv;
      tcv = tu;
    }
    ym_above = rb.out(p.c);  // y-(r0 - 1)
    // U(r0 - 1) for the top halo row
    const float tu = tcol[0];
    if (!VM) lcol[0] = lap5(tcol[kT32Stride - 1], tcv, tcol[kT32Stride + 1], tu, td);
  }

  // ---- down: L of rows r0-1 .. r1 in place of U ----------------------------
  const float lsc = p.lsc, b0 = p.b0, sg = p.sign;
  float tmax = 0.0f;
  {
    // top halo row r0 - 1: y+(r0-1) = c A^-1 uf(r0-1) - e1 U(r0-1)
    // U of lt row q: V mode reads V straight from the tile (row q + 1)
    auto Urow = [&](int q) { return VM ? tcol[(q + 1) * kT32Stride] : lcol[q * kT32Stride]; };
    if (r0 > 0) {
      const float u = Urow(0);
      float v = fmaf(-p.e1, u, rf.out_from(p.ci, fmaf(b0, u, sg * ym_above)));
      if (r0 - 1 == H - 1) v -= cbot;
      if (LSC) v *= lsc;
      lcol[0] = v;
    }
#pragma unroll
    for (int t = 0; t < kB32; ++t) {
      const int64_t r = r0 + t;
      const float u = Urow(t + 1);
      float v = rf.out_from(p.c, fmaf(b0, u, sg * park[t]));
      rf.step(p, u);
      if (r == 0) v += ctop;
      if (r == H - 1) v -= cbot;
      if (LSC) v *= lsc;
      lcol[(t + 1) * kT32Stride] = v;
      if (r < H) tmax = fmaxf(tmax, fabsf(v));
    }
    // bottom halo row r1: y+(r1) = c . uf(r1-1) (the walk's end state)
    {
      const float u = Urow(kB32 + 1);
      float v = rf.out_from(p.c, fmaf(b0, u, sg * ym_below));
      if (r1 == H - 1) v -= cbot;
      if (LSC) v *= lsc;
      lcol[(kB32 + 1) * kT32Stride] = v;
    }
  }
  pdl_trigger();
  // columns outside the image and the two halo columns each side never count
  if (j < 2 || j >= kC32 - 2 || col >= W) tmax = 0.0f;
  tmax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(tmax)));
  if (lane == 0) atomicMax(&S.cmax, __float_as_uint(tmax));
  __syncthreads();
  // publish this CTA's max now (later CTAs prune with it) and pick up what
  // earlier CTAs published since this one started
  if (j == 0) atomicMax(&st->absmax_bits, S.cmax);
  const float gnow = fmaxf(gbound, __uint_as_float(*(volatile unsigned *)&st->absmax_bits));

  // ---- store the owned L block (rows r0 .. min(r1, H)-1, cols c0 .. c0+123)
  // fused with the strict 3x3 NMS over frac * max(this CTA's max, the global
  // max so far): a lower bound of the final threshold -> a superset
  {
    const int64_t rhi = r1 < H ? r1 : H;
    const int nrow = (int)(rhi - r0);
    const int ncol = (int)(W - c0 < kC32Out ? W - c0 : kC32Out);
    const float th = p.frac > 0.0f ? p.frac * fmaxf(__uint_as_float(S.cmax), gnow)
                                   : __int_as_float(0x7f800000);
    auto test = [&](int q, int c, float v) -> bool {  // lt row q + 1, lt column 4 + c
      const int64_t r = r0 + q, cc = c0 + c;
      if (r < 1 || r > H - 2 || cc < 1 || cc > W - 2) return false;
      const int tr = q + 1, tcn = 4 + c;
      bool gt = true, lt = true;
#pragma unroll
      for (int di = -1; di <= 1; ++di)
#pragma unroll
        for (int dj = -1; dj <= 1; ++dj) {
          if (!di && !dj) continue;
          const float w = S.lt[tr + di][tcn + dj];
          gt &= v > w;
          lt &= v < w;
        }
      // a maximum counts when L >= t, a minimum when -L >= t
      return (gt && v >= th) || (lt && -v >= th);
    };
    if ((vec_out || !Lout) && ncol == kC32Out) {  // 31 float4 per row, one row per warp
      const bool act = lane < kC32Out / 4;
      const uint64_t lpol = l2_policy_evict_first();  // L streams out (if stored)
      float *dst = Lout ? Lout + r0 * ldl + c0 + 4 * lane : nullptr;
#pragma unroll 4
      for (int q = wid; q < nrow; q += kC32 / 32) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (act) {
          v = *reinterpret_cast<const float4 *>(&S.lt[q + 1][4 + 4 * lane]);
          if (dst) st_v4_hint(dst + q * ldl, v, lpol);
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
          cand_push_warp(&S.ccount, S.cy, S.cx, S.cv, kCand32, st, gy, gx, gv, gcap, m, (int)(r0 + q), (int)(c0 + 4 * lane), vv);
        }
      }
    } else {
      for (int q = wid; q < nrow; q += kC32 / 32)
        for (int cl = 0; cl < ncol; cl += 32) {
          const int c = cl + lane;
          float v = 0.0f;
          if (c < ncol) {
            v = S.lt[q + 1][4 + c];
            if (Lout) Lout[(r0 + q) * ldl + c0 + c] = v;
          }
          const unsigned m = c < ncol && fabsf(v) >= th && test(q, c, v) ? 1u : 0u;
          const float vv[4] = {v, 0.f, 0.f, 0.f};
          cand_push_warp(&S.ccount, S.cy, S.cx, S.cv, kCand32, st, gy, gx, gv, gcap, m, (int)(r0 + q), (int)(c0 + c), vv);
        }
    }
  }
  // ---- flush the shared candidates (they passed th; the finaliser applies
  // the final threshold) ----------------------------------------------------
  __syncthreads();
  __shared__ int flush_base;
  cand_flush(S.ccount < kCand32 ? S.ccount : kCand32, S.cy, S.cx, S.cv, st, gy, gx, gv, gcap,
             &flush_base);
}

// ---------------------------------------------------------------------------
// V mode (the input V is the fp32 row pass's R(Lap5 X): no horizontal
// neighbours needed, so the carry reads V straight from global memory)
// ---------------------------------------------------------------------------
// Carry: one CTA = 128 columns x one band, 256 threads; thread (j, half)
// loads its 32 rows (16 folded pairs) with coalesced independent loads --
// no staging, no shared tile, full occupancy -- rows past H read Vb.
template <int K>
__global__ void __launch_bounds__(2 * kC32) colcarry32v_kernel(const float *__restrict__ V,
                                                             int64_t ldv, Col32Params p,
                                                             float *__restrict__ R,
                                                             float *__restrict__ Mid,
                                                             CandState *__restrict__ cs,
                                                             const float *__restrict__ Vb) {
  __shared__ float part[3 * K][kC32];
  const int j = threadIdx.x & (kC32 - 1), half = threadIdx.x >> 7;
  const int b = blockIdx.y;
  const int64_t H = p.H, W = p.W;
  const int64_t col = (int64_t)blockIdx.x * kC32 + j;
  const int64_t cc = col < W ? col : W - 1;
  const int64_t r0 = (int64_t)b * kB32;
  pdl_wait();  // V comes from the row pass
  if (blockIdx.x == 0 && blockIdx.y == 0) cand_reset(cs);
  float xa[kB32 / 4], xb[kB32 / 4];
  const int t0 = half * (kB32 / 4);
  if (r0 + kB32 <= H) {  // (CTA-uniform) a full band: pointer steps, no row checks
    const float *pa = V + (r0 + t0) * ldv + cc, *pb = V + (r0 + kB32 - 1 - t0) * ldv + cc;
#pragma unroll
    for (int t = 0; t < kB32 / 4; ++t) {
      xa[t] = __ldg(pa + t * ldv);
      xb[t] = __ldg(pb - t * ldv);
    }
  } else {  // the last band: rows past H read the virtual row Vb
    auto ld = [&](int64_t r) { return r < H ? __ldg(V + r * ldv + cc) : __ldg(Vb + cc); };
#pragma unroll
    for (int t = 0; t < kB32 / 4; ++t) {
      xa[t] = ld(r0 + t0 + t);
      xb[t] = ld(r0 + kB32 - 1 - t0 - t);
    }
  }
  pdl_trigger();
  float P[K], Q[K], Mh[K];
#pragma unroll
  for (int i = 0; i < K; ++i) P[i] = Q[i] = Mh[i] = 0.0f;
  auto run = [&](auto HALF) {  // warp-uniform halves: compile-time weight indices
    constexpr int h0 = decltype(HALF)::value * (kB32 / 4);
#pragma unroll
    for (int t = 0; t < kB32 / 4; ++t) {
      const float s = xa[t] + xb[t], d = xa[t] - xb[t];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        P[i] = fmaf(p.SP[i][h0 + t], s, P[i]);
        Q[i] = fmaf(p.SQ[i][h0 + t], d, Q[i]);
        // the bottom half-band's backward zero-state carry (the apply's
        // top-half start): xb[t] is row r0 + 63 - h0 - t = r0 + 32 + (31 - h0 - t)
        Mh[i] = fmaf(p.Wh[kB32 / 2 - 1 - h0 - t][i], xb[t], Mh[i]);
      }
    }
  };
  if (half == 0)
    run(std::integral_constant<int, 0>());
  else
    run(std::integral_constant<int, 1>());
  if (half == 1) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
      part[i][j] = P[i];
      part[K + i][j] = Q[i];
      part[2 * K + i][j] = Mh[i];
    }
  }
  __syncthreads();
  if (half == 0 && col < W) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const float Pt = P[i] + part[i][j], Qt = Q[i] + part[K + i][j];
      R[ridx(b, i, K, W, col)] = Pt + Qt;      // forward
      R[ridx(b, K + i, K, W, col)] = Pt - Qt;  // backward
      Mid[((int64_t)b * K + i) * W + col] = Mh[i] + part[2 * K + i][j];
    }
  }
}

// One 32-row half of the apply with the two directions as the lanes of
// packed FMAs (the row pass's row_walks32_pair on a tile column): step j runs
// the forward recursion at half row j and the backward one at 31 - j; steps
// 0..15 park (fwd(j), bwd(31-j)) without the b0 V term, the state pairs swap
// halves, and steps 16..31 finish (L(31-j), L(j)) from the parked halves and
// write them over V in the tile (rows still to be read lie outside the
// written middle).  In: uf / ub the half's start states; out: the end states
// (uf after the half's last row, ub = ub(first row)).
template <int K, int KIND, bool SYM, bool LSC>
__device__ __forceinline__ void col_half_pair(float *tc, int base, const Col32Params &p,
                                              float (&uf)[K], float (&ub)[K], float &tmax) {
#define TVH(q) tc[(base + (q)) * kT32Stride]
  float2 u[K], cc[K], cx[K];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    u[i] = make_float2(uf[i], ub[i]);
    cc[i] = SYM ? make_float2(p.c[i], p.c[i]) : make_float2(p.c[i], p.cs[i]);
    cx[i] = SYM ? cc[i] : make_float2(p.cs[i], p.c[i]);
  }
  const float2 p2 = make_float2(p.p, p.p), q2 = make_float2(p.q, p.q),
               nq2 = make_float2(-p.q, -p.q), b02 = make_float2(p.b0, p.b0),
               l2 = make_float2(p.lsc, p.lsc);
  auto step = [&](float2 x2) {
    if (KIND == M32_JORDAN) {
      u[0] = ffma2(p2, u[0], x2);
#pragma unroll
      for (int i = 1; i < K; ++i) u[i] = ffma2(p2, u[i], u[i - 1]);
    } else {
      const float2 ur = u[0], ui = u[1];
      u[0] = ffma2(p2, ur, ffma2(nq2, ui, x2));
      u[1] = ffma2(q2, ur, fmul2(p2, ui));
    }
  };
  constexpr int N = kB32 / 2;
  float2 pk[N / 2];
#pragma unroll
  for (int j = 0; j < N / 2; ++j) {
    const float2 x2 = make_float2(TVH(j), TVH(N - 1 - j));
    float2 o = fmul2(cc[0], u[0]);
#pragma unroll
    for (int i = 1; i < K; ++i) o = ffma2(cc[i], u[i], o);
    pk[j] = o;
    step(x2);
  }
#pragma unroll
  for (int i = 0; i < K; ++i) u[i] = make_float2(u[i].y, u[i].x);  // (bwd, fwd)
#pragma unroll
  for (int j = N / 2; j < N; ++j) {
    const int m = N - 1 - j;
    const float2 x2 = make_float2(TVH(m), TVH(j));
    float2 o = ffma2(b02, x2, pk[m]);
#pragma unroll
    for (int i = 0; i < K; ++i) o = ffma2(cx[i], u[i], o);  // (L(m), L(j))
    step(x2);
    if (LSC) o = fmul2(l2, o);
    TVH(m) = o.x;
    TVH(j) = o.y;
    tmax = fmaxf(tmax, fmaxf(fabsf(o.x), fabsf(o.y)));
  }
#pragma unroll
  for (int i = 0; i < K; ++i) {
    ub[i] = u[i].x;
    uf[i] = u[i].y;
  }
#undef TVH
}

// Apply: one CTA = 128 columns x one band; the tile holds V rows r0-1 .. r1
// (TMA box at column c0-4); L is written in place (each column is private to
// its thread), then the owned 124 x 64 block leaves fused with the 3x3 NMS.
// The band is walked in two 32-row halves so only 32 backward values are
// parked in registers: the top half's backward start comes from a local
// zero-state carry over the bottom half (ub(r0+32) = A^32 ub(r1) + sum A^t b V).
struct Col32vSmem {
  float tile[kB32 + 2][kT32Stride];  // V, then L: rows r0-1 .. r1, cols c0-4 .. c0+127
  int cy[kCand32], cx[kCand32];
  float cv[kCand32];
  int ccount;
  unsigned int cmax;
};

template <int K, int KIND, bool LSC>
__global__ void __launch_bounds__(kC32, 5) colapply32v_kernel(
    const float *__restrict__ V, int64_t ldv, float *__restrict__ Lout, int64_t ldl,
    Col32Params p, const float *__restrict__ R, const float *__restrict__ Mid,
    const float *__restrict__ Ky, CandState *__restrict__ st, int *__restrict__ gy,
    int *__restrict__ gx, float *__restrict__ gv, int gcap,
    const __grid_constant__ CUtensorMap tmap, int use_tma, int vec_out,
    const float *__restrict__ Vb) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem_raw);
  Col32vSmem &S = *reinterpret_cast<Col32vSmem *>(smem_raw + ((128u - (sbase & 127u)) & 127u));
  __shared__ __align__(8) uint64_t tbar;
  const int j = threadIdx.x, lane = j & 31, wid = j >> 5;
  const int64_t H = p.H, W = p.W;
  const int64_t c0 = (int64_t)blockIdx.x * kC32Out;
  const int64_t col = c0 - 2 + j;
  const int64_t colc = col < 0 ? 0 : (col >= W ? W - 1 : col);
  const int b = blockIdx.y;
  const int64_t r0 = (int64_t)b * kB32, r1 = r0 + kB32;
  // every full band goes by TMA: the box's out-of-frame parts (the row above
  // band 0, the row below the last band, the columns left of column 0 and
  // right of W-1) arrive zero-filled and only feed outputs that are never
  // stored or tested (the halo rows / columns outside the frame)
  const bool tma = use_tma && r1 <= H;
  if (tma) {
    if (j == 0) {
      mbar_init(&tbar, 1);
      mbar_expect_tx(&tbar, (unsigned)((kB32 + 2) * kT32Stride * sizeof(float)));
      tma_load_2d_hint(&S.tile[0][0], &tmap, &tbar, (int)(c0 - 4), (int)(r0 - 1),
                       l2_policy_evict_first());  // last use of V
    }
  } else {  // clamped 4-byte async copies; below the image the virtual row Vb
    for (int e = j; e < (kB32 + 2) * kT32Stride; e += kC32) {
      const int tr = e / kT32Stride, tcn = e - tr * kT32Stride;
      int64_t r = r0 - 1 + tr, c = c0 - 4 + tcn;
      c = c < 0 ? 0 : (c >= W ? W - 1 : c);
      const float *src = r >= H ? Vb + c : V + (r < 0 ? 0 : r) * ldv + c;
      const unsigned sa = (unsigned)__cvta_generic_to_shared(&S.tile[tr][tcn]);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(src));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  }
  if (j == 0) {
    S.ccount = 0;
    S.cmax = 0u;
  }
  pdl_wait();  // band start states, Ky and the CandState come from earlier kernels
  // lower bounds of max |L|: the band scan's boundary rows, the earlier CTAs
  // (combined only where the threshold is formed: the loads' latency hides
  // behind the walks)
  const unsigned gb_scan = st->bound_bits, gb_max = st->absmax_bits;
  Rec32<K, KIND> rf, rbt;
  float ub1[K], mid[K];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    rf.u[i] = R[ridx(b, i, K, W, colc)];
    ub1[i] = R[ridx(b, K + i, K, W, colc)];
    mid[i] = Mid[((int64_t)b * K + i) * W + colc];
  }
  const float ctop = r0 == 0 ? Ky[colc] : 0.0f;
  const float cbot = (H - 1 >= r0 - 1 && H - 1 <= r1) ? Ky[W + colc] : 0.0f;
  if (tma) {
    __syncthreads();
    mbar_wait(&tbar, 0);
  } else {
    asm volatile("cp.async.wait_group 0;\n" ::);
  }
  __syncthreads();
  float *tc = &S.tile[0][j + 2];  // tile row q <-> image row r0 - 1 + q
#define TV(q) tc[(q) * kT32Stride]
  const float b0 = p.b0, lsc = p.lsc;
  float tmax = 0.0f;
  auto fin = [&](float v) { return LSC ? v * lsc : v; };
  // rows of this band (tile rows 1 .. nval) that lie inside the image
  const int nval = (int)(H - r0 < kB32 ? H - r0 : kB32);
  // top half's backward start: A^32 ub(r1) + sum_{t<32} A^t b V(r0 + 32 + t)
  // (the sum is the carry pass's half-band record)
#pragma unroll
  for (int i = 0; i < K; ++i) {
    float a = mid[i];
#pragma unroll
    for (int m = 0; m < K; ++m) a = fmaf(p.A32[i * K + m], ub1[m], a);
    rbt.u[i] = a;
  }
  // a fresher global maximum for the NMS threshold below, loaded now so its
  // latency hides behind the walks
  const unsigned gmid = *(volatile unsigned *)&st->absmax_bits;
  // ---- top half: rows r0 .. r0+31 (and the halo row r0-1)
  float uf[K], ub[K], hf = 0.0f;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    uf[i] = rf.u[i];
    ub[i] = rbt.u[i];
    hf = fmaf(p.ci[i], uf[i], hf);  // c A^-1 uf(r0-1): the halo row's forward part
  }
  auto walk_half = [&](int base) {
    if (p.sign > 0.0f)
      col_half_pair<K, KIND, true, LSC>(tc, base, p, uf, ub, tmax);
    else
      col_half_pair<K, KIND, false, LSC>(tc, base, p, uf, ub, tmax);
  };
  walk_half(1);
  if (r0 > 0) {  // L(r0-1): y+(r0-1) = c A^-1 uf(r0-1) - e1 V(r0-1); y-(r0-1) = c ub(r0)
    const float v = TV(0);
    float a = fmaf(b0, v, hf);
#pragma unroll
    for (int i = 0; i < K; ++i) a = fmaf(p.cs[i], ub[i], a);
    TV(0) = fin(fmaf(-p.e1, v, a));
  }
  // ---- bottom half: rows r0+32 .. r1-1 (and the halo row r1)
  float ym_below;
  {
    const float v = TV(kB32 + 1);  // y-(r1) = c A^-1 ub(r1) - e1 V(r1)
    float a = 0.0f;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      ub[i] = ub1[i];
      a = fmaf(p.ci[i], ub1[i], a);
    }
    ym_below = fmaf(-p.e1, v, a);
  }
  walk_half(kB32 / 2 + 1);
  {
    const float v = TV(kB32 + 1);
    float a = fmaf(b0, v, p.sign * ym_below);
#pragma unroll
    for (int i = 0; i < K; ++i) a = fmaf(p.c[i], uf[i], a);
    TV(kB32 + 1) = fin(a);
  }
  // the border rows' terms: L(0) += Ky[0], L(H-1) -= Ky[1] (tile row r - r0 + 1)
  const bool bot = H - 1 >= r0 - 1 && H - 1 <= r1;
  if (r0 == 0) TV(1) = TV(1) + fin(ctop);
  if (bot) {
    const int q = (int)(H - 1 - r0 + 1);
    TV(q) = TV(q) - fin(cbot);
  }
  // (CTA-uniform) bands with a corrected border row or rows past H: the
  // maximum is re-taken over the final values of the band's own rows
  if (nval < kB32 || r0 == 0 || bot) {
    tmax = 0.0f;
    for (int t = 0; t < nval; ++t) tmax = fmaxf(tmax, fabsf(TV(t + 1)));
  }
#undef TV
  pdl_trigger();
  if (j < 2 || j >= kC32 - 2 || col >= W) tmax = 0.0f;
  tmax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(tmax)));
  if (lane == 0) atomicMax(&S.cmax, __float_as_uint(tmax));
  __syncthreads();
  if (j == 0) atomicMax(&st->absmax_bits, S.cmax);
  const float gnow = fmaxf(fmaxf(__uint_as_float(gb_scan), __uint_as_float(gb_max)),
                           __uint_as_float(gmid));
  {
    const int64_t rhi = r1 < H ? r1 : H;
    const int nrow = (int)(rhi - r0);
    const int ncol = (int)(W - c0 < kC32Out ? W - c0 : kC32Out);
    const float th = p.frac > 0.0f ? p.frac * fmaxf(__uint_as_float(S.cmax), gnow)
                                   : __int_as_float(0x7f800000);
    auto test = [&](int q, int c, float v) -> bool {  // tile row q + 1, tile column 4 + c
      const int64_t r = r0 + q, cc = c0 + c;
      if (r < 1 || r > H - 2 || cc < 1 || cc > W - 2) return false;
      const int tr = q + 1, tcn = 4 + c;
      bool gt = true, lt = true;
#pragma unroll
      for (int di = -1; di <= 1; ++di)
#pragma unroll
        for (int dj = -1; dj <= 1; ++dj) {
          if (!di && !dj) continue;
          const float w = S.tile[tr + di][tcn + dj];
          gt &= v > w;
          lt &= v < w;
        }
      return (gt && v >= th) || (lt && -v >= th);
    };
    if ((vec_out || !Lout) && ncol == kC32Out) {
      // (Lout null: detections only -- L never leaves the tile)
      const bool act = lane < kC32Out / 4;
      const uint64_t lpol = l2_policy_evict_first();
      float *dst = Lout ? Lout + r0 * ldl + c0 + 4 * lane : nullptr;
      bool any = true;
      if (!dst) {  // detections only: one vote over the warp's rows first
        float mx = 0.0f;
        if (act) {
#pragma unroll 4
          for (int q = wid; q < nrow; q += kC32 / 32) {
            const float4 v = *reinterpret_cast<const float4 *>(&S.tile[q + 1][4 + 4 * lane]);
            mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
          }
        }
        any = __any_sync(0xffffffffu, mx >= th);
      }
#pragma unroll 4
      for (int q = wid; any && q < nrow; q += kC32 / 32) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (act) {
          v = *reinterpret_cast<const float4 *>(&S.tile[q + 1][4 + 4 * lane]);
          if (dst) st_v4_hint(dst + q * ldl, v, lpol);
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
          cand_push_warp(&S.ccount, S.cy, S.cx, S.cv, kCand32, st, gy, gx, gv, gcap, m, (int)(r0 + q), (int)(c0 + 4 * lane), vv);
        }
      }
    } else {
      for (int q = wid; q < nrow; q += kC32 / 32)
        for (int cl = 0; cl < ncol; cl += 32) {
          const int c = cl + lane;
          float v = 0.0f;
          if (c < ncol) {
            v = S.tile[q + 1][4 + c];
            if (Lout) Lout[(r0 + q) * ldl + c0 + c] = v;
          }
          const unsigned m = c < ncol && fabsf(v) >= th && test(q, c, v) ? 1u : 0u;
          const float vv[4] = {v, 0.f, 0.f, 0.f};
          cand_push_warp(&S.ccount, S.cy, S.cx, S.cv, kCand32, st, gy, gx, gv, gcap, m, (int)(r0 + q), (int)(c0 + c), vv);
        }
    }
  }
  // (the shared candidates already passed th; the finaliser applies the final
  // threshold, so no second, fresher read of the global maximum is needed)
  __syncthreads();
  __shared__ int flush_base;
  cand_flush(S.ccount < kCand32 ? S.ccount : kCand32, S.cy, S.cx, S.cv, st, gy, gx, gv, gcap,
             &flush_base);
}

// ---------------------------------------------------------------------------
// host: modal realisation (long double), plan, launches
// ---------------------------------------------------------------------------
struct Col32Plan {
  Col32Params p;
  Hm32 hm;
  int kind;
};

// Candidate capacity of the fp32 column pass: every candidate is a strict
// 3x3 extremum of L (maxima pairwise apart, minima too: at most
// ceil(h/2) ceil(w/2) of each), so the list cannot overflow and the
// finaliser never needs L itself -- L is stored only on request.
static int64_t cand32_capacity(int64_t h, int64_t w) {
  return 2 * cdiv(h, 2) * cdiv(w, 2) + 64;
}

size_t colpass32_workspace_bytes(int64_t h, int64_t w, int k) {
  const int64_t NB = cdiv(h, kB32);
  const size_t rec = (size_t)NB * (2 * k + 2) * w * sizeof(float);
  const size_t mid = (size_t)NB * k * w * sizeof(float);  // half-band carries (V mode)
  const int64_t gcap = cand32_capacity(h, w);
  return 4096 + ((rec + 255) & ~(size_t)255) + ((mid + 255) & ~(size_t)255) +
         ((2 * w * sizeof(float) + 255) & ~(size_t)255) + (size_t)gcap * 12 + 1024;
}

static int plan32(Col32Plan *P, int64_t h, int64_t w, const IirParams &ip) {
  Modal M;
  if (!modal_realise(ip.b, ip.a, ip.K, &M)) return fail(VMF_EVALUE, "no modal realisation");
  const int k = ip.K;
  Col32Params &p = P->p;
  memset(&p, 0, sizeof(p));
  P->kind = M.kind;
  p.K = k;
  p.p = (float)M.p;
  p.q = (float)M.q;
  for (int i = 0; i < k; ++i) p.c[i] = (float)M.c[i];
  // c A^-1: solve A^T x = c
  {
    ld At[16], x[4];
    for (int i = 0; i < k; ++i)
      for (int jj = 0; jj < k; ++jj) At[i * k + jj] = M.A[jj * k + i];
    for (int i = 0; i < k; ++i) x[i] = M.c[i];
    if (!solve(At, x, k)) return fail(VMF_EVALUE, "singular modal matrix");
    ld e1 = 0;
    for (int i = 0; i < k; ++i) {
      p.ci[i] = (float)x[i];
      e1 += x[i] * M.bv[i];
    }
    p.e1 = (float)e1;
  }
  p.b0 = (float)ip.b0;
  p.sign = (float)ip.sign;
  p.H = h;
  p.W = w;
  p.NB = (int)cdiv(h, kB32);
  if (p.NB > kMaxNB32) return fail(VMF_EVALUE, "image too tall for the fp32 column pass");
  // W(t) = A^t b, folded weights
  ld Wt[kB32][4];
  {
    ld v[4], t[4];
    for (int i = 0; i < k; ++i) v[i] = M.bv[i];
    for (int tt = 0; tt < kB32; ++tt) {
      for (int i = 0; i < k; ++i) Wt[tt][i] = v[i];
      for (int i = 0; i < k; ++i) {
        t[i] = 0;
        for (int jj = 0; jj < k; ++jj) t[i] += M.A[i * k + jj] * v[jj];
      }
      memcpy(v, t, sizeof(ld) * k);
    }
  }
  for (int i = 0; i < k; ++i)
    for (int t = 0; t < kB32 / 2; ++t) {
      p.SP[i][t] = (float)(0.5L * (Wt[t][i] + Wt[kB32 - 1 - t][i]));
      p.Wh[t][i] = (float)Wt[t][i];
      p.SQ[i][t] = (float)(0.5L * (Wt[kB32 - 1 - t][i] - Wt[t][i]));
    }
  {
    ld A32[16];
    matpow(M.A, kB32 / 2, A32, k);
    for (int i = 0; i < k * k; ++i) p.A32[i] = (float)A32[i];
    for (int i = 0; i < k; ++i) p.cs[i] = (float)(ip.sign * M.c[i]);
  }
  ld AL[16];
  matpow(M.A, kB32, AL, k);
  for (int i = 0; i < k * k; ++i) p.AL[i] = (double)AL[i];

  {
    ld IA[16], y[4];
    for (int i = 0; i < k; ++i) {
      for (int jj = 0; jj < k; ++jj) IA[i * k + jj] = (i == jj ? 1 : 0) - M.A[i * k + jj];
      y[i] = M.bv[i];
    }
    if (!solve(IA, y, k)) return fail(VMF_EVALUE, "pole on the unit circle");
    for (int i = 0; i < k; ++i) p.Iss[i] = (double)y[i];
  }
  // boundary-correction weights h(m) = c A^(m-1) b until the tail is
  // negligible (sum of |h| beyond Mh < 1e-9 of the total), at most H-1
  {
    std::vector<ld> hv(1, 0);
    ld v[4], t[4], tot = 0;
    for (int i = 0; i < k; ++i) v[i] = M.bv[i];
    const int64_t mmax = h - 1 < kHm32Max ? h - 1 : kHm32Max;
    for (int64_t m = 1; m <= mmax; ++m) {
      ld hm = 0;
      for (int i = 0; i < k; ++i) hm += M.c[i] * v[i];
      hv.push_back(hm);
      tot += fabsl(hm);
      for (int i = 0; i < k; ++i) {
        t[i] = 0;
        for (int jj = 0; jj < k; ++jj) t[i] += M.A[i * k + jj] * v[jj];
      }
      memcpy(v, t, sizeof(ld) * k);
    }
    // the tail beyond what h() holds must be negligible too (else the
    // caller keeps the fp64 pass)
    if (mmax == kHm32Max) {
      ld rest = 0;
      for (int64_t m = kHm32Max + 1; m <= kHm32Max + 4096 && m < h; ++m) {
        ld hm = 0;
        for (int i = 0; i < k; ++i) hm += M.c[i] * v[i];
        rest += fabsl(hm);
        for (int i = 0; i < k; ++i) {
          t[i] = 0;
          for (int jj = 0; jj < k; ++jj) t[i] += M.A[i * k + jj] * v[jj];
        }
        memcpy(v, t, sizeof(ld) * k);
      }
      if (rest >= 1e-9L * tot) return fail(VMF_EVALUE, "impulse response too long for h()");
    }
    int64_t Mh = (int64_t)hv.size() - 1;
    ld tail = 0;
    while (Mh > 1 && tail + fabsl(hv[Mh]) < 1e-9L * tot) tail += fabsl(hv[Mh--]);
    p.Mh = (int)Mh;
    memset(&P->hm, 0, sizeof(P->hm));
    for (int64_t m = 1; m <= Mh; ++m) P->hm.h[m] = (float)hv[m];
  }
  return VMF_OK;
}

template <int K, int KIND, bool VM>
static int launch32(const float *T, int64_t ldt, float *L, int64_t ldl, const Col32Plan &P,
                    const Col32VMode &vm, int32_t *det_yx, float *det_val, int64_t cap,
                    int64_t *n_det_dev, float *thr_dev, void *ws, cudaStream_t st) {
  const Col32Params &p = P.p;
  const int64_t h = p.H, w = p.W;
  char *base = (char *)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  CandState *cs = (CandState *)base;
  char *q = base + 4096;
  float *R = (float *)q;
  q += ((size_t)p.NB * (2 * K + 2) * w * sizeof(float) + 255) & ~(size_t)255;
  float *Mid = (float *)q;
  q += ((size_t)p.NB * K * w * sizeof(float) + 255) & ~(size_t)255;
  float *Cc = (float *)q;
  q += (2 * w * sizeof(float) + 255) & ~(size_t)255;
  const int64_t gcap = cand32_capacity(h, w);
  int *gy = (int *)q;
  int *gx = gy + gcap;
  float *gv = (float *)(gx + gcap);
  {
    Launch g(K_COL_CARRY, st);
    CUtensorMap cmap;
    memset(&cmap, 0, sizeof(cmap));
    const int ctma = make_tmap_2d_f32(&cmap, T, h, w, ldt, kCarryStride, kCarryRows) &&
                     !getenv("VMF_NO_TMA");
    cudaGetLastError();
    const int csm = kCarryRows * kCarryStride * (int)sizeof(float) + 128;
    static PerDevice attr;
    if (attr.first())
      cudaFuncSetAttribute(colcarry32_kernel<K, VM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           csm);
    if (VM)
      launch_pdl(colcarry32v_kernel<K>, dim3((unsigned)cdiv(w, kC32), (unsigned)p.NB),
                 dim3(2 * kC32), 0, st, T, ldt, p, R, Mid, cs, vm.vb);
    else
      launch_pdl(colcarry32_kernel<K, VM>, dim3((unsigned)cdiv(w, kC32), (unsigned)p.NB),
                 dim3(2 * kC32), csm, st, T, ldt, p, R, P.hm, cmap, ctma, cs, vm.vb);
  }
  {
    Launch g(K_COL_SCAN, st);
    // records, then (V mode) the last CTA's row-filter scratch
    const int ssm = p.NB * (2 * K + 2) * kScan32Cols * (int)sizeof(float);
    static PerDevice attr;
    if (attr.first())
      cudaFuncSetAttribute(colscan32_kernel<K, VM>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    launch_pdl(colscan32_kernel<K, VM>, dim3((unsigned)cdiv(w, kScan32Cols)), dim3(256), ssm, st,
               T, ldt, p, R, Cc, vm.vt, vm.vb, cs);
  }
  if (VM) {
    Launch g(K_COL_APPLY, st);
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    const int use_tma = make_tmap_2d_f32(&tmap, T, h, w, ldt, kT32Stride, kB32 + 2) &&
                        !getenv("VMF_NO_TMA");
    cudaGetLastError();
    const int sm = (int)sizeof(Col32vSmem) + 128;
    static PerDevice attr;
    if (attr.first()) {
      cudaFuncSetAttribute(colapply32v_kernel<K, KIND, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      cudaFuncSetAttribute(colapply32v_kernel<K, KIND, false>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    }
    auto kern = p.lsc == 1.0f ? colapply32v_kernel<K, KIND, false> : colapply32v_kernel<K, KIND, true>;
    launch_pdl(kern, dim3((unsigned)cdiv(w, kC32Out), (unsigned)p.NB), dim3(kC32), sm, st, T, ldt,
               L, ldl, p, (const float *)R, (const float *)Mid, vm.ky, cs, gy, gx, gv, (int)gcap,
               tmap, use_tma, (int)(L && ldl % 4 == 0 && (uintptr_t)L % 16 == 0), vm.vb);
  } else {
    Launch g(K_IIR_COLS_FUSED, st);
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    const int use_tma = make_tmap_2d_f32(&tmap, T, h, w, ldt, kT32Stride, kT32Rows) &&
                        !getenv("VMF_NO_TMA");
    cudaGetLastError();
    const int sm = (int)sizeof(Col32Smem) + 128;
    static PerDevice attr;
    if (attr.first()) {
      cudaFuncSetAttribute(colapply32_kernel<K, KIND, true, VM>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      cudaFuncSetAttribute(colapply32_kernel<K, KIND, false, VM>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    }
    auto kern = p.lsc == 1.0f ? colapply32_kernel<K, KIND, false, VM>
                              : colapply32_kernel<K, KIND, true, VM>;
    // border terms of rows 0 / H-1: T mode adds sign * Cc (T is row-filtered
    // already); V mode adds the row-filtered Ky (sign inside)
    launch_pdl(kern, dim3((unsigned)cdiv(w, kC32Out), (unsigned)p.NB), dim3(kC32), sm, st, T, ldt,
               L, ldl, p, (const float *)R, (const float *)(VM ? vm.ky : Cc), VM ? 1.0f : p.sign,
               cs, gy, gx, gv, (int)gcap, tmap, use_tma,
               (int)(L && ldl % 4 == 0 && (uintptr_t)L % 16 == 0), vm.vb);
  }
  if (p.frac > 0.0f)
    colfinal_launch(cs, gy, gx, gv, gcap, L, ldl, h, w, p.frac, det_yx, det_val, cap, n_det_dev,
                    thr_dev, st);
  return cuda_status("fp32 column pass");
}

static int get_plan32(int64_t h, int64_t w, const IirParams &ip, Col32Plan *out) {
  static PlanCache<Col32Plan> cache;
  std::vector<unsigned char> key;
  key_add(key, h);
  key_add(key, w);
  key_add(key, ip.K);
  key_add(key, ip.b0);
  key_add(key, ip.sign);
  key_add(key, ip.b, sizeof(double) * ip.K);
  key_add(key, ip.a, sizeof(double) * ip.K);
  if (cache.get(key, out)) return VMF_OK;
  const int rc = plan32(out, h, w, ip);
  if (rc) return rc;
  cache.put(key, *out);
  return VMF_OK;
}

bool colpass32_supported(int64_t h, int64_t w, const IirParams &ip) {
  if (getenv("VMF_NO_COLPASS32") || h < 64 || w < 1 || cdiv(h, kB32) > kMaxNB32) return false;
  Modal M;
  if (!modal_realise(ip.b, ip.a, ip.K, &M)) return false;
  static Col32Plan tmp;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  return get_plan32(h, w, ip, &tmp) == VMF_OK;  // else the caller keeps the fp64 pass
}

int colpass32_run(const float *T, int64_t ldt, float *L, int64_t ldl, const IirParams &ip,
                  int64_t h, int64_t w, float lap_scale, float frac, int32_t *det_yx,
                  float *det_val, int64_t cap, int64_t *n_det_dev, float *thr_dev, void *ws,
                  size_t ws_bytes, cudaStream_t st, const Col32VMode *vmode) {
  const size_t need = colpass32_workspace_bytes(h, w, ip.K);
  if (!ws || ws_bytes < need)
    return fail(VMF_EVALUE, "fp32 column-pass workspace too small: %zu < %zu bytes", ws_bytes,
                need);
  static Col32Plan run;  // (large: not on the stack)
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  const int rc = get_plan32(h, w, ip, &run);
  if (rc) return rc;
  run.p.lsc = lap_scale;
  run.p.frac = frac;
  const Col32VMode none = {};
  const Col32VMode &vm = vmode ? *vmode : none;
#define VMF_L32(KK, KD)                                                                       \
  (vmode ? launch32<KK, KD, true>(T, ldt, L, ldl, run, vm, det_yx, det_val, cap, n_det_dev,  \
                                  thr_dev, ws, st)                                            \
         : launch32<KK, KD, false>(T, ldt, L, ldl, run, vm, det_yx, det_val, cap, n_det_dev, \
                                   thr_dev, ws, st))
  if (run.kind == M32_CPAIR) return VMF_L32(2, M32_CPAIR);
  switch (ip.K) {
    case 2: return VMF_L32(2, M32_JORDAN);
    case 3: return VMF_L32(3, M32_JORDAN);
    case 4: return VMF_L32(4, M32_JORDAN);
  }
#undef VMF_L32
  return fail(VMF_EVALUE, "fp32 column pass supports K = 2..4, got %d", ip.K);
}

}  // namespace vmf
