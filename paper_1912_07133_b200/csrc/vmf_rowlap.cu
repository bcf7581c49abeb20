// vmf_rowlap.cu -- the first pass of the fp32 "Laplacian-first" path:
// V = R(U0), U0 = 5-point Laplacian of the input frame X, R the row filter
// (iir_rows, engine.py:137-155 / kernel 65-102) in fp32 modal form.
//
// Why.  The reference computes T = R X, B = C T and L = Lap5_rep(B)
// (engine.py:205-228, blob.py:161).  On the replicate-extended frame the three
// operators commute, so L = C R Lap5(X_ext) plus four border terms
// (tools/experiments/lapfirst_2d.py derives and checks them):
//   * left / right of the image Lap5(X_ext) is D02 X of column 0 / W-1,
//     constant along the row: the steady-state starts eL(r), eR(r) of R;
//   * above / below it is D20 X of row 0 / H-1 (zero past the columns):
//     the column pass starts from Vt = R0(D20 X(0, .)) / Vb (zero starts);
//   * L(r, 0) += C[dxl](r), dxl(r) = s sum_m h(m) (X(r, m) - X(r, m-1)) and
//     L(r, W-1) -= C[dxr](r): folded into V(r, 0) / V(r, W-1) (C is linear);
//   * L(0, c) += R[dyt](c), L(H-1, c) -= R[dyb](c): column sums of X's first
//     differences (the column carry pass), row-filtered by rowfix_kernel.
// Every quantity is then a Laplacian-size difference, so fp32 rounding is
// relative to |L| and the modal recursion (vmf_modal32.cuh) runs in fp32:
// the prototype's error is 1e-6 of max|L|, below the fp64 path's 3e-6..1e-5
// (which rounds T to fp32), at every config scale.
//
// Kernel: persistent CTAs own contiguous rows; thread = 32-sample chunk of
// the row (W = 32 C, C <= 256).  Input rows arrive by TMA (128-byte
// swizzled [C][32] boxes) into a ring of 4 buffers (rows r-1, r, r+1 and the
// prefetch of r+2); per row: U0 in registers, zero-state chunk carries by
// folded pairs, a Kogge-Stone chunk scan per direction (one warp each), the
// backward walk parked in registers, the forward walk writing V into one of
// two output buffers that leave by TMA store.
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "plan_cache.hpp"
#include "vmf_common.cuh"
#include "vmf_modal32.cuh"
#include "vmf_prof.cuh"
#include "vmf_rowlap.cuh"
#include "vmf_tma.cuh"

namespace vmf {

#ifndef VMF_ABL
#define VMF_ABL 0
#endif
#ifndef VMF_TIMELINE
#define VMF_TIMELINE 0
#endif
#if VMF_TIMELINE  // per-CTA / per-row globaltimer stamps (tools/row_ablation.py)
__device__ unsigned long long g_tl[4096];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TL(idx) \
  do {          \
    if (threadIdx.x == 0) g_tl[(idx)] = gtime(); \
  } while (0)
#define TLROW(i, ph) \
  do {               \
    if (blockIdx.x < 8 && (i) < 16) TL(2560 + (blockIdx.x * 16 + (i)) * 4 + (ph)); \
  } while (0)
#else
#define TL(idx) \
  do {          \
  } while (0)
#define TLROW(i, ph) \
  do {               \
  } while (0)
#endif
constexpr int kRLMaxC = 256;   // W <= 8192
constexpr int kRLBufs = 3;     // input ring: rows r-1, r, r+1 (r+2 lands in r-1's slot)

// TMA SWIZZLE_128B layout of a [C][32] fp32 row (see vmf_rowpass.cu)
struct SwzRow32 {
  char *base;
  __device__ __forceinline__ int off(int c, int q) const { return c * 128 + ((q ^ (c & 7)) << 4); }
  __device__ __forceinline__ float4 ld4(int c, int q) const {
    return *reinterpret_cast<const float4 *>(base + off(c, q));
  }
  __device__ __forceinline__ void st4(int c, int q, float4 v) const {
    *reinterpret_cast<float4 *>(base + off(c, q)) = v;
  }
  __device__ __forceinline__ float ld(int n) const {
    return *reinterpret_cast<const float *>(base + off(n >> 5, (n >> 2) & 7) + 4 * (n & 3));
  }
};

__device__ __forceinline__ int hidx(int n) { return n + (n >> 5); }  // padded h() copy

// ---------------------------------------------------------------------------
// the border kernel (every scale): the column direction's border sums,
// straight from the frame (column stage, modal fp32), in 64-row segments so
// the frame edge is covered by ~1k short CTAs:
//   Dy[0][c] = s_C sum_{m>=1} h_C(m) G(m, c),  Dy[1][c] = sum_{m>=1} h_C(m) G(H-m, c),
//   G(m, c) = X(m, c) - X(m-1, c),  h_C(m) = c A^(m-1) b.
// Segment k covers m = m0 .. m0+63 (m0 = 1 + 64 k): its share is
// (c A^(m0-1)) . sum_t A^t b G(m0 + t), the inner sum a zero-state
// recursion; S[which][k][c] holds the shares (summed in k order by the edge
// CTAs).  The last ns CTA rows compute each scale's row-direction chunk
// vectors vl(c) = c A^(32 c), vr(c) = c A^(W - 32 c - 33) (fp64 powers).
// It reads only X, so it runs first; the row pass depends on it.
// ---------------------------------------------------------------------------
constexpr int kSeg = 64;

template <int K, int KIND>
__global__ void __launch_bounds__(128, 7) sweep_border_kernel(const __grid_constant__ BorderMulti bm,
                                                           const float *__restrict__ X,
                                                           int64_t ldx, int64_t H, int64_t W,
                                                           SweepOut out) {
  // the frame may come from the kernel just before this one (the row pass
  // after this kernel then reads it with no wait of its own: this wait covers it)
  pdl_wait();
  int y = blockIdx.y;
  if (y >= 2 * bm.maxseg) {  // chunk-vector rows: y = scale
    y -= 2 * bm.maxseg;
    const BorderScale &b = bm.s[y];
    float *vlr = out.E(y) + kExVlr * W;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < b.C; c += gridDim.x * blockDim.x) {
      // vl = c_r A32^c; vr = ci A32^(C-1-c): binary powers in fp64
      double Pw[16], R[16], T[16];
      auto power = [&](int e) {
        for (int i = 0; i < K * K; ++i) {
          Pw[i] = b.A32[i];
          R[i] = (i % (K + 1) == 0) ? 1.0 : 0.0;
        }
        while (e > 0) {
          if (e & 1) {
            for (int i = 0; i < K; ++i)
              for (int jj = 0; jj < K; ++jj) {
                double a = 0.0;
                for (int m = 0; m < K; ++m) a = fma(R[i * K + m], Pw[m * K + jj], a);
                T[i * K + jj] = a;
              }
            for (int i = 0; i < K * K; ++i) R[i] = T[i];
          }
          for (int i = 0; i < K; ++i)
            for (int jj = 0; jj < K; ++jj) {
              double a = 0.0;
              for (int m = 0; m < K; ++m) a = fma(Pw[i * K + m], Pw[m * K + jj], a);
              T[i * K + jj] = a;
            }
          for (int i = 0; i < K * K; ++i) Pw[i] = T[i];
          e >>= 1;
        }
      };
      power(c);
      for (int jj = 0; jj < K; ++jj) {
        double a = 0.0;
        for (int i = 0; i < K; ++i) a = fma((double)b.cr[i], R[i * K + jj], a);
        vlr[c * 8 + jj] = (float)a;
      }
      power(b.C - 1 - c);
      for (int jj = 0; jj < K; ++jj) {
        double a = 0.0;
        for (int i = 0; i < K; ++i) a = fma((double)b.ci[i], R[i * K + jj], a);
        vlr[c * 8 + 4 + jj] = (float)a;
      }
    }
    return;
  }
  // segment k of side `which` for EVERY scale whose border reaches it: the
  // rows are loaded once, each scale runs its own recursion over them
  const int which = y / bm.maxseg, k = y % bm.maxseg;
  const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t cc = col < W ? col : W - 1;
  const int m0 = 1 + kSeg * k;
  const int n = (bm.maxMh - m0 + 1) < kSeg ? (bm.maxMh - m0 + 1) : kSeg;  // m = m0 .. m0+n-1
  // top: xs[t] = X(m0 - 1 + t); bottom: xs[t] = X(H - m0 - t).  The segment
  // goes in two 32-row halves (t = 32..64, then 0..32), each loaded whole
  // before the recursions (independent loads), every scale's state carried
  // across: 33 staged rows keep the kernel at 72 registers, so the ~1k CTAs
  // are one wave (the whole segment staged took 96 registers: 1.25 waves)
  constexpr int kH = kSeg / 2;
  float xs[kH + 1];
  const float *Xc = X + cc;
  // rows r(t) = r0 + dir t, t = 0..n; the common segment (whole, inside the
  // frame) walks one pointer by a 32-bit stride, the rest clamps per row
  const int64_t r0 = which == 0 ? m0 - 1 : H - m0;
  const int64_t rend = which == 0 ? r0 + n : r0 - n;
  const bool fast =
      n == kSeg && r0 >= 0 && r0 < H && rend >= 0 && rend < H && (int64_t)kSeg * ldx < (1 << 29);
  Rec32<K, KIND> u[kMaxScales];
#pragma unroll
  for (int s = 0; s < kMaxScales; ++s)
#pragma unroll
    for (int i = 0; i < K; ++i) u[s].u[i] = 0.0f;
#pragma unroll
  for (int hh = 1; hh >= 0; --hh) {
    const int t0 = kH * hh;
    if (fast) {
      const int step = which == 0 ? (int)ldx : -(int)ldx;
      const float *p = Xc + r0 * ldx + (int64_t)t0 * step;
#pragma unroll
      for (int t = 0; t <= kH; ++t) xs[t] = __ldg(p + t * step);
    } else {
#pragma unroll
      for (int t = 0; t <= kH; ++t) {  // t > n repeats row n: G = 0 there
        const int tt = t0 + t < n ? t0 + t : n;
        const int64_t r = which == 0 ? m0 - 1 + tt : H - m0 - tt;
        xs[t] = __ldg(Xc + (r < 0 ? 0 : (r >= H ? H - 1 : r)) * ldx);
      }
    }
#pragma unroll
    for (int s = 0; s < kMaxScales; ++s) {
      if (s >= bm.ns) break;
      const BorderScale &b = bm.s[s];
      if (k >= b.sv.nseg) continue;
      const int ns_ = (b.sv.Mh - m0 + 1) < kSeg ? (b.sv.Mh - m0 + 1) : kSeg;  // this scale's rows
      // G(m0 + t): top X(m0+t) - X(m0+t-1) = xs[t+1] - xs[t]; bottom
      // X(H-m0-t) - X(H-m0-t-1) = -(xs[t+1] - xs[t]): the sign goes on the share.
      // Steps t >= ns_ see G = 0 on a zero state.
      if (ns_ == kSeg) {
#pragma unroll
        for (int t = kH - 1; t >= 0; --t) u[s].step(b, xs[t + 1] - xs[t]);
      } else {
#pragma unroll
        for (int t = kH - 1; t >= 0; --t)
          u[s].step(b, t0 + t < ns_ ? xs[t + 1] - xs[t] : 0.0f);
      }
    }
  }
#pragma unroll
  for (int s = 0; s < kMaxScales; ++s) {
    if (s >= bm.ns) break;
    const BorderScale &b = bm.s[s];
    const int nseg = b.sv.nseg;
    if (k >= nseg) continue;
    float v = u[s].out(b.sv.v[k]);
    v *= which == 0 ? b.sign : -1.0f;
    if (col < W) out.E(s)[kExS * W + ((int64_t)which * nseg + k) * W + col] = v;
  }
}

// ---------------------------------------------------------------------------
// the row pass (every scale)
// ---------------------------------------------------------------------------
// Left / right border terms of one row for one scale: dxl = s sum_{n>=1}
// h(n) G(n), dxr = sum_{m>=1} h(m) G(W-m), G(n) = X(n) - X(n-1).  Per chunk
// (samples n = n0+1 .. n0+32) the sums are modal: h(n0+1+t) = (c A^n0) A^t b,
// h(W-n0-1-t) = (c A^(W-n0-33)) A^(31-t) b, so a chunk forms two zero-state
// sums with the uniform weights A^t b (g: its first differences) and dots
// them with its vectors vl, vr (the border kernel's table); chunks farther
// than Mh from an edge contribute nothing measurable and skip.
template <int K, int KIND>
__device__ __forceinline__ void dx_chunk(const RowLapParams &p, const RC32<K> &rc,
                                         const float *vlr, const float (&g)[kRChunk], float &pl,
                                         float &pr) {
  const int c = threadIdx.x;
  const int n0 = c * kRChunk;
  const int W = (int)p.W, Mh = p.Mh, C = p.C;
  pl = pr = 0.0f;
  const bool L = c < C && n0 < Mh, Rr = c < C && n0 + kRChunk >= W - Mh;
  if (L || Rr) {
    // zl = sum_t A^t b g_t (recursion from t = 31 down), zr = sum_t A^(31-t) b g_t;
    // a chunk near one edge only forms that side's sum
    if (L) {
      float v[K];
#pragma unroll
      for (int i = 0; i < K; ++i) v[i] = __ldg(vlr + c * 8 + i);  // (issued before the recursion)
      Rec32<K, KIND> z;
#pragma unroll
      for (int i = 0; i < K; ++i) z.u[i] = 0.0f;
#pragma unroll
      for (int t = 0; t < kRChunk; ++t) z.step(rc, g[kRChunk - 1 - t]);
#pragma unroll
      for (int i = 0; i < K; ++i) pl = fmaf(v[i], z.u[i], pl);
    }
    if (Rr) {
      float v[K];
#pragma unroll
      for (int i = 0; i < K; ++i) v[i] = __ldg(vlr + c * 8 + 4 + i);
      Rec32<K, KIND> z;
#pragma unroll
      for (int i = 0; i < K; ++i) z.u[i] = 0.0f;
#pragma unroll
      for (int t = 0; t < kRChunk; ++t) z.step(rc, g[t]);
#pragma unroll
      for (int i = 0; i < K; ++i) pr = fmaf(v[i], z.u[i], pr);
    }
  }
}

__device__ __forceinline__ void warp_sum2(float &a, float &b) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
}

// Grid: row CTAs (contiguous rows each) + one edge CTA per scale (the last
// ns): the virtual rows Vt / Vb and the column direction's border rows
// Ky = R_ss(Dy) of that scale (four single-row filters).  Per row, U = Lap5 X
// is formed once and every scale's carries go before one barrier, the 2 ns
// chunk scans share the warps, and each scale's walks write its V row.
template <int K, int KIND>
__global__ void __maxnreg__(168) sweep_rows_kernel(  // (3 CTAs of 128 threads per SM)
    const __grid_constant__ CUtensorMap xmap, const __grid_constant__ RowLapMulti rm,
    const SweepOut out) {
  extern __shared__ __align__(1024) unsigned char smem_rl[];
  __shared__ __align__(8) uint64_t bar[kRLBufs];
  __shared__ float red[kMaxScales][16], e2[2], dx2[kMaxScales][2];
  const int C = rm.C, c = threadIdx.x, nwarp = (int)(blockDim.x >> 5), lane = c & 31;
  const int ns = rm.ns;
  const bool live = c < C;  // the block is whole warps; threads c >= C carry no chunk
  const int rowbytes = C * 128;                // one row's TMA box
  const int rowb = (rowbytes + 1023) & ~1023;  // slot spacing: SWIZZLE_128B needs 1024-byte bases
  const unsigned sb = (unsigned)__cvta_generic_to_shared(smem_rl);
  char *xbuf = reinterpret_cast<char *>(smem_rl) + ((1024u - (sb & 1023u)) & 1023u);
  float *cfb = reinterpret_cast<float *>(xbuf + kRLBufs * rowb);  // [ns][2][blockDim][K]
  // every scale's parameters in shared memory: the scale loops index them at
  // run time (broadcast LDS instead of constant-cache misses)
  RowLapParams *sp = reinterpret_cast<RowLapParams *>(cfb + (size_t)rm.ns * 2 * blockDim.x * K);
  {
    // 16-byte words: a divergent constant-bank read costs one transaction per
    // distinct address, so wide words mean fewer of them
    static_assert(sizeof(RowLapParams) % 16 == 0, "RowLapParams: whole 16-byte words");
    const int nw = (int)(rm.ns * sizeof(RowLapParams) / sizeof(int4));
    const int4 *src = reinterpret_cast<const int4 *>(&rm.s[0]);
    int4 *dst = reinterpret_cast<int4 *>(sp);
    for (int e = threadIdx.x; e < nw; e += blockDim.x) dst[e] = src[e];
  }
  auto cfs = [&](int s) { return cfb + (size_t)s * 2 * blockDim.x * K; };
  auto cbs = [&](int s) { return cfb + (size_t)(2 * s + 1) * blockDim.x * K; };
  const int64_t H = rm.H;
  const int W = (int)rm.W;
  const int nrowctas = (int)gridDim.x - ns;
  const bool edge = (int)blockIdx.x >= nrowctas;
  const int64_t rlo = edge ? 0 : (int64_t)blockIdx.x * rm.rows_per;
  const int64_t rhi = edge ? 0 : (rlo + rm.rows_per < H ? rlo + rm.rows_per : H);
  const int nrows = (int)(rhi - rlo);
  auto issue_row = [&](int s, int64_t r) {
    mbar_expect_tx(&bar[s], (unsigned)rowbytes);
    tma_load_3d_hint(xbuf + s * rowb, &xmap, &bar[s], 0, 0, (int)r, l2_policy_evict_first());
  };
  auto clampr = [&](int64_t r) { return r < 0 ? (int64_t)0 : (r >= H ? H - 1 : r); };
  if (c == 0) {
    for (int s = 0; s < kRLBufs; ++s) mbar_init(&bar[s], 1);
    if (edge) {
      issue_row(0, 0);
      issue_row(1, H - 1);
    } else {
      for (int j = 0; j < kRLBufs && j <= nrows + 1; ++j) issue_row(j, clampr(rlo - 1 + j));
    }
  }
  __syncthreads();
  // the border kernel (this grid's predecessor) wrote the chunk vectors and
  // segment shares; the previous scale's column pass may still read V
  TL(2048 + (blockIdx.x & 511));
  pdl_wait();
  TL(blockIdx.x & 1023);
  float U[kRChunk], V[kRChunk], X[kRChunk];
  auto load_chunk = [&](int sl, float (&o)[kRChunk]) {
    const SwzRow32 r{xbuf + sl * rowb};
#pragma unroll
    for (int q = 0; q < kRChunk / 4; ++q) {
      const float4 v = live ? r.ld4(c, q) : make_float4(0.f, 0.f, 0.f, 0.f);
      o[4 * q] = v.x;
      o[4 * q + 1] = v.y;
      o[4 * q + 2] = v.z;
      o[4 * q + 3] = v.w;
    }
  };
  auto halos = [&](int sl, const float (&x)[kRChunk], float &xl, float &xr) {
    const SwzRow32 r{xbuf + sl * rowb};
    xl = c > 0 && live ? r.ld(c * kRChunk - 1) : x[0];
    xr = c < C - 1 ? r.ld(c * kRChunk + kRChunk) : x[kRChunk - 1];
  };
  // border partials of all scales (first differences g of this thread's
  // chunk), warp-reduced into red[s][warp] / red[s][8 + warp]
  auto dx_all = [&](const float (&x)[kRChunk], float xr) {
    float g[kRChunk];
#pragma unroll
    for (int t = 0; t < kRChunk; ++t) g[t] = (t < kRChunk - 1 ? x[t + 1] : xr) - x[t];
    const int cw0 = c & ~31;  // the warp's first chunk
    for (int s = 0; s < ns; ++s) {
      float pl = 0.0f, pr = 0.0f;
      const int Mh = sp[s].Mh;
      // (warp-uniform) only warps with a chunk within Mh of an edge contribute
      if (kRChunk * cw0 < Mh || kRChunk * (cw0 + 32) >= W - Mh) {
        dx_chunk<K, KIND>(sp[s], RC32<K>(sp[s]), out.E(s) + kExVlr * W, g, pl, pr);
        warp_sum2(pl, pr);
      }
      if (lane == 0) {
        red[s][c >> 5] = pl;
        red[s][8 + (c >> 5)] = pr;
      }
    }
  };
  auto reduce_dx = [&]() {  // (thread 0, after the barrier that follows dx_all)
    for (int s = 0; s < ns; ++s) {
      float a = 0.0f, b = 0.0f;
      for (int w = 0; w < nwarp; ++w) {
        a += red[s][w];
        b += red[s][8 + w];
      }
      dx2[s][0] = sp[s].sign * a;
      dx2[s][1] = b;
    }
  };

  if (edge) {
    const int s = (int)blockIdx.x - nrowctas;
    const RowLapParams &p = sp[s];
    float *E = out.E(s);
    float *cf = cfs(0), *cb = cbs(0);
    // virtual rows: Vt / Vb = R0(D20 X) of row 0 / H-1 (zero starts) with
    // that row's left / right border terms
    for (int which = 0; which < 2; ++which) {
      mbar_wait(&bar[which], 0);
      float xl, xr;
      load_chunk(which, X);
      halos(which, X, xl, xr);
#pragma unroll
      for (int t = 0; t < kRChunk; ++t) {
        const float l = t ? X[t - 1] : xl, r = t < kRChunk - 1 ? X[t + 1] : xr;
        U[t] = (l - X[t]) + (r - X[t]);
      }
      {
        float g[kRChunk];
#pragma unroll
        for (int t = 0; t < kRChunk; ++t) g[t] = (t < kRChunk - 1 ? X[t + 1] : xr) - X[t];
        float pl, pr;
        dx_chunk<K, KIND>(p, RC32<K>(p), E + kExVlr * W, g, pl, pr);
        warp_sum2(pl, pr);
        if (lane == 0) {
          red[0][c >> 5] = pl;
          red[0][8 + (c >> 5)] = pr;
        }
      }
      if (c == 0) e2[0] = e2[1] = 0.0f;
      row_carry32<K, KIND>(RC32<K>(p), U, cf, cb);
      __syncthreads();
      if (c == 0) {
        float a = 0.0f, b = 0.0f;
        for (int w = 0; w < nwarp; ++w) {
          a += red[0][w];
          b += red[0][8 + w];
        }
        dx2[0][0] = p.sign * a;
        dx2[0][1] = b;
      }
      row_scan_walk32<K, KIND>(p, U, V, cf, cb, e2, dx2[0]);
      float *dst = E + (which == 0 ? kExVt : kExVb) * W;
      if (live) {
#pragma unroll
        for (int q = 0; q < kRChunk / 4; ++q)
          *reinterpret_cast<float4 *>(dst + c * kRChunk + 4 * q) =
              make_float4(V[4 * q], V[4 * q + 1], V[4 * q + 2], V[4 * q + 3]);
      }
      __syncthreads();
    }
    // border rows: Ky = R_ss(dy), dy = the border kernel's segment shares
    float *rowp = reinterpret_cast<float *>(xbuf);  // (the input slots are idle now)
    const int nsg = p.nseg;
    for (int which = 0; which < 2; ++which) {
      // W <= 32 blockDim columns per thread, in groups of 8, each summed in k
      // order; a segment's 8 loads are in flight together
      for (int j0 = 0; j0 < kRChunk; j0 += 8) {
        float a[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = 0.0f;
        for (int k = 0; k < nsg; ++k) {
          const float *S = E + kExS * W + ((int64_t)which * nsg + k) * W + c;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int n = c + (j0 + j) * (int)blockDim.x;
            if (n < W) a[j] += __ldg(S + (j0 + j) * blockDim.x);
          }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int n = c + (j0 + j) * (int)blockDim.x;
          if (n < W) rowp[n + (n >> 5)] = a[j];
        }
      }
      if (c == 0) dx2[0][0] = dx2[0][1] = 0.0f;
      __syncthreads();
      if (c == 0) {
        e2[0] = rowp[0];
        e2[1] = rowp[(W - 1) + ((W - 1) >> 5)];
      }
#pragma unroll
      for (int t = 0; t < kRChunk; ++t) U[t] = live ? rowp[c * (kRChunk + 1) + t] : 0.0f;
      __syncthreads();
      row_filter<K, KIND>(p, U, V, cf, cb, e2, dx2[0]);
      if (live) {
#pragma unroll
        for (int t = 0; t < kRChunk; ++t) rowp[c * (kRChunk + 1) + t] = V[t];
      }
      __syncthreads();
      for (int n = c; n < W; n += blockDim.x) E[kExKy * W + (int64_t)which * W + n] = rowp[n + (n >> 5)];
      __syncthreads();
    }
    TL(1024 + (blockIdx.x & 1023));
    pdl_trigger();
    return;
  }
  if (nrows <= 0) return;

  for (int i = 0; i < nrows; ++i) {
    const int64_t r = rlo + i;
    // rows r-1, r, r+1 are logical rows i, i+1, i+2 (slots i%3, ...)
    const int su = i % kRLBufs, sc = (i + 1) % kRLBufs, sd = (i + 2) % kRLBufs;
    if (i == 0) {
      mbar_wait(&bar[0], 0);
      mbar_wait(&bar[1], 0);
    }
    mbar_wait(&bar[sd], (unsigned)(((i + 2) / kRLBufs) & 1));
    TLROW(i, 0);
    float xl, xr;
    load_chunk(sc, X);
    halos(sc, X, xl, xr);
    {
      float Xu[kRChunk];
      load_chunk(su, Xu);
#pragma unroll
      for (int t = 0; t < kRChunk; ++t) U[t] = Xu[t] - X[t];
      load_chunk(sd, Xu);
#pragma unroll
      for (int t = 0; t < kRChunk; ++t) {
        const float l = t ? X[t - 1] : xl, rr = t < kRChunk - 1 ? X[t + 1] : xr;
        U[t] = ((l - X[t]) + (rr - X[t])) + (U[t] + (Xu[t] - X[t]));
      }
    }
    dx_all(X, xr);
    if (c == 0 || c == C - 1) {  // D02 X of the end samples: the steady starts (every scale)
      const SwzRow32 ru{xbuf + su * rowb}, rd{xbuf + sd * rowb};
      const int n = c == 0 ? 0 : W - 1;
      const float xc = c == 0 ? X[0] : X[kRChunk - 1];
      e2[c == 0 ? 0 : 1] = (ru.ld(n) - xc) + (rd.ld(n) - xc);
    }
#if VMF_ABL != 3 && VMF_ABL != 6 && VMF_ABL != 7  // (VMF_ABL: timing ablations, tools/row_ablation.sh; results invalid)
    if (rm.carry_fold) {
      float2 sd[16];  // the folded sample pairs, shared by every scale's carries
#pragma unroll
      for (int t = 0; t < 16; ++t)
        sd[t] = make_float2(U[t] + U[kRChunk - 1 - t], U[t] - U[kRChunk - 1 - t]);
      for (int s = 0; s < ns; ++s) row_carry32_fold<K>(sp[s], sd, cfs(s), cbs(s));
    } else {
      for (int s = 0; s < ns; ++s) row_carry32<K, KIND>(RC32<K>(sp[s]), U, cfs(s), cbs(s));
    }
#endif
    __syncthreads();  // rows r-1 .. r+1 read; carries, e2, red published
    TLROW(i, 1);
    if (c == 0) {
      if (i + 3 <= nrows + 1) issue_row(su, clampr(rlo + 2 + i));  // row r+2 -> slot of r-1
      reduce_dx();
    }
    // the 2 ns chunk scans over the warps
#if VMF_ABL != 1 && VMF_ABL != 6 && VMF_ABL != 7
    for (int task = c >> 5; task < 2 * ns; task += nwarp)
      chunk_scan32<K>(sp[task >> 1], (task & 1) ? cbs(task >> 1) : cfs(task >> 1), task & 1,
                      e2[task & 1], lane);
#endif
    __syncthreads();
    TLROW(i, 2);
    for (int s = 0; s < ns; ++s) {
#if VMF_ABL == 0
      if (rm.store_inline == 2) {
        if (sp[s].sign > 0.f)
          row_walks32_pair<K, KIND, true>(sp[s], C, U, cfs(s), cbs(s), dx2[s],
                                          out.V(s) + r * out.ldv + c * kRChunk, live,
                                          l2_policy_evict_last());
        else
          row_walks32_pair<K, KIND, false>(sp[s], C, U, cfs(s), cbs(s), dx2[s],
                                           out.V(s) + r * out.ldv + c * kRChunk, live,
                                           l2_policy_evict_last());
        continue;
      }
      if (rm.store_inline) {
        row_walks32_store<K, KIND>(RC32<K>(sp[s]), C, U, cfs(s), cbs(s), dx2[s],
                                   out.V(s) + r * out.ldv + c * kRChunk, live,
                                   l2_policy_evict_last());
        continue;
      }
#endif
#if VMF_ABL != 2 && VMF_ABL != 6 && VMF_ABL != 7
      row_walks32<K, KIND>(RC32<K>(sp[s]), C, U, V, cfs(s), cbs(s), dx2[s]);
#else
      for (int t = 0; t < kRChunk; ++t) V[t] = U[t] * (float)s;
#endif
#if VMF_ABL == 4 || VMF_ABL == 7
      if (live && V[0] == 12345.678f && V[31] == -1.5f) {
#else
      if (live) {
#endif
        float *dst = out.V(s) + r * out.ldv + c * kRChunk;
#if VMF_ABL == 5
#pragma unroll
        for (int q = 0; q < kRChunk / 4; ++q)
          *reinterpret_cast<float4 *>(dst + 4 * q) =
              make_float4(V[4 * q], V[4 * q + 1], V[4 * q + 2], V[4 * q + 3]);
#else
        // V is read twice by the column pass; 256-bit stores: each lane fills
        // whole 32-byte sectors (the 128-byte lane stride of a chunk row
        // leaves 16-byte stores at half a sector each)
        const uint64_t pol = l2_policy_evict_last();
#pragma unroll
        for (int q = 0; q < kRChunk / 8; ++q) st_v8_hint(dst + 8 * q, V + 8 * q, pol);
#endif
      }
    }
    TLROW(i, 3);
  }
  TL(1024 + (blockIdx.x & 1023));
  pdl_trigger();
}

// ---------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------
static int rl_plan(RowLapPlan *P, int64_t h, int64_t w, const double *b, const double *a, int k,
                   double b0, int sign) {
  Modal M;
  if (!modal_realise(b, a, k, &M)) return fail(VMF_EVALUE, "no modal realisation");
  RowLapParams &p = P->p;
  memset(&p, 0, sizeof(p));
  P->kind = M.kind;
  p.K = k;
  p.p = (float)M.p;
  p.q = (float)M.q;
  for (int i = 0; i < k; ++i) {
    p.c[i] = (float)M.c[i];
    p.cs[i] = (float)(sign * M.c[i]);
  }
  p.b0 = (float)b0;
  p.sign = (float)sign;
  p.H = h;
  p.W = w;
  p.C = (int)(w / kRChunk);
  p.cpl = (p.C + 31) / 32;
  ld Wt[kRChunk][4];
  {
    ld v[4], t[4];
    for (int i = 0; i < k; ++i) v[i] = M.bv[i];
    for (int tt = 0; tt < kRChunk; ++tt) {
      for (int i = 0; i < k; ++i) Wt[tt][i] = v[i];
      for (int i = 0; i < k; ++i) {
        t[i] = 0;
        for (int jj = 0; jj < k; ++jj) t[i] += M.A[i * k + jj] * v[jj];
      }
      memcpy(v, t, sizeof(ld) * k);
    }
  }
  for (int i = 0; i < k; ++i)
    for (int t = 0; t < kRChunk / 2; ++t) {
      p.SPQ[i][t][0] = (float)(0.5L * (Wt[t][i] + Wt[kRChunk - 1 - t][i]));
      p.SPQ[i][t][1] = (float)(0.5L * (Wt[kRChunk - 1 - t][i] - Wt[t][i]));
    }
  {  // c A^-1: the right border's vector of the last chunk
    ld At[16], x[4];
    for (int i = 0; i < k; ++i)
      for (int jj = 0; jj < k; ++jj) At[i * k + jj] = M.A[jj * k + i];
    for (int i = 0; i < k; ++i) x[i] = M.c[i];
    if (!solve(At, x, k)) return fail(VMF_EVALUE, "singular modal matrix");
    for (int i = 0; i < k; ++i) P->ci[i] = (float)x[i];
  }
  ld A32[16];
  matpow(M.A, kRChunk, A32, k);
  for (int i = 0; i < k * k; ++i) p.A32[i] = (float)A32[i];
  for (int l = 0; l < 5; ++l) {
    ld X[16];
    matpow(A32, (int64_t)p.cpl << l, X, k);
    for (int i = 0; i < k * k; ++i) p.Apow[l][i] = (float)X[i];
  }
  {
    ld IA[16], y[4];
    for (int i = 0; i < k; ++i) {
      for (int jj = 0; jj < k; ++jj) IA[i * k + jj] = (i == jj ? 1 : 0) - M.A[i * k + jj];
      y[i] = M.bv[i];
    }
    if (!solve(IA, y, k)) return fail(VMF_EVALUE, "pole on the unit circle");
    for (int i = 0; i < k; ++i) p.Iss[i] = (float)y[i];
  }
  // border weights h(1..Mh) along the row (tail below 1e-9 of sum |h|)
  {
    std::vector<ld> hv(1, 0);
    ld v[4], t[4], tot = 0;
    for (int i = 0; i < k; ++i) v[i] = M.bv[i];
    const int64_t mmax = w - 1 < kHmRowMax ? w - 1 : kHmRowMax;
    for (int64_t m = 1; m <= mmax; ++m) {
      ld hmv = 0;
      for (int i = 0; i < k; ++i) hmv += M.c[i] * v[i];
      hv.push_back(hmv);
      tot += fabsl(hmv);
      for (int i = 0; i < k; ++i) {
        t[i] = 0;
        for (int jj = 0; jj < k; ++jj) t[i] += M.A[i * k + jj] * v[jj];
      }
      memcpy(v, t, sizeof(ld) * k);
    }
    if (mmax == kHmRowMax && w - 1 > kHmRowMax) {
      ld rest = 0;
      for (int64_t m = kHmRowMax + 1; m < w && m <= kHmRowMax + 4096; ++m) {
        ld hmv = 0;
        for (int i = 0; i < k; ++i) hmv += M.c[i] * v[i];
        rest += fabsl(hmv);
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
    // (border terms: a tail below 1e-8 of sum |h| is ~1e-8 of the edge
    // gradients -- far below fp32 L)
    while (Mh > 1 && tail + fabsl(hv[Mh]) < 1e-8L * tot) tail += fabsl(hv[Mh--]);
    p.Mh = (int)Mh;
  }
  return VMF_OK;
}

int rowlap_get_plan(int64_t h, int64_t w, const double *b, const double *a, int k, double b0,
                    int sign, RowLapPlan *out) {
  static PlanCache<RowLapPlan> cache;
  std::vector<unsigned char> key;
  key_add(key, h);
  key_add(key, w);
  key_add(key, k);
  key_add(key, b0);
  key_add(key, sign);
  key_add(key, b, sizeof(double) * k);
  key_add(key, a, sizeof(double) * k);
  if (cache.get(key, out)) return VMF_OK;
  const int rc = rl_plan(out, h, w, b, a, k, b0, sign);
  if (rc) return rc;
  cache.put(key, *out);
  return VMF_OK;
}

bool rowlap_supported(int64_t h, int64_t w, const double *b, const double *a, int k, double b0,
                      int sign) {
  if (getenv("VMF_NO_ROWLAP") || h < 2 || w < 64 || w % kRChunk || w / kRChunk > kRLMaxC)
    return false;
  static RowLapPlan tmp;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  return rowlap_get_plan(h, w, b, a, k, b0, sign, &tmp) == VMF_OK;
}

static int rl_block(int C) { return (C + 31) / 32 * 32; }

static size_t rl_smem(int C, int k, int ns) {
  return 1024 + (size_t)kRLBufs * ((C * 128 + 1023) & ~1023) +
         (size_t)ns * 2 * rl_block(C) * k * sizeof(float) + (size_t)ns * sizeof(RowLapParams) + 16;
}

// segment vectors c A^(m0-1) of a column stage (m0 = 1 + 64 k)
static int seg_vectors(const double *b, const double *a, int k, int Mh, SegVec *sv) {
  Modal M;
  if (!modal_realise(b, a, k, &M)) return fail(VMF_EVALUE, "no modal realisation");
  memset(sv, 0, sizeof(*sv));
  sv->Mh = Mh;
  sv->nseg = (int)cdiv(sv->Mh, kSeg);
  if (sv->nseg > kMaxSeg) return fail(VMF_EVALUE, "border too long");
  ld v[4], t[4];
  for (int i = 0; i < k; ++i) v[i] = M.c[i];  // c A^0
  int m = 1;
  for (int s = 0; s < sv->nseg; ++s) {
    for (; m < 1 + kSeg * s; ++m) {  // v <- v A
      for (int j = 0; j < k; ++j) {
        t[j] = 0;
        for (int i = 0; i < k; ++i) t[j] += v[i] * M.A[i * k + j];
      }
      memcpy(v, t, sizeof(ld) * k);
    }
    for (int i = 0; i < k; ++i) sv->v[s][i] = (float)v[i];
  }
  return VMF_OK;
}

struct SweepPlan {
  RowLapMulti rm;
  BorderMulti bm;
  int kind, nseg_total;
};

static int sweep_plan(int64_t h, int64_t w, int k, int ns, const SweepStage *st, SweepPlan *P) {
  if (ns < 1 || ns > kMaxScales) return fail(VMF_EVALUE, "1..%d scales per sweep", kMaxScales);
  memset(P, 0, sizeof(*P));
  P->rm.ns = P->bm.ns = ns;
  P->rm.H = h;
  P->rm.W = w;
  P->rm.C = (int)(w / kRChunk);
  P->kind = -1;
  for (int s = 0; s < ns; ++s) {
    RowLapPlan R, Cp;
    int rc = rowlap_get_plan(h, w, st[s].rb, st[s].ra, k, st[s].rb0, st[s].rsign, &R);
    if (rc) return rc;
    // the column stage along the columns (length h): modal form, border length
    rc = rowlap_get_plan(w, h, st[s].cb, st[s].ca, k, st[s].cb0, st[s].csign, &Cp);
    if (rc) return rc;
    if (R.kind != Cp.kind || (P->kind >= 0 && R.kind != P->kind))
      return fail(VMF_EVALUE, "sweep: every stage needs the same modal structure");
    P->kind = R.kind;
    P->rm.s[s] = R.p;
    BorderScale &b = P->bm.s[s];
    b.p = Cp.p.p;
    b.q = Cp.p.q;
    b.sign = Cp.p.sign;
    for (int i = 0; i < 4; ++i) {
      b.c[i] = Cp.p.c[i];
      b.cr[i] = R.p.c[i];
      b.ci[i] = R.ci[i];
    }
    for (int i = 0; i < 16; ++i) b.A32[i] = R.p.A32[i];
    b.C = R.p.C;
    b.Mh = R.p.Mh;
    rc = seg_vectors(st[s].cb, st[s].ca, k, Cp.p.Mh, &b.sv);
    if (rc) return rc;
    P->rm.s[s].nseg = b.sv.nseg;
    P->nseg_total += 2 * b.sv.nseg;
    if (b.sv.nseg > P->bm.maxseg) P->bm.maxseg = b.sv.nseg;
    if (b.sv.Mh > P->bm.maxMh) P->bm.maxMh = b.sv.Mh;
  }
  return VMF_OK;
}

bool sweep_supported(const void *x, int64_t h, int64_t w, int64_t ldx, int k, int ns,
                     const SweepStage *st) {
  if (getenv("VMF_NO_ROWLAP") || h < 2 || w < 64 || w % kRChunk || w / kRChunk > kRLMaxC)
    return false;
  if (((uintptr_t)x & 15) || ((ldx * 4) & 15)) return false;
  static SweepPlan P;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  return sweep_plan(h, w, k, ns, st, &P) == VMF_OK &&
         rl_smem((int)(w / kRChunk), k, ns) <= 220 * 1024;
}

template <int K, int KIND>
static int launch_sweep(const float *x, int64_t ldx, SweepPlan &P, const SweepOut &out,
                        cudaStream_t st) {
  RowLapMulti &rm = P.rm;
  CUtensorMap xm;
  memset(&xm, 0, sizeof(xm));
  if (!make_tmap_rows_swz_f32(&xm, x, rm.H, rm.W, ldx, 1)) {
    cudaGetLastError();
    return fail(VMF_EVALUE, "row pass: TMA descriptor unavailable");
  }
  {
    Launch g(K_ROW_BORDER, st);  // the border kernel (reads X only)
    launch_pdl(sweep_border_kernel<K, KIND>,
               dim3((unsigned)cdiv(rm.W, 128), (unsigned)(2 * P.bm.maxseg + rm.ns)), dim3(128), 0, st,
               P.bm, x, ldx, rm.H, rm.W, out);
  }
  const size_t smem = rl_smem(rm.C, K, rm.ns);
  const int block = rl_block(rm.C);
  static std::map<std::pair<int, size_t>, int> slot_cache;
  const int dev = current_device();
  int &slots = slot_cache[std::make_pair(dev, smem)];
  static PerDevice attr;
  if (attr.first()) {  // the largest dynamic footprint next to the static shared memory
    cudaFuncAttributes fa;
    memset(&fa, 0, sizeof(fa));
    cudaFuncGetAttributes(&fa, sweep_rows_kernel<K, KIND>);
    cudaFuncSetAttribute(sweep_rows_kernel<K, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024 - (int)fa.sharedSizeBytes);
    cudaGetLastError();
  }
  if (!slots) {
    int occ = 0, nsm = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep_rows_kernel<K, KIND>, block, smem);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaGetLastError();
    if (const char *e = getenv("VMF_ROW_OCC")) {  // experiment: fewer resident CTAs per SM
      const int o = atoi(e);
      if (o > 0 && o < occ) occ = o;
    }
    slots = (occ > 0 ? occ : 1) * nsm;
  }
  // ns slots are the edge CTAs (virtual and border rows of each scale)
  const int rslots = slots > rm.ns ? slots - rm.ns : 1;
  rm.rows_per = (int)cdiv(rm.H, rslots);
  rm.carry_fold = getenv("VMF_CARRY_REC") ? 0 : 1;
  rm.store_inline = getenv("VMF_STORE_AFTER") ? 0 : getenv("VMF_WALK_SEQ") ? 1 : 2;
  const int grid = (int)cdiv(rm.H, rm.rows_per) + rm.ns;
  Launch g(K_SWEEP_ROWS, st);
  launch_pdl(sweep_rows_kernel<K, KIND>, dim3(grid), dim3(block), smem, st, xm,
             (const RowLapMulti)rm, out);
  return cuda_status("fp32 row pass");
}

#if VMF_TIMELINE
}  // namespace vmf
extern "C" int vmf_debug_timeline(unsigned long long *host, int n) {
  return (int)cudaMemcpyFromSymbol(host, vmf::g_tl, sizeof(unsigned long long) * (n < 4096 ? n : 4096));
}
extern "C" int vmf_debug_timeline_reset(void) {
  static unsigned long long z[4096];
  return (int)cudaMemcpyToSymbol(vmf::g_tl, z, sizeof(z));
}
namespace vmf {
#endif
int sweep_rows(const float *x, int64_t ldx, int64_t h, int64_t w, int k, int ns,
               const SweepStage *st, const SweepOut &out, cudaStream_t stream) {
  static SweepPlan P;  // (large: not on the stack)
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  int rc = sweep_plan(h, w, k, ns, st, &P);
  if (rc) return rc;
  if (P.kind == M32_CPAIR) return launch_sweep<2, M32_CPAIR>(x, ldx, P, out, stream);
  switch (k) {
    case 2: return launch_sweep<2, M32_JORDAN>(x, ldx, P, out, stream);
    case 3: return launch_sweep<3, M32_JORDAN>(x, ldx, P, out, stream);
    case 4: return launch_sweep<4, M32_JORDAN>(x, ldx, P, out, stream);
  }
  return fail(VMF_EVALUE, "fp32 row pass supports K = 2..4, got %d", k);
}

}  // namespace vmf
