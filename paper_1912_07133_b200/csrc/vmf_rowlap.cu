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
// the border kernel: the column direction's border sums, straight from the
// frame (column stage, modal fp32), in 64-row segments so the whole frame
// edge is covered by ~1k short CTAs:
//   Dy[0][c] = s_C sum_{m>=1} h_C(m) G(m, c),  Dy[1][c] = sum_{m>=1} h_C(m) G(H-m, c),
//   G(m, c) = X(m, c) - X(m-1, c),  h_C(m) = c A^(m-1) b.
// Segment k covers m = m0 .. m0+63 (m0 = 1 + 64 k): its share is
// (c A^(m0-1)) . sum_t A^t b G(m0 + t), the inner sum a zero-state
// recursion; S[which][k][c] holds the shares, summed in k order by the row
// pass.  It reads only X, so it runs first and the row pass waits for it
// (griddepcontrol) only before its first store.
// ---------------------------------------------------------------------------
constexpr int kSeg = 64;

template <int K, int KIND>
__global__ void __launch_bounds__(128) rowborder_kernel(const __grid_constant__ RowLapParams pc,
                                                        const __grid_constant__ SegVec sv,
                                                        const float *__restrict__ X, int64_t ldx,
                                                        int64_t H, int64_t W,
                                                        float *__restrict__ S) {
  // (no early trigger: the row pass's CTAs would take the registers this
  // grid needs and stretch it; it launches when this grid completes)
  const int nseg = sv.nseg;
  const int which = (int)blockIdx.y / nseg, k = (int)blockIdx.y % nseg;
  const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t cc = col < W ? col : W - 1;
  const int Mh = sv.Mh;
  const int m0 = 1 + kSeg * k;
  const int n = (Mh - m0 + 1) < kSeg ? (Mh - m0 + 1) : kSeg;  // m = m0 .. m0+n-1
  // rows holding G(m) for m = m0 + t: top rows m (G = X(m) - X(m-1)); bottom
  // rows H - m (G = X(H-m) - X(H-m-1)); the samples X(r) for the n+1 rows
  // involved, all loaded before the recursion (independent loads)
  float xs[kSeg + 1];
  const float *Xc = X + cc;
#pragma unroll
  for (int t = 0; t <= kSeg; ++t) {
    // top: xs[t] = X(m0 - 1 + t); bottom: xs[t] = X(H - m0 - t)
    const int64_t r = which == 0 ? m0 - 1 + t : H - m0 - t;
    xs[t] = t <= n ? __ldg(Xc + (r < 0 ? 0 : (r >= H ? H - 1 : r)) * ldx) : 0.0f;
  }
  Rec32<K, KIND> u;
#pragma unroll
  for (int i = 0; i < K; ++i) u.u[i] = 0.0f;
#pragma unroll
  for (int t = kSeg - 1; t >= 0; --t) {
    if (t < n) {
      // G(m0 + t): top X(m0+t) - X(m0+t-1) = xs[t+1] - xs[t];
      //            bottom X(H-m0-t) - X(H-m0-t-1) = xs[t] - xs[t+1]
      const float g = which == 0 ? xs[t + 1] - xs[t] : xs[t] - xs[t + 1];
      u.step(pc, g);
    }
  }
  float v = u.out(sv.v[k]);
  if (which == 0) v *= pc.sign;
  if (col < W) S[((int64_t)which * nseg + k) * W + col] = v;
}

// ---------------------------------------------------------------------------
// the row pass
// ---------------------------------------------------------------------------
// Left / right border terms of one row: dxl = s sum_{n>=1} h(n) G(n),
// dxr = sum_{m>=1} h(m) G(W-m), G(n) = X(n) - X(n-1).  Per chunk (samples
// n = n0+1 .. n0+32) the sums are modal: h(n0+1+t) = (c A^n0) A^t b and
// h(W-n0-1-t) = (c A^(W-n0-33)) A^(31-t) b, so each chunk forms two zero-state
// sums with the uniform weights A^t b and dots them with its own vectors
// vl(c) = c A^n0, vr(c) = c A^(W-n0-33) (smem); chunks farther than Mh from
// the edge contribute nothing measurable and skip.  Reduced over the CTA in
// a fixed order into red[0..nwarp) / red[8..).
template <int K>
__device__ __forceinline__ void dx_partials(const RowLapParams &p, const float *vlr,
                                            const float (&X)[kRChunk], float xr, float *red) {
  const int c = threadIdx.x, lane = c & 31, warp = c >> 5;
  const int n0 = c * kRChunk;
  const int W = (int)p.W, Mh = p.Mh, C = p.C;
  float pl = 0.0f, pr = 0.0f;
  const bool L = c < C && n0 < Mh, Rr = c < C && n0 + kRChunk >= W - Mh;
  if (L || Rr) {
    float zl[K], zr[K];
#pragma unroll
    for (int i = 0; i < K; ++i) zl[i] = zr[i] = 0.0f;
#pragma unroll
    for (int t = 0; t < kRChunk; ++t) {
      const float g = (t < kRChunk - 1 ? X[t + 1] : xr) - X[t];  // G(n0 + 1 + t)
#pragma unroll
      for (int i = 0; i < K; ++i) {
        zl[i] = fmaf(p.Wt[t][i], g, zl[i]);
        zr[i] = fmaf(p.Wt[kRChunk - 1 - t][i], g, zr[i]);
      }
    }
    if (L)
#pragma unroll
      for (int i = 0; i < K; ++i) pl = fmaf(vlr[c * 8 + i], zl[i], pl);
    if (Rr)
#pragma unroll
      for (int i = 0; i < K; ++i) pr = fmaf(vlr[c * 8 + 4 + i], zr[i], pr);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    pl += __shfl_xor_sync(0xffffffffu, pl, o);
    pr += __shfl_xor_sync(0xffffffffu, pr, o);
  }
  if (lane == 0) {
    red[warp] = pl;
    red[8 + warp] = pr;
  }
}

// Grid: row CTAs (contiguous rows each) + one edge CTA (the last) for the
// four single-row filters: the virtual rows Vt / Vb and, once the border
// kernel has completed, the column direction's border rows Ky = R_ss(Dy).
template <int K, int KIND>
__global__ void __launch_bounds__(kRLMaxC) rowlap_kernel(
    const __grid_constant__ CUtensorMap xmap, const __grid_constant__ RowLapParams p,
    float *__restrict__ Vout, int64_t ldv, const __grid_constant__ VlrTab vtab,
    float *__restrict__ Vt, float *__restrict__ Vb, const float *__restrict__ S, int nseg,
    float *__restrict__ Ky) {
  extern __shared__ __align__(1024) unsigned char smem_rl[];
  __shared__ __align__(8) uint64_t bar[kRLBufs];
  __shared__ float red[16], e2[2], dx2[2];
  const int C = p.C, c = threadIdx.x, nwarp = (int)(blockDim.x >> 5);
  const bool live = c < C;  // the block is whole warps; threads c >= C carry no chunk
  const int rowbytes = C * 128;                // one row's TMA box
  const int rowb = (rowbytes + 1023) & ~1023;  // slot spacing: SWIZZLE_128B needs 1024-byte bases
  const unsigned sb = (unsigned)__cvta_generic_to_shared(smem_rl);
  char *xbuf = reinterpret_cast<char *>(smem_rl) + ((1024u - (sb & 1023u)) & 1023u);
  float *cf = reinterpret_cast<float *>(xbuf + kRLBufs * rowb);
  float *cb = cf + blockDim.x * K;
  float *vlr = cb + blockDim.x * K;  // [C][8]: vl (4), vr (4)
  const int64_t H = p.H;
  const int W = (int)p.W;
  for (int e = c; e < C * 8; e += blockDim.x) vlr[e] = vtab.v[e];
  const bool edge = blockIdx.x == gridDim.x - 1;
  const int64_t rlo = edge ? 0 : (int64_t)blockIdx.x * p.rows_per;
  const int64_t rhi = edge ? 0 : (rlo + p.rows_per < H ? rlo + p.rows_per : H);
  const int nrows = (int)(rhi - rlo);
  auto issue_row = [&](int s, int64_t r) {
    mbar_expect_tx(&bar[s], (unsigned)rowbytes);
    tma_load_3d_hint(xbuf + s * rowb, &xmap, &bar[s], 0, 0, (int)r, l2_policy_evict_first());
  };
  // row CTAs: logical input row j = clamp(rlo - 1 + j), j = 0 .. nrows + 1,
  // in slot j % 3; the edge CTA: rows 0 and H-1 in slots 0 / 1
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
  float U[kRChunk], V[kRChunk], X[kRChunk];
  auto load_chunk = [&](int s, float (&o)[kRChunk]) {
    const SwzRow32 r{xbuf + s * rowb};
#pragma unroll
    for (int q = 0; q < kRChunk / 4; ++q) {
      const float4 v = live ? r.ld4(c, q) : make_float4(0.f, 0.f, 0.f, 0.f);
      o[4 * q] = v.x;
      o[4 * q + 1] = v.y;
      o[4 * q + 2] = v.z;
      o[4 * q + 3] = v.w;
    }
  };
  auto halos = [&](int s, const float (&x)[kRChunk], float &xl, float &xr) {
    const SwzRow32 r{xbuf + s * rowb};
    xl = c > 0 && live ? r.ld(c * kRChunk - 1) : x[0];
    xr = c < C - 1 ? r.ld(c * kRChunk + kRChunk) : x[kRChunk - 1];
  };
  auto reduce_dx = [&]() {  // (thread 0, after a barrier that follows dx_partials)
    float a = 0.0f, b = 0.0f;
    for (int w = 0; w < nwarp; ++w) {
      a += red[w];
      b += red[8 + w];
    }
    dx2[0] = p.sign * a;
    dx2[1] = b;
  };

  if (edge) {
    // virtual rows: Vt / Vb = R0(D20 X) of row 0 / H-1 (zero starts), with
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
      dx_partials<K>(p, vlr, X, xr, red);
      if (c == 0) e2[0] = e2[1] = 0.0f;
      row_carry32<K>(p, U, cf, cb);
      __syncthreads();
      if (c == 0) reduce_dx();
      row_scan_walk32<K, KIND>(p, U, V, cf, cb, e2, dx2);
      float *dst = which == 0 ? Vt : Vb;
      if (live) {
#pragma unroll
        for (int q = 0; q < kRChunk / 4; ++q)
          *reinterpret_cast<float4 *>(dst + c * kRChunk + 4 * q) =
              make_float4(V[4 * q], V[4 * q + 1], V[4 * q + 2], V[4 * q + 3]);
      }
      __syncthreads();
    }
    // border rows: Ky = R_ss(dy), dy = sum of the border kernel's segment
    // shares (the border kernel is this grid's predecessor)
    pdl_wait();
    float *rowp = reinterpret_cast<float *>(xbuf);  // (the input slots are idle now)
    for (int which = 0; which < 2; ++which) {
      for (int n = c; n < W; n += blockDim.x) {
        float a = 0.0f;
        for (int k = 0; k < nseg; ++k) a += __ldg(S + ((int64_t)which * nseg + k) * W + n);
        rowp[n + (n >> 5)] = a;
      }
      if (c == 0) dx2[0] = dx2[1] = 0.0f;
      __syncthreads();
      if (c == 0) {
        e2[0] = rowp[0];
        e2[1] = rowp[(W - 1) + ((W - 1) >> 5)];
      }
#pragma unroll
      for (int t = 0; t < kRChunk; ++t) U[t] = live ? rowp[c * (kRChunk + 1) + t] : 0.0f;
      __syncthreads();
      row_filter<K, KIND>(p, U, V, cf, cb, e2, dx2);
      if (live) {
#pragma unroll
        for (int t = 0; t < kRChunk; ++t) rowp[c * (kRChunk + 1) + t] = V[t];
      }
      __syncthreads();
      for (int n = c; n < W; n += blockDim.x) Ky[(int64_t)which * W + n] = rowp[n + (n >> 5)];
      __syncthreads();
    }
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
    dx_partials<K>(p, vlr, X, xr, red);
    if (c == 0 || c == C - 1) {  // D02 X of the end samples: the steady starts
      const SwzRow32 ru{xbuf + su * rowb}, rd{xbuf + sd * rowb};
      const int n = c == 0 ? 0 : W - 1;
      const float xc = X[c == 0 ? 0 : kRChunk - 1];
      e2[c == 0 ? 0 : 1] = (ru.ld(n) - xc) + (rd.ld(n) - xc);
    }
    row_carry32<K>(p, U, cf, cb);
    __syncthreads();  // rows r-1 .. r+1 read; carries, e2, red published
    if (c == 0) {
      if (i + 3 <= nrows + 1) issue_row(su, clampr(rlo + 2 + i));  // row r+2 -> slot of r-1
      reduce_dx();
    }
    row_scan_walk32<K, KIND>(p, U, V, cf, cb, e2, dx2);
    if (i == 0) pdl_wait();  // V may still be read by the previous scale's column pass
    if (live) {
      float *dst = Vout + r * ldv + c * kRChunk;
      const uint64_t pol = l2_policy_evict_last();  // V is read twice by the column pass
#pragma unroll
      for (int q = 0; q < kRChunk / 4; ++q)
        st_v4_hint(dst + 4 * q, make_float4(V[4 * q], V[4 * q + 1], V[4 * q + 2], V[4 * q + 3]),
                   pol);
    }
  }
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
      p.SP[i][t] = (float)(0.5L * (Wt[t][i] + Wt[kRChunk - 1 - t][i]));
      p.SQ[i][t] = (float)(0.5L * (Wt[kRChunk - 1 - t][i] - Wt[t][i]));
    }
  for (int t = 0; t < kRChunk; ++t)
    for (int i = 0; i < k; ++i) p.Wt[t][i] = (float)Wt[t][i];
  // border-term chunk vectors vl(c) = c A^(32 c), vr(c) = c A^(W - 32 c - 33)
  {
    ld Ainv[16], IA[16];
    for (int i = 0; i < k * k; ++i) IA[i] = M.A[i];
    for (int col = 0; col < k; ++col) {  // A^-1 column by column
      ld M2[16], y[4];
      memcpy(M2, IA, sizeof(ld) * k * k);
      for (int i = 0; i < k; ++i) y[i] = (i == col) ? 1 : 0;
      if (!solve(M2, y, k)) return fail(VMF_EVALUE, "singular modal matrix");
      for (int i = 0; i < k; ++i) Ainv[i * k + col] = y[i];
    }
    memset(&P->vlr, 0, sizeof(P->vlr));
    ld A32[16];
    matpow(M.A, kRChunk, A32, k);
    ld v[4], t4[4];
    for (int i = 0; i < k; ++i) v[i] = M.c[i];  // c A^0
    for (int cc = 0; cc < p.C; ++cc) {          // vl(cc) = c A^(32 cc)
      for (int i = 0; i < k; ++i) P->vlr.v[cc * 8 + i] = (float)v[i];
      for (int jj = 0; jj < k; ++jj) {
        t4[jj] = 0;
        for (int i = 0; i < k; ++i) t4[jj] += v[i] * A32[i * k + jj];
      }
      memcpy(v, t4, sizeof(ld) * k);
    }
    for (int i = 0; i < k; ++i) {  // vr(C-1) = c A^-1, then x A^32 going left
      v[i] = 0;
      for (int jj = 0; jj < k; ++jj) v[i] += M.c[jj] * Ainv[jj * k + i];
    }
    for (int cc = p.C - 1; cc >= 0; --cc) {
      for (int i = 0; i < k; ++i) P->vlr.v[cc * 8 + 4 + i] = (float)v[i];
      for (int jj = 0; jj < k; ++jj) {
        t4[jj] = 0;
        for (int i = 0; i < k; ++i) t4[jj] += v[i] * A32[i * k + jj];
      }
      memcpy(v, t4, sizeof(ld) * k);
    }
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
    memset(&P->hm, 0, sizeof(P->hm));
    for (int64_t m = 1; m <= Mh; ++m) P->hm.h[m] = (float)hv[m];
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

static size_t rl_smem(int C, int k) {
  return 1024 + (size_t)kRLBufs * ((C * 128 + 1023) & ~1023) +
         2 * (size_t)rl_block(C) * k * sizeof(float) + (size_t)C * 8 * sizeof(float);
}

template <int K, int KIND>
static int launch_rowlap(const float *x, int64_t ldx, float *V, int64_t ldv, float *vrows,
                         RowLapPlan &P, const RowLapPlan &PC, const SegVec &sv, cudaStream_t st) {
  RowLapParams &p = P.p;
  CUtensorMap xm;
  memset(&xm, 0, sizeof(xm));
  if (!make_tmap_rows_swz_f32(&xm, x, p.H, p.W, ldx, 1)) {
    cudaGetLastError();
    return fail(VMF_EVALUE, "row pass: TMA descriptor unavailable");
  }
  float *Vt = vrows, *Vb = vrows + p.W, *Ky = vrows + 2 * p.W, *S = vrows + 4 * p.W;
  {
    Launch g(K_ROW_BORDER, st);  // the border kernel (reads X only)
    launch_pdl(rowborder_kernel<K, KIND>, dim3((unsigned)cdiv(p.W, 128), (unsigned)(2 * sv.nseg)),
               dim3(128), 0, st, PC.p, sv, x, ldx, p.H, p.W, S);
  }
  const size_t smem = rl_smem(p.C, K);
  const int block = rl_block(p.C);
  static std::map<std::pair<int, size_t>, int> slot_cache;
  const int dev = current_device();
  int &slots = slot_cache[std::make_pair(dev, smem)];
  static PerDevice attr;
  if (attr.first())  // the largest footprint (C = 256), so every width may launch
    cudaFuncSetAttribute(rowlap_kernel<K, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)rl_smem(kRLMaxC, K));
  if (!slots) {
    int occ = 0, nsm = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rowlap_kernel<K, KIND>, block, smem);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaGetLastError();
    slots = (occ > 0 ? occ : 1) * nsm;
  }
  // one slot is the edge CTA (virtual and border rows)
  p.rows_per = (int)cdiv(p.H, slots > 1 ? slots - 1 : 1);
  const int grid = (int)cdiv(p.H, p.rows_per) + 1;
  Launch g(K_IIR_ROWS_FUSED, st);
  launch_pdl(rowlap_kernel<K, KIND>, dim3(grid), dim3(block), smem, st, xm, (const RowLapParams)p,
             V, ldv, P.vlr, Vt, Vb, (const float *)S, sv.nseg, Ky);
  return cuda_status("fp32 row pass");
}

// segment vectors c A^(m0-1) of the column stage (m0 = 1 + 64 k)
static int seg_vectors(const double *b, const double *a, int k, const RowLapPlan &PC, SegVec *sv) {
  Modal M;
  if (!modal_realise(b, a, k, &M)) return fail(VMF_EVALUE, "no modal realisation");
  memset(sv, 0, sizeof(*sv));
  sv->Mh = PC.p.Mh;
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

int rowlap_run(const float *x, int64_t ldx, float *V, int64_t ldv, float *vrows, int64_t h,
               int64_t w, const double *b, const double *a, int k, double b0, int sign,
               const double *cb_, const double *ca, double cb0, int csign, cudaStream_t st) {
  static RowLapPlan P, PC;  // (large: not on the stack)
  static SegVec sv;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  int rc = rowlap_get_plan(h, w, b, a, k, b0, sign, &P);
  if (rc) return rc;
  // the column stage's modal form and border length along the columns
  rc = rowlap_get_plan(w, h, cb_, ca, k, cb0, csign, &PC);
  if (rc) return rc;
  if (PC.kind != P.kind) return fail(VMF_EVALUE, "fp32 path: stages of different structure");
  rc = seg_vectors(cb_, ca, k, PC, &sv);
  if (rc) return rc;
  if (P.kind == M32_CPAIR) return launch_rowlap<2, M32_CPAIR>(x, ldx, V, ldv, vrows, P, PC, sv, st);
  switch (k) {
    case 2: return launch_rowlap<2, M32_JORDAN>(x, ldx, V, ldv, vrows, P, PC, sv, st);
    case 3: return launch_rowlap<3, M32_JORDAN>(x, ldx, V, ldv, vrows, P, PC, sv, st);
    case 4: return launch_rowlap<4, M32_JORDAN>(x, ldx, V, ldv, vrows, P, PC, sv, st);
  }
  return fail(VMF_EVALUE, "fp32 row pass supports K = 2..4, got %d", k);
}

}  // namespace vmf
