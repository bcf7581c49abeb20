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
#include <map>
#include <cstdlib>
#include <cstring>

#include "vmf_common.cuh"
#include "vmf_dfi.cuh"
#include "vmf_iir.cuh"
#include "vmf_prof.cuh"
#include "vmf_rowpass.cuh"
#include "plan_cache.hpp"
#include "vmf_tma.cuh"

namespace vmf {

// ---------------------------------------------------------------------------
// shared-memory row layouts
// ---------------------------------------------------------------------------
__device__ __forceinline__ int sidx(int n) { return n + 4 * (n >> 5); }

// Padded layout (cp.async staging): a 4-float pad after every 32 samples, so
// thread c reading chunk c with 16-byte loads is bank-conflict free.
struct PadRow {
  float *xr;
  __device__ float4 ld4(int c, int q) const {
    return *reinterpret_cast<const float4 *>(xr + 36 * c + 4 * q);
  }
  __device__ void st4(int c, int q, float4 v) const {
    *reinterpret_cast<float4 *>(xr + 36 * c + 4 * q) = v;
  }
  __device__ float ld(int n) const { return xr[sidx(n)]; }
};

// TMA SWIZZLE_128B layout of a [C][32] fp32 box: 16-byte unit q of chunk c
// sits at unit q ^ (c & 7) of the chunk's 128 bytes (1024-byte aligned base),
// which is again conflict free for per-chunk 16-byte loads.
struct SwzRow {
  char *base;
  __device__ int off(int c, int q) const { return c * 128 + ((q ^ (c & 7)) << 4); }
  __device__ float4 ld4(int c, int q) const {
    return *reinterpret_cast<const float4 *>(base + off(c, q));
  }
  __device__ void st4(int c, int q, float4 v) const {
    *reinterpret_cast<float4 *>(base + off(c, q)) = v;
  }
  __device__ float ld(int n) const {
    return *reinterpret_cast<const float *>(base + off(n >> 5, (n >> 2) & 7) + 4 * (n & 3));
  }
};

// ---------------------------------------------------------------------------
// the three phases of one row (thread = chunk c of row rr)
// ---------------------------------------------------------------------------
// b. zero-state chunk carries (folded sample pairs) -> scan inputs d_c =
//    Yzs_c + Tx X_{c-1} in cf / cb (x history before the chunk in scan
//    order; the first chunk adds Ty E_{-1}, E_{-1} = yss * end sample).
template <int K, class Row>
__device__ __forceinline__ void row_carry(const RowParams &p, const Row &xr, int c, int C, int Wp,
                                          double *cfr, double *cbr) {
  double P[K], Q[K];
#pragma unroll
  for (int i = 0; i < K; ++i) P[i] = Q[i] = 0.0;
  float xv[kChunk];  // fp32 copies; the pair sums are formed in fp64
#pragma unroll
  for (int q = 0; q < kChunk / 4; ++q) {
    float4 v = xr.ld4(c, q);
    xv[4 * q] = v.x;
    xv[4 * q + 1] = v.y;
    xv[4 * q + 2] = v.z;
    xv[4 * q + 3] = v.w;
  }
#pragma unroll
  for (int t = 0; t < kChunk / 2; ++t) {
    // pair sums in fp32 (one conversion per sum instead of per sample; the
    // rounding is that of an fp32 input)
    const double u = (double)(xv[t] + xv[kChunk - 1 - t]);
    const double v = (double)(xv[t] - xv[kChunk - 1 - t]);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      P[i] = fma(p.SP32[i][t], u, P[i]);
      Q[i] = fma(p.SQ32[i][t], v, Q[i]);
    }
  }
  const int n0 = c * kChunk;
  double Xf[K], Xb[K];
  const double x0 = (double)xr.ld(0), xl = (double)xr.ld(Wp - 1);
#pragma unroll
  for (int i = 0; i < K; ++i) {
    Xf[i] = c > 0 ? (double)xr.ld(n0 - 1 - i) : x0;
    Xb[i] = c < C - 1 ? (double)xr.ld(n0 + kChunk + i) : xl;
  }
#pragma unroll
  for (int i = 0; i < K; ++i) {
    double df = P[i] + Q[i], db = P[i] - Q[i];
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
    cfr[c * K + i] = df;
    cbr[c * K + i] = db;
  }
}

// c. scan of one (row, direction) by one warp: E_c = d_c + Ty E_{c-1}
//    (c in scan order; the backward direction scans chunks from the right
//    end).  Lane l owns cpl consecutive chunks: local sequential scan,
//    Kogge-Stone across lanes with Ty^(cpl*2^j), then a sequential re-scan
//    from the carry-in.  Leaves the END history of every chunk in cc.
template <int K>
__device__ __forceinline__ void row_scan(const RowParams &p, double *cc, int dir, int C, int lane) {
  const int cpl = p.cpl;
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
        cc[ch * K + i] = En[i];
      }
    }
  }
}

// d. apply, backward half: DF-I recursion from the true history, sign*y-
//    parked in 32 fp32 registers per row (its rounding is smoothed away by
//    the column pass, tools/experiments/park_precision.py); also returns the
//    forward start history.  Reads only x.  NR rows are walked in lockstep so
//    the scheduler sees NR independent recursion chains.
template <int K, int NR, class Row, typename PT>
__device__ __forceinline__ void row_apply_bwd(const RowParams &p, const Row *xr, int c, int C,
                                              int Wp, double *const *cfr, double *const *cbr,
                                              PT (*park)[kChunk], double (*Xf)[K],
                                              double (*Yf)[K]) {
  const int n0 = c * kChunk;
  double Xb[NR][K], Yb[NR][K];
#pragma unroll
  for (int g = 0; g < NR; ++g) {
    const double xl = (double)xr[g].ld(Wp - 1), x0 = (double)xr[g].ld(0);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      int qb = n0 + kChunk + i;
      Xb[g][i] = (double)xr[g].ld(qb > Wp - 1 ? Wp - 1 : qb);
      Yb[g][i] = p.sign * (c < C - 1 ? cbr[g][(c + 1) * K + i] : p.yss * xl);  // of sign*y-
      int qf = n0 - 1 - i;
      Xf[g][i] = (double)xr[g].ld(qf < 0 ? 0 : qf);
      Yf[g][i] = c > 0 ? cfr[g][(c - 1) * K + i] : p.yss * x0;
    }
  }
  DfiRun<K> rb[NR];
#pragma unroll
  for (int g = 0; g < NR; ++g) rb[g].init(p.bwd, Yb[g], Xb[g]);
#pragma unroll
  for (int q = kChunk / 4 - 1; q >= 0; --q) {
    float e[NR][4];
#pragma unroll
    for (int g = 0; g < NR; ++g) {
      float4 v = xr[g].ld4(c, q);
      e[g][0] = v.x;
      e[g][1] = v.y;
      e[g][2] = v.z;
      e[g][3] = v.w;
    }
#pragma unroll
    for (int u = 3; u >= 0; --u) {
#pragma unroll
      for (int g = 0; g < NR; ++g) {
        park[g][4 * q + u] = (PT)rb[g].step(p.bwd, (double)e[g][u]);  // sign*y-
      }
    }
  }
}

// d. apply, forward half: out(n) = b0 x + y+ + parked sign*y-, in place.
template <int K, int NR, class Row, typename PT>
__device__ __forceinline__ void row_apply_fwd(const RowParams &p, const Row *xr, int c,
                                              const PT (*park)[kChunk], double (*Xf)[K],
                                              double (*Yf)[K]) {
  DfiRun<K> rf[NR];
#pragma unroll
  for (int g = 0; g < NR; ++g) rf[g].init(p, Yf[g], Xf[g]);
#pragma unroll
  for (int q = 0; q < kChunk / 4; ++q) {
    float e[NR][4], o[NR][4];
#pragma unroll
    for (int g = 0; g < NR; ++g) {
      float4 v = xr[g].ld4(c, q);
      e[g][0] = v.x;
      e[g][1] = v.y;
      e[g][2] = v.z;
      e[g][3] = v.w;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int g = 0; g < NR; ++g) {
        const double xv = (double)e[g][u];
        const double s = rf[g].step(p, xv);
        o[g][u] = (float)(fma(p.b0, xv, s) + (double)park[g][4 * q + u]);
      }
    }
#pragma unroll
    for (int g = 0; g < NR; ++g) xr[g].st4(c, q, make_float4(o[g][0], o[g][1], o[g][2], o[g][3]));
  }
}

// ---------------------------------------------------------------------------
// kernel 1: one CTA = R whole rows, staged with cp.async (any width / dtype)
// ---------------------------------------------------------------------------
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
  } else if (sizeof(T) < 4 && p.vec8) {  // integer samples: 8 per vector load
    for (int r = 0; r < nrows; ++r)
      for (int n = 8 * tid; n < W; n += 8 * blockDim.x) {
        float o[8];
        ld8f(x + (row0 + r) * ldx + n, o);
        float *d = xs + r * rowf + sidx(n);  // 8 samples of one 32-chunk: contiguous
        *reinterpret_cast<float4 *>(d) = make_float4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<float4 *>(d + 4) = make_float4(o[4], o[5], o[6], o[7]);
      }
  } else {
    for (int r = 0; r < nrows; ++r)
      for (int n = tid; n < W; n += blockDim.x)
        xs[r * rowf + sidx(n)] = ldf32(x + (row0 + r) * ldx + n);
  }
  __syncthreads();
  // Each row is padded to C*32 samples with copies of x[W-1]: a steady state
  // fed a constant stays steady, so the backward recursion may start at the
  // padded end in the steady state of x[W-1].
  for (int r = 0; r < nrows; ++r)
    for (int n = W + tid; n < Wp; n += blockDim.x) xs[r * rowf + sidx(n)] = xs[r * rowf + sidx(W - 1)];
  __syncthreads();

  const bool active = rr < nrows;
  const PadRow xr{xs + rr * rowf};
  if (active) row_carry<K>(p, xr, c, C, Wp, cf + rr * C * K, cb + rr * C * K);
  __syncthreads();
  {
    const int lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    for (int task = warp; task < 2 * nrows; task += nwarps) {
      const int r = task >> 1, dir = task & 1;
      row_scan<K>(p, (dir == 0 ? cf : cb) + r * C * K, dir, C, lane);
      __syncwarp();
    }
  }
  __syncthreads();
  float park[1][kChunk];
  double Xf[1][K], Yf[1][K];
  double *cfr[1] = {cf + rr * C * K}, *cbr[1] = {cb + rr * C * K};
  if (active) row_apply_bwd<K, 1>(p, &xr, c, C, Wp, cfr, cbr, park, Xf, Yf);
  __syncthreads();  // every halo read before any chunk is overwritten
  if (active) row_apply_fwd<K, 1>(p, &xr, c, (const float(*)[kChunk])park, Xf, Yf);
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

#ifdef VMF_PHASE_PROF
__device__ unsigned long long g_row_phase[8];
#define PH(i)                                                        \
  do {                                                               \
    if (c == 0) {                                                    \
      long long t_ = clock64();                                      \
      atomicAdd(&g_row_phase[i], (unsigned long long)(t_ - ph_t0)); \
      ph_t0 = t_;                                                    \
    }                                                                \
  } while (0)
#else
#define PH(i) \
  do {        \
  } while (0)
#endif

// ---------------------------------------------------------------------------
// kernel 2 (fp32, W = 32 C): persistent, NR rows per step, TMA in and out.
// A step's rows are one SWIZZLE_128B box [NR][C][32]; the box of the next
// step is loaded while the current one is computed, and the result leaves
// with a TMA store from the same buffer (two buffers, one mbarrier each).
// With NR = 2 every thread walks two independent recursions and the four
// (row, direction) scans keep all four warps busy.
// ---------------------------------------------------------------------------
template <int K, int NR, int NBUF>
__global__ void __launch_bounds__(kRowThreads, NR == 1 ? (NBUF == 2 ? 5 : 4) : 3)
    rowpass_tma_kernel(const __grid_constant__ CUtensorMap xmap,
                       const __grid_constant__ CUtensorMap ymap, RowParams p) {
  extern __shared__ __align__(1024) unsigned char smem_tma[];
  __shared__ __align__(8) uint64_t bar[NBUF];
  const int C = p.C, Wp = C * kChunk;
  const int rowb = Wp * (int)sizeof(float);
  const int stepb = NR * rowb;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem_tma);
  char *buf0 = reinterpret_cast<char *>(smem_tma) + ((1024u - (sbase & 1023u)) & 1023u);
  double *cf = reinterpret_cast<double *>(buf0 + NBUF * stepb);  // [NR][C][K]
  double *cb = cf + NR * C * K;
  const int c = threadIdx.x;
  const int64_t H = p.H;
  const int64_t per = p.rows_per;  // multiple of NR
  const int64_t rlo = (int64_t)blockIdx.x * per;
  const int64_t rhi = rlo + per < H ? rlo + per : H;
  if (rlo >= rhi) return;
  // x may come from the kernel just before this one on the stream (a dtype
  // conversion, say): wait for it before the prologue reads it
  pdl_wait();
  if (c == 0) {
    for (int q = 0; q < NBUF; ++q) mbar_init(&bar[q], 1);
    // prologue: the first NBUF-1 steps in flight
    for (int q = 0; q < NBUF - 1 && rlo + (int64_t)q * NR < rhi; ++q) {
      mbar_expect_tx(&bar[q], (unsigned)stepb);
      tma_load_3d_hint(buf0 + q * stepb, &xmap, &bar[q], 0, 0, (int)(rlo + (int64_t)q * NR),
                       l2_policy_evict_first());
    }
  }
  __syncthreads();
  int b = 0;
  unsigned phases = 0u;
  double *cfr[NR], *cbr[NR];
#pragma unroll
  for (int g = 0; g < NR; ++g) {
    cfr[g] = cf + g * C * K;
    cbr[g] = cb + g * C * K;
  }
#ifdef VMF_PHASE_PROF
  long long ph_t0 = clock64();
#endif
  for (int64_t r = rlo; r < rhi; r += NR, b = (b + 1 == NBUF ? 0 : b + 1)) {
    SwzRow xr[NR];
#pragma unroll
    for (int g = 0; g < NR; ++g) xr[g].base = buf0 + b * stepb + g * rowb;
    mbar_wait(&bar[b], (phases >> b) & 1u);
    phases ^= 1u << b;
    PH(0);
#pragma unroll
    for (int g = 0; g < NR; ++g) row_carry<K>(p, xr[g], c, C, Wp, cfr[g], cbr[g]);
    __syncthreads();
    PH(1);
    const int64_t rn = r + (int64_t)(NBUF - 1) * NR;  // the step this refill serves
    if (c == 0 && rn < rhi) {
      // buffer bn last held the previous step, whose TMA store was issued a
      // full step ago: wait until it has been read out, then refill
      const int bn = b == 0 ? NBUF - 1 : b - 1;
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      mbar_expect_tx(&bar[bn], (unsigned)stepb);
      tma_load_3d_hint(buf0 + bn * stepb, &xmap, &bar[bn], 0, 0, (int)rn,
                       l2_policy_evict_first());
    }
    for (int task = c >> 5; task < 2 * NR; task += (int)(blockDim.x >> 5))
      row_scan<K>(p, (task & 1) == 0 ? cfr[task >> 1] : cbr[task >> 1], task & 1, C, c & 31);
    __syncthreads();
    PH(2);
#ifdef VMF_PARK32
    typedef float ParkT;
#else
    typedef double ParkT;  // fp64 park: no F2F pair per sample (the XU pipe is the busy one)
#endif
    ParkT park[NR][kChunk];
    double Xf[NR][K], Yf[NR][K];
    row_apply_bwd<K, NR>(p, xr, c, C, Wp, cfr, cbr, park, Xf, Yf);
    __syncthreads();  // every halo read (and cf / cb) before chunks are overwritten
    PH(3);
    row_apply_fwd<K, NR>(p, xr, c, (const ParkT(*)[kChunk])park, Xf, Yf);
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> TMA
    __syncthreads();
    PH(4);
    if (c == 0) {
      if (r == rlo) pdl_wait();  // T may still be read by the previous scale's column pass
      tma_store_3d_hint(&ymap, buf0 + b * stepb, 0, 0, (int)r, l2_policy_evict_last());
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
    PH(5);
  }
  pdl_trigger();
  if (c == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
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
  for (int m = 0; m < k; ++m) {
    p->bwd.b[m] = ip.sign * ip.b[m];
    p->bwd.a[m] = ip.a[m];
  }
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
  static PerDevice attr;
  if (attr.first()) {
    cudaFuncSetAttribute(rowpass_kernel<K, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
  }
  p.vec4 = (sizeof(T) == 4) && (p.W % 4 == 0) && (ldx % 4 == 0) && (ldy % 4 == 0) &&
           ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0);
  if (sizeof(T) != 4) p.vec4 = (p.W % 4 == 0) && (ldy % 4 == 0) && ((uintptr_t)y % 16 == 0);
  p.vec8 = (sizeof(T) < 4) && (p.W % 8 == 0) && (ldx % 8 == 0) &&
           ((uintptr_t)x % (8 * sizeof(T)) == 0);
  int grid = (int)cdiv(p.H, p.R);
  Launch g(K_IIR_ROWS_FUSED, st);
  rowpass_kernel<K, T><<<grid, p.R * p.C, smem, st>>>(x, ldx, y, ldy, p);
  return cuda_status("row pass");
}

// Persistent TMA variant: fp32, w = 32 C exactly (no padding), aligned
// pitches; NR = 2 rows per step when the height is even.
template <int K, int NR, int NBUF>
static int launch_rowpass_tma(const CUtensorMap &xm, const CUtensorMap &ym, RowParams p,
                              cudaStream_t st) {
  const size_t smem = 1024 + NBUF * (size_t)NR * p.C * kChunk * sizeof(float) +
                      2 * (size_t)NR * p.C * K * sizeof(double);
  // resident CTAs over the device: per device and per shared-memory size
  // (the width sets the CTA's footprint)
  static std::map<std::pair<int, size_t>, int> slot_cache;
  const int dev_now = current_device();
  int &slots = slot_cache[std::make_pair(dev_now, smem)];
  if (!slots) {
    cudaFuncSetAttribute(rowpass_tma_kernel<K, NR, NBUF>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int occ = 0, dev = dev_now, nsm = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rowpass_tma_kernel<K, NR, NBUF>,
                                                  kRowThreads, smem);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaGetLastError();
    slots = (occ > 0 ? occ : 1) * nsm;
  }
  // equal row counts per CTA (a multiple of NR)
  p.rows_per = cdiv(cdiv(p.H, slots), NR) * NR;
  const int grid = (int)cdiv(p.H, p.rows_per);
  Launch g(K_IIR_ROWS_FUSED, st);
  launch_pdl(rowpass_tma_kernel<K, NR, NBUF>, dim3(grid), dim3(p.C), smem, st, xm, ym, p);
  return cuda_status("row pass");
}

template <int K>
static int launch_rowpass_tma_any(const float *x, int64_t ldx, float *y, int64_t ldy,
                                  const RowParams &p, cudaStream_t st, bool *done) {
  // NR = 2 (two interleaved rows per thread) needs twice the registers and
  // shared memory and measured slower on B200 (2 CTAs/SM instead of 5);
  // VMF_ROW_NR2 selects it for experiments.
  const int nr = (p.H % 2 == 0 && getenv("VMF_ROW_NR2")) ? 2 : 1;
  CUtensorMap xm, ym;
  memset(&xm, 0, sizeof(xm));
  memset(&ym, 0, sizeof(ym));
  *done = make_tmap_rows_swz_f32(&xm, x, p.H, p.W, ldx, nr) &&
          make_tmap_rows_swz_f32(&ym, y, p.H, p.W, ldy, nr);
  cudaGetLastError();
  if (!*done) return VMF_OK;
  if (nr == 2) return launch_rowpass_tma<K, 2, 2>(xm, ym, p, st);
  static const bool three = getenv("VMF_ROW_NBUF3") != nullptr;  // experiment: prefetch 2 ahead
  return three ? launch_rowpass_tma<K, 1, 3>(xm, ym, p, st) : launch_rowpass_tma<K, 1, 2>(xm, ym, p, st);
}

template <typename T>
int rowpass_run(const T *x, int64_t ldx, float *y, int64_t ldy, const IirParams &ip, int64_t h,
                int64_t w, cudaStream_t st) {
  RowParams p;
  {
    static PlanCache<RowParams> cache;
    std::vector<unsigned char> key;
    key_add(key, h);
    key_add(key, w);
    key_add(key, ip.K);
    key_add(key, ip.b0);
    key_add(key, ip.sign);
    key_add(key, ip.b, sizeof(double) * ip.K);
    key_add(key, ip.a, sizeof(double) * ip.K);
    if (!cache.get(key, &p)) {
      rowpass_plan(&p, ip, h, w);
      cache.put(key, p);
    }
  }
  if (sizeof(T) == 4 && w == (int64_t)p.C * kChunk && p.C >= 32 && p.C <= kRowThreads &&
      !getenv("VMF_ROW_NO_TMA")) {
    const float *xf = (const float *)x;
    bool done = false;
    int rc = VMF_OK;
    switch (ip.K) {
      case 1: rc = launch_rowpass_tma_any<1>(xf, ldx, y, ldy, p, st, &done); break;
      case 2: rc = launch_rowpass_tma_any<2>(xf, ldx, y, ldy, p, st, &done); break;
      case 3: rc = launch_rowpass_tma_any<3>(xf, ldx, y, ldy, p, st, &done); break;
      case 4: rc = launch_rowpass_tma_any<4>(xf, ldx, y, ldy, p, st, &done); break;
      case 5: rc = launch_rowpass_tma_any<5>(xf, ldx, y, ldy, p, st, &done); break;
      case 6: rc = launch_rowpass_tma_any<6>(xf, ldx, y, ldy, p, st, &done); break;
      case 7: rc = launch_rowpass_tma_any<7>(xf, ldx, y, ldy, p, st, &done); break;
      case 8: rc = launch_rowpass_tma_any<8>(xf, ldx, y, ldy, p, st, &done); break;
    }
    if (done) return rc;
  }
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
template int rowpass_run<uint8_t>(const uint8_t *, int64_t, float *, int64_t, const IirParams &,
                                  int64_t, int64_t, cudaStream_t);
template int rowpass_run<u16be>(const u16be *, int64_t, float *, int64_t, const IirParams &,
                                int64_t, int64_t, cudaStream_t);

}  // namespace vmf

#ifdef VMF_PHASE_PROF
extern "C" int vmf_debug_row_phases(double *out, int n) {
  unsigned long long h[8] = {0};
  cudaMemcpyFromSymbol(h, vmf::g_row_phase, sizeof(h));
  unsigned long long z[8] = {0};
  cudaMemcpyToSymbol(vmf::g_row_phase, z, sizeof(z));
  for (int i = 0; i < n && i < 8; ++i) out[i] = (double)h[i];
  return 8;
}
#endif
