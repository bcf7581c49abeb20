// vmf_firpass.cu -- the FIR blur of the hot path on B200 (SURVEY.md §8 a3/a4,
// north star: "a tiled shared-memory FIR kernel ... for impulse responses up
// to hundreds of taps" and the fused second pass + Laplacian + NMS).
//
//   out(n) = sum_{m=-k..k} taps[k+m] x(clamp(n-m))   (_conv_rows_kernel,
//   engine.py:35-62; conv_cols engine.py:124-126 for the columns)
//
// fp64 accumulation (a 257-tap Gaussian misses the 1e-4 Laplacian tolerance
// with fp32 accumulation), fp32 in and out.  Both kernels
// are register-blocked: a thread owns 8 consecutive outputs along the filter
// direction and slides a 16-value fp64 window over the staged input, so every
// input read from shared memory feeds 8 DFMAs and every tap (a uniform
// constant-bank load) feeds 8 DFMAs; the FMA pipe, not the LSU, is the limit.
//
// fir_rows_fast_kernel: CTA = 1024 outputs of one row; the input window (1024
//   + taps, edge-clamped) is staged in shared memory once.
// firapply_kernel: the column pass fused with the Laplacian and detection:
//   CTA = 128 computed (124 owned) columns x 32 B rows (28 owned L rows).  The
//   column window (32 + taps rows x 132 columns, edge-clamped, fp32) is staged
//   with cp.async; B is kept in fp64 in shared memory (it never rounds to fp32
//   before the Laplacian), L = lsc (Bl + Br + Bu + Bd - 4 Bc) is formed from it
//   with replicate edges, and the owned block is stored as float4 rows fused
//   with the strict 3x3 NMS over frac * max(CTA max, global max so far) -- the
//   same candidate protocol as the IIR column pass, finished by colfinal.
#include <cstdlib>
#include <cstring>

#include "vmf_colpass.cuh"
#include "vmf_common.cuh"
#include "vmf_firpass.cuh"
#include "vmf_prof.cuh"
#include "vmf_tma.cuh"

namespace vmf {

constexpr int kFirTapsPad = kFirMaxFast + 15;  // reversed taps, zero-padded to a multiple of 8

struct FirTapsP {
  double t[kFirTapsPad];  // t[i] = taps[n-1-i] (i < n), 0 beyond
  int n, np;              // taps; rounded up to a multiple of 8 (window sizes)
};

static void fir_plan(FirTapsP *tp, const double *taps, int ntaps) {
  memset(tp, 0, sizeof(*tp));
  for (int i = 0; i < ntaps; ++i) tp->t[i] = taps[ntaps - 1 - i];
  tp->n = ntaps;
  tp->np = (ntaps + 7) / 8 * 8;
}

// acc[j] += sum_i t[i] * w(base + j + i), w(q) read through `ld` (fp32 -> fp64)
template <class LD>
__device__ __forceinline__ void fir8(const FirTapsP &tp, LD ld, double *acc) {
  double xw[16];
#pragma unroll
  for (int j = 0; j < 8; ++j) xw[j] = ld(j);
  auto block8 = [&](int mb) {
#pragma unroll
    for (int j = 0; j < 8; ++j) xw[8 + j] = ld(mb + 8 + j);
#pragma unroll
    for (int mm = 0; mm < 8; ++mm) {
      const double tap = tp.t[mb + mm];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = fma(tap, xw[j + mm], acc[j]);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) xw[j] = xw[8 + j];
  };
  int mb = 0;
  for (; mb + 8 <= tp.n; mb += 8) block8(mb);
  // the last n % 8 taps without padding DFMAs: 2k + 1 taps with k % 4 == 0
  // (every Gaussian / SG kernel of the configs) leave exactly one, whose
  // samples are already in the window; 2..4 use a half block; 5..7 one more
  // full block over the zero-padded taps
  const int rem = tp.n - mb;
  if (rem == 1) {
    const double tap = tp.t[mb];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = fma(tap, xw[j], acc[j]);
  } else if (rem > 1 && rem <= 4) {
#pragma unroll
    for (int j = 0; j < 4; ++j) xw[8 + j] = ld(mb + 8 + j);
#pragma unroll
    for (int mm = 0; mm < 4; ++mm) {
      const double tap = tp.t[mb + mm];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = fma(tap, xw[j + mm], acc[j]);
    }
  } else if (rem > 4) {
    block8(mb);
  }
}

// ---------------------------------------------------------------------------
// row pass
// ---------------------------------------------------------------------------
constexpr int kFrSeg = 1024, kFrThreads = 128;

template <typename T>
__global__ void __launch_bounds__(kFrThreads) fir_rows_fast_kernel(const T *__restrict__ x,
                                                                   int64_t ldx,
                                                                   float *__restrict__ y,
                                                                   int64_t ldy, int64_t h,
                                                                   int64_t w, FirTapsP tp,
                                                                   int vec_out, int vec_in) {
  extern __shared__ __align__(16) float fwin_raw[];  // [kFrSeg + np + 16]
  const int k = (tp.n - 1) / 2;
  const int nwin = kFrSeg + tp.np + 16;
  const int64_t n0 = (int64_t)blockIdx.x * kFrSeg;
  const int base = 8 * threadIdx.x;
  // window sample q = image column s0 + q at fwin[q]; with s0 a multiple of
  // 4 (k % 4 == 0: every Gaussian / SG kernel of the configs) the window is
  // staged in 16-byte units.  fwin stays 16-byte aligned either way: the
  // 8-output register blocks then read it as LDS.128.
  const int64_t s0 = n0 - k;
  const int nv = (nwin + 3) / 4;
  const bool vec = sizeof(T) == 4 && vec_in && (k & 3) == 0;
  // units entirely inside the row: [vlo, vhi)
  const int vlo = s0 >= 0 ? 0 : (int)((3 - s0) / 4);
  const int vhi = (int)((w - s0) / 4 < nv ? (w - s0) / 4 : nv);
  float *fwin = fwin_raw;
  for (int64_t row = blockIdx.y; row < h; row += gridDim.y) {
    __syncthreads();
    const T *xr = x + row * ldx;
    if (vec) {  // 16-byte asynchronous copies; units crossing an edge are clamped per sample
      const float *xf = reinterpret_cast<const float *>(xr);
      const float *src = xf + s0;  // unit v = samples s0 + 4v .. s0 + 4v + 3
      for (int v = threadIdx.x; v < nv; v += blockDim.x) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(fwin_raw + 4 * v);
        if (v >= vlo && v < vhi) {
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src + 4 * v));
        } else {
          const int64_t g = s0 + 4 * v;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int64_t c = g + e < 0 ? 0 : (g + e >= w ? w - 1 : g + e);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa + 4 * e),
                         "l"(xf + c));
          }
        }
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
    } else if (sizeof(T) == 4) {  // asynchronous 4-byte copies: the whole window in flight at once
      for (int q = threadIdx.x; q < nwin; q += blockDim.x) {
        int64_t c = s0 + q;
        c = c < 0 ? 0 : (c >= w ? w - 1 : c);
        const unsigned sa = (unsigned)__cvta_generic_to_shared(fwin + q);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(xr + c));
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
    } else {
      for (int q = threadIdx.x; q < nwin; q += blockDim.x) {
        int64_t c = s0 + q;
        c = c < 0 ? 0 : (c >= w ? w - 1 : c);
        fwin[q] = ldf32(xr + c);
      }
    }
    __syncthreads();
    if (n0 + base >= w) continue;
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0;
    const float *wp = fwin + base;
    fir8(tp, [&](int q) { return (double)wp[q]; }, acc);
    float *yr = y + row * ldy + n0 + base;
    if (vec_out && n0 + base + 8 <= w) {
      reinterpret_cast<float4 *>(yr)[0] = make_float4((float)acc[0], (float)acc[1],
                                                       (float)acc[2], (float)acc[3]);
      reinterpret_cast<float4 *>(yr)[1] = make_float4((float)acc[4], (float)acc[5],
                                                       (float)acc[6], (float)acc[7]);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (n0 + base + j < w) yr[j] = (float)acc[j];
    }
  }
}

template <typename T>
int fir_rows_fast(const T *x, int64_t ldx, float *y, int64_t ldy, int64_t h, int64_t w,
                  const double *taps, int ntaps, cudaStream_t st) {
  FirTapsP tp;
  fir_plan(&tp, taps, ntaps);
  const size_t smem = (size_t)(kFrSeg + tp.np + 16) * sizeof(float);
  const int vec = (ldy % 4 == 0) && ((uintptr_t)y % 16 == 0);
  const int vin = (ldx % 4 == 0) && ((uintptr_t)x % 16 == 0);
  dim3 grid((unsigned)cdiv(w, kFrSeg), (unsigned)(h < 65535 ? h : 65535));
  Launch g(K_FIR_ROWS, st);
  fir_rows_fast_kernel<T><<<grid, kFrThreads, smem, st>>>(x, ldx, y, ldy, h, w, tp, vec, vin);
  return cuda_status("fir row pass");
}

template int fir_rows_fast<float>(const float *, int64_t, float *, int64_t, int64_t, int64_t,
                                  const double *, int, cudaStream_t);
template int fir_rows_fast<uint8_t>(const uint8_t *, int64_t, float *, int64_t, int64_t, int64_t,
                                    const double *, int, cudaStream_t);
template int fir_rows_fast<u16be>(const u16be *, int64_t, float *, int64_t, int64_t, int64_t,
                                  const double *, int, cudaStream_t);
template int fir_rows_fast<uint16_t>(const uint16_t *, int64_t, float *, int64_t, int64_t,
                                     int64_t, const double *, int, cudaStream_t);

// ---------------------------------------------------------------------------
// fused column pass
// ---------------------------------------------------------------------------
// Tile shapes: COLS computed columns (COLS-4 owned), GROUPS groups of 8 B rows
// (8 GROUPS - 4 owned L rows).  Every tap count uses 64 x 8 (512 threads):
// the 2k-row halo of the column window is shared by 60 B rows.  Measured per
// scale on 4096^2 (tools/fir_ab.py): 64 x 4 ties at 33 taps and is 9-23 %
// slower at 17 and >= 65 taps; 128 x 4, 32 x 8 and 64 x 16 are slower at
// every tap count.
template <int COLS, int GROUPS>
struct FcShape {
  static constexpr int kCols = COLS, kOut = COLS - 4, kGroups = GROUPS;
  static constexpr int kThreads = COLS * GROUPS;
  static constexpr int kRB = 8 * GROUPS;  // B rows r0-2 .. r0+kRB-3
  static constexpr int kOwn = kRB - 4;    // owned L rows r0 .. r0+kOwn-1
  static constexpr int kLR = kRB - 2;     // L rows r0-1 .. r0+kOwn
  static constexpr int kStride = COLS + 4;
  static size_t region_bytes(int np) {
    const size_t win = (size_t)(kRB + np + 8) * kStride * sizeof(float);
    const size_t bl = (size_t)kRB * kCols * sizeof(double) + (size_t)kLR * kStride * sizeof(float);
    return win > bl ? win : bl;
  }
};
using FcLong = FcShape<64, 8>;
constexpr int kFcCand = 256;

struct FcSmall {
  int cy[kFcCand], cx[kFcCand];
  float cv[kFcCand];
  int ccount;
  unsigned cmax;
  float thr_end;
};

// Hessian detector outputs (MODE 1, blob.py:109-128,158-163)
struct HessOut {
  double sigma4, t1;
  int polarity;           // +1 dark (trace > 0), -1 bright (trace < 0)
  float *nd_field;        // nullable: sigma^4 (D20 D02 - D11^2), pitch ldn
  float *trace_field;     // nullable: D20 + D02
  int64_t ldn;
  int *cy, *cx;           // candidates: nd > t1 with the polarity
  double *cnd;
  float *cdx, *cdy;       // stationary-point displacement (NaN if |det| < 1e-12)
  int cap;
  int *count;             // appended candidates (may exceed cap: overflow)
  float *deriv[6];        // MODE 2: D00 D10 D01 D20 D02 D11 (pitch ldn), any may be null
};

// Owned pixels of a fused FIR tile -> derivative bank fir_vm_bank(3) of B
// (replicate edges: rows clamped here, columns by the clamped inputs), the
// scale-normalised Hessian determinant, trace and displacement; candidates
// appended with one atomic per warp.
template <class SH>
__device__ __forceinline__ void hess_tile(const double *Bs, int64_t r0, int64_t c0, int64_t H,
                                          int64_t W, const HessOut &ho) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t rB0 = r0 - 2;
  for (int base = 0; base < SH::kOwn * SH::kOut; base += SH::kThreads) {
    const int idx = base + tid;
    bool cand = false;
    int64_t r = 0, c = 0;
    double nd = 0.0, dxv = 0.0, dyv = 0.0;
    if (idx < SH::kOwn * SH::kOut) {
      const int q = idx / SH::kOut, cl = idx - q * SH::kOut;
      r = r0 + q;
      c = c0 + cl;
      if (r < H && c < W) {
        const int jj = cl + 2;  // B tile column of image column c
        const int64_t tr = r - rB0;
        const int64_t tu = (r > 0 ? r - 1 : 0) - rB0, td = (r + 1 < H ? r + 1 : H - 1) - rB0;
        const double *rc = Bs + tr * SH::kCols + jj, *ru = Bs + tu * SH::kCols + jj,
                     *rd = Bs + td * SH::kCols + jj;
        // conv taps in the reference's accumulation order (m ascending)
        const double d10 = fma(-0.5, rc[-1], 0.5 * rc[1]);
        const double d01 = fma(-0.5, ru[0], 0.5 * rd[0]);
        const double d20 = (rc[1] - 2.0 * rc[0]) + rc[-1];
        const double d02 = (rd[0] - 2.0 * rc[0]) + ru[0];
        const double d10u = fma(-0.5, ru[-1], 0.5 * ru[1]), d10d = fma(-0.5, rd[-1], 0.5 * rd[1]);
        const double d11 = fma(-0.5, d10u, 0.5 * d10d);
        const double det = d20 * d02 - d11 * d11;
        nd = ho.sigma4 * det;
        const double tr2 = d20 + d02;
        if (ho.nd_field) ho.nd_field[r * ho.ldn + c] = (float)nd;
        if (ho.trace_field) ho.trace_field[r * ho.ldn + c] = (float)tr2;
        cand = nd > ho.t1 && (ho.polarity > 0 ? tr2 > 0.0 : tr2 < 0.0);
        if (cand) {
          if (fabs(det) < 1e-12) {
            dxv = dyv = __longlong_as_double(0x7ff8000000000000ll);
          } else {
            dxv = (d01 * d11 - d02 * d10) / det;
            dyv = (d10 * d11 - d20 * d01) / det;
          }
        }
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, cand);
    if (!bal) continue;
    int basek = 0;
    if (lane == 0) basek = atomicAdd(ho.count, __popc(bal));
    basek = __shfl_sync(0xffffffffu, basek, 0);
    if (cand) {
      const int k = basek + __popc(bal & ((1u << lane) - 1u));
      if (k < ho.cap) {
        ho.cy[k] = (int)r;
        ho.cx[k] = (int)c;
        ho.cnd[k] = nd;
        ho.cdx[k] = (float)dxv;
        ho.cdy[k] = (float)dyv;
      }
    }
  }
}

// MODE 2: the derivative bank fir_vm_bank(3) of the fp64 blur as fp32 images
// (engine.derivative_field, engine.py:205-228, in one pass)
template <class SH>
__device__ __forceinline__ void deriv_tile(const double *Bs, int64_t r0, int64_t c0, int64_t H,
                                           int64_t W, const HessOut &ho) {
  const int64_t rB0 = r0 - 2;
  for (int idx = threadIdx.x; idx < SH::kOwn * SH::kOut; idx += SH::kThreads) {
    const int q = idx / SH::kOut, cl = idx - q * SH::kOut;
    const int64_t r = r0 + q, c = c0 + cl;
    if (r >= H || c >= W) continue;
    const int jj = cl + 2;
    const int64_t tr = r - rB0;
    const int64_t tu = (r > 0 ? r - 1 : 0) - rB0, td = (r + 1 < H ? r + 1 : H - 1) - rB0;
    const double *rc = Bs + tr * SH::kCols + jj, *ru = Bs + tu * SH::kCols + jj,
                 *rd = Bs + td * SH::kCols + jj;
    const double d10u = fma(-0.5, ru[-1], 0.5 * ru[1]), d10d = fma(-0.5, rd[-1], 0.5 * rd[1]);
    const double v[6] = {rc[0],
                         fma(-0.5, rc[-1], 0.5 * rc[1]),
                         fma(-0.5, ru[0], 0.5 * rd[0]),
                         (rc[1] - 2.0 * rc[0]) + rc[-1],
                         (rd[0] - 2.0 * rc[0]) + ru[0],
                         fma(-0.5, d10u, 0.5 * d10d)};
    const int64_t o = r * ho.ldn + c;
#pragma unroll
    for (int d = 0; d < 6; ++d)
      if (ho.deriv[d]) ho.deriv[d][o] = (float)v[d];
  }
}

// One tile of the fused column pass on a staged window `fsm` (B and L reuse
// the window's space once the taps are done).  Every thread of the CTA calls
// it; it contains block barriers.
template <class SH, int MODE>
__device__ __forceinline__ void fc_tile(
    unsigned char *fsm, FcSmall &S, int64_t c0, int64_t r0, float *__restrict__ Lout, int64_t ldl,
    int64_t H, int64_t W, const FirTapsP &tp, float lap_scale, float frac,
    CandState *__restrict__ st, int *__restrict__ gy, int *__restrict__ gx, float *__restrict__ gv,
    int gcap, int vec_out, const HessOut &ho, float gbound) {
  const float *win = reinterpret_cast<const float *>(fsm);  // [kRB + np + 8][kStride]
  double *Bs = reinterpret_cast<double *>(fsm);              // [kRB][kCols]
  float *Ls = reinterpret_cast<float *>(fsm + (size_t)SH::kRB * SH::kCols * sizeof(double));
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int j = tid & (SH::kCols - 1), g = tid / SH::kCols;
  const int64_t rB0 = r0 - 2;  // image row of B tile row 0
  // ---- B rows 8g .. 8g+7 of column j (tile column j + 2) -------------------
  double acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0.0;
  {
    const float *wp = win + (8 * g) * SH::kStride + j + 2;
    fir8(tp, [&](int q) { return (double)wp[q * SH::kStride]; }, acc);
  }
  __syncthreads();  // the window is dead: B and L reuse its space
#pragma unroll
  for (int q = 0; q < 8; ++q) Bs[(8 * g + q) * SH::kCols + j] = acc[q];
  __syncthreads();
  if (MODE == 1) {
    hess_tile<SH>(Bs, r0, c0, H, W, ho);
    return;
  }
  if (MODE == 2) {
    deriv_tile<SH>(Bs, r0, c0, H, W, ho);
    return;
  }
  if (MODE == 3) {  // the conv_cols leaf: the owned blur rows, rounded to fp32
    for (int idx = tid; idx < SH::kOwn * SH::kOut; idx += SH::kThreads) {
      const int q = idx / SH::kOut, cl = idx - q * SH::kOut;
      const int64_t r = r0 + q, c = c0 + cl;
      if (r < H && c < W) Lout[r * ldl + c] = (float)Bs[(q + 2) * SH::kCols + cl + 2];
    }
    return;
  }
  // ---- L rows r0-1 .. r0+kOwn (B tile rows 1 .. kRB-2), replicate edges ---
  // Thread (g, j) forms L at its own 8 B rows: centre and (inside the group)
  // vertical neighbours from registers, horizontal ones from Bs.  Columns
  // outside the image were filtered from clamped inputs, so they already
  // hold the replicated edge column.
  const double lsc = (double)lap_scale;
  float tmax = 0.0f;
  // rows r0-1 .. r0+kOwn and their vertical neighbours all inside the image
  // (every tile but the first and last row band): no per-row edge logic
  const bool rows_in = rB0 >= 0 && rB0 + SH::kRB <= H;
  if (j != 0 && j != SH::kCols - 1 && rows_in) {
    const int64_t c = c0 - 2 + j;
    const bool cin = c >= 0 && c < W;
    const double *bcol = Bs + (8 * g) * SH::kCols + j;  // B(tile row 8g, column j)
    float *lcol = Ls + (8 * g - 1) * SH::kStride + j + 2;
    float m = 0.0f;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if ((q == 0 && g == 0) || (q == 7 && g == SH::kGroups - 1)) continue;  // tile rows 0, kRB-1
      const double bc = acc[q];
      const double bu = q > 0 ? acc[q - 1] : bcol[-SH::kCols];
      const double bd = q < 7 ? acc[q + 1] : bcol[8 * SH::kCols];
      const double bl = bcol[q * SH::kCols - 1], br = bcol[q * SH::kCols + 1];
      const float v = (float)(lsc * fma(-4.0, bc, (bl + br) + (bu + bd)));
      lcol[q * SH::kStride] = v;
      m = fmaxf(m, fabsf(v));
    }
    if (cin) tmax = m;
  } else if (j != 0 && j != SH::kCols - 1) {
    const int64_t c = c0 - 2 + j;
    const bool cin = c >= 0 && c < W;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int tr = 8 * g + q;
      if (tr == 0 || tr == SH::kRB - 1) continue;
      const int64_t r = rB0 + tr;
      if (r < 0 || r >= H) continue;
      const double bc = acc[q];
      const double bu = r == 0 ? bc : (q > 0 ? acc[q - 1] : Bs[(tr - 1) * SH::kCols + j]);
      const double bd = r + 1 >= H ? bc : (q < 7 ? acc[q + 1] : Bs[(tr + 1) * SH::kCols + j]);
      const double bl = Bs[tr * SH::kCols + j - 1], br = Bs[tr * SH::kCols + j + 1];
      const float v = (float)(lsc * fma(-4.0, bc, (bl + br) + (bu + bd)));
      Ls[(tr - 1) * SH::kStride + j + 2] = v;
      if (cin) tmax = fmaxf(tmax, fabsf(v));
    }
  }
  tmax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(tmax)));
  if (lane == 0) atomicMax(&S.cmax, __float_as_uint(tmax));
  pdl_trigger();
  __syncthreads();
  // publish this tile's max; the previous global max comes back while the
  // block is stored and only the flush needs it
  unsigned old = 0u;
  if (tid == 0) old = atomicMax(&st->absmax_bits, S.cmax);
  // ---- owned block out (float4 rows) + strict 3x3 NMS ---------------------
  {
    const int nrow = (int)(H - r0 < SH::kOwn ? H - r0 : SH::kOwn);
    const int ncol = (int)(W - c0 < SH::kOut ? W - c0 : SH::kOut);
    // frac <= 0: L only (scale-space stacks), no candidates
    const float th = frac > 0.0f ? frac * fmaxf(__uint_as_float(S.cmax), gbound)
                                 : __int_as_float(0x7f800000);
    auto test = [&](int q, int c, float v) -> bool {  // L tile row q + 1, tile column 4 + c
      const int64_t r = r0 + q, cc = c0 + c;
      if (r < 1 || r > H - 2 || cc < 1 || cc > W - 2) return false;
      const float *lp = Ls + (q + 1) * SH::kStride + 4 + c;
      bool gt = true, lt = true;
#pragma unroll
      for (int di = -1; di <= 1; ++di)
#pragma unroll
        for (int dj = -1; dj <= 1; ++dj) {
          if (!di && !dj) continue;
          const float u = lp[di * SH::kStride + dj];
          gt &= v > u;
          lt &= v < u;
        }
      // a maximum counts when L >= t, a minimum when -L >= t (|L| >= t alone
      // would admit a maximum of a negative region)
      return (gt && v >= th) || (lt && -v >= th);
    };
    // warp-ballot compaction over the lanes that reach it together
    auto push = [&](unsigned m, int q, int c, const float (&vv)[4]) {
      const unsigned mem = __activemask();
      cand_push_warp(&S.ccount, S.cy, S.cx, S.cv, kFcCand, st, gy, gx, gv, gcap, m,
                     (int)(r0 + q), (int)(c0 + c), vv, mem);
    };
    if ((vec_out || !Lout) && ncol == SH::kOut) {
      // a row is kOut / 4 float4 (15 for the 64-column tile): with <= 16 a
      // warp takes two rows per step (half-warps), else one.  (Lout null:
      // detections only, L never leaves the tile)
      constexpr int kRpw = SH::kOut / 4 <= 16 ? 2 : 1;
      const int u = kRpw == 2 ? (lane & 15) : lane;
      if (u < SH::kOut / 4) {
        float *dst = Lout ? Lout + r0 * ldl + c0 + 4 * u : nullptr;
        for (int q = kRpw * wid + (kRpw == 2 ? lane >> 4 : 0); q < nrow;
             q += kRpw * (SH::kThreads / 32)) {
          const float4 v = *reinterpret_cast<const float4 *>(Ls + (q + 1) * SH::kStride + 4 + 4 * u);
          if (dst) *reinterpret_cast<float4 *>(dst + q * ldl) = v;
          const float m4 = fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
          const float vv[4] = {v.x, v.y, v.z, v.w};
          unsigned m = 0u;
          if (m4 >= th) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (fabsf(vv[i]) >= th && test(q, 4 * u + i, vv[i])) m |= 1u << i;
          }
          push(m, q, 4 * u, vv);
        }
      }
    } else {
      for (int q = wid; q < nrow; q += SH::kThreads / 32)
        for (int cl = lane; cl < ncol; cl += 32) {
          const float v = Ls[(q + 1) * SH::kStride + 4 + cl];
          if (Lout) Lout[(r0 + q) * ldl + c0 + cl] = v;
          const float vv[4] = {v, 0.f, 0.f, 0.f};
          push(fabsf(v) >= th && test(q, cl, v) ? 1u : 0u, q, cl, vv);
        }
    }
  }
  __syncthreads();
  // ---- flush the candidates that survive the best threshold known now -----
  if (tid == 0) {
    S.thr_end = frac * fmaxf(__uint_as_float(old), __uint_as_float(S.cmax));
  }
  __syncthreads();
  const int n = S.ccount < kFcCand ? S.ccount : kFcCand;
  for (int q = tid; q < n; q += SH::kThreads) {
    if (!(fabsf(S.cv[q]) >= S.thr_end)) continue;
    int kk = atomicAdd(&st->count, 1);
    if (kk < gcap) {
      gy[kk] = S.cy[q];
      gx[kk] = S.cx[q];
      gv[kk] = S.cv[q];
    } else {
      st->overflow = 1;
    }
  }
}

// Fused column pass: one CTA per tile (tile = row-band-major over ntx column
// tiles).  The window of an interior tile is one TMA transfer (tma_boxes
// boxes), edge tiles are staged with clamped cp.async copies.  (A persistent
// variant that stages the next tile's window into a second buffer while the
// current one is filtered measured 2-12 % slower at every tap count: the
// other resident CTAs already hide the staging, and the second buffer costs
// occupancy.)
template <class SH, int MODE>  // MODE 0: Laplacian + 3x3 NMS, 1: Hessian detector, 2: derivatives,
                               // 3: the blur only (fp32)
__global__ void __launch_bounds__(SH::kThreads, 1024 / SH::kThreads) firapply_kernel(
    const float *__restrict__ T, int64_t ldt, float *__restrict__ Lout, int64_t ldl, int64_t H,
    int64_t W, FirTapsP tp, float lap_scale, float frac, CandState *__restrict__ st,
    int *__restrict__ gy, int *__restrict__ gx, float *__restrict__ gv, int gcap, int vec_out,
    const __grid_constant__ CUtensorMap tmap, int tma_rows, int tma_boxes, HessOut ho) {
  extern __shared__ __align__(128) unsigned char fsm_raw[];
  __shared__ FcSmall S;
  __shared__ __align__(8) uint64_t fbar;
  // 128-byte aligned base (TMA destination), derived from the shared array
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(fsm_raw);
  unsigned char *fsm = fsm_raw + ((128u - (sbase & 127u)) & 127u);
  float *win = reinterpret_cast<float *>(fsm);
  const int tid = threadIdx.x;
  const int k = (tp.n - 1) / 2;
  const int wrows = SH::kRB + tp.np + 8;
  const int64_t c0 = (int64_t)blockIdx.x * SH::kOut;
  const int64_t r0 = (int64_t)blockIdx.y * SH::kOwn;
  if (tid == 0) {
    S.ccount = 0;
    S.cmax = 0u;
  }
  pdl_wait();
  // global max |L| published so far (a lower bound of the final one; read
  // now so the load hides under the staging and the taps)
  const float gbound = MODE == 0 ? __uint_as_float(*(volatile unsigned *)&st->absmax_bits) : 0.0f;
  // ---- stage the column window: row w <-> image row r0 - 2 - k + w, column
  //      cc <-> image column c0 - 4 + cc, both edge-clamped ----------------
  const int64_t rw0 = r0 - 2 - k;
  const bool tma = tma_boxes > 0 && rw0 >= 0 && rw0 + (int64_t)tma_boxes * tma_rows <= H &&
                   c0 >= 4 && c0 - 4 + SH::kStride <= W;
  if (tma) {  // interior tile: tma_boxes boxes of tma_rows x kStride
    if (tid == 0) {
      mbar_init(&fbar, 1);
      mbar_expect_tx(&fbar, (unsigned)(tma_boxes * tma_rows * SH::kStride * sizeof(float)));
      for (int bx = 0; bx < tma_boxes; ++bx)
        tma_load_2d_hint(win + bx * tma_rows * SH::kStride, &tmap, &fbar, (int)(c0 - 4),
                         (int)(rw0 + bx * tma_rows), l2_policy_evict_first());
    }
    __syncthreads();
    mbar_wait(&fbar, 0);
  } else {
    for (int idx = tid; idx < wrows * SH::kStride; idx += SH::kThreads) {
      const int wr = idx / SH::kStride, cc = idx - wr * SH::kStride;
      int64_t r = rw0 + wr, c = c0 - 4 + cc;
      r = r < 0 ? 0 : (r >= H ? H - 1 : r);
      c = c < 0 ? 0 : (c >= W ? W - 1 : c);
      const unsigned sa = (unsigned)__cvta_generic_to_shared(win + idx);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(T + r * ldt + c));
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
  }
  __syncthreads();
  fc_tile<SH, MODE>(fsm, S, c0, r0, Lout, ldl, H, W, tp, lap_scale, frac, st, gy, gx, gv, gcap,
                    vec_out, ho, gbound);
}

template <class SH>
static size_t fc_smem(int np) {
  // + room for the rounded-up TMA boxes and the 128-byte alignment
  const size_t box = (size_t)(SH::kRB + np + 8 + 8 * ((SH::kRB + np + 8 + 255) / 256)) *
                     SH::kStride * sizeof(float);
  const size_t r = SH::region_bytes(np);
  return (r > box ? r : box) + 128;
}
static size_t fc_smem_any(int np) {
  return fc_smem<FcLong>(np);
}

bool firpass_supported(int64_t h, int64_t w, int ntaps) {
  if (ntaps < 1 || ntaps > kFirMaxFast || h < 4 || w < 4) return false;
  const int np = (ntaps + 7) / 8 * 8;
  return fc_smem_any(np) + sizeof(FcSmall) + 1024 <= 227 * 1024;
}

// every candidate is a strict 3x3 extremum of L (at most ceil(h/2) ceil(w/2)
// maxima and as many minima): the list cannot overflow, so L is stored only
// on request (the finaliser's full-scan fallback is never needed)
static int64_t fir_cand_capacity(int64_t h, int64_t w) {
  return 2 * cdiv(h, 2) * cdiv(w, 2) + 64;
}

size_t firpass_workspace_bytes(int64_t h, int64_t w) {
  return 4096 + (size_t)fir_cand_capacity(h, w) * 12 + 256;
}

// window rows staged by TMA: nbox boxes of `rows` (<= 256, a multiple of 8)
template <class SH>
static void fc_boxes(int np, int *rows, int *nbox) {
  const int wrows = SH::kRB + np + 8;
  *nbox = (wrows + 255) / 256;
  *rows = ((wrows + *nbox - 1) / *nbox + 7) / 8 * 8;
}

template <class SH, int MODE = 0>
static void launch_firapply(const float *T, int64_t ldt, float *L, int64_t ldl, int64_t h,
                            int64_t w, const FirTapsP &tp, float lap_scale, float frac,
                            CandState *cs, int *gy, int *gx, float *gv, int64_t gcap, int vec,
                            cudaStream_t st, const HessOut *hop = nullptr) {
  HessOut ho;
  memset(&ho, 0, sizeof(ho));
  if (hop) ho = *hop;
  const size_t smem = fc_smem<SH>(tp.np);
  int rows = 0, nbox = 0;
  fc_boxes<SH>(tp.np, &rows, &nbox);
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  if (!make_tmap_2d_f32(&tmap, T, h, w, ldt, SH::kStride, rows) || getenv("VMF_NO_TMA")) nbox = 0;
  cudaGetLastError();
  cudaFuncSetAttribute(firapply_kernel<SH, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  dim3 grid((unsigned)cdiv(w, SH::kOut), (unsigned)cdiv(h, SH::kOwn));
  launch_pdl(firapply_kernel<SH, MODE>, grid, dim3(SH::kThreads), smem, st, T, ldt, L, ldl, h, w,
             tp, lap_scale, frac, cs, gy, gx, gv, (int)gcap, vec, tmap, rows, nbox, ho);
}

int fir_cols_blur(const float *T, int64_t ldt, float *y, int64_t ldy, const double *taps,
                  int ntaps, int64_t h, int64_t w, cudaStream_t st) {
  if (!firpass_supported(h, w, ntaps))
    return fail(VMF_EVALUE, "FIR column tile does not support %d taps at %lldx%lld", ntaps,
                (long long)h, (long long)w);
  FirTapsP tp;
  fir_plan(&tp, taps, ntaps);
  Launch g(K_FIR_COLS, st);
  launch_firapply<FcLong, 3>(T, ldt, y, ldy, h, w, tp, 1.0f, 0.0f, nullptr, nullptr, nullptr,
                             nullptr, 0, 0, st);
  return cuda_status("fir column blur");
}

int firpass_run(const float *T, int64_t ldt, float *L, int64_t ldl, const double *taps, int ntaps,
                int64_t h, int64_t w, float lap_scale, float frac, int32_t *det_yx,
                float *det_val, int64_t cap, int64_t *n_det_dev, float *thr_dev, void *ws,
                size_t ws_bytes, cudaStream_t st) {
  if (!firpass_supported(h, w, ntaps))
    return fail(VMF_EVALUE, "fused FIR column pass does not support %d taps at %lldx%lld", ntaps,
                (long long)h, (long long)w);
  if (!ws || ws_bytes < firpass_workspace_bytes(h, w))
    return fail(VMF_EVALUE, "FIR column-pass workspace too small");
  FirTapsP tp;
  fir_plan(&tp, taps, ntaps);
  char *base = (char *)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  CandState *cs = (CandState *)base;
  const int64_t gcap = fir_cand_capacity(h, w);
  int *gy = (int *)(base + 4096);
  int *gx = gy + gcap;
  float *gv = (float *)(gx + gcap);
  cudaMemsetAsync(cs, 0, sizeof(CandState), st);
  {
    Launch g(K_FIR_COLS, st);
    const int vec = (int)(L && ldl % 4 == 0 && (uintptr_t)L % 16 == 0);
    launch_firapply<FcLong>(T, ldt, L, ldl, h, w, tp, lap_scale, frac, cs, gy, gx, gv, gcap, vec,
                            st);
  }
  int rc = cuda_status("fir column pass");
  if (rc) return rc;
  if (frac <= 0.0f) return VMF_OK;
  return colfinal_launch(cs, gy, gx, gv, gcap, L, ldl, h, w, frac, det_yx, det_val, cap,
                         n_det_dev, thr_dev, st);
}

// Hessian detector candidates from the row-pass output T and a FIR column
// stage (blob.detect's derivative field, fused; B stays fp64).
int hesspass_run(const float *T, int64_t ldt, const double *taps, int ntaps, int64_t h,
                 int64_t w, double sigma, double t1, int polarity, float *nd_field,
                 float *trace_field, int64_t ldn, int *cy, int *cx, double *cnd, float *cdx,
                 float *cdy, int64_t cap, int *count, cudaStream_t st) {
  if (!firpass_supported(h, w, ntaps))
    return fail(VMF_EVALUE, "Hessian detector: %d-tap column stage unsupported", ntaps);
  FirTapsP tp;
  fir_plan(&tp, taps, ntaps);
  HessOut ho;
  memset(&ho, 0, sizeof(ho));
  ho.sigma4 = sigma * sigma * sigma * sigma;
  ho.t1 = t1;
  ho.polarity = polarity >= 0 ? 1 : -1;
  ho.nd_field = nd_field;
  ho.trace_field = trace_field;
  ho.ldn = ldn;
  ho.cy = cy;
  ho.cx = cx;
  ho.cnd = cnd;
  ho.cdx = cdx;
  ho.cdy = cdy;
  ho.cap = (int)(cap < 0x7fffffff ? cap : 0x7fffffff);
  ho.count = count;
  cudaMemsetAsync(count, 0, sizeof(int), st);
  Launch g(K_FIR_COLS, st);
  launch_firapply<FcLong, 1>(T, ldt, nullptr, 0, h, w, tp, 1.0f, 0.0f, nullptr, nullptr,
                             nullptr, nullptr, 0, 0, st, &ho);
  return cuda_status("hessian pass");
}

// ---------------------------------------------------------------------------
// the same Hessian / derivative outputs from an fp64 blur in global memory
// (the IIR column pass's MODE 2 output): one thread per pixel, 3x3
// neighbourhood with replicate edges
// ---------------------------------------------------------------------------
template <int MODE>  // 1: Hessian detector, 2: derivative images
__global__ void __launch_bounds__(256) b64_kernel(const double *__restrict__ B, int64_t H,
                                                  int64_t W, HessOut ho) {
  const int lane = threadIdx.x & 31;
  const int64_t npx = H * W;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < npx;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t idx = base + threadIdx.x;
    bool cand = false;
    int64_t r = 0, c = 0;
    double nd = 0.0, dxv = 0.0, dyv = 0.0;
    if (idx < npx) {
      r = idx / W;
      c = idx - r * W;
      const int64_t ru = r > 0 ? r - 1 : 0, rd = r + 1 < H ? r + 1 : H - 1;
      const int64_t cl = c > 0 ? c - 1 : 0, cr = c + 1 < W ? c + 1 : W - 1;
      const double *pc = B + r * W, *pu = B + ru * W, *pd = B + rd * W;
      const double b00 = pc[c], bl = pc[cl], br = pc[cr], bu = pu[c], bd = pd[c];
      const double d10 = fma(-0.5, bl, 0.5 * br);
      const double d01 = fma(-0.5, bu, 0.5 * bd);
      const double d20 = (br - 2.0 * b00) + bl;
      const double d02 = (bd - 2.0 * b00) + bu;
      const double d10u = fma(-0.5, pu[cl], 0.5 * pu[cr]), d10d = fma(-0.5, pd[cl], 0.5 * pd[cr]);
      const double d11 = fma(-0.5, d10u, 0.5 * d10d);
      const int64_t o = r * ho.ldn + c;
      if (MODE == 2) {
        const double v[6] = {b00, d10, d01, d20, d02, d11};
#pragma unroll
        for (int d = 0; d < 6; ++d)
          if (ho.deriv[d]) ho.deriv[d][o] = (float)v[d];
      } else {
        const double det = d20 * d02 - d11 * d11;
        nd = ho.sigma4 * det;
        const double tr2 = d20 + d02;
        if (ho.nd_field) ho.nd_field[o] = (float)nd;
        if (ho.trace_field) ho.trace_field[o] = (float)tr2;
        cand = nd > ho.t1 && (ho.polarity > 0 ? tr2 > 0.0 : tr2 < 0.0);
        if (cand) {
          if (fabs(det) < 1e-12) {
            dxv = dyv = __longlong_as_double(0x7ff8000000000000ll);
          } else {
            dxv = (d01 * d11 - d02 * d10) / det;
            dyv = (d10 * d11 - d20 * d01) / det;
          }
        }
      }
    }
    if (MODE != 1) continue;
    const unsigned bal = __ballot_sync(0xffffffffu, cand);
    if (!bal) continue;
    int basek = 0;
    if (lane == 0) basek = atomicAdd(ho.count, __popc(bal));
    basek = __shfl_sync(0xffffffffu, basek, 0);
    if (cand) {
      const int k = basek + __popc(bal & ((1u << lane) - 1u));
      if (k < ho.cap) {
        ho.cy[k] = (int)r;
        ho.cx[k] = (int)c;
        ho.cnd[k] = nd;
        ho.cdx[k] = (float)dxv;
        ho.cdy[k] = (float)dyv;
      }
    }
  }
}

static HessOut hess_out(double sigma, double t1, int polarity, float *nd_field, float *trace_field,
                        int64_t ldn, int *cy, int *cx, double *cnd, float *cdx, float *cdy,
                        int64_t cap, int *count) {
  HessOut ho;
  memset(&ho, 0, sizeof(ho));
  ho.sigma4 = sigma * sigma * sigma * sigma;
  ho.t1 = t1;
  ho.polarity = polarity >= 0 ? 1 : -1;
  ho.nd_field = nd_field;
  ho.trace_field = trace_field;
  ho.ldn = ldn;
  ho.cy = cy;
  ho.cx = cx;
  ho.cnd = cnd;
  ho.cdx = cdx;
  ho.cdy = cdy;
  ho.cap = (int)(cap < 0x7fffffff ? cap : 0x7fffffff);
  ho.count = count;
  return ho;
}

int hess_from_b64(const double *B, int64_t h, int64_t w, double sigma, double t1, int polarity,
                  float *nd_field, float *trace_field, int64_t ldn, int *cy, int *cx, double *cnd,
                  float *cdx, float *cdy, int64_t cap, int *count, cudaStream_t st) {
  HessOut ho = hess_out(sigma, t1, polarity, nd_field, trace_field, ldn, cy, cx, cnd, cdx, cdy,
                        cap, count);
  cudaMemsetAsync(count, 0, sizeof(int), st);
  const int64_t nb = cdiv(h * w, 256);
  Launch g(K_LAPLACIAN, st);
  b64_kernel<1><<<(unsigned)(nb < 148 * 16 ? nb : 148 * 16), 256, 0, st>>>(B, h, w, ho);
  return cuda_status("hessian (fp64 blur)");
}

int deriv_from_b64(const double *B, int64_t h, int64_t w, float *const *outs, int64_t ldo,
                   cudaStream_t st) {
  HessOut ho;
  memset(&ho, 0, sizeof(ho));
  ho.ldn = ldo;
  for (int d = 0; d < 6; ++d) ho.deriv[d] = outs[d];
  const int64_t nb = cdiv(h * w, 256);
  Launch g(K_LAPLACIAN, st);
  b64_kernel<2><<<(unsigned)(nb < 148 * 16 ? nb : 148 * 16), 256, 0, st>>>(B, h, w, ho);
  return cuda_status("derivatives (fp64 blur)");
}

// engine.derivative_field (order 3, FIR blur) in one fused column pass
int derivpass_run(const float *T, int64_t ldt, const double *taps, int ntaps, int64_t h,
                  int64_t w, float *const *outs, int64_t ldo, cudaStream_t st) {
  if (!firpass_supported(h, w, ntaps))
    return fail(VMF_EVALUE, "fused derivative bank: %d-tap column stage unsupported", ntaps);
  FirTapsP tp;
  fir_plan(&tp, taps, ntaps);
  HessOut ho;
  memset(&ho, 0, sizeof(ho));
  ho.ldn = ldo;
  for (int d = 0; d < 6; ++d) ho.deriv[d] = outs[d];
  Launch g(K_FIR_COLS, st);
  launch_firapply<FcLong, 2>(T, ldt, nullptr, 0, h, w, tp, 1.0f, 0.0f, nullptr, nullptr,
                             nullptr, nullptr, 0, 0, st, &ho);
  return cuda_status("derivative pass");
}

}  // namespace vmf
