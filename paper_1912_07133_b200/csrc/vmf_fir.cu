// vmf_fir.cu -- centred FIR along rows or columns with replicate edges,
// fp32/u16 in, fp32 out, fp64 accumulation.
//
// Replaces _conv_rows_kernel (engine.py:35-62) and conv_rows / conv_cols
// (engine.py:112-126):  out(n) = sum_{m=-k..k} taps[k+m] x(clamp(n-m)),
// accumulated with m ascending like the reference.  fp64 accumulation: with
// fp32 accumulation a 257-tap Gaussian misses the 1e-4 Laplacian tolerance
// (SURVEY.md §8(a3)).
//
// Tiling: a CTA owns a tile of outputs and stages the input window (tile +
// 2k halo, edge-clamped) in shared memory once, so each input element is read
// from L2/HBM once per tile instead of (2k+1) times.
#include <cstdlib>

#include "vmf_common.cuh"
#include "vmf_firpass.cuh"
#include "vmf_iir.cuh"
#include "vmf_prof.cuh"

namespace vmf {

template <int MAXT>
struct FirTaps {
  double t[MAXT];
  int n;
};

constexpr int kFirRowTile = 256;  // outputs per CTA along a row
constexpr int kFirColTileW = 32;  // columns per CTA (one warp wide)
constexpr int kFirColTileH = 64;  // rows per CTA

// ROWS: CTA = (row segment of kFirRowTile outputs) x (one row per blockIdx.y
// step).  Shared: taps + window of kFirRowTile + 2k samples (fp64).
template <int MAXT, typename T>
__global__ void __launch_bounds__(kFirRowTile) fir_rows_kernel(const T *__restrict__ x,
                                                               int64_t ldx, float *__restrict__ y,
                                                               int64_t ldy, int64_t h, int64_t w,
                                                               FirTaps<MAXT> taps) {
  extern __shared__ double sm[];
  const int nt = taps.n, k = (nt - 1) / 2;
  double *st = sm;           // [nt]
  double *win = sm + nt;     // [kFirRowTile + 2k]
  for (int i = threadIdx.x; i < nt; i += blockDim.x) st[i] = taps.t[i];
  int64_t n0 = (int64_t)blockIdx.x * kFirRowTile;
  for (int64_t row = blockIdx.y; row < h; row += gridDim.y) {
    __syncthreads();
    const T *xr = x + row * ldx;
    for (int i = threadIdx.x; i < kFirRowTile + 2 * k; i += blockDim.x) {
      int64_t q = n0 - k + i;
      q = q < 0 ? 0 : (q >= w ? w - 1 : q);
      win[i] = ld64(xr + q);
    }
    __syncthreads();
    int64_t n = n0 + threadIdx.x;
    if (n < w) {
      // out(n) = sum_m t[k+m] x(n-m); x(n-m) = win[threadIdx.x + k - m]
      const double *wp = win + threadIdx.x + 2 * k;
      double acc = 0.0;
      for (int j = 0; j < nt; ++j) acc = fma(st[j], wp[-j], acc);
      y[row * ldy + n] = (float)acc;
    }
  }
}

// COLS: CTA = kFirColTileW columns x kFirColTileH rows of outputs.
template <int MAXT, typename T>
__global__ void __launch_bounds__(256) fir_cols_kernel(const T *__restrict__ x, int64_t ldx,
                                                       float *__restrict__ y, int64_t ldy,
                                                       int64_t h, int64_t w,
                                                       FirTaps<MAXT> taps) {
  extern __shared__ double sm[];
  const int nt = taps.n, k = (nt - 1) / 2;
  double *st = sm;
  double *win = sm + nt;  // [kFirColTileH + 2k][kFirColTileW]
  for (int i = threadIdx.x; i < nt; i += blockDim.x) st[i] = taps.t[i];
  int64_t j0 = (int64_t)blockIdx.x * kFirColTileW, r0 = (int64_t)blockIdx.y * kFirColTileH;
  int tx = threadIdx.x % kFirColTileW, ty = threadIdx.x / kFirColTileW;
  int64_t j = j0 + tx;
  int64_t jc = j < w ? j : w - 1;
  int rows = kFirColTileH + 2 * k;
  for (int i = ty; i < rows; i += blockDim.x / kFirColTileW) {
    int64_t q = r0 - k + i;
    q = q < 0 ? 0 : (q >= h ? h - 1 : q);
    win[i * kFirColTileW + tx] = ld64(x + q * ldx + jc);
  }
  __syncthreads();
  if (j >= w) return;
  for (int r = ty; r < kFirColTileH; r += blockDim.x / kFirColTileW) {
    int64_t n = r0 + r;
    if (n >= h) break;
    const double *wp = win + (r + 2 * k) * kFirColTileW + tx;
    double acc = 0.0;
    for (int m = 0; m < nt; ++m) acc = fma(st[m], wp[-m * kFirColTileW], acc);
    y[n * ldy + j] = (float)acc;
  }
}

template <int MAXT, int O, typename T>
static int launch_fir(const T *x, int64_t ldx, float *y, int64_t ldy, int64_t h, int64_t w,
                      const double *taps, int ntaps, cudaStream_t st) {
  FirTaps<MAXT> tp;
  for (int i = 0; i < ntaps; ++i) tp.t[i] = taps[i];
  tp.n = ntaps;
  int k = (ntaps - 1) / 2;
  if (O == ROWS) {
    size_t smem = (size_t)(ntaps + kFirRowTile + 2 * k) * sizeof(double);
    cudaFuncSetAttribute(fir_rows_kernel<MAXT, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    dim3 grid((unsigned)cdiv(w, kFirRowTile), (unsigned)(h < 65535 ? h : 65535));
    Launch g(K_FIR_ROWS, st);
    fir_rows_kernel<MAXT, T><<<grid, kFirRowTile, smem, st>>>(x, ldx, y, ldy, h, w, tp);
  } else {
    size_t smem = (size_t)(ntaps + (kFirColTileH + 2 * k) * kFirColTileW) * sizeof(double);
    if (smem > 200 * 1024) return fail(VMF_EVALUE, "FIR too long for column tile (%d taps)", ntaps);
    cudaFuncSetAttribute(fir_cols_kernel<MAXT, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    dim3 grid((unsigned)cdiv(w, kFirColTileW), (unsigned)cdiv(h, kFirColTileH));
    Launch g(K_FIR_COLS, st);
    fir_cols_kernel<MAXT, T><<<grid, 256, smem, st>>>(x, ldx, y, ldy, h, w, tp);
  }
  return cuda_status("fir pass");
}

template <int O, typename T>
static int fir_bucket(const T *x, int64_t ldx, float *y, int64_t ldy, int64_t h, int64_t w,
                      const double *taps, int ntaps, cudaStream_t st) {
  if (ntaps <= 33) return launch_fir<33, O, T>(x, ldx, y, ldy, h, w, taps, ntaps, st);
  if (ntaps <= 129) return launch_fir<129, O, T>(x, ldx, y, ldy, h, w, taps, ntaps, st);
  if (ntaps <= 513) return launch_fir<513, O, T>(x, ldx, y, ldy, h, w, taps, ntaps, st);
  return launch_fir<VMF_MAX_FIR_TAPS, O, T>(x, ldx, y, ldy, h, w, taps, ntaps, st);
}

template <int O>
int fir_pass(const void *x, int x_dtype, float *y, int64_t h, int64_t w, int64_t ldx,
             int64_t ldy, const double *taps, int ntaps, cudaStream_t st) {
  if (h < 1 || w < 1) return fail(VMF_EVALUE, "image must be a 2-D array");
  if (ldx < w || ldy < w)
    return fail(VMF_EVALUE, "row pitch smaller than width (ldx=%lld ldy=%lld w=%lld)",
                (long long)ldx, (long long)ldy, (long long)w);
  if (ntaps < 1 || ntaps % 2 == 0) return fail(VMF_EVALUE, "taps must have odd length 2K+1");
  if (ntaps > VMF_MAX_FIR_TAPS)
    return fail(VMF_EVALUE, "kernel length %d exceeds the %d-tap limit", ntaps, VMF_MAX_FIR_TAPS);
  int64_t length = O == ROWS ? w : h;
  if (ntaps > length)
    return fail(VMF_EVALUE, "kernel length %d exceeds row length %lld", ntaps, (long long)length);
  // rows up to kFirMaxFast taps: the register-blocked kernel (vmf_firpass.cu)
  const bool fast = O == ROWS && ntaps <= kFirMaxFast && !getenv("VMF_FIR_GENERIC");
  // fp32 columns: the fused column pass's tiles (window staged once per
  // 60-row block, 8 outputs per thread) instead of the generic kernel
  if (O == COLS && x_dtype == VMF_F32 && firpass_supported(h, w, ntaps) &&
      !getenv("VMF_FIR_GENERIC"))
    return fir_cols_blur((const float *)x, ldx, y, ldy, taps, ntaps, h, w, st);
  return with_sample_type(x_dtype, x, [&](auto xt) {
    if (fast) return fir_rows_fast(xt, ldx, y, ldy, h, w, taps, ntaps, st);
    return fir_bucket<O>(xt, ldx, y, ldy, h, w, taps, ntaps, st);
  });
}

template int fir_pass<ROWS>(const void *, int, float *, int64_t, int64_t, int64_t, int64_t,
                            const double *, int, cudaStream_t);
template int fir_pass<COLS>(const void *, int, float *, int64_t, int64_t, int64_t, int64_t,
                            const double *, int, cudaStream_t);

}  // namespace vmf
