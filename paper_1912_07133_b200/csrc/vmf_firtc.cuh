// vmf_firtc.cuh -- the FIR blur -> Laplacian path on the 5th-generation
// tensor cores (tcgen05.mma kind::tf32, 3xTF32 split), "Laplacian first".
//
// Why.  The reference's FIR blur (conv_rows / conv_cols, engine.py:35-62 /
// 112-135) is one multiply-add per tap per pixel per pass: 770 for the
// 385-tap SG kernel of config 5.  On CUDA cores in fp64 (vmf_firpass.cu) that
// runs at ~80 % of the DFMA peak.  As a matrix product it fits the tensor
// cores: per 128 x 128 output tile, D = A . B^T with A the 128 input lines x
// a window of 128 + 2k samples and B the banded Toeplitz matrix of the taps
// (B[n][q] = t[n + 2k - q]).  TF32 alone is 1e-3 of max|L| off; the 3xTF32
// split (hi*hi + hi*lo + lo*hi) with fp32 accumulation in TMEM is fp32-grade,
// and filtering the Laplacian of the frame instead of the frame (the
// identity of vmf_rowlap.cu, here with h(m) = the taps) keeps every rounding
// relative to |L|: tools/experiments/fir_blocked_fp32.py measures 4e-7 ..
// 1.2e-6 of max|L| for 65 .. 385 taps.
//
// Passes (all on the caller's stream):
//   1. prep: U = Lap5 X (replicate) and the four border rows (D20 X of rows
//      0 / H-1, the column sums dyt / dyb), split into tf32 hi / lo; the
//      per-line edge table {eL, eR, dL, dR}; the banded tap tables.
//   2. rows: V = R(U) on the tensor cores; the epilogue adds the edge terms
//      (constant extension eL / eR through the tap tail sums, the border
//      terms dL / dR on the end samples) and writes V transposed (hi / lo),
//      the virtual rows Vt / Vb and the row-filtered Ky rows.
//   3. columns: L = C(V^T) the same way (edge terms Vt / Vb, Ky), scaled,
//      written row-major with |L|max for stage 4.
#pragma once
#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace vmf {

constexpr int kTcMaxK = 192;       // FIR half-length (taps <= 385)
// below, the fp64 CUDA-core FIR (vmf_firpass.cu) is faster: at 4096^2, 17 taps
// 124.9k vs 117.0k Mpixel/s on the tensor cores; 33 taps 104.6k vs 117.4k
constexpr int kFirTcMinTaps = 33;

// true if the tensor-core FIR path takes this frame and these stages
bool firtc_supported(int64_t h, int64_t w, int64_t ldx, int row_taps, int col_taps);
size_t firtc_workspace_bytes(int64_t h, int64_t w, int row_taps, int col_taps);

// L (h x w, pitch ldl) = lap_scale * Lap5_rep(C_rep R_rep X) for FIR stages,
// then (frac > 0) stage 4 into det_yx / det_val / n_det_dev / thr_dev (the
// column pass's candidate list and sorting finaliser).
int firtc_detect(const float *x, int64_t ldx, int64_t h, int64_t w, const double *rtaps, int rn,
                 const double *ctaps, int cn, float lap_scale, float frac, float *L, int64_t ldl,
                 int32_t *det_yx, float *det_val, int64_t cap, int64_t *n_det_dev, float *thr_dev,
                 void *ws, size_t ws_bytes, cudaStream_t st);

}  // namespace vmf
