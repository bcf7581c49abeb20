// vmf_rowpass.cuh -- single-kernel row pass (vmf_rowpass.cu).
#pragma once
#include "vmf_iir.cuh"
#include "vmf_dfi.cuh"

namespace vmf {

constexpr int kChunk = 32;          // samples per thread (one chunk)
constexpr int kRowThreads = 128;    // target threads per CTA (R rows x C chunks)
constexpr int kRowMaxThreads = 256; // rows up to 8192 samples (C <= 256)
constexpr int kRowMinBlocks = 3;    // with 256 threads -> <= 85 registers
constexpr int64_t kRowTileBytes = 40 * 1024;

struct RowParams {
  double b[VMF_MAX_IIR_ORDER], a[VMF_MAX_IIR_ORDER];
  double b0, sign, yss;
  double h[kChunk + 1];  // causal impulse response h[0..32], h[0] = 0
  double Ty[VMF_MAX_IIR_ORDER * VMF_MAX_IIR_ORDER];  // DF-I history transfer over 32 samples
  double Tx[VMF_MAX_IIR_ORDER * VMF_MAX_IIR_ORDER];
  double Tpow[5][VMF_MAX_IIR_ORDER * VMF_MAX_IIR_ORDER];  // Ty^(cpl*2^j)
  double SP32[VMF_MAX_IIR_ORDER][kChunk / 2], SQ32[VMF_MAX_IIR_ORDER][kChunk / 2];  // folded
  int64_t H, W;
  int C, R, cpl;
  int vec4, vec8;  // 16-byte fp32 / 8-sample integer vector loads
  int64_t rows_per;  // TMA variant: rows per CTA
  DfiCoef bwd;       // b_minus = sign * b, a: the backward run yields sign * y- directly
};

bool rowpass_supported(int64_t w, int k);
template <typename T>
int rowpass_run(const T *x, int64_t ldx, float *y, int64_t ldy, const IirParams &ip, int64_t h,
                int64_t w, cudaStream_t st);

}  // namespace vmf
