// vmf_iir.cuh -- IIR pass planning structures (see vmf_iir.cu).
#pragma once
#include "vmf_common.cuh"

namespace vmf {

constexpr int64_t kIirChunk = 64;      // samples per chunk (lines x chunks fill the GPU)
constexpr int kIirApplyThreads = 128;
constexpr int kIirHmax = (int)kIirChunk + 2 * VMF_MAX_IIR_ORDER;  // > longest chunk

// Everything a pass needs, passed by value as a kernel parameter.
struct IirParams {
  double b[VMF_MAX_IIR_ORDER], a[VMF_MAX_IIR_ORDER];
  double b0, sign, yss;  // yss = sum(b)/(1 + sum(a)): steady-state y+ per unit step
  double T[2][VMF_MAX_IIR_ORDER * 2 * VMF_MAX_IIR_ORDER];  // [L, Llast] transfer matrices
  double h[kIirHmax];  // causal impulse response, h[0] = 0
  int64_t M, N, L, C, Llast;
  int K;
};

bool poles_inside_unit_circle(const double *a_plus, int k);
void iir_geometry(int64_t n, int k, int64_t *L, int64_t *C, int64_t *Llast);
size_t iir_workspace_bytes(int64_t lines, int64_t length, int k);
int iir_plan(IirParams *p, int64_t lines, int64_t length, const double *b_plus,
             const double *a_plus, int k, double b_zero, int sign);

template <int O>
int iir_pass(const void *x, int x_dtype, float *y, int64_t h, int64_t w, int64_t ldx,
             int64_t ldy, const double *b_plus, const double *a_plus, int k, double b_zero,
             int sign, void *ws, size_t ws_bytes, cudaStream_t st);

template <int O>
int fir_pass(const void *x, int x_dtype, float *y, int64_t h, int64_t w, int64_t ldx,
             int64_t ldy, const double *taps, int ntaps, cudaStream_t st);

}  // namespace vmf
