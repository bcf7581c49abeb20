// vmf_firpass.cuh -- the FIR hot path: register-blocked row FIR and the fused
// column FIR + Laplacian + 3x3 NMS (vmf_firpass.cu).
#pragma once
#include "vmf_common.cuh"

namespace vmf {

constexpr int kFirMaxFast = 385;  // taps of the fast FIR paths (longer: generic kernels)

bool firpass_supported(int64_t h, int64_t w, int ntaps);
size_t firpass_workspace_bytes(int64_t h, int64_t w);

// row pass: y = conv_rows(x, taps) (fp32 / u16 in, fp32 out, fp64 accumulation)
template <typename T>
int fir_rows_fast(const T *x, int64_t ldx, float *y, int64_t ldy, int64_t h, int64_t w,
                  const double *taps, int ntaps, cudaStream_t st);

// column FIR of T + Laplacian + threshold / 3x3 NMS; L (pitch ldl) and the
// sorted detections like colpass_run
int firpass_run(const float *T, int64_t ldt, float *L, int64_t ldl, const double *taps, int ntaps,
                int64_t h, int64_t w, float lap_scale, float frac, int32_t *det_yx,
                float *det_val, int64_t cap, int64_t *n_det_dev, float *thr_dev, void *ws,
                size_t ws_bytes, cudaStream_t st);

// Hessian blob-detector candidates (fused FIR column pass, B in fp64)
int hesspass_run(const float *T, int64_t ldt, const double *taps, int ntaps, int64_t h,
                 int64_t w, double sigma, double t1, int polarity, float *nd_field,
                 float *trace_field, int64_t ldn, int *cy, int *cx, double *cnd, float *cdx,
                 float *cdy, int64_t cap, int *count, cudaStream_t st);

// derivative bank fir_vm_bank(3) of the (fp64) FIR blur: outs = D00 D10 D01
// D20 D02 D11 (any may be null), fp32, pitch ldo
int derivpass_run(const float *T, int64_t ldt, const double *taps, int ntaps, int64_t h,
                  int64_t w, float *const *outs, int64_t ldo, cudaStream_t st);

// the same outputs from an fp64 blur B (pitch w) in global memory
int hess_from_b64(const double *B, int64_t h, int64_t w, double sigma, double t1, int polarity,
                  float *nd_field, float *trace_field, int64_t ldn, int *cy, int *cx, double *cnd,
                  float *cdx, float *cdy, int64_t cap, int *count, cudaStream_t st);
int deriv_from_b64(const double *B, int64_t h, int64_t w, float *const *outs, int64_t ldo,
                   cudaStream_t st);

// the conv_cols leaf on the fused column tiles: y = taps (*) T along columns,
// fp64 accumulation, fp32 out (firpass_supported shapes)
int fir_cols_blur(const float *T, int64_t ldt, float *y, int64_t ldy, const double *taps,
                  int ntaps, int64_t h, int64_t w, cudaStream_t st);

}  // namespace vmf
