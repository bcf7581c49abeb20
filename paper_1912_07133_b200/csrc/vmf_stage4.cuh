// vmf_stage4.cuh -- Laplacian + threshold/NMS entry points (vmf_stage4.cu).
#pragma once
#include "vmf_common.cuh"

namespace vmf {

int laplacian(const float *b, int64_t ldb, float *l, int64_t ldl, int64_t h, int64_t w,
              float scale, float *absmax, cudaStream_t st);
size_t detect_workspace_bytes(int64_t ns, int64_t h, int64_t w);
// absmax lives in the first slot of the detect workspace; callers that
// already reduced |L| there pass have_absmax = true.
float *detect_absmax_slot(void *ws);
// Ordered full-frame NMS whose kernels do nothing unless *gate != 0 (the
// fallback of the fused column pass); absmax is a device float.
int detect_if(const float *l, int64_t ld, int64_t h, int64_t w, float frac, float *absmax,
              const int *gate, int32_t *det_yx, float *det_val, int64_t cap, int64_t *n_det_dev,
              float *thr_dev, void *ws, size_t ws_bytes, cudaStream_t st);
// the scale-space rule from the per-scale candidate lists of the fused
// column passes (see vmf_detect3x3x3_cands); *n_det = -1 when a list was cut
int detect3x3x3_cands(const float *l, int64_t ld, int64_t plane, int ns, int64_t h, int64_t w,
                      const int32_t *cyx, const float *cval, int64_t cstride,
                      const int64_t *cscal, int32_t *det, float *dval, int64_t cap,
                      int64_t *n_det, float *thr_out, cudaStream_t st);
int detect(const float *l, int64_t ld, int64_t plane, int64_t ns, int64_t h, int64_t w,
           float frac, bool have_absmax, int32_t *det_idx, int idx_stride, float *det_val,
           int64_t cap, int64_t *n_det_dev, float *thr_dev, int64_t *n_det_host, void *ws,
           size_t ws_bytes, cudaStream_t st);

}  // namespace vmf
