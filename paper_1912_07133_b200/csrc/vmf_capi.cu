// vmf_capi.cu -- extern "C" entry points of libvmfilt_b200.so (declared in
// include/vmfilt_b200.h).  Host-side validation mirrors the reference
// wrappers (engine.py:105-109, 115-118, 139-142) before anything is launched.
#include <cstdlib>
#include <cstring>

#include "vmf_common.cuh"
#include "vmf_iir.cuh"
#include "vmf_colpass.cuh"
#include "vmf_rowlap.cuh"
#include "vmf_modal32.cuh"
#include "vmf_firpass.cuh"
#include "vmf_firtc.cuh"

namespace vmf {
size_t greedy_nms_workspace_bytes(int64_t n, int64_t h, int64_t w, double r2);
int greedy_nms(const int *cy, const int *cx, const double *nd, int64_t n, int64_t h, int64_t w,
               double r2, int *order, int *nkept, void *ws, size_t ws_bytes, cudaStream_t st);
}  // namespace vmf
#include "vmf_stage4.cuh"

namespace vmf {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_status(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(VMF_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return VMF_OK;
}

static size_t align256(size_t n) { return (n + 255) & ~(size_t)255; }

static int check_stage(const vmf_stage *s, int64_t length, const char *axis) {
  if (!s) return fail(VMF_EVALUE, "%s stage is NULL", axis);
  if (s->kind == VMF_STAGE_FIR) {
    if (!s->taps || s->n < 1 || s->n % 2 == 0)
      return fail(VMF_EVALUE, "taps must have odd length 2K+1");
    if (s->n > length)
      return fail(VMF_EVALUE, "kernel length %d exceeds row length %lld", s->n, (long long)length);
    return VMF_OK;
  }
  if (s->kind == VMF_STAGE_IIR) {
    if (s->n < 0 || s->n > VMF_MAX_IIR_ORDER)
      return fail(VMF_EVALUE, "IIR order %d outside 0..%d", s->n, VMF_MAX_IIR_ORDER);
    if (s->n > 0 && (!s->b_plus || !s->a_plus)) return fail(VMF_EVALUE, "IIR coefficients NULL");
    if (length < 2 * s->n + 1)
      return fail(VMF_EVALUE, "row length %lld < 2K+1 = %d", (long long)length, 2 * s->n + 1);
    if (s->n > 0 && !poles_inside_unit_circle(s->a_plus, s->n))
      return fail(VMF_ESTABILITY, "recursion has a pole on or outside the unit circle");
    return VMF_OK;
  }
  return fail(VMF_EVALUE, "unsupported stage type %d", s->kind);
}

static size_t stage_ws(const vmf_stage *s, int64_t lines, int64_t length) {
  if (s && s->kind == VMF_STAGE_IIR) return iir_workspace_bytes(lines, length, s->n);
  return 0;
}

template <int O>
static int run_stage(const vmf_stage *s, const void *x, int dt, float *y, int64_t h, int64_t w,
                     int64_t ldx, int64_t ldy, void *ws, size_t wsb, cudaStream_t st) {
  if (s->kind == VMF_STAGE_FIR) return fir_pass<O>(x, dt, y, h, w, ldx, ldy, s->taps, s->n, st);
  return iir_pass<O>(x, dt, y, h, w, ldx, ldy, s->b_plus, s->a_plus, s->n, s->b_zero, s->sign,
                     ws, wsb, st);
}

}  // namespace vmf

using namespace vmf;

extern "C" {

const char *vmf_last_error(void) { return g_err; }
int vmf_abi_version(void) { return 1; }

size_t vmf_iir_workspace_bytes(int64_t lines, int64_t length, int k) {
  return iir_workspace_bytes(lines, length, k);
}

size_t vmf_iir_cols_workspace_bytes(int64_t h, int64_t w, int k) {
  size_t g = iir_workspace_bytes(w, h, k);
  if (!colpass_supported(h, w, k)) return g;
  size_t c = colpass_workspace_bytes(h, w, k, 0) + 256;
  return c > g ? c : g;
}

int vmf_iir_rows(const void *x, int x_dtype, float *y, int64_t h, int64_t w, int64_t ldx,
                 int64_t ldy, const double *b_plus, const double *a_plus, int k, double b_zero,
                 int sign, void *ws, size_t ws_bytes, void *stream) {
  return iir_pass<ROWS>(x, x_dtype, y, h, w, ldx, ldy, b_plus, a_plus, k, b_zero, sign, ws,
                        ws_bytes, (cudaStream_t)stream);
}

int vmf_iir_cols(const void *x, int x_dtype, float *y, int64_t h, int64_t w, int64_t ldx,
                 int64_t ldy, const double *b_plus, const double *a_plus, int k, double b_zero,
                 int sign, void *ws, size_t ws_bytes, void *stream) {
  return iir_pass<COLS>(x, x_dtype, y, h, w, ldx, ldy, b_plus, a_plus, k, b_zero, sign, ws,
                        ws_bytes, (cudaStream_t)stream);
}

int vmf_conv_rows(const void *x, int x_dtype, float *y, int64_t h, int64_t w, int64_t ldx,
                  int64_t ldy, const double *taps, int ntaps, void *stream) {
  return fir_pass<ROWS>(x, x_dtype, y, h, w, ldx, ldy, taps, ntaps, (cudaStream_t)stream);
}

int vmf_conv_cols(const void *x, int x_dtype, float *y, int64_t h, int64_t w, int64_t ldx,
                  int64_t ldy, const double *taps, int ntaps, void *stream) {
  return fir_pass<COLS>(x, x_dtype, y, h, w, ldx, ldy, taps, ntaps, (cudaStream_t)stream);
}

int vmf_laplacian(const float *b, float *l, int64_t h, int64_t w, int64_t ldb, int64_t ldl,
                  float lap_scale, void *stream) {
  if (h < 1 || w < 1) return fail(VMF_EVALUE, "image must be a 2-D array");
  if (ldb < w || ldl < w) return fail(VMF_EVALUE, "row pitch smaller than width");
  return laplacian(b, ldb, l, ldl, h, w, lap_scale, nullptr, (cudaStream_t)stream);
}

size_t vmf_detect_workspace_bytes(int64_t h, int64_t w) { return detect_workspace_bytes(1, h, w); }

int vmf_detect3x3(const float *l, int64_t h, int64_t w, int64_t ldl, float frac, int32_t *det_yx,
                  float *det_val, int64_t cap, int64_t *n_det_dev, float *thr_dev,
                  int64_t *n_det_host, void *ws, size_t ws_bytes, void *stream) {
  if (h < 1 || w < 1) return fail(VMF_EVALUE, "image must be a 2-D array");
  if (ldl < w) return fail(VMF_EVALUE, "row pitch smaller than width");
  return detect(l, ldl, h * ldl, 1, h, w, frac, false, det_yx, 2, det_val, cap, n_det_dev,
                thr_dev, n_det_host, ws, ws_bytes, (cudaStream_t)stream);
}

size_t vmf_detect3x3x3_workspace_bytes(int64_t ns, int64_t h, int64_t w) {
  return detect_workspace_bytes(ns, h, w);
}

int vmf_detect3x3x3(const float *n, int64_t ns, int64_t h, int64_t w, int64_t ldn,
                    int64_t plane_stride, float frac, int32_t *det_syx, float *det_val,
                    int64_t cap, int64_t *n_det_dev, float *thr_dev, int64_t *n_det_host,
                    void *ws, size_t ws_bytes, void *stream) {
  if (ns < 1 || h < 1 || w < 1) return fail(VMF_EVALUE, "stack must be 3-D and non-empty");
  if (ldn < w || plane_stride < h * ldn) return fail(VMF_EVALUE, "bad stack strides");
  return detect(n, ldn, plane_stride, ns, h, w, frac, false, det_syx, 3, det_val, cap, n_det_dev,
                thr_dev, n_det_host, ws, ws_bytes, (cudaStream_t)stream);
}

int vmf_detect3x3x3_cands(const float *n, int64_t ns, int64_t h, int64_t w, int64_t ldn,
                          int64_t plane_stride, const int32_t *cand_yx, const float *cand_val,
                          int64_t cand_stride, const int64_t *cand_scal, int32_t *det_syx,
                          float *det_val, int64_t cap, int64_t *n_det_dev, float *thr_dev,
                          void *stream) {
  if (ns < 1 || ns > 64 || h < 1 || w < 1) return fail(VMF_EVALUE, "stack must be 3-D and non-empty");
  if (ldn < w || plane_stride < h * ldn) return fail(VMF_EVALUE, "bad stack strides");
  if (!cand_yx || !cand_val || !cand_scal || cand_stride < 1 || !n_det_dev)
    return fail(VMF_EVALUE, "candidate lists missing");
  if (cap > 0 && (!det_syx || !det_val)) return fail(VMF_EVALUE, "detection buffers are NULL");
  return detect3x3x3_cands(n, ldn, plane_stride, (int)ns, h, w, cand_yx, cand_val, cand_stride,
                           cand_scal, det_syx, det_val, cap, n_det_dev, thr_dev,
                           (cudaStream_t)stream);
}

int vmf_detect3x3x3_absmax(const float *n, int64_t ns, int64_t h, int64_t w, int64_t ldn,
                           int64_t plane_stride, float frac, const float *absmax_dev,
                           int32_t *det_syx, float *det_val, int64_t cap, int64_t *n_det_dev,
                           float *thr_dev, int64_t *n_det_host, void *ws, size_t ws_bytes,
                           void *stream) {
  if (ns < 1 || h < 1 || w < 1) return fail(VMF_EVALUE, "stack must be 3-D and non-empty");
  if (ldn < w || plane_stride < h * ldn) return fail(VMF_EVALUE, "bad stack strides");
  if (!absmax_dev) return fail(VMF_EVALUE, "absmax_dev must not be NULL");
  if (!ws || ws_bytes < detect_workspace_bytes(ns, h, w))
    return fail(VMF_EVALUE, "detect workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemcpyAsync(detect_absmax_slot(ws), absmax_dev, sizeof(float), cudaMemcpyDeviceToDevice, st);
  return detect(n, ldn, plane_stride, ns, h, w, frac, true, det_syx, 3, det_val, cap, n_det_dev,
                thr_dev, n_det_host, ws, ws_bytes, st);
}

static bool iir_b64(const vmf_stage *col_stage, int64_t h, int64_t w) {
  return col_stage && col_stage->kind == VMF_STAGE_IIR && colpass_supported(h, w, col_stage->n);
}

size_t vmf_hessian_detect_workspace_bytes(int64_t h, int64_t w, const vmf_stage *row_stage,
                                          const vmf_stage *col_stage) {
  size_t b = align256((size_t)h * w * sizeof(float)) + align256(stage_ws(row_stage, h, w)) + 256;
  if (iir_b64(col_stage, h, w))  // fp64 blur + the IIR column-pass workspace
    b += align256((size_t)h * w * sizeof(double)) +
         align256(colpass_workspace_bytes(h, w, col_stage->n, 0));
  return b;
}

// row stage into T, then the fp64 blur B64 of an IIR column stage
static int blur64_iir(const void *x, int x_dtype, int64_t h, int64_t w, int64_t ldx,
                      const vmf_stage *row_stage, const vmf_stage *col_stage, void *ws,
                      double **b64, cudaStream_t st) {
  char *p = (char *)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  float *T = (float *)p;
  p += align256((size_t)h * w * sizeof(float));
  const size_t rws = align256(stage_ws(row_stage, h, w));
  int rc = run_stage<ROWS>(row_stage, x, x_dtype, T, h, w, ldx, w, p, rws, st);
  if (rc) return rc;
  p += rws;
  *b64 = (double *)p;
  p += align256((size_t)h * w * sizeof(double));
  IirParams ip;
  rc = iir_plan(&ip, w, h, col_stage->b_plus, col_stage->a_plus, col_stage->n, col_stage->b_zero,
                col_stage->sign);
  if (rc) return rc;
  return colpass_run(T, w, nullptr, 0, *b64, ip, h, w, 1.0f, 0.0f, nullptr, nullptr, 0, nullptr,
                     nullptr, p, align256(colpass_workspace_bytes(h, w, col_stage->n, 0)), st);
}

int vmf_hessian_detect(const void *x, int x_dtype, int64_t h, int64_t w, int64_t ldx,
                       const vmf_stage *row_stage, const vmf_stage *col_stage, double sigma,
                       double t1, int polarity, float *nd_field, float *trace_field,
                       int64_t ldn, int32_t *cy, int32_t *cx, double *cnd, float *cdx,
                       float *cdy, int64_t cap, int32_t *count_dev, void *ws, size_t ws_bytes,
                       void *stream) {
  if (h < 1 || w < 1) return fail(VMF_EVALUE, "image must be a 2-D array");
  if (ldx < w) return fail(VMF_EVALUE, "row pitch smaller than width");
  int rc = check_stage(row_stage, w, "row");
  if (rc) return rc;
  rc = check_stage(col_stage, h, "column");
  if (rc) return rc;
  const bool iir = iir_b64(col_stage, h, w);
  if (!iir && (col_stage->kind != VMF_STAGE_FIR || !firpass_supported(h, w, col_stage->n)))
    return fail(VMF_EVALUE, "Hessian detector: column stage unsupported (FIR <= %d taps or "
                "IIR K = 2..4)", kFirMaxFast);
  if ((nd_field || trace_field) && ldn < w) return fail(VMF_EVALUE, "field pitch smaller than width");
  if (!count_dev || (cap > 0 && (!cy || !cx || !cnd || !cdx || !cdy)))
    return fail(VMF_EVALUE, "candidate outputs missing");
  size_t need = vmf_hessian_detect_workspace_bytes(h, w, row_stage, col_stage);
  if (!ws || ws_bytes < need)
    return fail(VMF_EVALUE, "workspace too small: %zu < %zu bytes", ws_bytes, need);
  cudaStream_t st = (cudaStream_t)stream;
  if (iir) {
    double *b64 = nullptr;
    rc = blur64_iir(x, x_dtype, h, w, ldx, row_stage, col_stage, ws, &b64, st);
    if (rc) return rc;
    return hess_from_b64(b64, h, w, sigma, t1, polarity, nd_field, trace_field, ldn, cy, cx, cnd,
                         cdx, cdy, cap, count_dev, st);
  }
  char *p = (char *)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  float *T = (float *)p;
  p += align256((size_t)h * w * sizeof(float));
  rc = run_stage<ROWS>(row_stage, x, x_dtype, T, h, w, ldx, w, p,
                       align256(stage_ws(row_stage, h, w)), st);
  if (rc) return rc;
  return hesspass_run(T, w, col_stage->taps, col_stage->n, h, w, sigma, t1, polarity, nd_field,
                      trace_field, ldn, cy, cx, cnd, cdx, cdy, cap, count_dev, st);
}

int vmf_derivative_field(const void *x, int x_dtype, int64_t h, int64_t w, int64_t ldx,
                         const vmf_stage *row_stage, const vmf_stage *col_stage, float *d00,
                         float *d10, float *d01, float *d20, float *d02, float *d11, int64_t ldo,
                         void *ws, size_t ws_bytes, void *stream) {
  if (h < 1 || w < 1) return fail(VMF_EVALUE, "image must be a 2-D array");
  if (ldx < w || ldo < w) return fail(VMF_EVALUE, "row pitch smaller than width");
  int rc = check_stage(row_stage, w, "row");
  if (rc) return rc;
  rc = check_stage(col_stage, h, "column");
  if (rc) return rc;
  const bool iir = iir_b64(col_stage, h, w);
  if (!iir && (col_stage->kind != VMF_STAGE_FIR || !firpass_supported(h, w, col_stage->n)))
    return fail(VMF_EVALUE, "derivative bank: column stage unsupported (FIR <= %d taps or IIR "
                "K = 2..4)", kFirMaxFast);
  size_t need = vmf_hessian_detect_workspace_bytes(h, w, row_stage, col_stage);
  if (!ws || ws_bytes < need)
    return fail(VMF_EVALUE, "workspace too small: %zu < %zu bytes", ws_bytes, need);
  cudaStream_t st = (cudaStream_t)stream;
  if (iir) {
    double *b64 = nullptr;
    rc = blur64_iir(x, x_dtype, h, w, ldx, row_stage, col_stage, ws, &b64, st);
    if (rc) return rc;
    float *outs[6] = {d00, d10, d01, d20, d02, d11};
    return deriv_from_b64(b64, h, w, outs, ldo, st);
  }
  char *p = (char *)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  float *T = (float *)p;
  p += align256((size_t)h * w * sizeof(float));
  rc = run_stage<ROWS>(row_stage, x, x_dtype, T, h, w, ldx, w, p,
                       align256(stage_ws(row_stage, h, w)), st);
  if (rc) return rc;
  float *outs[6] = {d00, d10, d01, d20, d02, d11};
  return derivpass_run(T, w, col_stage->taps, col_stage->n, h, w, outs, ldo, st);
}

size_t vmf_greedy_nms_workspace_bytes(int64_t n, int64_t h, int64_t w, double r2) {
  return greedy_nms_workspace_bytes(n, h, w, r2);
}

int vmf_greedy_nms(const int32_t *cy, const int32_t *cx, const double *cnd, int64_t n, int64_t h,
                   int64_t w, double r2, int32_t *order, int32_t *n_kept_dev, void *ws,
                   size_t ws_bytes, void *stream) {
  if (h < 1 || w < 1) return fail(VMF_EVALUE, "image must be a 2-D array");
  if (!n_kept_dev || (n > 0 && (!cy || !cx || !cnd || !order)))
    return fail(VMF_EVALUE, "NMS inputs missing");
  return greedy_nms(cy, cx, cnd, n, h, w, r2, order, n_kept_dev, ws, ws_bytes,
                    (cudaStream_t)stream);
}

static bool fused_col(const vmf_stage *col_stage, int64_t h, int64_t w) {
  return col_stage && col_stage->kind == VMF_STAGE_IIR && colpass_supported(h, w, col_stage->n) &&
         !getenv("VMF_FORCE_GENERIC");
}

static bool fused_fir_col(const vmf_stage *col_stage, int64_t h, int64_t w) {
  return col_stage && col_stage->kind == VMF_STAGE_FIR &&
         firpass_supported(h, w, col_stage->n) && !getenv("VMF_FORCE_GENERIC");
}

// workspace: [T row-pass out][B if blur_out NULL][L if lap_out NULL][iir carry][detect]
size_t vmf_blur_lap_detect_workspace_bytes(int64_t h, int64_t w, const vmf_stage *row_stage,
                                           const vmf_stage *col_stage) {
  size_t img = align256((size_t)h * w * sizeof(float));
  size_t carry = stage_ws(row_stage, h, w);
  size_t c2 = stage_ws(col_stage, w, h);
  if (c2 > carry) carry = c2;
  if (fused_col(col_stage, h, w)) {
    size_t c3 = colpass_workspace_bytes(h, w, col_stage->n, 0);
    if (c3 > carry) carry = c3;
    c3 = colpass32_workspace_bytes(h, w, col_stage->n);
    if (c3 > carry) carry = c3;
  }
  if (fused_fir_col(col_stage, h, w)) {
    size_t c4 = firpass_workspace_bytes(h, w);
    if (c4 > carry) carry = c4;
  }
  if (row_stage && col_stage && row_stage->kind == VMF_STAGE_FIR &&
      col_stage->kind == VMF_STAGE_FIR) {
    size_t c5 = firtc_workspace_bytes(h, w, row_stage->n, col_stage->n);
    if (c5 > carry) carry = c5;
  }
  return 3 * img + align256(carry) + align256(detect_workspace_bytes(1, h, w)) + 256 +
         align256((size_t)sweep_extras_floats(w) * sizeof(float));  // fp32 row pass extras
}

// The all-fp32 "Laplacian-first" path (vmf_rowlap.cu + vmf_colpass32.cu V
// mode): fp32 frames with W = 32 C (C <= 256), 16-byte aligned rows, IIR row
// and column stages with a modal fp32 realisation.
static SweepStage sweep_stage(const vmf_stage *row, const vmf_stage *col) {
  SweepStage s;
  s.rb = row->b_plus;
  s.ra = row->a_plus;
  s.rb0 = row->b_zero;
  s.rsign = row->sign;
  s.cb = col->b_plus;
  s.ca = col->a_plus;
  s.cb0 = col->b_zero;
  s.csign = col->sign;
  return s;
}

// The all-fp32 "Laplacian-first" path (vmf_rowlap.cu + vmf_colpass32.cu V
// mode): fp32 frames with W = 32 C (C <= 256), 16-byte aligned rows, IIR row
// and column stages of one order with a modal fp32 realisation.
static bool lapfirst_ok(const void *x, int x_dtype, int64_t h, int64_t w, int64_t ldx, int ns,
                        const vmf_stage *rows, const vmf_stage *cols) {
  if (x_dtype != VMF_F32 || getenv("VMF_FORCE_GENERIC") || ns < 1 || ns > kMaxScales) return false;
  SweepStage st[kMaxScales];
  for (int s = 0; s < ns; ++s) {
    const vmf_stage *r = rows + s, *cl = cols + s;
    if (r->kind != VMF_STAGE_IIR || cl->kind != VMF_STAGE_IIR || r->n != cl->n ||
        r->n != rows[0].n)
      return false;
    IirParams ip;
    if (iir_plan(&ip, w, h, cl->b_plus, cl->a_plus, cl->n, cl->b_zero, cl->sign)) {
      cudaGetLastError();
      return false;
    }
    if (!colpass32_supported(h, w, ip)) return false;
    st[s] = sweep_stage(r, cl);
  }
  return sweep_supported(x, h, w, ldx, rows[0].n, ns, st);
}

static size_t sweep_ws_bytes(int64_t h, int64_t w, int ns) {
  return (size_t)ns * (align256((size_t)h * w * sizeof(float)) +
                       align256((size_t)sweep_extras_floats(w) * sizeof(float))) + 256;
}

static SweepOut sweep_layout(void *sws, int64_t h, int64_t w, int ns) {
  (void)ns;
  SweepOut o;
  memset(&o, 0, sizeof(o));
  char *p = (char *)(((uintptr_t)sws + 255) & ~(uintptr_t)255);
  const size_t vb = align256((size_t)h * w * sizeof(float));
  const size_t eb = align256((size_t)sweep_extras_floats(w) * sizeof(float));
  o.V0 = (float *)p;
  o.E0 = (float *)(p + vb);
  o.vstride = o.estride = (int64_t)((vb + eb) / sizeof(float));
  o.ldv = w;
  return o;
}

// the column pass of scale s of a sweep (V mode) into L + detections
static int sweep_cols(const SweepOut &o, int s, int64_t h, int64_t w, const vmf_stage *col,
                      float lap_scale, float frac, float *L, int64_t ldl, int32_t *det_yx,
                      float *det_val, int64_t cap, int64_t *n_det_dev, float *thr_dev, void *cws,
                      size_t cws_b, cudaStream_t st) {
  IirParams ip;
  int rc = iir_plan(&ip, w, h, col->b_plus, col->a_plus, col->n, col->b_zero, col->sign);
  if (rc) return rc;
  const float *E = o.E(s);
  const Col32VMode vm = {E + kExVt * w, E + kExVb * w, E + kExKy * w};
  return colpass32_run(o.V(s), o.ldv, L, ldl, ip, h, w, lap_scale, frac, det_yx, det_val, cap,
                       n_det_dev, thr_dev, cws, cws_b, st, &vm);
}

int vmf_blur_lap_detect(const void *x, int x_dtype, int64_t h, int64_t w, int64_t ldx,
                        const vmf_stage *row_stage, const vmf_stage *col_stage, float lap_scale,
                        float frac, float *blur_out, float *lap_out, int32_t *det_yx,
                        float *det_val, int64_t cap, int64_t *n_det_dev, float *thr_dev,
                        int64_t *n_det_host, void *ws, size_t ws_bytes, void *stream) {
  if (h < 1 || w < 1) return fail(VMF_EVALUE, "image must be a 2-D array");
  if (ldx < w) return fail(VMF_EVALUE, "row pitch smaller than width");
  int rc = check_stage(row_stage, w, "row");
  if (rc) return rc;
  rc = check_stage(col_stage, h, "column");
  if (rc) return rc;
  size_t need = vmf_blur_lap_detect_workspace_bytes(h, w, row_stage, col_stage);
  if (!ws || ws_bytes < need)
    return fail(VMF_EVALUE, "workspace too small: %zu < %zu bytes", ws_bytes, need);
  cudaStream_t st = (cudaStream_t)stream;
  char *p = (char *)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  size_t img = align256((size_t)h * w * sizeof(float));
  float *T = (float *)p;
  p += img;
  float *B = blur_out ? blur_out : (float *)p;
  p += img;
  float *L = lap_out ? lap_out : (float *)p;
  p += img;
  const size_t vrows_b = align256((size_t)sweep_extras_floats(w) * sizeof(float));
  size_t carry_b = align256(vmf_blur_lap_detect_workspace_bytes(h, w, row_stage, col_stage) -
                            3 * img - align256(detect_workspace_bytes(1, h, w)) - 256 - vrows_b);
  void *carry = p;
  p += carry_b;
  void *dws = p;
  size_t dws_b = align256(detect_workspace_bytes(1, h, w));
  p += dws_b;
  float *vrows = (float *)p;
  if (lapfirst_ok(x, x_dtype, h, w, ldx, 1, row_stage, col_stage)) {
    // V = R(Lap5 X) into T's slot (a one-scale sweep), then the column pass
    // in V mode
    SweepOut o;
    memset(&o, 0, sizeof(o));
    o.V0 = T;
    o.E0 = vrows;
    o.ldv = w;
    SweepStage sst = sweep_stage(row_stage, col_stage);
    rc = sweep_rows((const float *)x, ldx, h, w, row_stage->n, 1, &sst, o, st);
    if (rc) return rc;
    rc = sweep_cols(o, 0, h, w, col_stage, lap_scale, frac, lap_out, w, det_yx, det_val, cap,
                    n_det_dev, thr_dev, carry, carry_b, st);
    if (rc) return rc;
    if (blur_out) {  // B on request: T into the (unused) B slot, then the column leaf
      float *Tb = T + img / sizeof(float);
      rc = run_stage<ROWS>(row_stage, x, x_dtype, Tb, h, w, ldx, w, carry, carry_b, st);
      if (rc) return rc;
      rc = run_stage<COLS>(col_stage, Tb, VMF_F32, blur_out, h, w, w, w, carry, carry_b, st);
      if (rc) return rc;
    }
    if (n_det_host && frac > 0.0f) {
      cudaMemcpyAsync(n_det_host, n_det_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      return cuda_status("detect readback");
    }
    return VMF_OK;
  }
  // the tensor-core FIR path beats the fp64 CUDA-core one from ~65 taps
  // (profiles/README.md); VMF_FORCE_FIRTC takes it for any length (tests)
  const bool force_tc = getenv("VMF_FORCE_FIRTC") != nullptr;
  if (x_dtype == VMF_F32 && row_stage->kind == VMF_STAGE_FIR && col_stage->kind == VMF_STAGE_FIR &&
      !getenv("VMF_FORCE_GENERIC") && firtc_supported(h, w, ldx, row_stage->n, col_stage->n) &&
      ((uintptr_t)x & 15) == 0 &&
      !getenv("VMF_NO_FIRTC") &&  // (tests: the fp64 fused FIR pass at any length)
      (force_tc || (row_stage->n > col_stage->n ? row_stage->n : col_stage->n) >= kFirTcMinTaps)) {
    // both FIR passes on the tensor cores, Laplacian first, then stage 4
    // (vmf_firtc.cu)
    rc = firtc_detect((const float *)x, ldx, h, w, row_stage->taps, row_stage->n, col_stage->taps,
                      col_stage->n, lap_scale, frac, L, w, det_yx, det_val, cap, n_det_dev, thr_dev,
                      carry, carry_b, st);
    if (rc) return rc;
    if (blur_out) {  // B on request: the two FIR leaves (T in T's slot)
      rc = run_stage<ROWS>(row_stage, x, x_dtype, T, h, w, ldx, w, carry, carry_b, st);
      if (rc) return rc;
      rc = run_stage<COLS>(col_stage, T, VMF_F32, blur_out, h, w, w, w, carry, carry_b, st);
      if (rc) return rc;
    }
    if (n_det_host && frac > 0.0f) {
      cudaMemcpyAsync(n_det_host, n_det_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      return cuda_status("detect readback");
    }
    return VMF_OK;
  }
  rc = run_stage<ROWS>(row_stage, x, x_dtype, T, h, w, ldx, w, carry, carry_b, st);
  if (rc) return rc;
  if (fused_col(col_stage, h, w)) {
    // column IIR + Laplacian + NMS in one pass over T (vmf_colpass.cu)
    IirParams ip;
    rc = iir_plan(&ip, w, h, col_stage->b_plus, col_stage->a_plus, col_stage->n,
                  col_stage->b_zero, col_stage->sign);
    if (rc) return rc;
    if (colpass32_supported(h, w, ip))  // fp32 "Laplacian first" (vmf_colpass32.cu)
      rc = colpass32_run(T, w, lap_out, w, ip, h, w, lap_scale, frac, det_yx, det_val, cap,
                         n_det_dev, thr_dev, carry, carry_b, st);
    else
      rc = colpass_run(T, w, L, w, nullptr, ip, h, w, lap_scale, frac, det_yx, det_val, cap,
                       n_det_dev, thr_dev, carry, carry_b, st);
    if (rc) return rc;
    if (blur_out) {  // B is not materialised by the fused pass; recompute on request
      rc = run_stage<COLS>(col_stage, T, VMF_F32, blur_out, h, w, w, w, carry, carry_b, st);
      if (rc) return rc;
    }
    if (n_det_host && frac > 0.0f) {
      cudaMemcpyAsync(n_det_host, n_det_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      return cuda_status("detect readback");
    }
    return VMF_OK;
  }
  if (fused_fir_col(col_stage, h, w)) {
    // column FIR + Laplacian + NMS in one pass over T (vmf_firpass.cu)
    rc = firpass_run(T, w, lap_out, w, col_stage->taps, col_stage->n, h, w, lap_scale, frac,
                     det_yx, det_val, cap, n_det_dev, thr_dev, carry, carry_b, st);
    if (rc) return rc;
    if (blur_out) {
      rc = run_stage<COLS>(col_stage, T, VMF_F32, blur_out, h, w, w, w, carry, carry_b, st);
      if (rc) return rc;
    }
    if (n_det_host && frac > 0.0f) {
      cudaMemcpyAsync(n_det_host, n_det_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      return cuda_status("detect readback");
    }
    return VMF_OK;
  }
  rc = run_stage<COLS>(col_stage, T, VMF_F32, B, h, w, w, w, carry, carry_b, st);
  if (rc) return rc;
  float *absmax = detect_absmax_slot(dws);
  cudaMemsetAsync(absmax, 0, sizeof(float), st);
  rc = laplacian(B, w, L, w, h, w, lap_scale, absmax, st);
  if (rc) return rc;
  if (frac <= 0.0f) return VMF_OK;
  return detect(L, w, h * w, 1, h, w, frac, true, det_yx, 2, det_val, cap, n_det_dev, thr_dev,
                n_det_host, dws, dws_b, st);
}

// ---------------------------------------------------------------------------
// multi-scale sweep: one fp32 row pass over X for every scale, then one
// column pass per scale (any stream ordered after vmf_sweep_rows)
// ---------------------------------------------------------------------------
size_t vmf_sweep_workspace_bytes(int64_t h, int64_t w, int nscales) {
  return sweep_ws_bytes(h, w, nscales);
}

size_t vmf_sweep_detect_workspace_bytes(int64_t h, int64_t w, const vmf_stage *col_stage) {
  return align256(colpass32_workspace_bytes(h, w, col_stage ? col_stage->n : 4)) + 256;
}

int vmf_sweep_supported(const void *x, int x_dtype, int64_t h, int64_t w, int64_t ldx,
                        int nscales, const vmf_stage *row_stages, const vmf_stage *col_stages) {
  if (!row_stages || !col_stages || h < 1 || w < 1 || ldx < w) return 0;
  for (int s = 0; s < nscales; ++s)
    if (check_stage(row_stages + s, w, "row") || check_stage(col_stages + s, h, "column")) {
      set_error("%s", "");
      return 0;
    }
  return lapfirst_ok(x, x_dtype, h, w, ldx, nscales, row_stages, col_stages) ? 1 : 0;
}

int vmf_sweep_rows(const void *x, int x_dtype, int64_t h, int64_t w, int64_t ldx, int nscales,
                   const vmf_stage *row_stages, const vmf_stage *col_stages, void *sweep_ws,
                   size_t sweep_ws_bytes_, void *stream) {
  if (!vmf_sweep_supported(x, x_dtype, h, w, ldx, nscales, row_stages, col_stages))
    return fail(VMF_EVALUE, "sweep: frame / stages not supported by the fp32 path");
  if (!sweep_ws || sweep_ws_bytes_ < sweep_ws_bytes(h, w, nscales))
    return fail(VMF_EVALUE, "sweep workspace too small");
  SweepStage st[kMaxScales];
  for (int s = 0; s < nscales; ++s) st[s] = sweep_stage(row_stages + s, col_stages + s);
  const SweepOut o = sweep_layout(sweep_ws, h, w, nscales);
  return sweep_rows((const float *)x, ldx, h, w, row_stages[0].n, nscales, st, o,
                    (cudaStream_t)stream);
}

int vmf_sweep_detect(int scale, int64_t h, int64_t w, int nscales, const vmf_stage *col_stage,
                     float lap_scale, float frac, float *lap_out, int32_t *det_yx,
                     float *det_val, int64_t cap, int64_t *n_det_dev, float *thr_dev,
                     void *sweep_ws, size_t sweep_ws_bytes_, void *ws, size_t ws_bytes,
                     void *stream) {
  if (scale < 0 || scale >= nscales) return fail(VMF_EVALUE, "scale index out of range");
  int rc = check_stage(col_stage, h, "column");
  if (rc) return rc;
  if (!sweep_ws || sweep_ws_bytes_ < sweep_ws_bytes(h, w, nscales))
    return fail(VMF_EVALUE, "sweep workspace too small");
  const size_t need = vmf_sweep_detect_workspace_bytes(h, w, col_stage);
  if (!ws || ws_bytes < need)
    return fail(VMF_EVALUE, "workspace too small: %zu < %zu bytes", ws_bytes, need);
  if (frac > 0.0f && (!n_det_dev || !thr_dev || (cap > 0 && (!det_yx || !det_val))))
    return fail(VMF_EVALUE, "detection outputs missing");
  const SweepOut o = sweep_layout(sweep_ws, h, w, nscales);
  char *p = (char *)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  // lap_out null: detections only, L stays in the column pass's tiles
  return sweep_cols(o, scale, h, w, col_stage, lap_scale, frac, lap_out, w, det_yx, det_val, cap,
                    n_det_dev, thr_dev, p, align256(colpass32_workspace_bytes(h, w, col_stage->n)),
                    (cudaStream_t)stream);
}

}  // extern "C"
