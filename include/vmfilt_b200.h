/*
 * vmfilt_b200.h -- C ABI of the B200-native hot path of `vmfilt`
 * (Kennedy, "vanishing-moment shape filters", arXiv 1912.07133).
 *
 * Each entry point replaces one native kernel (or wrapper + kernel) of the
 * reference package; file:line below are relative to
 * /root/reference/pkg/src/vmfilt/.  The reference crosses Python -> numba
 * native code at exactly these points (engine.py:120, engine.py:145); the
 * matching ctypes binding is shown in INTEGRATION.md.
 *
 * Conventions:
 *   - every array pointer is a DEVICE pointer (cudaMalloc / torch CUDA
 *     tensor); images are row-major [h][w] with row pitches ldx/ldy in
 *     ELEMENTS; outputs are caller-allocated and fully written; inputs are
 *     never modified;
 *   - work is enqueued on `stream` (a cudaStream_t, NULL = legacy default)
 *     and is asynchronous; no entry point synchronises the host except
 *     vmf_detect* when n_det_host != NULL;
 *   - return codes: VMF_OK, VMF_EVALUE (the reference raises ValueError),
 *     VMF_ESTABILITY (the reference raises StabilityError, errors.py:32),
 *     VMF_ECUDA (CUDA launch/runtime failure).  vmf_last_error() gives the
 *     message of the last failure on the calling thread;
 *   - results do not depend on launch configuration (chunk count, block
 *     size): the analogue of tests/test_engine.py:119-128.
 *   - arithmetic: fp32 loads/stores, fp64 recurrence state and fp64
 *     accumulation.
 */
#ifndef VMFILT_B200_H
#define VMFILT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { VMF_OK = 0, VMF_EVALUE = 2, VMF_ESTABILITY = 3, VMF_ECUDA = 4 };
/* input element types of the first (row) pass: fp32, u16 in host order,
   u8, and big-endian u16 -- the sample bytes of a PGM P5 file with
   maxval > 255 (pgmio.py:40-45), byte-swapped inside the row pass */
enum { VMF_F32 = 0, VMF_U16 = 1, VMF_U8 = 2, VMF_U16BE = 3 };
/* stage kinds for vmf_stage */
enum { VMF_STAGE_FIR = 0, VMF_STAGE_IIR = 1 };

#define VMF_MAX_IIR_ORDER 8    /* polyz.py:494-495 allows K <= 8 */
#define VMF_MAX_FIR_TAPS 2049   /* taps travel as kernel parameters */

/* A separable stage: FirKernel (design.py:40-77) or ThreePartIIR
 * (polyz.py:348-405), flattened to plain arrays.  Host pointers. */
typedef struct vmf_stage {
  int kind;               /* VMF_STAGE_FIR | VMF_STAGE_IIR               */
  int n;                  /* FIR: number of taps 2K+1; IIR: order K       */
  const double *taps;     /* FIR taps h(-K..K) (FirKernel.taps)           */
  const double *b_plus;   /* IIR b_plus[0..K-1]  (m = 1..K)              */
  const double *a_plus;   /* IIR a_plus[0..K-1]                          */
  double b_zero;          /* IIR b_zero                                   */
  int sign;               /* IIR +1 parity "sym", -1 parity "anti"        */
} vmf_stage;

const char *vmf_last_error(void);
int vmf_abi_version(void);

/* Workspace (bytes, device memory) needed by one IIR pass over `lines`
 * lines of `length` samples of order k. */
size_t vmf_iir_workspace_bytes(int64_t lines, int64_t length, int k);
/* workspace of vmf_iir_cols that also admits its fast path (fp32 input,
   K 2..4: the band-parallel column pass); vmf_iir_workspace_bytes(w, h, k)
   still works with the generic column kernel */
size_t vmf_iir_cols_workspace_bytes(int64_t h, int64_t w, int k);

/* Three-part IIR along rows: replaces iir_rows (engine.py:137-153) and
 * _iir_rows_kernel (engine.py:65-102).  Validation identical to
 * engine.py:139-142: w >= 2K+1 else VMF_EVALUE; all poles strictly inside
 * the unit circle else VMF_ESTABILITY. */
int vmf_iir_rows(const void *x, int x_dtype, float *y, int64_t h, int64_t w,
                 int64_t ldx, int64_t ldy, const double *b_plus,
                 const double *a_plus, int k, double b_zero, int sign,
                 void *ws, size_t ws_bytes, void *stream);

/* Three-part IIR along columns: replaces iir_cols (engine.py:156-158)
 * without the two transposed copies.  Requires h >= 2K+1. */
int vmf_iir_cols(const void *x, int x_dtype, float *y, int64_t h, int64_t w,
                 int64_t ldx, int64_t ldy, const double *b_plus,
                 const double *a_plus, int k, double b_zero, int sign,
                 void *ws, size_t ws_bytes, void *stream);

/* Centred FIR along rows with replicate edges: replaces conv_rows
 * (engine.py:112-121) and _conv_rows_kernel (engine.py:35-62).  ntaps odd,
 * ntaps <= w else VMF_EVALUE (engine.py:115-118). */
int vmf_conv_rows(const void *x, int x_dtype, float *y, int64_t h, int64_t w,
                  int64_t ldx, int64_t ldy, const double *taps, int ntaps,
                  void *stream);

/* FIR along columns: replaces conv_cols (engine.py:124-126). ntaps <= h. */
int vmf_conv_cols(const void *x, int x_dtype, float *y, int64_t h, int64_t w,
                  int64_t ldx, int64_t ldy, const double *taps, int ntaps,
                  void *stream);

/* Laplacian L = lap_scale * (D20 + D02) with the (1,-2,1) stencil of
 * fir_vm_bank(3)[2] and replicate edges: replaces derivative_field's
 * D20/D02 pair (engine.py:218-227) and the trace of blob.py:161.
 * lap_scale = 1 reproduces the reference; sigma^2 gives the scale-normalised
 * response used by the scale-space NMS. */
int vmf_laplacian(const float *b, float *l, int64_t h, int64_t w, int64_t ldb,
                  int64_t ldl, float lap_scale, void *stream);

/* Workspace for vmf_detect3x3 / vmf_blur_lap_detect. */
size_t vmf_detect_workspace_bytes(int64_t h, int64_t w);

/* Threshold + 3x3 NMS (stage 4; conventions of
 * blob.py:162-168): a pixel is a detection iff it is strictly greater (or
 * strictly smaller) than its 8 edge-replicated neighbours and
 * |L| >= frac * max|L| over the frame.  Detections are written sorted by
 * (y, x): det_yx[2i] = y, det_yx[2i+1] = x, det_val[i] = L(y, x).
 * *n_det_dev (device int64) receives the total count (may exceed cap);
 * *thr_dev (device float, may be NULL) the threshold used.  If n_det_host
 * is non-NULL the call synchronises `stream` and stores the count there. */
int vmf_detect3x3(const float *l, int64_t h, int64_t w, int64_t ldl,
                  float frac, int32_t *det_yx, float *det_val, int64_t cap,
                  int64_t *n_det_dev, float *thr_dev, int64_t *n_det_host,
                  void *ws, size_t ws_bytes, void *stream);

/* Whole hot path in one call: B = cols(rows(x, row_stage), col_stage);
 * L = lap_scale * Laplacian(B); detections as vmf_detect3x3 (frac <= 0
 * skips detection).  blur_out / lap_out may be NULL (pitch = w).  This is derivative_field + trace + stage 4 fused
 * (engine.py:205-228, blob.py:158-168). */
size_t vmf_blur_lap_detect_workspace_bytes(int64_t h, int64_t w,
                                           const vmf_stage *row_stage,
                                           const vmf_stage *col_stage);
int vmf_blur_lap_detect(const void *x, int x_dtype, int64_t h, int64_t w,
                        int64_t ldx, const vmf_stage *row_stage,
                        const vmf_stage *col_stage, float lap_scale, float frac,
                        float *blur_out, float *lap_out, int32_t *det_yx,
                        float *det_val, int64_t cap, int64_t *n_det_dev,
                        float *thr_dev, int64_t *n_det_host, void *ws,
                        size_t ws_bytes, void *stream);

/* Multi-scale sweep (config 3's scale sweep; engine.py:205-228 per scale):
 * the same blur -> Laplacian -> threshold + NMS per scale as
 * vmf_blur_lap_detect, with one row pass over x for every scale.
 * vmf_sweep_supported: nonzero when the fp32 "Laplacian-first" path takes
 * the sweep (fp32 x, w a multiple of 32 up to 8192, 16-byte aligned rows,
 * IIR row and column stages of one order with an fp32 modal realisation,
 * 1..8 scales).  vmf_sweep_rows: the row pass of every scale into
 * sweep_ws (vmf_sweep_workspace_bytes).  vmf_sweep_detect: the column pass
 * of one scale (any stream ordered after vmf_sweep_rows; scales are
 * independent and may run concurrently, each with its own ws of
 * vmf_sweep_detect_workspace_bytes); outputs as vmf_blur_lap_detect.
 * lap_out may be NULL: the detections are then made from the column pass's
 * tiles and L is never written (the candidate list is sized for every
 * strict 3x3 extremum of the frame, so no fallback needs L). */
size_t vmf_sweep_workspace_bytes(int64_t h, int64_t w, int nscales);
size_t vmf_sweep_detect_workspace_bytes(int64_t h, int64_t w, const vmf_stage *col_stage);
int vmf_sweep_supported(const void *x, int x_dtype, int64_t h, int64_t w, int64_t ldx,
                        int nscales, const vmf_stage *row_stages, const vmf_stage *col_stages);
int vmf_sweep_rows(const void *x, int x_dtype, int64_t h, int64_t w, int64_t ldx, int nscales,
                   const vmf_stage *row_stages, const vmf_stage *col_stages, void *sweep_ws,
                   size_t sweep_ws_bytes, void *stream);
int vmf_sweep_detect(int scale, int64_t h, int64_t w, int nscales, const vmf_stage *col_stage,
                     float lap_scale, float frac, float *lap_out, int32_t *det_yx,
                     float *det_val, int64_t cap, int64_t *n_det_dev, float *thr_dev,
                     void *sweep_ws, size_t sweep_ws_bytes, void *ws, size_t ws_bytes,
                     void *stream);

/* Scale-space 3x3x3 NMS over a stack of ns normalised responses
 * N[s] (each h x w, pitch ldn, planes spaced plane_stride elements):
 * strict extremum against the 8 in-scale and the 9+9 adjacent-scale
 * neighbours (one-sided at the first/last scale), |N| >= frac*max|N| over
 * the whole stack.  Detections sorted by (s, y, x): det_syx[3i..3i+2]. */
size_t vmf_detect3x3x3_workspace_bytes(int64_t ns, int64_t h, int64_t w);
/* The same with the stack maximum supplied (max |n| of a larger stack this
 * one is a slab of -- the scale-sharded sweep: each rank's
 * slab carries one halo plane of each neighbour and the all-reduced max):
 * threshold = frac * *absmax_dev. */
int vmf_detect3x3x3_absmax(const float *n, int64_t ns, int64_t h, int64_t w, int64_t ldn,
                           int64_t plane_stride, float frac, const float *absmax_dev,
                           int32_t *det_syx, float *det_val, int64_t cap, int64_t *n_det_dev,
                           float *thr_dev, int64_t *n_det_host, void *ws, size_t ws_bytes,
                           void *stream);
/* The same rule from the candidate lists of the stack's fused column passes
 * (vmf_sweep_detect with lap_out = plane s and frac > 0: plane s's strict
 * 3x3 extrema above frac * max|N_s|, sorted by (y, x); cand_yx[s][i][2],
 * cand_val[s][i] with cand_stride entries per scale, cand_scal[s] = {count,
 * threshold bits}): the stack threshold is the largest scale threshold and a
 * candidate is kept when it also clears the 9 + 9 adjacent-scale neighbours
 * -- the exact result of vmf_detect3x3x3 without a pass over the stack.
 * *n_det_dev = -1 when a scale's list was cut short (count > cand_stride):
 * run vmf_detect3x3x3 then. */
int vmf_detect3x3x3_cands(const float *n, int64_t ns, int64_t h, int64_t w, int64_t ldn,
                          int64_t plane_stride, const int32_t *cand_yx, const float *cand_val,
                          int64_t cand_stride, const int64_t *cand_scal, int32_t *det_syx,
                          float *det_val, int64_t cap, int64_t *n_det_dev, float *thr_dev,
                          void *stream);
int vmf_detect3x3x3(const float *n, int64_t ns, int64_t h, int64_t w,
                    int64_t ldn, int64_t plane_stride, float frac,
                    int32_t *det_syx, float *det_val, int64_t cap,
                    int64_t *n_det_dev, float *thr_dev, int64_t *n_det_host,
                    void *ws, size_t ws_bytes, void *stream);

/* Hessian blob detector: replaces the field stage of blob.detect
 * (blob.py:143-166; hessian_det blob.py:109-111, displacement
 * blob.py:114-128): row stage (IIR or FIR), then the
 * column stage -- fused with the derivative bank fir_vm_bank(3)
 * (design.py:250-280) on the fp64 blur for a FIR, or the fused IIR column
 * pass writing the fp64 blur followed by the bank -- giving
 * nd = sigma^4 (D20 D02 - D11^2), trace D20 + D02 and the stationary-point
 * displacement.  Candidates nd > t1 with the polarity
 * (+1 dark: trace > 0, -1 bright: trace < 0) are appended unordered:
 * (cy, cx, cnd, cdx, cdy)[0 .. min(count, cap)), *count_dev = all found.
 * nd_field / trace_field (pitch ldn) are optional fp32 outputs.
 * vmf_greedy_nms: replaces the suppression loop of blob.detect
 * (blob.py:168-176): greedy suppression within r (d^2 <= r2) in the order
 * (nd desc, y asc, x asc) of lexsort((x, y, -nd)); order[0 .. *n_kept_dev)
 * = kept candidate indices, strongest first (parallel rounds that keep
 * exactly the sequential greedy set). */
size_t vmf_hessian_detect_workspace_bytes(int64_t h, int64_t w, const vmf_stage *row_stage,
                                          const vmf_stage *col_stage);
int vmf_hessian_detect(const void *x, int x_dtype, int64_t h, int64_t w, int64_t ldx,
                       const vmf_stage *row_stage, const vmf_stage *col_stage, double sigma,
                       double t1, int polarity, float *nd_field, float *trace_field,
                       int64_t ldn, int32_t *cy, int32_t *cx, double *cnd, float *cdx,
                       float *cdy, int64_t cap, int32_t *count_dev, void *ws, size_t ws_bytes,
                       void *stream);
/* engine.derivative_field(order=3) (engine.py:205-228) for a FIR (one fused pass) or IIR
 * (fp64 blur, then the bank) column stage: D00 (the blur) D10 D01 D20 D02 D11 of the fp64 blur, fp32, pitch
 * ldo (any output may be NULL); workspace = vmf_hessian_detect_workspace_bytes. */
int vmf_derivative_field(const void *x, int x_dtype, int64_t h, int64_t w, int64_t ldx,
                         const vmf_stage *row_stage, const vmf_stage *col_stage, float *d00,
                         float *d10, float *d01, float *d20, float *d02, float *d11, int64_t ldo,
                         void *ws, size_t ws_bytes, void *stream);
size_t vmf_greedy_nms_workspace_bytes(int64_t n, int64_t h, int64_t w, double r2);
int vmf_greedy_nms(const int32_t *cy, const int32_t *cx, const double *cnd, int64_t n, int64_t h,
                   int64_t w, double r2, int32_t *order, int32_t *n_kept_dev, void *ws,
                   size_t ws_bytes, void *stream);

/* Launch accounting / in-situ kernel timing (used by bench.py).
 * vmf_launch_count: kernels launched by this library since load.
 * vmf_profile_begin: start bracketing every launch with CUDA events on its
 * stream (record nodes when the stream is being captured into a graph).
 * vmf_profile_stop: stop bracketing new launches.  vmf_profile_read: wait
 * for the recorded events and write, per kernel id, the summed duration (ms)
 * and launch count (the latest replay for graph-captured launches); returns
 * the number of ids.  vmf_profile_end = stop + read. */
long long vmf_launch_count(void);
int vmf_num_kernel_ids(void);
const char *vmf_kernel_name(int id);
void vmf_profile_begin(void);
void vmf_profile_stop(void);
int vmf_profile_read(double *ms, long long *counts, int n);
int vmf_profile_end(double *ms, long long *counts, int n);
/* The recorded launches in order: kernel id, start / end in ms after the
 * first recorded start (a concurrent replay's timeline); returns the count. */
int vmf_profile_timeline(int *ids, float *t0, float *t1, int n);

#ifdef __cplusplus
}
#endif
#endif /* VMFILT_B200_H */
