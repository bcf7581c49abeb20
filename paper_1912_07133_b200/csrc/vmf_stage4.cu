// vmf_stage4.cu -- Laplacian (stage 3) and threshold + NMS blob extraction
// (stage 4) with deterministic, order-preserving compaction.
//
// Laplacian: L = s * (D20 + D02), D20 = conv_rows(B, (1,-2,1)),
// D02 = conv_cols(B, (1,-2,1)) with replicate edges (engine.py:218-227,
// fir_vm_bank(3)[2] from design.py:250-280, trace at blob.py:161).
//
// Detection rule (conventions from blob.py:162-168): a
// pixel is kept iff it is strictly greater (smaller) than all 8
// edge-replicated neighbours and L >= t (-L >= t), t = frac * max|L|.
// Border pixels are their own replicated neighbours and never qualify.
// Scale-space variant: additionally strict against the 3x3 patches of the
// adjacent scales that exist.
//
// Compaction is three short launches (count per CTA, scan, ordered write) so
// the list comes out sorted by linear index (s, y, x) with no atomics on the
// data path: deterministic for any launch configuration.
#include "vmf_common.cuh"
#include "vmf_stage4.cuh"
#include "vmf_prof.cuh"

namespace vmf {

constexpr int kLapThreads = 256;
constexpr int kNmsThreads = 256;
constexpr int kNmsPerThread = 8;
constexpr int64_t kNmsPerBlock = (int64_t)kNmsThreads * kNmsPerThread;

__device__ __forceinline__ float block_max(float v, float *red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0f;
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  }
  return v;
}

__global__ void __launch_bounds__(kLapThreads) laplacian_kernel(
    const float *__restrict__ b, int64_t ldb, float *__restrict__ l, int64_t ldl, int64_t h,
    int64_t w, float scale, float *__restrict__ absmax) {
  __shared__ float red[kLapThreads / 32];
  float mx = 0.0f;
  for (int64_t i = blockIdx.x; i < h; i += gridDim.x) {  // one row per CTA step
    const int64_t iu = i > 0 ? i - 1 : 0, id = i < h - 1 ? i + 1 : h - 1;
    const float *bc = b + i * ldb, *bu = b + iu * ldb, *bd = b + id * ldb;
    for (int64_t j = threadIdx.x; j < w; j += blockDim.x) {
      const int64_t jl = j > 0 ? j - 1 : 0, jr = j < w - 1 ? j + 1 : w - 1;
      double c = (double)bc[j];
      double dx = (double)bc[jr] - 2.0 * c + (double)bc[jl];
      double dy = (double)bd[j] - 2.0 * c + (double)bu[j];
      float v = (float)((double)scale * (dx + dy));
      l[i * ldl + j] = v;
      mx = fmaxf(mx, fabsf(v));
    }
  }
  mx = block_max(mx, red);
  if (threadIdx.x == 0 && absmax) atomic_max_nonneg(absmax, mx);
}

// Is pixel (s, i, j) a detection?  v = its value (already loaded).
__device__ __forceinline__ bool is_det(const float *__restrict__ l, int64_t ld, int64_t plane,
                                       int64_t ns, int64_t h, int64_t w, int64_t s, int64_t i,
                                       int64_t j, float v, float thr) {
  if (i <= 0 || j <= 0 || i >= h - 1 || j >= w - 1) return false;
  if (!(fabsf(v) >= thr)) return false;
  const float *P = l + s * plane;
  bool gt = true, lt = true;
#pragma unroll
  for (int di = -1; di <= 1; ++di)
#pragma unroll
    for (int dj = -1; dj <= 1; ++dj) {
      if (di == 0 && dj == 0) continue;
      float u = P[(i + di) * ld + j + dj];
      gt &= v > u;
      lt &= v < u;
    }
  if (!gt && !lt) return false;
  for (int64_t t = s - 1; t <= s + 1; t += 2) {
    if (t < 0 || t >= ns) continue;
    const float *Q = l + t * plane;
#pragma unroll
    for (int di = -1; di <= 1; ++di)
#pragma unroll
      for (int dj = -1; dj <= 1; ++dj) {
        float u = Q[(i + di) * ld + j + dj];
        gt &= v > u;
        lt &= v < u;
      }
  }
  return (gt && v >= thr) || (lt && -v >= thr);
}

// Ranges of the compaction: kNmsPerBlock consecutive pixels of one row
// (rows in (s, i) order, segments left to right), so a range's pixels are
// contiguous in memory and the output order stays linear (s, i, j).  One
// division per range, none per pixel.
struct NmsRange {
  int64_t s, i, j0;
};
__device__ __forceinline__ NmsRange nms_range(int64_t rg, int64_t h, int64_t nseg) {
  const int64_t row = rg / nseg, seg = rg - row * nseg;
  NmsRange r;
  r.s = row / h;
  r.i = row - r.s * h;
  r.j0 = seg * kNmsPerBlock;
  return r;
}

// 8 consecutive values of a row from column j (vector loads when aligned)
__device__ __forceinline__ void ld_row8(const float *__restrict__ row, int64_t j, int64_t w,
                                        float *v) {
  if (j + 8 <= w && (((uintptr_t)(row + j)) & 15) == 0) {
    const float4 a = __ldg(reinterpret_cast<const float4 *>(row + j));
    const float4 b = __ldg(reinterpret_cast<const float4 *>(row + j + 4));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = j + e < w ? __ldg(row + j + e) : 0.0f;
  }
}

__global__ void __launch_bounds__(kNmsThreads) nms_count_kernel(
    const float *__restrict__ l, int64_t ld, int64_t plane, int64_t ns, int64_t h, int64_t w,
    float frac, const float *__restrict__ absmax, float *thr_out, int *__restrict__ counts,
    const int *gate) {
  if (gate && !*gate) return;
  float thr = frac * *absmax;
  if (blockIdx.x == 0 && threadIdx.x == 0 && thr_out) *thr_out = thr;
  const int64_t nseg = (w + kNmsPerBlock - 1) / kNmsPerBlock;
  const int64_t nranges = ns * h * nseg;
  __shared__ int sc;
  for (int64_t rg = blockIdx.x; rg < nranges; rg += gridDim.x) {  // grid-stride over ranges
    const NmsRange r = nms_range(rg, h, nseg);
    const int64_t j = r.j0 + (int64_t)threadIdx.x * kNmsPerThread;
    int c = 0;
    if (j < w) {
      float v[kNmsPerThread];
      ld_row8(l + r.s * plane + r.i * ld, j, w, v);
#pragma unroll
      for (int e = 0; e < kNmsPerThread; ++e)
        if (j + e < w && is_det(l, ld, plane, ns, h, w, r.s, r.i, j + e, v[e], thr)) ++c;
    }
    if (threadIdx.x == 0) sc = 0;
    __syncthreads();
    if (c) atomicAdd(&sc, c);
    __syncthreads();
    if (threadIdx.x == 0) counts[rg] = sc;
    __syncthreads();
  }
}

// Single CTA: exclusive scan of per-CTA counts, total -> *n_det.
__global__ void __launch_bounds__(1024) nms_scan_kernel(int *__restrict__ counts, int64_t nb,
                                                        int64_t *__restrict__ n_det,
                                                        const int *gate) {
  if (gate && !*gate) return;
  __shared__ int64_t part[1024];
  int64_t per = (nb + blockDim.x - 1) / blockDim.x;
  int64_t lo = threadIdx.x * per, hi = lo + per < nb ? lo + per : nb;
  int64_t s = 0;
  for (int64_t i = lo; i < hi; ++i) s += counts[i];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      int64_t t = part[i];
      part[i] = run;
      run += t;
    }
    *n_det = run;
    counts[nb] = (int)run;  // sentinel: range rg is empty iff counts[rg + 1] == counts[rg]
  }
  __syncthreads();
  int64_t run = part[threadIdx.x];
  for (int64_t i = lo; i < hi; ++i) {
    int64_t t = counts[i];
    counts[i] = (int)run;  // offsets fit: detections <= pixels per launch < 2^31
    run += t;
  }
}

__global__ void __launch_bounds__(kNmsThreads) nms_write_kernel(
    const float *__restrict__ l, int64_t ld, int64_t plane, int64_t ns, int64_t h, int64_t w,
    float frac, const float *__restrict__ absmax, const int *__restrict__ offsets,
    int32_t *__restrict__ det_idx, int idx_stride, float *__restrict__ det_val, int64_t cap,
    const int *gate) {
  if (gate && !*gate) return;
  float thr = frac * *absmax;
  const int64_t nseg = (w + kNmsPerBlock - 1) / kNmsPerBlock;
  const int64_t nranges = ns * h * nseg;
  __shared__ int wsum[kNmsThreads / 32];
  for (int64_t rg = blockIdx.x; rg < nranges; rg += gridDim.x) {  // grid-stride over ranges
    if (offsets[rg + 1] == offsets[rg]) continue;  // no detection in this range (uniform)
    const NmsRange r = nms_range(rg, h, nseg);
    const int64_t j = r.j0 + (int64_t)threadIdx.x * kNmsPerThread;
    unsigned flags = 0;
    float vals[kNmsPerThread];
    if (j < w) {
      ld_row8(l + r.s * plane + r.i * ld, j, w, vals);
#pragma unroll
      for (int e = 0; e < kNmsPerThread; ++e)
        if (j + e < w && is_det(l, ld, plane, ns, h, w, r.s, r.i, j + e, vals[e], thr))
          flags |= 1u << e;
    }
    int c = __popc(flags);
    // block exclusive scan of c (thread order == pixel order)
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    __syncthreads();
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      int v = lane < kNmsThreads / 32 ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
      }
      if (lane < kNmsThreads / 32) wsum[lane] = v;
    }
    __syncthreads();
    int64_t pos = (int64_t)offsets[rg] + (wid ? wsum[wid - 1] : 0) + inc - c;
#pragma unroll
    for (int e = 0; e < kNmsPerThread; ++e) {
      if (!(flags >> e & 1u)) continue;
      if (pos < cap) {
        int32_t *o = det_idx + pos * idx_stride;
        if (idx_stride == 3) {
          o[0] = (int32_t)r.s;
          o[1] = (int32_t)r.i;
          o[2] = (int32_t)(j + e);
        } else {
          o[0] = (int32_t)r.i;
          o[1] = (int32_t)(j + e);
        }
        det_val[pos] = vals[e];
      }
      ++pos;
    }
  }
}

__global__ void absmax_kernel(const float *__restrict__ l, int64_t ld, int64_t plane,
                              int64_t ns, int64_t h, int64_t w, float *__restrict__ absmax) {
  __shared__ float red[32];
  float mx = 0.0f;
  const int64_t rows = ns * h;
  const bool vec = (w % 4 == 0) && (ld % 4 == 0) && (plane % 4 == 0) &&
                   (((uintptr_t)l & 15) == 0);
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const int64_t s = row / h, i = row - s * h;
    const float *R = l + s * plane + i * ld;
    if (vec) {
      for (int64_t j = 4 * threadIdx.x; j < w; j += 4 * blockDim.x) {
        const float4 v = __ldg(reinterpret_cast<const float4 *>(R + j));
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
      }
    } else {
      for (int64_t j = threadIdx.x; j < w; j += blockDim.x) mx = fmaxf(mx, fabsf(R[j]));
    }
  }
  mx = block_max(mx, red);
  if (threadIdx.x == 0) atomic_max_nonneg(absmax, mx);
}

// ---------------------------------------------------------------------------
// the scale-space rule from per-scale candidates: each scale's fused column
// pass wrote its plane of the stack and listed its strict 3x3 extrema above
// frac * its own max (sorted by (y, x)); the stack threshold is the largest
// of those thresholds, and a 3x3x3 detection is one of those candidates that
// also clears the adjacent planes' 9 + 9 neighbours and the stack threshold
// -- so only the candidates are tested, in (s, y, x) order, by one CTA
// (block-wide ordered compaction); no pass over the whole stack.
// ---------------------------------------------------------------------------
constexpr int kCandThreads = 1024;
__global__ void __launch_bounds__(kCandThreads) detect3x3x3_cands_kernel(
    const float *__restrict__ l, int64_t ld, int64_t plane, int ns, int64_t h, int64_t w,
    const int32_t *__restrict__ cyx, const float *__restrict__ cval, int64_t cstride,
    const int64_t *__restrict__ cscal, int32_t *__restrict__ det, float *__restrict__ dval,
    int64_t cap, int64_t *__restrict__ n_det, float *__restrict__ thr_out) {
  __shared__ int wsum[kCandThreads / 32];
  __shared__ float sthr;
  __shared__ int overflow;
  pdl_wait();  // the column passes' candidate lists and the stack
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    float t = 0.0f;
    int ov = 0;
    for (int s = 0; s < ns; ++s) {
      t = fmaxf(t, __int_as_float((int)(cscal[2 * s + 1] & 0xffffffffll)));
      ov |= cscal[2 * s] > cstride;
    }
    sthr = t;
    overflow = ov;
    if (thr_out) *thr_out = t;
  }
  __syncthreads();
  if (overflow) {  // a list was cut short: the caller runs the full-stack rule
    if (tid == 0) *n_det = -1;
    return;
  }
  const float thr = sthr;
  int64_t base = 0;
  for (int s = 0; s < ns; ++s) {
    const int64_t n = cscal[2 * s];
    for (int64_t q0 = 0; q0 < n; q0 += kCandThreads) {
      const int64_t q = q0 + tid;
      int keep = 0;
      int32_t y = 0, x = 0;
      float v = 0.0f;
      if (q < n) {
        y = cyx[(s * cstride + q) * 2];
        x = cyx[(s * cstride + q) * 2 + 1];
        v = cval[s * cstride + q];
        if (fabsf(v) >= thr) {
          bool gt = v > 0.0f, lt = v < 0.0f;  // (the in-plane test already passed)
          for (int t = s - 1; t <= s + 1; t += 2) {
            if (t < 0 || t >= ns) continue;
            const float *Q = l + (int64_t)t * plane;
#pragma unroll
            for (int di = -1; di <= 1; ++di)
#pragma unroll
              for (int dj = -1; dj <= 1; ++dj) {
                const float u = Q[(int64_t)(y + di) * ld + x + dj];
                gt &= v > u;
                lt &= v < u;
              }
          }
          keep = (gt && v >= thr) || (lt && -v >= thr);
        }
      }
      // ordered block compaction
      int inc = keep;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
      }
      if (lane == 31) wsum[wid] = inc;
      __syncthreads();
      if (wid == 0) {
        int v2 = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, v2, o);
          if (lane >= o) v2 += t;
        }
        wsum[lane] = v2;
      }
      __syncthreads();
      const int64_t pos = base + (wid ? wsum[wid - 1] : 0) + inc - keep;
      if (keep && pos < cap) {
        det[3 * pos] = s;
        det[3 * pos + 1] = y;
        det[3 * pos + 2] = x;
        dval[pos] = v;
      }
      base += wsum[kCandThreads / 32 - 1];
      __syncthreads();
    }
  }
  if (tid == 0) *n_det = base;
}

int detect3x3x3_cands(const float *l, int64_t ld, int64_t plane, int ns, int64_t h, int64_t w,
                      const int32_t *cyx, const float *cval, int64_t cstride,
                      const int64_t *cscal, int32_t *det, float *dval, int64_t cap,
                      int64_t *n_det, float *thr_out, cudaStream_t st) {
  Launch g(K_NMS_WRITE, st);
  launch_pdl(detect3x3x3_cands_kernel, dim3(1), dim3(kCandThreads), 0, st, l, ld, plane, ns, h, w,
             cyx, cval, cstride, cscal, det, dval, cap, n_det, thr_out);
  return cuda_status("scale-space detect (candidates)");
}

// ---------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------
static int sm_count() {
  static int by_dev[64];
  const int dev = current_device();
  int tmp = 0;
  int &n = dev >= 0 && dev < 64 ? by_dev[dev] : tmp;
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int laplacian(const float *b, int64_t ldb, float *l, int64_t ldl, int64_t h, int64_t w,
              float scale, float *absmax, cudaStream_t st) {
  int64_t cap = (int64_t)sm_count() * 8;
  {
    Launch g(K_LAPLACIAN, st);
    laplacian_kernel<<<(int)(h < cap ? h : cap), kLapThreads, 0, st>>>(b, ldb, l, ldl, h, w,
                                                                        scale, absmax);
  }
  return cuda_status("laplacian");
}

static int64_t nms_ranges(int64_t ns, int64_t h, int64_t w) {
  return ns * h * cdiv(w, kNmsPerBlock);
}

size_t detect_workspace_bytes(int64_t ns, int64_t h, int64_t w) {
  int64_t nb = nms_ranges(ns, h, w);
  return 256 + 256 + (size_t)(nb + 1) * sizeof(int) + 256;
}

// ws layout: [0,256) absmax float; [256,512) scratch; [512, ...) counts
static int detect_core(const float *l, int64_t ld, int64_t plane, int64_t ns, int64_t h,
                       int64_t w, float frac, float *absmax, const int *gate, int32_t *det_idx,
                       int idx_stride, float *det_val, int64_t cap, int64_t *n_det_dev,
                       float *thr_dev, int *counts, cudaStream_t st) {
  int64_t nb = nms_ranges(ns, h, w);
  if (nb > 0x7fffffff) return fail(VMF_EVALUE, "frame stack too large");
  // grid-stride launch: a gated (fallback) launch costs a few hundred idle CTAs
  const unsigned grid = (unsigned)(nb < (int64_t)sm_count() * 8 ? nb : (int64_t)sm_count() * 8);
  {
    Launch g(K_NMS_COUNT, st);
    nms_count_kernel<<<grid, kNmsThreads, 0, st>>>(l, ld, plane, ns, h, w, frac, absmax,
                                                           thr_dev, counts, gate);
  }
  {
    Launch g(K_NMS_SCAN, st);
    nms_scan_kernel<<<1, 1024, 0, st>>>(counts, nb, n_det_dev, gate);
  }
  {
    Launch g(K_NMS_WRITE, st);
    nms_write_kernel<<<grid, kNmsThreads, 0, st>>>(l, ld, plane, ns, h, w, frac, absmax,
                                                           counts, det_idx, idx_stride, det_val,
                                                           cap, gate);
  }
  return cuda_status("detect");
}

int detect(const float *l, int64_t ld, int64_t plane, int64_t ns, int64_t h, int64_t w,
           float frac, bool have_absmax, int32_t *det_idx, int idx_stride, float *det_val,
           int64_t cap, int64_t *n_det_dev, float *thr_dev, int64_t *n_det_host, void *ws,
           size_t ws_bytes, cudaStream_t st) {
  size_t need = detect_workspace_bytes(ns, h, w);
  if (!ws || ws_bytes < need)
    return fail(VMF_EVALUE, "detect workspace too small: %zu < %zu bytes", ws_bytes, need);
  if (!n_det_dev) return fail(VMF_EVALUE, "n_det_dev must not be NULL");
  if (cap > 0 && (!det_idx || !det_val)) return fail(VMF_EVALUE, "detection buffers are NULL");
  char *base = (char *)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  float *absmax = (float *)base;
  int *counts = (int *)(base + 512);
  if (!have_absmax) {
    cudaMemsetAsync(absmax, 0, sizeof(float), st);
    Launch g(K_ABSMAX, st);
    absmax_kernel<<<sm_count() * 4, 256, 0, st>>>(l, ld, plane, ns, h, w, absmax);
  }
  int rc = detect_core(l, ld, plane, ns, h, w, frac, absmax, nullptr, det_idx, idx_stride,
                       det_val, cap, n_det_dev, thr_dev, counts, st);
  if (rc) return rc;
  if (n_det_host) {
    cudaMemcpyAsync(n_det_host, n_det_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    return cuda_status("detect readback");
  }
  return VMF_OK;
}

int detect_if(const float *l, int64_t ld, int64_t h, int64_t w, float frac, float *absmax,
              const int *gate, int32_t *det_yx, float *det_val, int64_t cap, int64_t *n_det_dev,
              float *thr_dev, void *ws, size_t ws_bytes, cudaStream_t st) {
  size_t need = detect_workspace_bytes(1, h, w);
  if (!ws || ws_bytes < need) return fail(VMF_EVALUE, "detect workspace too small");
  char *base = (char *)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  return detect_core(l, ld, h * ld, 1, h, w, frac, absmax, gate, det_yx, 2, det_val, cap,
                     n_det_dev, thr_dev, (int *)(base + 512), st);
}

float *detect_absmax_slot(void *ws) {
  return (float *)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
}

}  // namespace vmf
