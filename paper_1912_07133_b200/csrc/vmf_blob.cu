// vmf_blob.cu -- deterministic greedy non-maximum suppression of the Hessian
// blob detector (blob.py:168-176):
//
//   order = lexsort((x, y, -score));  keep a candidate iff no kept candidate
//   lies within r (squared distance <= r^2), visiting in that order.
//
// The sequential greedy is computed in parallel rounds on a uniform grid of
// cells of side ceil(r): an undecided candidate with a kept neighbour is
// removed; one with no undecided neighbour of higher priority is kept.  A
// candidate is only decided after every higher-priority neighbour is, so the
// kept set is exactly the greedy one (and independent of thread order); the
// highest-priority undecided candidate is always decidable, so the rounds
// terminate.  The kept candidates are then ranked by priority (strongest
// first, ties by y then x like the lexsort).
#include <cmath>

#include "vmf_common.cuh"
#include "vmf_prof.cuh"

namespace vmf {

namespace {

constexpr unsigned char kUnd = 0, kKept = 1, kGone = 2;

__device__ __forceinline__ bool higher(const int *cy, const int *cx, const double *nd, int j,
                                       int i) {
  if (nd[j] != nd[i]) return nd[j] > nd[i];
  if (cy[j] != cy[i]) return cy[j] < cy[i];
  return cx[j] < cx[i];
}

struct Grid {
  int cs, gw, gh;
  __device__ int cell(int y, int x) const { return (y / cs) * gw + x / cs; }
};

__global__ void nms_cell_count(const int *cy, const int *cx, int n, Grid g, int *cnt) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    atomicAdd(&cnt[g.cell(cy[i], cx[i])], 1);
}

// one CTA: exclusive scan of the cell counts (start), fill counters zeroed
__global__ void __launch_bounds__(1024) nms_cell_scan(const int *cnt, int *start, int *fill,
                                                      int ncell) {
  __shared__ int wsum[32];
  __shared__ int carry;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < ncell; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int v = i < ncell ? cnt[i] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int s = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      wsum[lane] = s;
    }
    __syncthreads();
    const int excl = carry + (wid ? wsum[wid - 1] : 0) + x - v;
    if (i < ncell) {
      start[i] = excl;
      fill[i] = 0;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
}

__global__ void nms_cell_scatter(const int *cy, const int *cx, int n, Grid g, const int *start,
                                 int *fill, int *perm) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int c = g.cell(cy[i], cx[i]);
    perm[start[c] + atomicAdd(&fill[c], 1)] = i;
  }
}

// one CTA: greedy rounds; then the kept indices are compacted into `kept`
__global__ void __launch_bounds__(1024) nms_rounds(const int *cy, const int *cx, const double *nd,
                                                   int n, Grid g, long long r2, const int *start,
                                                   const int *cnt, const int *perm,
                                                   unsigned char *state, int *kept, int *nkept) {
  __shared__ int und, nk;
  for (int i = threadIdx.x; i < n; i += blockDim.x) state[i] = kUnd;
  if (threadIdx.x == 0) nk = 0;
  __syncthreads();
  while (true) {
    if (threadIdx.x == 0) und = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      if (state[i] != kUnd) continue;
      const int yi = cy[i], xi = cx[i];
      const int gy0 = yi / g.cs, gx0 = xi / g.cs;
      bool kept_near = false, wait = false;
      for (int gy = gy0 - 1; gy <= gy0 + 1 && !kept_near; ++gy) {
        if (gy < 0 || gy >= g.gh) continue;
        for (int gx = gx0 - 1; gx <= gx0 + 1 && !kept_near; ++gx) {
          if (gx < 0 || gx >= g.gw) continue;
          const int c = gy * g.gw + gx;
          for (int p = start[c], e = start[c] + cnt[c]; p < e; ++p) {
            const int jj = perm[p];
            if (jj == i) continue;
            const long long dy = cy[jj] - yi, dx = cx[jj] - xi;
            if (dy * dy + dx * dx > r2) continue;
            const unsigned char sj = state[jj];
            if (sj == kKept) {
              kept_near = true;
              break;
            }
            if (sj == kUnd && higher(cy, cx, nd, jj, i)) wait = true;
          }
        }
      }
      if (kept_near) {
        state[i] = kGone;
      } else if (!wait) {
        state[i] = kKept;
        kept[atomicAdd(&nk, 1)] = i;
      } else {
        atomicAdd(&und, 1);
      }
    }
    __syncthreads();
    const int u = und;
    __syncthreads();
    if (u == 0) break;
  }
  if (threadIdx.x == 0) *nkept = nk;
}

// rank of each kept candidate among the kept ones -> order[rank] = index
__global__ void nms_rank(const int *cy, const int *cx, const double *nd, const int *kept,
                         const int *nkept, int *order) {
  const int k = *nkept;
  for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < k; a += gridDim.x * blockDim.x) {
    const int i = kept[a];
    int rank = 0;
    for (int b = 0; b < k; ++b) rank += higher(cy, cx, nd, kept[b], i);
    order[rank] = i;
  }
}

Grid make_grid(int64_t h, int64_t w, double r2) {
  Grid g;
  g.cs = (int)std::ceil(std::sqrt(r2 > 0 ? r2 : 0.0));
  if (g.cs < 1) g.cs = 1;
  g.gw = (int)((w + g.cs - 1) / g.cs);
  g.gh = (int)((h + g.cs - 1) / g.cs);
  return g;
}

}  // namespace

size_t greedy_nms_workspace_bytes(int64_t n, int64_t h, int64_t w, double r2) {
  const Grid g = make_grid(h, w, r2);
  const size_t ncell = (size_t)g.gw * g.gh;
  return 256 + 3 * ncell * sizeof(int) + 2 * (size_t)n * sizeof(int) + (size_t)n + 1024;
}

int greedy_nms(const int *cy, const int *cx, const double *nd, int64_t n, int64_t h, int64_t w,
               double r2, int *order, int *nkept, void *ws, size_t ws_bytes, cudaStream_t st) {
  if (n < 0 || n > 0x7fffffff) return fail(VMF_EVALUE, "candidate count out of range");
  if (ws_bytes < greedy_nms_workspace_bytes(n, h, w, r2))
    return fail(VMF_EVALUE, "greedy NMS workspace too small");
  const Grid g = make_grid(h, w, r2);
  const int ncell = g.gw * g.gh;
  char *p = (char *)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  int *cnt = (int *)p;
  int *start = cnt + ncell;
  int *fill = start + ncell;
  int *perm = fill + ncell;
  int *kept = perm + n;
  unsigned char *state = (unsigned char *)(kept + n);
  cudaMemsetAsync(cnt, 0, (size_t)ncell * sizeof(int), st);
  cudaMemsetAsync(nkept, 0, sizeof(int), st);
  if (n == 0) return cuda_status("greedy nms");
  const int nb = (int)((n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184);
  const long long r2i = (long long)std::floor(r2);  // integer offsets: d^2 <= r^2 <=> d^2 <= floor(r^2)
  Launch lg(K_NMS_WRITE, st);
  nms_cell_count<<<nb, 256, 0, st>>>(cy, cx, (int)n, g, cnt);
  nms_cell_scan<<<1, 1024, 0, st>>>(cnt, start, fill, ncell);
  nms_cell_scatter<<<nb, 256, 0, st>>>(cy, cx, (int)n, g, start, fill, perm);
  nms_rounds<<<1, 1024, 0, st>>>(cy, cx, nd, (int)n, g, r2i, start, cnt, perm, state, kept, nkept);
  nms_rank<<<nb, 256, 0, st>>>(cy, cx, nd, kept, nkept, order);
  return cuda_status("greedy nms");
}

}  // namespace vmf
