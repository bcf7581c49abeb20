// vmf_rowlap.cuh -- the fp32 "Laplacian-first" row pass (vmf_rowlap.cu).
#pragma once
#include <vector>
#include "vmf_common.cuh"
#include "vmf_modal32.cuh"

namespace vmf {

constexpr int kHmRowMax = 2048;  // border weights h(1..Mh) along a row

struct RowLapParams {
  float p, q;           // modal pole (JORDAN: p; CPAIR: p + i q)
  float c[4], cs[4];    // y+ = c . u(n-1); cs = sign * c (the anticausal part)
  float b0, sign;
  float SP[4][16], SQ[4][16];  // folded 32-sample chunk-carry weights
  float Wt[32][4];      // A^t b, t < 32 (border-term chunk sums)
  float A32[16];        // A^32
  float Apow[5][16];    // A^(32 cpl 2^l): the chunk scan's Kogge-Stone steps
  float Iss[4];         // (I - A)^-1 b
  int64_t H, W;
  int C, cpl, rows_per, Mh, K;
};

constexpr int kMaxSeg = 32;  // border segments of 64 rows (Mh <= 2048)
struct SegVec {             // c A^(m0-1) per border segment (column stage)
  float v[kMaxSeg][4];
  int nseg, Mh;
};

struct HmRow {
  float h[kHmRowMax + 1];
};

struct VlrTab {  // [C][8]: the border-term chunk vectors vl(c) (4), vr(c) (4)
  float v[256 * 8];
};

struct RowLapPlan {
  RowLapParams p;
  HmRow hm;
  VlrTab vlr;
  int kind;
};

constexpr int kRChunk = 32;

// One row through R, in two phases around a block barrier:
//   row_carry32: this thread's chunk U -> its zero-state carries in cf / cb;
//   row_scan_walk32: (after the barrier) chunk scans, then the walks -> V.
// e2: steady-state inputs left / right of the row; cf / cb: [blockDim][K]
// scratch; dx2: the row's border terms (added to V(0) / subtracted from
// V(W-1)), read only after the scan's barrier.
template <int K>
__device__ __forceinline__ void row_carry32(const RowLapParams &p, const float (&U)[kRChunk],
                                            float *cf, float *cb) {
  const int c = threadIdx.x;
  // zero-state chunk carries: forward end state P + Q, backward start P - Q
  {
    float P[K], Q[K];
#pragma unroll
    for (int i = 0; i < K; ++i) P[i] = Q[i] = 0.0f;
#pragma unroll
    for (int t = 0; t < kRChunk / 2; ++t) {
      const float s = U[t] + U[kRChunk - 1 - t], d = U[t] - U[kRChunk - 1 - t];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        P[i] = fmaf(p.SP[i][t], s, P[i]);
        Q[i] = fmaf(p.SQ[i][t], d, Q[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < K; ++i) {
      cf[c * K + i] = P[i] + Q[i];
      cb[c * K + i] = P[i] - Q[i];
    }
  }
}

template <int K, int KIND>
__device__ __forceinline__ void row_scan_walk32(const RowLapParams &p, const float (&U)[kRChunk],
                                                float (&V)[kRChunk], float *cf, float *cb,
                                                const float *e2, const float *dx2) {
  const int c = threadIdx.x, C = p.C, lane = c & 31, warp = c >> 5;
  // chunk scans: task 0 forward (chunks 0..C-1), task 1 backward
  for (int task = warp; task < 2; task += (int)(blockDim.x >> 5)) {
    float *cc = task == 0 ? cf : cb;
    const int cpl = p.cpl;
    const float e = e2[task];
    float A[K];
#pragma unroll
    for (int i = 0; i < K; ++i) A[i] = 0.0f;
    for (int q = 0; q < cpl; ++q) {
      const int sp = lane * cpl + q;
      if (sp >= C) break;
      const int ch = task == 0 ? sp : C - 1 - sp;
      float d[K];
#pragma unroll
      for (int i = 0; i < K; ++i) d[i] = cc[ch * K + i];
      if (sp == 0) {  // + A^32 u_ss(e): the steady start enters with the first chunk
#pragma unroll
        for (int i = 0; i < K; ++i)
#pragma unroll
          for (int m = 0; m < K; ++m) d[i] = fmaf(p.A32[i * K + m], p.Iss[m] * e, d[i]);
      }
      float An[K];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        float a = d[i];
#pragma unroll
        for (int m = 0; m < K; ++m) a = fmaf(p.A32[i * K + m], A[m], a);
        An[i] = a;
      }
#pragma unroll
      for (int i = 0; i < K; ++i) A[i] = An[i];
    }
#pragma unroll
    for (int lv = 0; lv < 5; ++lv) {
      const int o = 1 << lv;
      float Bv[K];
#pragma unroll
      for (int i = 0; i < K; ++i) Bv[i] = __shfl_up_sync(0xffffffffu, A[i], o);
      if (lane >= o) {
#pragma unroll
        for (int i = 0; i < K; ++i) {
          float a = A[i];
#pragma unroll
          for (int m = 0; m < K; ++m) a = fmaf(p.Apow[lv][i * K + m], Bv[m], a);
          A[i] = a;
        }
      }
    }
    float E[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const float v = __shfl_up_sync(0xffffffffu, A[i], 1);
      E[i] = lane ? v : p.Iss[i] * e;
    }
    // each chunk's start state over its carry
    for (int q = 0; q < cpl; ++q) {
      const int sp = lane * cpl + q;
      if (sp >= C) break;
      const int ch = task == 0 ? sp : C - 1 - sp;
      float d[K];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        d[i] = cc[ch * K + i];
        cc[ch * K + i] = E[i];
      }
      // (chunk 0: E is the steady start itself, so A^32 E brings it in once)
      float En[K];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        float a = d[i];
#pragma unroll
        for (int m = 0; m < K; ++m) a = fmaf(p.A32[i * K + m], E[m], a);
        En[i] = a;
      }
#pragma unroll
      for (int i = 0; i < K; ++i) E[i] = En[i];
    }
  }
  __syncthreads();
  // walks: backward parked (b0 U + s y-), forward adds y+
  float park[kRChunk];
  {
    Rec32<K, KIND> rb;
#pragma unroll
    for (int i = 0; i < K; ++i) rb.u[i] = cb[c * K + i];
#pragma unroll
    for (int t = kRChunk - 1; t >= 0; --t) {
      park[t] = rb.out_from(p.cs, p.b0 * U[t]);
      rb.step(p, U[t]);
    }
  }
  {
    Rec32<K, KIND> rf;
#pragma unroll
    for (int i = 0; i < K; ++i) rf.u[i] = cf[c * K + i];
#pragma unroll
    for (int t = 0; t < kRChunk; ++t) {
      V[t] = rf.out_from(p.c, park[t]);
      rf.step(p, U[t]);
    }
  }
  if (c == 0) V[0] += dx2[0];
  if (c == C - 1) V[kRChunk - 1] -= dx2[1];
}

int rowlap_get_plan(int64_t h, int64_t w, const double *b, const double *a, int k, double b0,
                    int sign, RowLapPlan *out);

// both phases (contains two block barriers)
template <int K, int KIND>
__device__ __forceinline__ void row_filter(const RowLapParams &p, const float (&U)[kRChunk],
                                           float (&V)[kRChunk], float *cf, float *cb,
                                           const float *e2, const float *dx2) {
  row_carry32<K>(p, U, cf, cb);
  __syncthreads();
  row_scan_walk32<K, KIND>(p, U, V, cf, cb, e2, dx2);
}

bool rowlap_supported(int64_t h, int64_t w, const double *b, const double *a, int k, double b0,
                      int sign);
// X (fp32, pitch ldx; 16-byte aligned rows) -> V = R(Lap5 X) (pitch ldv) with
// the left / right border terms folded in; vrows = [Vt | Vb | Ky(2) | S(2 x 32)]
// x w floats: the virtual rows above / below the image, the column
// direction's border rows Ky = R_ss(Dy) (column stage (cb_, ca, cb0, csign),
// same order k) and the border kernel's segment shares S.
int rowlap_run(const float *x, int64_t ldx, float *V, int64_t ldv, float *vrows, int64_t h,
               int64_t w, const double *b, const double *a, int k, double b0, int sign,
               const double *cb_, const double *ca, double cb0, int csign, cudaStream_t st);
constexpr int kRowLapVrows = 4 + 2 * kMaxSeg;  // floats per column of vrows

}  // namespace vmf
