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
  alignas(16) float SPQ[4][16][2];  // folded 32-sample chunk-carry weights (SP, SQ) pairs:
                       // fwd = sum SP s + SQ d, bwd = sum SP s - SQ d over the
                       // pairs s = U(t) + U(31-t), d = U(t) - U(31-t)
  float A32[16];        // A^32
  float Apow[5][16];    // A^(32 cpl 2^l): the chunk scan's Kogge-Stone steps
  float Iss[4];         // (I - A)^-1 b
  int64_t H, W;
  int C, cpl, rows_per, Mh, K;
  int nseg;             // (sweep) the column stage's border segments of this scale
};

constexpr int kMaxSeg = 32;  // border segments of 64 rows (Mh <= 2048)
struct SegVec {             // c A^(m0-1) per border segment (column stage)
  float v[kMaxSeg][4];
  int nseg, Mh;
};

struct RowLapPlan {  // (POD: cached by value)
  RowLapParams p;
  float ci[4];        // c A^-1 (the right border's last-chunk vector)
  int kind;
};

// ---------------------------------------------------------------------------
// multi-scale sweep (vmf_rowlap.cu): one pass over X feeds every scale's row
// filter (U = Lap5 X, the X staging and the barriers are shared), then one
// column pass per scale
// ---------------------------------------------------------------------------
constexpr int kMaxScales = 5;  // (one row-pass instantiation per count)

struct RowLapMulti {
  RowLapParams s[kMaxScales];  // per scale: the row stage
  int ns;
  int64_t H, W;
  int C, rows_per;
  int carry_fold;              // chunk carries as folded packed-FMA sums (else recursions)
  int store_inline;            // V stored in 8-sample groups during the walk (2: the two
                               // directions paired on packed FMAs, 1: walked in turn)
};

struct BorderScale {   // per scale, for the border kernel
  float p, q, c[4], sign;   // the column stage (column-direction recursion)
  SegVec sv;                // its segment vectors
  float A32[16], cr[4], ci[4];  // the row stage: A^32, c, c A^-1 (chunk vectors)
  int C, Mh;                // chunks; the row stage's border length
};
struct BorderMulti {
  BorderScale s[kMaxScales];
  int ns;
  int maxseg, maxMh;  // the longest scale's segments / border length
};

// Per-scale extras, floats, w = frame width: Vt [w] | Vb [w] | Ky [2w] |
// S [2 x kMaxSeg x w] | vlr [C x 8]
constexpr int64_t kExVt = 0, kExVb = 1, kExKy = 2, kExS = 4, kExVlr = 4 + 2 * kMaxSeg;
inline int64_t sweep_extras_floats(int64_t w) { return (kExVlr + 1) * w; }

struct SweepOut {          // scale s: V_s = V0 + s vstride, extras_s = E0 + s estride
  float *V0, *E0;
  int64_t vstride, estride;  // floats
  int64_t ldv;
  __host__ __device__ float *V(int s) const { return V0 + s * vstride; }
  __host__ __device__ float *E(int s) const { return E0 + s * estride; }
};

constexpr int kRChunk = 32;

// The coefficients a chunk's recursions use, in registers (loaded once per
// scale and row from the kernel parameters): pole, output vectors, b0.
template <int K>
struct RC32 {
  float p, q, c[K], cs[K], b0;
  __device__ __forceinline__ explicit RC32(const RowLapParams &P) {
    p = P.p;
    q = P.q;
    b0 = P.b0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      c[i] = P.c[i];
      cs[i] = P.cs[i];
    }
  }
};

// One row through R, in two phases around a block barrier:
//   row_carry32: this thread's chunk U -> its zero-state carries in cf / cb
//     (the forward end state and the backward start state of the chunk, by
//     running the recursion from zero over the chunk: only the pole is
//     needed, so nothing but registers is read);
//   row_scan_walk32: (after the barrier) chunk scans, then the walks -> V.
// e2: steady-state inputs left / right of the row; cf / cb: [blockDim][K]
// scratch; dx2: the row's border terms (added to V(0) / subtracted from
// V(W-1)), read only after the scan's barrier.
template <int K, int KIND>
__device__ __forceinline__ void row_carry32(const RC32<K> &rc, const float (&U)[kRChunk],
                                            float *cf, float *cb) {
  const int c = threadIdx.x;
  Rec32<K, KIND> f, b;
#pragma unroll
  for (int i = 0; i < K; ++i) f.u[i] = b.u[i] = 0.0f;
#pragma unroll
  for (int t = 0; t < kRChunk; ++t) {
    f.step(rc, U[t]);
    b.step(rc, U[kRChunk - 1 - t]);
  }
#pragma unroll
  for (int i = 0; i < K; ++i) {
    cf[c * K + i] = f.u[i];
    cb[c * K + i] = b.u[i];
  }
}

// The zero-state chunk carries of one scale from the row's folded sample
// pairs sd[t] = (U(t) + U(31-t), U(t) - U(31-t)) (formed once per row for
// every scale): (P_i, Q_i) = sum_t (SP_it, SQ_it) * sd[t] as packed FMAs
// with the (SP, SQ) pairs read two at a time from shared memory;
// forward carry P + Q, backward P - Q (the recursion's end states, as
// independent sums instead of a chain).
template <int K>
__device__ __forceinline__ void row_carry32_fold(const RowLapParams &p, const float2 (&sd)[16],
                                                 float *cf, float *cb) {
  const int c = threadIdx.x;
  float2 pq[K];
#pragma unroll
  for (int i = 0; i < K; ++i) pq[i] = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int t = 0; t < 16; t += 2) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const float4 w = *reinterpret_cast<const float4 *>(&p.SPQ[i][t][0]);
      pq[i] = ffma2(make_float2(w.x, w.y), sd[t], pq[i]);
      pq[i] = ffma2(make_float2(w.z, w.w), sd[t + 1], pq[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < K; ++i) {
    cf[c * K + i] = pq[i].x + pq[i].y;
    cb[c * K + i] = pq[i].x - pq[i].y;
  }
}

// One chunk scan (one warp): direction dir (0: chunks 0..C-1, 1: backward)
// over the zero-state carries in cc, steady start e; leaves every chunk's
// start state in cc.
template <int K>
__device__ __forceinline__ void chunk_scan32(const RowLapParams &p, float *cc, int dir, float e,
                                             int lane) {

    const int cpl = p.cpl, C = p.C;
    float A[K];
#pragma unroll
    for (int i = 0; i < K; ++i) A[i] = 0.0f;
    for (int q = 0; q < cpl; ++q) {
      const int sp = lane * cpl + q;
      if (sp >= C) break;
      const int ch = dir == 0 ? sp : C - 1 - sp;
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
      const int ch = dir == 0 ? sp : C - 1 - sp;
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

// The walks of one row (after the scans): backward parked (b0 U + s y-),
// forward adds y+; the row's border terms on the end samples.
template <int K, int KIND>
__device__ __forceinline__ void row_walks32(const RC32<K> &rc, int C, const float (&U)[kRChunk],
                                            float (&V)[kRChunk], const float *cf, const float *cb,
                                            const float *dx2) {
  const int c = threadIdx.x;
  float park[kRChunk];
  {
    Rec32<K, KIND> rb;
#pragma unroll
    for (int i = 0; i < K; ++i) rb.u[i] = cb[c * K + i];
#pragma unroll
    for (int t = kRChunk - 1; t >= 0; --t) {
      park[t] = rb.out_from(rc.cs, rc.b0 * U[t]);
      rb.step(rc, U[t]);
    }
  }
  {
    Rec32<K, KIND> rf;
#pragma unroll
    for (int i = 0; i < K; ++i) rf.u[i] = cf[c * K + i];
#pragma unroll
    for (int t = 0; t < kRChunk; ++t) {
      V[t] = rf.out_from(rc.c, park[t]);
      rf.step(rc, U[t]);
    }
  }
  if (c == 0) V[0] += dx2[0];
  if (c == C - 1) V[kRChunk - 1] -= dx2[1];
}

// row_walks32 with V leaving as it is produced: each group of 8 outputs goes
// out as one 256-bit store, so the stores spread over the forward walk and
// release their registers long before the next scale reuses them
template <int K, int KIND>
__device__ __forceinline__ void row_walks32_store(const RC32<K> &rc, int C,
                                                  const float (&U)[kRChunk], const float *cf,
                                                  const float *cb, const float *dx2, float *dst,
                                                  bool live, uint64_t pol) {
  const int c = threadIdx.x;
  float park[kRChunk];
  {
    Rec32<K, KIND> rb;
#pragma unroll
    for (int i = 0; i < K; ++i) rb.u[i] = cb[c * K + i];
#pragma unroll
    for (int t = kRChunk - 1; t >= 0; --t) {
      park[t] = rb.out_from(rc.cs, rc.b0 * U[t]);
      rb.step(rc, U[t]);
    }
  }
  Rec32<K, KIND> rf;
#pragma unroll
  for (int i = 0; i < K; ++i) rf.u[i] = cf[c * K + i];
#pragma unroll
  for (int q = 0; q < kRChunk / 8; ++q) {
    float v[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      v[t] = rf.out_from(rc.c, park[8 * q + t]);
      rf.step(rc, U[8 * q + t]);
    }
    if (q == 0 && c == 0) v[0] += dx2[0];
    if (q == kRChunk / 8 - 1 && c == C - 1) v[7] -= dx2[1];
    if (live) st_v8_hint(dst + 8 * q, v, pol);
  }
}

// row_walks32_store with the two directions as the lanes of packed FMAs:
// step j runs the forward recursion at sample j and the backward one at
// 31 - j on the same pole (a broadcast operand), so each step is 2K + 1
// FFMA2 for both walks (4K + 1 FFMA per sample when walked one after the
// other).  Steps 0..15 park the pairs (fwd(j), bwd(31-j)) -- outputs without
// the b0 U term; at step 16 the state pairs swap halves, and steps 16..31
// start from the parked halves plus b0 U (both lanes, broadcast b0), so the
// pair of step j is (V(31-j), V(j)) and V completes from the middle out (two
// 8-sample groups after step 23, the last two after step 31).  The park
// stays 32 registers.  Per lane the terms are the single-walk ones; only the
// order in which b0 U and the two directions' sums are added differs.
// SYM (sign +1, every blur): cs = c, so the output vectors broadcast too.
template <int K, int KIND, bool SYM>
__device__ __forceinline__ void row_walks32_pair(const RowLapParams &P, int C,
                                                 const float (&U)[kRChunk], const float *cf,
                                                 const float *cb, const float *dx2, float *dst,
                                                 bool live, uint64_t pol) {
  const int c = threadIdx.x;
  float2 u[K], cc[K], cx[K];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    u[i] = make_float2(cf[c * K + i], cb[c * K + i]);
    cc[i] = SYM ? make_float2(P.c[i], P.c[i]) : make_float2(P.c[i], P.cs[i]);
    cx[i] = SYM ? cc[i] : make_float2(P.cs[i], P.c[i]);
  }
  const float2 p2 = make_float2(P.p, P.p), q2 = make_float2(P.q, P.q),
               nq2 = make_float2(-P.q, -P.q), b02 = make_float2(P.b0, P.b0);
  auto step = [&](float2 x2) {
    if (KIND == M32_JORDAN) {
      u[0] = ffma2(p2, u[0], x2);
#pragma unroll
      for (int i = 1; i < K; ++i) u[i] = ffma2(p2, u[i], u[i - 1]);
    } else {
      const float2 ur = u[0], ui = u[1];
      u[0] = ffma2(p2, ur, ffma2(nq2, ui, x2));
      u[1] = ffma2(q2, ur, fmul2(p2, ui));
    }
  };
  float2 pk[kRChunk / 2];
#pragma unroll
  for (int j = 0; j < kRChunk / 2; ++j) {
    const float2 x2 = make_float2(U[j], U[kRChunk - 1 - j]);
    float2 o = fmul2(cc[0], u[0]);
#pragma unroll
    for (int i = 1; i < K; ++i) o = ffma2(cc[i], u[i], o);
    pk[j] = o;  // (fwd(j), bwd(31-j)) without b0 U
    step(x2);
  }
#pragma unroll
  for (int i = 0; i < K; ++i) u[i] = make_float2(u[i].y, u[i].x);  // (bwd, fwd)
  float lo[8], hi[8];
#pragma unroll
  for (int j = kRChunk / 2; j < kRChunk; ++j) {
    const int m = kRChunk - 1 - j;
    const float2 x2 = make_float2(U[m], U[j]);
    float2 o = ffma2(b02, x2, pk[m]);  // (fwd(m) + b0 U(m), bwd(j) + b0 U(j))
#pragma unroll
    for (int i = 0; i < K; ++i) o = ffma2(cx[i], u[i], o);  // (V(m), V(j))
    step(x2);
    const int g = (j - kRChunk / 2) & 7;
    lo[7 - g] = o.x;  // V(m): m = 15 - g (first group) or 7 - g (second)
    hi[g] = o.y;      // V(j): j = 16 + g or 24 + g
    if (g == 7) {
      const bool last = j == kRChunk - 1;
      if (last && c == 0) lo[0] += dx2[0];
      if (last && c == C - 1) hi[7] -= dx2[1];
      if (live) {
        st_v8_hint(dst + (last ? 0 : 8), lo, pol);
        st_v8_hint(dst + (last ? 24 : 16), hi, pol);
      }
    }
  }
}

template <int K, int KIND>
__device__ __forceinline__ void row_scan_walk32(const RowLapParams &p, const float (&U)[kRChunk],
                                                float (&V)[kRChunk], float *cf, float *cb,
                                                const float *e2, const float *dx2) {
  const int c = threadIdx.x, lane = c & 31, warp = c >> 5;
  for (int task = warp; task < 2; task += (int)(blockDim.x >> 5))
    chunk_scan32<K>(p, task == 0 ? cf : cb, task, e2[task], lane);
  __syncthreads();
  row_walks32<K, KIND>(RC32<K>(p), p.C, U, V, cf, cb, dx2);
}

// both phases (contains two block barriers)
template <int K, int KIND>
__device__ __forceinline__ void row_filter(const RowLapParams &p, const float (&U)[kRChunk],
                                           float (&V)[kRChunk], float *cf, float *cb,
                                           const float *e2, const float *dx2) {
  row_carry32<K, KIND>(RC32<K>(p), U, cf, cb);
  __syncthreads();
  row_scan_walk32<K, KIND>(p, U, V, cf, cb, e2, dx2);
}

int rowlap_get_plan(int64_t h, int64_t w, const double *b, const double *a, int k, double b0,
                    int sign, RowLapPlan *out);
bool rowlap_supported(int64_t h, int64_t w, const double *b, const double *a, int k, double b0,
                      int sign);

// One sweep's stage pair per scale (row stage, column stage), all of one
// order k and one modal kind.  sweep_rows: the border kernel, then the
// multi-scale row pass: V_s and the extras of every scale.
struct SweepStage {
  const double *rb, *ra, *cb, *ca;
  double rb0, cb0;
  int rsign, csign;
};
bool sweep_supported(const void *x, int64_t h, int64_t w, int64_t ldx, int k, int ns,
                     const SweepStage *st);
int sweep_rows(const float *x, int64_t ldx, int64_t h, int64_t w, int k, int ns,
               const SweepStage *st, const SweepOut &out, cudaStream_t stream);

}  // namespace vmf
