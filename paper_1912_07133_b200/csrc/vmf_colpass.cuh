// vmf_colpass.cuh -- the fused column pass: column IIR + Laplacian + 3x3 NMS
// (vmf_colpass.cu).
#pragma once
#include "vmf_iir.cuh"
#include "vmf_dfi.cuh"
#include "vmf_rowlap.cuh"

namespace vmf {

constexpr int kSub = 32;            // rows per sub-chunk (one recursion run)
constexpr int kBand = 64;           // rows per band (carry granularity)
constexpr int kMaxCpl = 4;          // bands per lane in the band scan (H <= 8192)
constexpr int kColThreads = 128;    // computed columns per CTA
constexpr int kColHalo = 2;         // halo columns each side (Laplacian + NMS)
constexpr int kColOut = kColThreads - 2 * kColHalo;  // 124 output columns per CTA
constexpr int kCandSmem = 512;      // per-CTA candidate buffer
constexpr int kHMax = kBand + 2 * VMF_MAX_IIR_ORDER + 2;

struct ColParams {
  double b[VMF_MAX_IIR_ORDER], a[VMF_MAX_IIR_ORDER];
  double b0, sign, yss;
  double h[kHMax];        // causal impulse response, h[0] = 0
  double Ty[VMF_MAX_IIR_ORDER * VMF_MAX_IIR_ORDER];   // over one 32-row sub-chunk
  double Tx[VMF_MAX_IIR_ORDER * VMF_MAX_IIR_ORDER];
  double TyB[2][VMF_MAX_IIR_ORDER * VMF_MAX_IIR_ORDER];  // over a band / the last band
  double TxB[2][VMF_MAX_IIR_ORDER * VMF_MAX_IIR_ORDER];
  double TyBp[5][VMF_MAX_IIR_ORDER * VMF_MAX_IIR_ORDER];  // TyB^(cpl 2^l)
  double SP[4][kBand / 2], SQ[4][kBand / 2];  // folded band-carry weights (K <= 4)
  int64_t H, W, Hp;       // Hp = H rounded up to 32 (rows >= H replicate row H-1)
  double TyBc[VMF_MAX_IIR_ORDER * VMF_MAX_IIR_ORDER];  // TyB^cpb (one scan group)
  int NB, Blast, cpl, cpb;  // bands; rows in the last band; bands per lane / scan group
  float lap_scale, frac;
  DfiCoef bwd;  // b_minus = sign * b, a: the backward run yields sign * y- directly
};

constexpr int kFinCtas = 128;       // CTAs of the finaliser's large-list path

// Device-side bookkeeping shared by the fused column pass and the finaliser
// (zeroed by the first kernel of every pass).
struct CandState {
  unsigned int absmax_bits;  // max |L| (float bits)
  int count;                 // candidates appended
  int overflow;              // the global candidate list overflowed
  int ticket;                // CTAs done (the fp32 column scan's last-CTA step)
  unsigned int bound_bits;   // a lower bound of max |L| known before the apply
                             // (the fp32 band scan: |L| on the band-boundary rows)
  // decoupled look-back of the finaliser's large-list path: per CTA
  // (status << 62) | count, status 1 = own count, 2 = inclusive prefix
  unsigned long long look[kFinCtas];
};

// A candidate goes to the CTA's shared buffer, or straight to the global list
// once that is full (a superset either way: the finaliser applies the final
// threshold), so a busy tile never forces the ordered full-frame fallback.
__device__ __forceinline__ void cand_push(int *ccount, int *cy, int *cx, float *cv, int smem_cap,
                                          CandState *st, int *gy, int *gx, float *gv, int gcap,
                                          int y, int x, float v) {
  const int k = atomicAdd(ccount, 1);
  if (k < smem_cap) {
    cy[k] = y;
    cx[k] = x;
    cv[k] = v;
    return;
  }
  const int g = atomicAdd(&st->count, 1);
  if (g < gcap) {
    gy[g] = y;
    gx[g] = x;
    gv[g] = v;
  } else {
    st->overflow = 1;
  }
}

// Warp-ballot compaction: the lanes of `mem` (the converged lanes calling
// together; the whole warp by default) append up to 4 candidates each,
// (y, x0 + i, v[i]) for the set bits i of `mask`.  One ballot per candidate
// slot ranks every lane's candidates among the warp's, and the lowest lane
// reserves the warp's block in the CTA's shared buffer with ONE atomicAdd
// (past the buffer, the global list, as cand_push).
__device__ __forceinline__ void cand_push_warp(int *ccount, int *cy, int *cx, float *cv,
                                               int smem_cap, CandState *st, int *gy, int *gx,
                                               float *gv, int gcap, unsigned mask, int y, int x0,
                                               const float (&v)[4], unsigned mem = 0xffffffffu) {
  if (!__ballot_sync(mem, mask != 0u)) return;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  int before = 0, tot = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const unsigned bal = __ballot_sync(mem, (mask >> i) & 1u);
    before += __popc(bal & lt);
    tot += __popc(bal);
  }
  const int leader = __ffs(mem) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(ccount, tot);
  int k = __shfl_sync(mem, base, leader) + before;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (!((mask >> i) & 1u)) continue;
    if (k < smem_cap) {
      cy[k] = y;
      cx[k] = x0 + i;
      cv[k] = v[i];
    } else {
      const int g = atomicAdd(&st->count, 1);
      if (g < gcap) {
        gy[g] = y;
        gx[g] = x0 + i;
        gv[g] = v[i];
      } else {
        st->overflow = 1;
      }
    }
    ++k;
  }
}

// Flush a CTA's n shared candidates (n uniform over the CTA, read after a
// barrier) to the global list with ONE reservation per CTA: a per-candidate
// atomicAdd on the single global counter serialises in L2 when thresholds
// are low and thousands of candidates arrive (frac = 0.05).  All threads of
// the CTA must call it; sbase is a __shared__ int.
__device__ __forceinline__ void cand_flush(int n, const int *cy, const int *cx, const float *cv,
                                           CandState *st, int *gy, int *gx, float *gv, int gcap,
                                           int *sbase) {
  if (n <= 0) return;
  if (threadIdx.x == 0) *sbase = atomicAdd(&st->count, n);
  __syncthreads();
  const int base = *sbase;
  for (int q = threadIdx.x; q < n; q += blockDim.x) {
    const int k = base + q;
    if (k < gcap) {
      gy[k] = cy[q];
      gx[k] = cx[q];
      gv[k] = cv[q];
    } else {
      st->overflow = 1;
    }
  }
}

// Zero the CandState (one CTA's threads; after the pass's pdl_wait).
__device__ __forceinline__ void cand_reset(CandState *st) {
  unsigned *w = reinterpret_cast<unsigned *>(st);
  for (int i = threadIdx.x; i < (int)(sizeof(CandState) / 4); i += blockDim.x) w[i] = 0u;
}

bool colpass_supported(int64_t h, int64_t w, int k);
// candidate list capacity of the fused column passes (IIR and FIR)
int64_t colpass_cand_capacity(int64_t h, int64_t w);
// final threshold + (y, x) order of the candidates a fused column pass appended
int colfinal_launch(CandState *cs, const int *gy, const int *gx, const float *gv, int64_t gcap,
                    const float *L, int64_t ldl, int64_t H, int64_t W, float frac,
                    int32_t *det_yx, float *det_val, int64_t cap, int64_t *n_det_dev,
                    float *thr_dev, cudaStream_t st);
size_t colpass_workspace_bytes(int64_t h, int64_t w, int k, int64_t cand_cap);
// T (fp32, h x w, pitch ldt) -> L (pitch ldl) + detections (sorted by y, x).
// b64 != null: only the fp64 blur B (pitch w) is produced (no L / detections);
// blur_only: only the blur B, rounded to fp32, into L (the iir_cols leaf)
int colpass_run(const float *T, int64_t ldt, float *L, int64_t ldl, double *b64,
                const IirParams &ip,
                int64_t h, int64_t w, float lap_scale, float frac, int32_t *det_yx,
                float *det_val, int64_t cap, int64_t *n_det_dev, float *thr_dev, void *ws,
                size_t ws_bytes, cudaStream_t st, bool blur_only = false);

// fp32 "Laplacian-first" fused column pass (vmf_colpass32.cu): the detect
// path's column pass for IIR stages with a modal fp32 realisation (repeated
// real pole, K = 2..4, or a complex pair, K = 2); L (* lap_scale) +
// detections, no blur output.
// V mode: the input is V = R(Lap5 X) from the fp32 row pass (vmf_rowlap.cu)
// instead of T; x = the frame (border partials), vt / vb = its virtual rows,
// (rb, ra, rk, rb0, rsign) = the ROW stage (the border rows are row-filtered).
struct Col32VMode {
  const float *vt, *vb;       // the row pass's virtual rows (steady inputs, padded rows)
  const float *ky;            // its border rows Ky[2][w] (added to L rows 0 / H-1)
};
bool colpass32_supported(int64_t h, int64_t w, const IirParams &ip);
size_t colpass32_workspace_bytes(int64_t h, int64_t w, int k);
int colpass32_run(const float *T, int64_t ldt, float *L, int64_t ldl, const IirParams &ip,
                  int64_t h, int64_t w, float lap_scale, float frac, int32_t *det_yx,
                  float *det_val, int64_t cap, int64_t *n_det_dev, float *thr_dev, void *ws,
                  size_t ws_bytes, cudaStream_t st, const Col32VMode *vmode = nullptr);

}  // namespace vmf
