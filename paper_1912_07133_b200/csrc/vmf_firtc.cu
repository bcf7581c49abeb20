// vmf_firtc.cu -- see vmf_firtc.cuh.
//
// Geometry of one pass (rows or columns alike): the lines m (image rows for
// the row pass, image columns for the column pass), the outputs n along a
// line, K the input window of a 128 x 128 tile; the accumulator is
//   D[n][m] = sum_q A[n][q] B[m][q],  A[n][q] = t[n + 2k - q] (the band,
//   zero outside 0 <= n + 2k - q <= 2k),  B[m][q] = in[m0 + m][n0 - k + q]
// which is out[n] = sum_j t[j] in[n + k - j] (engine.py:35-62's conv with
// j = k + m).  Input samples outside the line read as zero (TMA OOB fill);
// the constant extension the Laplacian-first identity needs there enters in
// the epilogue through the tap tail sums: left of the line the extension is
// eL, so out[n] += eL sum_{j > n + k} t[j] (n < k), right of it eR,
// out[n] += eR sum_{j <= n + k - len} t[j].
//
// Per K-slice of 32 the MMA issuer runs 4 x 3 tcgen05.mma kind::tf32 (M 128,
// N 128, K 8; hi*hi, hi*lo, lo*hi) on operands the producer brought in by TMA
// with 128-byte swizzle (the K-major SWIZZLE_128B layout: 8-row x 128-byte
// atoms, 1024 bytes apart; +32 bytes per K step inside the atom).
#include <cmath>
#include <cstring>
#include <mutex>

#include "vmf_colpass.cuh"
#include "vmf_common.cuh"
#include "vmf_firtc.cuh"
#include "vmf_prof.cuh"
#include "vmf_tma.cuh"

#ifndef VMF_TC_ABL  // timing ablations (tools/gpu): 1 no split, 2 no stores, 3 one MMA step,
                    // 4 no MMA, 5 every tile loads tile 0's lines
#define VMF_TC_ABL 0
#endif

namespace vmf {

#ifdef VMF_TC_TL  // per-tile globaltimer stamps of CTA 0 (tools/diag/tl_firtc.py)
__device__ unsigned long long g_tctl[1024];
#define TCTL(i, ph)                                                             \
  do {                                                                          \
    if (blockIdx.x == 0 && (i) < 64) {                                          \
      unsigned long long t_;                                                    \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                   \
      g_tctl[(i) * 8 + (ph)] = t_;                                              \
    }                                                                           \
  } while (0)
#define TCS(g, ph)                                                             \
  do {                                                                          \
    if (blockIdx.x == 0 && (g) < 96) {                                          \
      unsigned long long t_;                                                    \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                   \
      g_tctl[512 + (g) * 5 + (ph)] = t_;                                        \
    }                                                                           \
  } while (0)
#else
#define TCTL(i, ph) \
  do {              \
  } while (0)
#define TCS(g, ph) \
  do {             \
  } while (0)
#endif

namespace {

constexpr int kTile = 128;    // M = N = 128
constexpr int kSlice = 32;    // K per pipeline stage (one 128-byte swizzle atom)
constexpr int kMaxStages = 6;
constexpr int kOpBytes = kTile * kSlice * 4;      // one operand slice: 16 KB
constexpr int kStageBytes = 2 * kOpBytes;         // the lines' slice: raw -> hi, lo
constexpr int kSmemBudget = 220 * 1024;           // dynamic shared memory per CTA
constexpr uint32_t kIdesc = (1u << 4)             // D fp32
                            | (2u << 7)           // A tf32
                            | (2u << 10)          // B tf32 (both K-major)
                            | ((uint32_t)(kTile >> 3) << 17)   // N
                            | ((uint32_t)(kTile >> 4) << 24);  // M

struct FirTcStage {
  float t[2 * kTcMaxK + 1];
  float ctl[kTcMaxK];  // ctl[n] = sum_{j > n + k} t[j]        (outputs n < k)
  float ctr[kTcMaxK];  // ctr[i] = sum_{j <= i} t[j]           (outputs len - k + i)
  int T, k, KW;        // taps, half-length, window (multiple of 32)
  int gr;              // rows of the tall band G (128 + 32 (KW / 32 - 1))
};

struct FirTcPass {
  int mrows;            // GEMM rows (lines)
  int len;              // outputs per line
  int H;                // (row pass) image rows: lines H .. H+3 are the border rows
  int k, nslices, nstages;
  const float4 *edge;   // per line {eL, eR, dL, dR}
  // row pass outputs
  float *vt;            // V^T [W][ldvt] (fp32)
  int64_t ldvt;
  float4 *edge2;        // the column pass's edge table {Vt, Vb, Kyt, Kyb} per column
  // column pass outputs
  float *L;
  int64_t ldl;
  float lap_scale;
  unsigned *absmax;     // CandState::absmax_bits (max |L| as float bits)
  int vec;              // L rows 32-byte (2) / 16-byte (1) aligned: vector stores
};

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);   // start address
  d |= (uint64_t)1 << 16;                    // LBO (unused: swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;          // SBO: 8-row groups 1024 B apart
  d |= (uint64_t)1 << 46;                    // sm_100 descriptor version
  d |= (uint64_t)2 << 61;                    // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t dt, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(bar)));
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

// ---------------------------------------------------------------------------
// prep: one launch, three block ranges (U quads | border sums | band tables)
// ---------------------------------------------------------------------------
struct PrepArgs {
  const float *X;
  int64_t ldx;
  int H, W;
  float *u;  // U [H + 4][ldu] (fp32)
  int64_t ldu;
  float4 *edge;
  float *b1h, *b1l, *b2h, *b2l;
  int nbu, nbe;  // blocks of the U and border ranges
};

__device__ __forceinline__ void put_split(float *h, float *l, int64_t i, float u) {
  const float hi = tf32_hi(u);
  h[i] = hi;
  l[i] = tf32_hi(u - hi);
}

// U rows 0 .. H-1: 5-point Laplacian (replicate), a block = 1024 samples x 4
// rows (the 6 input rows' quads loaded up front); rows H, H+1: D20 X of rows
// 0 and H-1 (the virtual rows' input, zero beyond the columns).
__device__ __forceinline__ void prep_u4(const PrepArgs &a, int blk) {
  const int bpr = (a.W + 1023) / 1024;
  const int rg = blk / bpr, c = 4 * ((blk - rg * bpr) * 256 + (int)threadIdx.x);
  const int r0 = 4 * rg;
  if (r0 >= a.H || c >= a.W) return;
  const int H = a.H, W = a.W;
  auto rowp = [&](int r) { return a.X + (int64_t)(r < 0 ? 0 : (r > H - 1 ? H - 1 : r)) * a.ldx; };
  if (c + 4 <= W) {
    float4 x[6];
    float hl[4], hr[4];
#pragma unroll
    for (int q = 0; q < 6; ++q) x[q] = __ldg(reinterpret_cast<const float4 *>(rowp(r0 - 1 + q) + c));
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float *rp = rowp(r0 + q);
      hl[q] = __ldg(rp + (c > 0 ? c - 1 : 0));
      hr[q] = __ldg(rp + (c + 4 < W ? c + 4 : W - 1));
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (r0 + q >= H) break;
      const float4 m = x[q + 1], u = x[q], d = x[q + 2];
      const float xs[6] = {hl[q], m.x, m.y, m.z, m.w, hr[q]};
      const float us[4] = {u.x, u.y, u.z, u.w}, ds[4] = {d.x, d.y, d.z, d.w};
      float o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        o[j] = ((xs[j] - xs[j + 1]) + (xs[j + 2] - xs[j + 1])) +
               ((us[j] - xs[j + 1]) + (ds[j] - xs[j + 1]));
      *reinterpret_cast<float4 *>(a.u + (int64_t)(r0 + q) * a.ldu + c) =
          make_float4(o[0], o[1], o[2], o[3]);
    }
  } else {
    for (int q = 0; q < 4 && r0 + q < H; ++q) {
      const int r = r0 + q;
      const float *row = rowp(r), *up = rowp(r - 1), *dn = rowp(r + 1);
      for (int cc = c; cc < W; ++cc) {
        const float x = __ldg(row + cc);
        a.u[(int64_t)r * a.ldu + cc] =
            ((__ldg(row + (cc > 0 ? cc - 1 : 0)) - x) + (__ldg(row + (cc < W - 1 ? cc + 1 : W - 1)) - x)) +
            ((__ldg(up + cc) - x) + (__ldg(dn + cc) - x));
      }
    }
  }
}
__device__ __forceinline__ void prep_d20(const PrepArgs &a, int which, int c) {
  if (c >= a.W) return;
  const int W = a.W;
  const float *row = a.X + (int64_t)(which == 0 ? 0 : a.H - 1) * a.ldx;
  const float x = __ldg(row + c);
  a.u[(int64_t)(a.H + which) * a.ldu + c] =
      (__ldg(row + (c > 0 ? c - 1 : 0)) - x) + (__ldg(row + (c < W - 1 ? c + 1 : W - 1)) - x);
}

// Border sums (fp32, k terms), one warp per sum: lane l takes m = 1 + l,
// 1 + l + 32, ..., then a butterfly reduction.  Forward:
// sum_{m>=1} t[k-m] (x(m) - x(m-1)); backward: sum_{m>=1} t[k+m] (x(n-m) - x(n-1-m)),
// along a line of n samples at p, step apart.
__device__ __forceinline__ float wsum(const FirTcStage &s, const float *p, int64_t step, int n,
                                      bool fwd, int lane) {
  const int m1 = s.k < n - 1 ? s.k : n - 1;
  float a = 0.0f;
  for (int m = 1 + lane; m <= m1; m += 32) {
    const float g = fwd ? __ldg(p + m * step) - __ldg(p + (m - 1) * step)
                        : __ldg(p + (int64_t)(n - m) * step) - __ldg(p + (int64_t)(n - 1 - m) * step);
    a = fmaf(s.t[fwd ? s.k - m : s.k + m], g, a);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  return a;
}

// warp task i < H+4: the row pass's edge table {eL, eR, dL, dR} of line i
__device__ __forceinline__ void prep_edge(const PrepArgs &a, const FirTcStage &rs,
                                          const FirTcStage &cs, int64_t i, int lane) {
  const int H = a.H, W = a.W;
  const float *X = a.X;
  const int64_t ldx = a.ldx;
  auto d02 = [&](int r, int c) {  // vertical second difference (replicate)
    const float x = __ldg(X + (int64_t)r * ldx + c);
    return (__ldg(X + (int64_t)(r > 0 ? r - 1 : 0) * ldx + c) - x) +
           (__ldg(X + (int64_t)(r < H - 1 ? r + 1 : H - 1) * ldx + c) - x);
  };
  auto dxl = [&](int r) { return wsum(rs, X + (int64_t)r * ldx, 1, W, true, lane); };
  auto dxr = [&](int r) { return wsum(rs, X + (int64_t)r * ldx, 1, W, false, lane); };
  auto dyt = [&](int c) { return wsum(cs, X + c, ldx, H, true, lane); };
  auto dyb = [&](int c) { return wsum(cs, X + c, ldx, H, false, lane); };
  if (i < H + 4) {
    float4 e;
    if (i < H) {
      const float l = dxl((int)i), r = dxr((int)i);
      e = make_float4(d02((int)i, 0), d02((int)i, W - 1), l, r);
    } else if (i < H + 2) {  // virtual rows: zero extension, the border row's dx terms
      const int rr = i == H ? 0 : H - 1;
      const float l = dxl(rr), r = dxr(rr);
      e = make_float4(0.0f, 0.0f, l, r);
    } else if (i == H + 2) {  // Ky top: R(dyt) with replicate ends
      const float l = dyt(0), r = dyt(W - 1);
      e = make_float4(l, r, 0.0f, 0.0f);
    } else {
      const float l = dyb(0), r = dyb(W - 1);
      e = make_float4(l, r, 0.0f, 0.0f);
    }
    if (lane == 0) a.edge[i] = e;
    return;
  }
}

// the column sums dyt / dyb of 32 columns per 256-thread block (coalesced:
// thread (c, g) sums rows m = 1 + g, 1 + g + 8, ...; partials summed in g
// order) into U rows H+2 / H+3
__device__ __forceinline__ void prep_cols(const PrepArgs &a, const FirTcStage &cs, int blk) {
  __shared__ float part[2][8][32];
  const int cx = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int c = 32 * blk + cx;
  const int H = a.H, W = a.W;
  const int m1 = cs.k < H - 1 ? cs.k : H - 1;
  float t = 0.0f, b = 0.0f;
  if (c < W) {
    const float *p = a.X + c;
    for (int m = 1 + g; m <= m1; m += 8) {
      t = fmaf(cs.t[cs.k - m], __ldg(p + (int64_t)m * a.ldx) - __ldg(p + (int64_t)(m - 1) * a.ldx), t);
      b = fmaf(cs.t[cs.k + m],
               __ldg(p + (int64_t)(H - m) * a.ldx) - __ldg(p + (int64_t)(H - 1 - m) * a.ldx), b);
    }
  }
  part[0][g][cx] = t;
  part[1][g][cx] = b;
  __syncthreads();
  if (g < 2 && c < W) {
    float v = 0.0f;
#pragma unroll
    for (int q = 0; q < 8; ++q) v += part[g][q][cx];
    a.u[(int64_t)(H + 2 + g) * a.ldu + c] = v;
  }
}

// the tall band G[row][q] = t[row + 2k - 32 (ns - 1) - q] (hi / lo, [gr][32]):
// slice sl's band A_sl[n][q] = t[n + 2k - 32 sl - q] is G's rows from (ns - 1 - sl) 32
__device__ __forceinline__ void prep_band(const FirTcStage &s, float *bh, float *bl, int64_t i) {
  if (i >= (int64_t)s.gr * kSlice) return;
  const int row = (int)(i / kSlice), q = (int)(i % kSlice);
  const int j = row + 2 * s.k - kSlice * (s.KW / kSlice - 1) - q;
  put_split(bh, bl, i, (j >= 0 && j < s.T) ? s.t[j] : 0.0f);
}

__global__ void __launch_bounds__(256) firtc_prep_kernel(const __grid_constant__ PrepArgs a,
                                                         const __grid_constant__ FirTcStage rs,
                                                         const __grid_constant__ FirTcStage cs) {
  // block ranges, the latency-bound border sums first: [column sums][row
  // edge table][band tables][U]
  int b = blockIdx.x;
  const int nbc = (a.W + 31) / 32, nbr = (a.H + 4 + 7) / 8;
  if (b < nbc) {
    prep_cols(a, cs, b);
    return;
  }
  b -= nbc;
  if (b < nbr) {
    const int64_t task = (int64_t)b * 8 + (threadIdx.x >> 5);
    if (task < a.H + 4) prep_edge(a, rs, cs, task, threadIdx.x & 31);
    return;
  }
  b -= nbr;
  const int nbb = (int)(((int64_t)kSlice * (rs.gr + cs.gr) + 255) / 256);
  if (b < nbb) {
    const int64_t i = (int64_t)b * blockDim.x + threadIdx.x;
    const int64_t n1 = (int64_t)rs.gr * kSlice;
    if (i < n1)
      prep_band(rs, a.b1h, a.b1l, i);
    else
      prep_band(cs, a.b2h, a.b2l, i - n1);
    return;
  }
  b -= nbb;
  const int nbd = (a.W + 255) / 256;
  if (b < 2 * nbd) {
    prep_d20(a, b / nbd, (b % nbd) * 256 + threadIdx.x);
    return;
  }
  prep_u4(a, b - 2 * nbd);
}

// ---------------------------------------------------------------------------
// the tensor-core pass
// ---------------------------------------------------------------------------
// Persistent, warp-specialised: warp 0 (one lane) streams the K-slices of
// every tile this CTA owns through the smem ring; warp 1 (one lane) issues
// the MMAs into one of two TMEM accumulators (128 columns each) so the next
// tile accumulates while warps 2..5 drain the previous one.  The accumulator
// is D^T: A = the band (M = 128 outputs), B = the 128 lines' windows (N), so
// TMEM lane = output sample and the columns run along the lines -- each
// epilogue thread writes 16 consecutive lines of its output row (V^T rows,
// L rows) as wide stores.
constexpr int kEpiWarps = 4;
constexpr int kCvtWarps = 4;  // split the lines' fp32 slice into tf32 hi / lo in smem
constexpr int kThreads = 64 + 32 * (kEpiWarps + kCvtWarps);

__device__ __forceinline__ void st_v4(float *p, float a, float b, float c, float d) {
  *reinterpret_cast<float4 *>(p) = make_float4(a, b, c, d);
}

template <int MODE>  // 1: rows (-> V^T hi / lo, border rows), 2: columns (-> L)
__global__ void __launch_bounds__(kThreads, 1) firtc_mma_kernel(
    const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb_h,
    const __grid_constant__ CUtensorMap tb_l, const __grid_constant__ FirTcStage s,
    const __grid_constant__ FirTcPass P) {
  // ta: the lines' fp32 data [mrows][len] (B operand, split here); tb_*: the
  // band [128][KW] as tf32 hi / lo (A operand)
  extern __shared__ __align__(1024) unsigned char smem_tc[];
  __shared__ __align__(8) uint64_t full[kMaxStages], conv[kMaxStages], empty[kMaxStages],
      tfull[2], tempty[2], bandbar;
  __shared__ uint32_t tbase;
  __shared__ float4 edge_s[2][kTile];
  const uint32_t sb0 = (uint32_t)__cvta_generic_to_shared(smem_tc);
  const uint32_t pad = (1024u - (sb0 & 1023u)) & 1023u;
  // [tall band hi][tall band lo][ring of nstages x (raw / hi, lo)]
  const int gbytes = s.gr * 128;  // (multiple of 1024: gr is a multiple of 32)
  const uint32_t band_s = sb0 + pad;
  unsigned char *ring = smem_tc + pad + 2 * gbytes;
  const uint32_t ring_s = band_s + 2 * gbytes;
  const int nst = P.nstages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntn = (int)((P.len + kTile - 1) / kTile), ntm = (int)((P.mrows + kTile - 1) / kTile);
  const int ntiles = ntn * ntm;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(
        (unsigned)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 32) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&conv[i], kCvtWarps);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&bandbar, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiWarps);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t dt = tbase;
  pdl_wait();  // the operands come from the previous kernels
  const int ns = P.nslices;
  if (warp == 0) {
    if (lane == 0) {  // producer
      const uint64_t pol_a = l2_policy_evict_first(), pol_b = l2_policy_evict_last();
      // the tall band, once: G[row][q] = t[row + 2k - 32 (ns - 1) - q]; slice
      // sl's band A_sl is G's rows (ns - 1 - sl) 32 .. +127 (4096 bytes per 32 rows)
      mbar_expect_tx(&bandbar, 2 * gbytes);
      for (int r0 = 0; r0 < s.gr; r0 += kSlice) {  // (32-row boxes: gr is a multiple of 32)
        tma_load_2d_hint(smem_tc + pad + r0 * 128, &tb_h, &bandbar, 0, r0, pol_b);
        tma_load_2d_hint(smem_tc + pad + gbytes + r0 * 128, &tb_l, &bandbar, 0, r0, pol_b);
      }
      int g = 0;  // slices issued by this CTA
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int n0 = (t % ntn) * kTile, m0 = (t / ntn) * kTile;
        for (int sl = 0; sl < ns; ++sl, ++g) {
          const int st = g % nst;
          if (g >= nst) mbar_wait(&empty[st], (unsigned)(((g / nst) - 1) & 1));
          if (sl == 0) TCTL((t - (int)blockIdx.x) / (int)gridDim.x, 0);
          if (sl == ns - 1) TCTL((t - (int)blockIdx.x) / (int)gridDim.x, 1);
          TCS(g, 0);
          mbar_expect_tx(&full[st], kOpBytes);
          tma_load_2d_hint(ring + st * kStageBytes, &ta, &full[st],
                           VMF_TC_ABL == 5 ? kSlice * sl : n0 - P.k + kSlice * sl,
                           VMF_TC_ABL == 5 ? 0 : m0, pol_a);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      mbar_wait(&bandbar, 0);
      int g = 0, i = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int buf = i & 1;
        if (i >= 2) mbar_wait(&tempty[buf], (unsigned)(((i >> 1) - 1) & 1));
        TCTL(i, 2);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const uint32_t d = dt + buf * kTile;
        for (int sl = 0; sl < ns; ++sl, ++g) {
          const int st = g % nst;
          mbar_wait(&conv[st], (unsigned)((g / nst) & 1));
          TCS(g, 3);
          asm volatile("tcgen05.fence::after_thread_sync;\n");
          const uint32_t ga = band_s + (uint32_t)(ns - 1 - sl) * 4096u;
          const uint64_t ah = sw128_desc(ga), al = sw128_desc(ga + gbytes);
          const uint32_t b = ring_s + st * kStageBytes;
          const uint64_t bh = sw128_desc(b), bl = sw128_desc(b + kOpBytes);
#pragma unroll
          for (int kk = 0; kk < (VMF_TC_ABL == 3 ? 1 : VMF_TC_ABL == 4 ? 0 : kSlice / 8); ++kk) {  // K = 8 (32 bytes) per instruction
            const uint64_t o = 2 * kk;
            mma_tf32(d, ah + o, bh + o, (sl > 0 || kk > 0) ? 1u : 0u);
            mma_tf32(d, ah + o, bl + o, 1u);
            mma_tf32(d, al + o, bh + o, 1u);
          }
          mma_commit(&empty[st]);  // the slot is free once these MMAs have read it
          TCS(g, 4);
        }
        TCTL(i, 3);
        mma_commit(&tfull[buf]);
      }
    }
  } else if (warp >= 2 + kEpiWarps) {
    // ---- converters: the lines' slice (fp32, swizzled) -> tf32 hi in place
    // and lo into the next slot (same swizzled offsets: same layout)
    const int ct = threadIdx.x - 32 * (2 + kEpiWarps);
    int g = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int sl = 0; sl < ns; ++sl, ++g) {
        const int st = g % nst;
        mbar_wait(&full[st], (unsigned)((g / nst) & 1));
        if (ct == 0) TCS(g, 1);
        float4 *raw = reinterpret_cast<float4 *>(ring + st * kStageBytes);
        float4 *lo = reinterpret_cast<float4 *>(ring + st * kStageBytes + kOpBytes);
#pragma unroll
        for (int u = 0; u < (VMF_TC_ABL == 1 ? 0 : kOpBytes / 16 / (32 * kCvtWarps)); ++u) {
          const int e = ct + u * 32 * kCvtWarps;
          const float4 v = raw[e];
          float4 h, l;
          h.x = tf32_hi(v.x);
          h.y = tf32_hi(v.y);
          h.z = tf32_hi(v.z);
          h.w = tf32_hi(v.w);
          l.x = tf32_hi(v.x - h.x);
          l.y = tf32_hi(v.y - h.y);
          l.z = tf32_hi(v.z - h.z);
          l.w = tf32_hi(v.w - h.w);
          raw[e] = h;
          lo[e] = l;
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // visible to the MMA
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[st]);
        if (ct == 0) TCS(g, 2);
      }
    }
  } else {
    // ---- epilogue warps: thread = TMEM lane = output sample n0 + q
    const int quarter = warp & 3;  // the TMEM lanes this warp may access
    const int q = 32 * quarter + lane;
    const int et = threadIdx.x - 64;  // 0..127
    const int len = P.len, k = P.k;
    float amax = 0.0f;
    int i = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const int buf = i & 1;
      const int n0 = (t % ntn) * kTile, m0 = (t / ntn) * kTile;
      edge_s[buf][et] = m0 + et < P.mrows ? P.edge[m0 + et] : make_float4(0.f, 0.f, 0.f, 0.f);
      asm volatile("bar.sync 1, %0;\n" ::"n"(32 * kEpiWarps));
      mbar_wait(&tfull[buf], (unsigned)((i >> 1) & 1));
      if (et == 0) TCTL(i, 4);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const int n = n0 + q;
      const bool nlive = n < len;
      // the edge weights of this output sample
      const float cl = n < k ? s.ctl[n] : 0.0f;
      const float cr = (n >= len - k && n < len) ? s.ctr[n - (len - k)] : 0.0f;
      const float f0 = n == 0 ? 1.0f : 0.0f, f1 = n == len - 1 ? 1.0f : 0.0f;
      const bool edges = n0 < k || n0 + kTile > len - k;
      const uint32_t trow = dt + ((uint32_t)(32 * quarter) << 16) + buf * kTile;
#pragma unroll 1
      for (int c0 = 0; c0 < kTile; c0 += 16) {
        float v[16];
        tmem_ld16(trow + c0, v);
        if (edges) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float4 e = edge_s[buf][c0 + j];
            v[j] = fmaf(e.x, cl, fmaf(e.y, cr, fmaf(f0, e.z, fmaf(-f1, e.w, v[j]))));
          }
        }
        const int mb = m0 + c0;  // first line of this chunk
        if (!nlive || mb >= P.mrows || VMF_TC_ABL == 2) continue;
        if (MODE == 1) {
          const int nimg = P.H - mb;  // lines of the chunk that are image rows
          float *dv = P.vt + (int64_t)n * P.ldvt + mb;
          if (nimg >= 16) {
            // 256-bit stores: a whole 32-byte sector per lane (rows are 32-byte aligned)
            const uint64_t pol = l2_policy_evict_last();  // read by the column pass next
            st_v8_hint(dv, v, pol);
            st_v8_hint(dv + 8, v + 8, pol);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int m = mb + j;
              if (m >= P.mrows) break;
              if (m < P.H)
                dv[j] = v[j];
              else
                reinterpret_cast<float *>(P.edge2 + n)[m - P.H] = v[j];
            }
          }
        } else {
          float *dst = P.L + (int64_t)n * P.ldl + mb;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            v[j] *= P.lap_scale;
            if (mb + j < P.mrows) amax = fmaxf(amax, fabsf(v[j]));
          }
          if (mb + 16 <= P.mrows && P.vec == 2) {
            const uint64_t pol = l2_policy_evict_last();  // read by stage 4 next
            st_v8_hint(dst, v, pol);
            st_v8_hint(dst + 8, v + 8, pol);
          } else if (mb + 16 <= P.mrows && P.vec) {
#pragma unroll
            for (int j = 0; j < 16; j += 4) st_v4(dst + j, v[j], v[j + 1], v[j + 2], v[j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (mb + j < P.mrows) dst[j] = v[j];
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      if (et == 0) TCTL(i, 5);
    }
    if (MODE == 2) {
      amax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(amax)));
      if (lane == 0) atomicMax(P.absmax, __float_as_uint(amax));
    }
  }
  pdl_trigger();
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tbase));
}

// ---------------------------------------------------------------------------
// stage 4 on L: thresholded 3x3 non-maximum suppression (the restated rule of
// |v| >= frac max|L|, strictly above (or below) all eight
// neighbours, the one-pixel frame border excluded), one 32 x 128 tile per CTA
// from shared memory; survivors go through the column pass's candidate
// machinery (per-CTA buffer, global list) to the sorting finaliser.
// ---------------------------------------------------------------------------
constexpr int kNmsR = 32, kNmsC = 128, kNmsCand = 256;
constexpr int kNmsP = kNmsC + 8;  // tile pitch: halo column 3, interior 4 .. 131, halo 132
__global__ void __launch_bounds__(256) firtc_nms_kernel(const float *__restrict__ L, int64_t ldl,
                                                        int H, int W, float frac,
                                                        CandState *__restrict__ st,
                                                        int *__restrict__ gy, int *__restrict__ gx,
                                                        float *__restrict__ gv, int gcap, int vec) {
  __shared__ __align__(16) float t[kNmsR + 2][kNmsP];
  __shared__ int cy[kNmsCand], cx[kNmsCand];
  __shared__ float cv[kNmsCand];
  __shared__ int ccount;
  const int r0 = blockIdx.y * kNmsR, c0 = blockIdx.x * kNmsC;
  const int tid = threadIdx.x;
  if (tid == 0) ccount = 0;
  pdl_wait();  // L and its max come from the column pass
  const float thr = frac * __uint_as_float(st->absmax_bits);
  // tile rows r0-1 .. r0+32 (clamped): the 128 interior columns by 16-byte
  // asynchronous copies (all in flight together), the two halo columns apart
  const bool v4 = vec && c0 + kNmsC <= W;
  for (int e = tid; e < (kNmsR + 2) * (kNmsC / 4); e += blockDim.x) {
    const int tr = e >> 5, q = e & 31;
    int r = r0 - 1 + tr;
    r = r < 0 ? 0 : (r >= H ? H - 1 : r);
    const float *row = L + (int64_t)r * ldl;
    if (v4) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(&t[tr][4 + 4 * q]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(row + c0 + 4 * q));
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + 4 * q + u;
        t[tr][4 + 4 * q + u] = __ldg(row + (c < W ? c : W - 1));
      }
    }
  }
  if (v4) asm volatile("cp.async.commit_group;\n" ::);
  if (tid < 2 * (kNmsR + 2)) {
    const int tr = tid >> 1, side = tid & 1;
    int r = r0 - 1 + tr;
    r = r < 0 ? 0 : (r >= H ? H - 1 : r);
    int c = side ? c0 + kNmsC : c0 - 1;
    c = c < 0 ? 0 : (c >= W ? W - 1 : c);
    t[tr][side ? 4 + kNmsC : 3] = __ldg(L + (int64_t)r * ldl + c);
  }
  if (v4) asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  // warp w takes rows w, w+8, w+16, w+24; a lane 4 adjacent columns: the
  // warp votes on each row's 128 values before any neighbour is read
  const int w = tid >> 5, lane = tid & 31;
  for (int q = w; q < kNmsR; q += 8) {
    const int r = r0 + q;
    const float4 x = *reinterpret_cast<const float4 *>(&t[q + 1][4 + 4 * lane]);
    const float vv[4] = {x.x, x.y, x.z, x.w};
    const float m4 = fmaxf(fmaxf(fabsf(x.x), fabsf(x.y)), fmaxf(fabsf(x.z), fabsf(x.w)));
    const bool live = r >= 1 && r <= H - 2 && m4 >= thr;
    if (!__any_sync(0xffffffffu, live)) continue;  // (warp-uniform)
    unsigned m = 0u;
    if (live) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int cc = c0 + 4 * lane + i, tc = 4 + 4 * lane + i;
        const float v = vv[i];
        if (!(fabsf(v) >= thr) || cc < 1 || cc > W - 2) continue;
        bool gt = true, lt = true;
#pragma unroll
        for (int di = 0; di < 3; ++di)
#pragma unroll
          for (int dj = -1; dj <= 1; ++dj) {
            if (di == 1 && dj == 0) continue;
            const float u = t[q + di][tc + dj];
            gt &= v > u;
            lt &= v < u;
          }
        // a maximum counts when positive, a minimum when negative (|v| >= thr
        // alone would admit a positive local minimum)
        if ((gt && v >= thr) || (lt && -v >= thr)) m |= 1u << i;
      }
    }
    cand_push_warp(&ccount, cy, cx, cv, kNmsCand, st, gy, gx, gv, gcap, m, r, c0 + 4 * lane, vv);
  }
  __syncthreads();
  __shared__ int flush_base;
  cand_flush(ccount < kNmsCand ? ccount : kNmsCand, cy, cx, cv, st, gy, gx, gv, gcap, &flush_base);
  pdl_trigger();
}

size_t align_up(size_t n) { return (n + 255) & ~(size_t)255; }
int64_t ld4(int64_t n) { return (n + 7) & ~(int64_t)7; }  // (32-byte rows)
int kw_of(int T) { return (int)cdiv(kTile + T - 1, kSlice) * kSlice; }
int gr_of(int T) { return kTile + kSlice * (kw_of(T) / kSlice - 1); }
// data stages that fit next to the resident band (hi + lo)
int stages_of(const FirTcStage &s) {
  int n = (kSmemBudget - 1024 - 2 * s.gr * 128) / kStageBytes;
  return n > kMaxStages ? kMaxStages : n;
}

bool stage_of(const double *taps, int n, FirTcStage *s) {
  if (n < 1 || !(n & 1) || (n - 1) / 2 > kTcMaxK) return false;
  memset(s, 0, sizeof(*s));
  s->T = n;
  s->k = (n - 1) / 2;
  s->KW = kw_of(n);
  s->gr = kTile + kSlice * (s->KW / kSlice - 1);
  for (int j = 0; j < n; ++j) s->t[j] = (float)taps[j];
  for (int i = 0; i < s->k; ++i) {  // tail / prefix sums in fp64, one rounding
    double a = 0.0, b = 0.0;
    for (int j = i + s->k + 1; j < n; ++j) a += taps[j];
    for (int j = 0; j <= i; ++j) b += taps[j];
    s->ctl[i] = (float)a;
    s->ctr[i] = (float)b;
  }
  return true;
}

struct Layout {
  float *u, *vt, *b1h, *b1l, *b2h, *b2l;
  float4 *edge1, *edge2;
  CandState *cs;
  int *gy, *gx;
  float *gv;
  int64_t ldu, ldvt, gcap;
  size_t bytes;
};

Layout layout(void *ws, int64_t h, int64_t w, int rt, int ct) {
  Layout o;
  memset(&o, 0, sizeof(o));
  o.ldu = ld4(w);
  o.ldvt = ld4(h);
  char *p = (char *)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  char *p0 = p;
  auto take = [&](size_t b) {
    char *q = p;
    p += align_up(b);
    return q;
  };
  o.u = (float *)take((size_t)(h + 4) * o.ldu * 4);
  o.vt = (float *)take((size_t)w * o.ldvt * 4);
  o.edge1 = (float4 *)take((size_t)(h + 4) * 16);
  o.edge2 = (float4 *)take((size_t)w * 16);
  o.b1h = (float *)take((size_t)gr_of(rt) * kSlice * 4);
  o.b1l = (float *)take((size_t)gr_of(rt) * kSlice * 4);
  o.b2h = (float *)take((size_t)gr_of(ct) * kSlice * 4);
  o.b2l = (float *)take((size_t)gr_of(ct) * kSlice * 4);
  o.cs = (CandState *)take(sizeof(CandState));
  o.gcap = colpass_cand_capacity(h, w);
  o.gy = (int *)take((size_t)o.gcap * 4);
  o.gx = (int *)take((size_t)o.gcap * 4);
  o.gv = (float *)take((size_t)o.gcap * 4);
  o.bytes = (size_t)(p - p0) + 256;
  return o;
}

template <int MODE>
int launch_pass(const CUtensorMap *tm, const FirTcStage &s, const FirTcPass &P, cudaStream_t st) {
  static PerDevice attr;
  if (attr.first())
    cudaFuncSetAttribute(firtc_mma_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSmemBudget);
  const size_t smem = 1024 + 2 * (size_t)s.gr * 128 + (size_t)P.nstages * kStageBytes;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, current_device());
  const int64_t tiles = cdiv(P.len, kTile) * cdiv(P.mrows, kTile);
  const int grid = (int)(tiles < nsm ? tiles : nsm);
  Launch g(MODE == 1 ? K_FIRTC_ROWS : K_FIRTC_COLS, st);
  launch_pdl(firtc_mma_kernel<MODE>, dim3(grid), dim3(kThreads), smem, st, tm[0], tm[1], tm[2], s,
             P);
  return cuda_status(MODE == 1 ? "tensor-core FIR rows" : "tensor-core FIR columns");
}

}  // namespace

bool firtc_supported(int64_t h, int64_t w, int64_t ldx, int row_taps, int col_taps) {
  if (getenv("VMF_NO_FIRTC")) return false;
  if (h < 3 || w < 3 || h > (1 << 20) || w > (1 << 20) || (ldx & 3)) return false;
  if (!(row_taps & 1) || !(col_taps & 1)) return false;
  if ((row_taps - 1) / 2 > kTcMaxK || (col_taps - 1) / 2 > kTcMaxK) return false;
  // every line holds the whole kernel (the reference's own requirement)
  return row_taps <= w && col_taps <= h;
}

#ifdef VMF_TC_TL
}  // namespace vmf
extern "C" int vmf_debug_tctl(unsigned long long *host) {
  return (int)cudaMemcpyFromSymbol(host, vmf::g_tctl, sizeof(unsigned long long) * 1024);
}
namespace vmf {
#endif

size_t firtc_workspace_bytes(int64_t h, int64_t w, int row_taps, int col_taps) {
  return layout(nullptr, h, w, row_taps, col_taps).bytes;
}

int firtc_detect(const float *x, int64_t ldx, int64_t h, int64_t w, const double *rtaps, int rn,
                 const double *ctaps, int cn, float lap_scale, float frac, float *L, int64_t ldl,
                 int32_t *det_yx, float *det_val, int64_t cap, int64_t *n_det_dev, float *thr_dev,
                 void *ws, size_t ws_bytes, cudaStream_t st) {
  if (!firtc_supported(h, w, ldx, rn, cn) || ((uintptr_t)x & 15))
    return fail(VMF_EVALUE, "tensor-core FIR: unsupported frame or kernel");
  Layout o = layout(ws, h, w, rn, cn);
  if (ws_bytes < o.bytes) return fail(VMF_EVALUE, "tensor-core FIR: workspace too small");
  cudaMemsetAsync(o.cs, 0, sizeof(CandState), st);
  static FirTcStage rs, cs;  // (large: not on the stack; host-side, guarded)
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (!stage_of(rtaps, rn, &rs) || !stage_of(ctaps, cn, &cs))
    return fail(VMF_EVALUE, "tensor-core FIR: taps must be odd and <= %d", 2 * kTcMaxK + 1);
  const int H = (int)h, W = (int)w;
  {
    PrepArgs a;
    a.X = x;
    a.ldx = ldx;
    a.H = H;
    a.W = W;
    a.u = o.u;
    a.ldu = o.ldu;
    a.edge = o.edge1;
    a.b1h = o.b1h;
    a.b1l = o.b1l;
    a.b2h = o.b2h;
    a.b2l = o.b2l;
    a.nbu = (int)(cdiv(H, 4) * cdiv(W, 1024) + 2 * cdiv(W, 256));
    a.nbe = 0;
    const int nblk = (int)(cdiv(W, 32) + cdiv(H + 4, 8) +
                           cdiv((int64_t)kSlice * (rs.gr + cs.gr), 256) + a.nbu);
    Launch g(K_FIRTC_PREP, st);
    firtc_prep_kernel<<<nblk, 256, 0, st>>>(a, rs, cs);
  }
  int rc = cuda_status("tensor-core FIR prep");
  if (rc) return rc;
  CUtensorMap tm[3];
  // row pass: lines = U [H + 4][W], band = the row stage's [128][KW1]
  if (!make_tmap_2d_f32_sw128(&tm[0], o.u, H + 4, W, o.ldu, kTile) ||
      !make_tmap_2d_f32_sw128(&tm[1], o.b1h, rs.gr, kSlice, kSlice, kSlice) ||
      !make_tmap_2d_f32_sw128(&tm[2], o.b1l, rs.gr, kSlice, kSlice, kSlice))
    return fail(VMF_EVALUE, "tensor-core FIR: TMA descriptor unavailable");
  FirTcPass P;
  memset(&P, 0, sizeof(P));
  P.mrows = H + 4;
  P.len = W;
  P.H = H;
  P.k = rs.k;
  P.nslices = rs.KW / kSlice;
  P.nstages = stages_of(rs);
  P.edge = o.edge1;
  P.vt = o.vt;
  P.ldvt = o.ldvt;
  P.edge2 = o.edge2;
  rc = launch_pass<1>(tm, rs, P, st);
  if (rc) return rc;
  // column pass: lines = V^T [W][H], band = the column stage's
  if (!make_tmap_2d_f32_sw128(&tm[0], o.vt, W, H, o.ldvt, kTile) ||
      !make_tmap_2d_f32_sw128(&tm[1], o.b2h, cs.gr, kSlice, kSlice, kSlice) ||
      !make_tmap_2d_f32_sw128(&tm[2], o.b2l, cs.gr, kSlice, kSlice, kSlice))
    return fail(VMF_EVALUE, "tensor-core FIR: TMA descriptor unavailable");
  memset(&P, 0, sizeof(P));
  P.mrows = W;
  P.len = H;
  P.H = H;
  P.k = cs.k;
  P.nslices = cs.KW / kSlice;
  P.nstages = stages_of(cs);
  P.edge = o.edge2;
  P.L = L;
  P.ldl = ldl;
  P.lap_scale = lap_scale;
  P.absmax = &o.cs->absmax_bits;
  P.vec = (ldl % 8 == 0 && ((uintptr_t)L & 31) == 0) ? 2 : (ldl % 4 == 0 && ((uintptr_t)L & 15) == 0) ? 1 : 0;
  rc = launch_pass<2>(tm, cs, P, st);
  if (rc || frac <= 0.0f) return rc;
  {
    Launch g(K_NMS_WRITE, st);
    launch_pdl(firtc_nms_kernel, dim3((unsigned)cdiv(W, kNmsC), (unsigned)cdiv(H, kNmsR)), dim3(256),
               0, st, (const float *)L, ldl, H, W, frac, o.cs, o.gy, o.gx, o.gv, (int)o.gcap,
               (ldl % 4 == 0 && ((uintptr_t)L & 15) == 0) ? 1 : 0);
  }
  rc = cuda_status("tensor-core FIR stage 4");
  if (rc) return rc;
  return colfinal_launch(o.cs, o.gy, o.gx, o.gv, o.gcap, L, ldl, h, w, frac, det_yx, det_val, cap,
                         n_det_dev, thr_dev, st);
}

}  // namespace vmf
