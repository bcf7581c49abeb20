// vmf_rowlap.cuh -- the fp32 "Laplacian-first" row pass (vmf_rowlap.cu).
#pragma once
#include "vmf_common.cuh"

namespace vmf {

constexpr int kHmRowMax = 2048;  // border weights h(1..Mh) along a row

struct RowLapParams {
  float p, q;           // modal pole (JORDAN: p; CPAIR: p + i q)
  float c[4], cs[4];    // y+ = c . u(n-1); cs = sign * c (the anticausal part)
  float b0, sign;
  float SP[4][16], SQ[4][16];  // folded 32-sample chunk-carry weights
  float A32[16];        // A^32
  float Apow[5][16];    // A^(32 cpl 2^l): the chunk scan's Kogge-Stone steps
  float Iss[4];         // (I - A)^-1 b
  int64_t H, W;
  int C, cpl, rows_per, Mh, K;
};

struct HmRow {
  float h[kHmRowMax + 1];
};

struct RowLapPlan {
  RowLapParams p;
  HmRow hm;
  int kind;
};

bool rowlap_supported(int64_t h, int64_t w, const double *b, const double *a, int k, double b0,
                      int sign);
// X (fp32, pitch ldx; 16-byte aligned rows) -> V = R(Lap5 X) (pitch ldv) with
// the left / right border terms folded in, and the virtual rows Vt / Vb [w]
int rowlap_run(const float *x, int64_t ldx, float *V, int64_t ldv, float *Vt, float *Vb,
               int64_t h, int64_t w, const double *b, const double *a, int k, double b0, int sign,
               cudaStream_t st);
// Ky[2][w] = R_ss(s Cc[0]), R_ss(Cc[1]): the top / bottom border terms of the
// column direction (Cc from the column scan; s = sign of the column stage)
int rowfix_run(const float *Cc, float *Ky, int64_t h, int64_t w, const double *b,
               const double *a, int k, double b0, int sign, float col_sign, cudaStream_t st);

}  // namespace vmf
