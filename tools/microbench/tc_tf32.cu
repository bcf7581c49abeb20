// tcgen05.mma kind::tf32 probe: one CTA, D[128x128] (+)= A[128xK] . B[128xK]^T
// with A, B K-major fp32 tiles loaded by TMA (SWIZZLE_128B, box {32, 128}),
// K = 32 per slice, NS slices; 1xTF32 and 3xTF32 (hi/lo split) against an
// fp64 host reference.  Pins the smem / instruction descriptor encodings the
// tensor-core FIR (vmf_firtc.cu) uses.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O2 -I../../paper_1912_07133_b200/csrc \
//        tc_tf32.cu ../../paper_1912_07133_b200/csrc/vmf_tma.cu -o tc_tf32
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "vmf_tma.cuh"

using namespace vmf;

__device__ __forceinline__ uint64_t sw128_desc(const void *smem) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(smem);
  uint64_t d = 0;
  d |= (uint64_t)((a & 0x3FFFF) >> 4);          // start address
  d |= (uint64_t)1 << 16;                        // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;              // SBO: 8-row groups 1024 B apart
  d |= (uint64_t)1 << 46;                        // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                        // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t dt, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

constexpr int M = 128, N = 128;
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
                            ((uint32_t)(M >> 4) << 24);

// mode 1: D = A B^T (tf32); mode 3: D = Ah Bh + Ah Bl + Al Bh
__global__ void __launch_bounds__(128) probe(const __grid_constant__ CUtensorMap ta_h,
                                             const __grid_constant__ CUtensorMap ta_l,
                                             const __grid_constant__ CUtensorMap tb_h,
                                             const __grid_constant__ CUtensorMap tb_l, int ns,
                                             int mode, float *D) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char *sm = sm_raw + ((1024 - ((uint32_t)__cvta_generic_to_shared(sm_raw) & 1023)) & 1023);
  float *Ah = (float *)sm, *Al = Ah + M * 32, *Bh = Al + M * 32, *Bl = Bh + N * 32;
  __shared__ __align__(8) uint64_t bar_ld, bar_mma;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(
        (unsigned)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar_ld, 1);
    mbar_init(&bar_mma, 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t dt = tbase;
  for (int s = 0; s < ns; ++s) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(&bar_ld, 4 * M * 32 * 4);
      tma_load_2d(Ah, &ta_h, &bar_ld, 32 * s, 0);
      tma_load_2d(Al, &ta_l, &bar_ld, 32 * s, 0);
      tma_load_2d(Bh, &tb_h, &bar_ld, 32 * s, 0);
      tma_load_2d(Bl, &tb_l, &bar_ld, 32 * s, 0);
    }
    mbar_wait(&bar_ld, s & 1);
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (threadIdx.x == 0) {
      for (int k = 0; k < 4; ++k) {  // K = 8 per instruction: +32 bytes in the atom
        const uint64_t ah = sw128_desc(Ah) + 2 * k, al = sw128_desc(Al) + 2 * k;
        const uint64_t bh = sw128_desc(Bh) + 2 * k, bl = sw128_desc(Bl) + 2 * k;
        const uint32_t acc = (s > 0 || k > 0) ? 1u : 0u;
        mma_tf32(dt, ah, bh, kIdesc, acc);
        if (mode == 3) {
          mma_tf32(dt, ah, bl, kIdesc, 1u);
          mma_tf32(dt, al, bh, kIdesc, 1u);
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(&bar_mma)));
    }
    mbar_wait(&bar_mma, s & 1);  // (smem reused by the next slice)
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  // epilogue: lane = row, 128 columns
  const int row = threadIdx.x;
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(dt + ((uint32_t)(32 * warp) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(tbase));
}

static float tf32r(float x) {  // round to nearest even at 10 mantissa bits
  uint32_t u;
  memcpy(&u, &x, 4);
  u = (u + 0xFFF + ((u >> 13) & 1)) & ~0x1FFFu;
  memcpy(&x, &u, 4);
  return x;
}

int main() {
  const int ns = 4, K = 32 * ns;
  std::vector<float> A(M * K), B(N * K), Ah(M * K), Al(M * K), Bh(N * K), Bl(N * K);
  srand(7);
  for (auto &v : A) v = (float)rand() / RAND_MAX - 0.5f;
  for (auto &v : B) v = (float)rand() / RAND_MAX - 0.5f;
  for (int i = 0; i < M * K; ++i) { Ah[i] = tf32r(A[i]); Al[i] = tf32r(A[i] - Ah[i]); }
  for (int i = 0; i < N * K; ++i) { Bh[i] = tf32r(B[i]); Bl[i] = tf32r(B[i] - Bh[i]); }
  float *d[5];
  const std::vector<float> *src[4] = {&Ah, &Al, &Bh, &Bl};
  for (int i = 0; i < 4; ++i) {
    cudaMalloc(&d[i], src[i]->size() * 4);
    cudaMemcpy(d[i], src[i]->data(), src[i]->size() * 4, cudaMemcpyHostToDevice);
  }
  cudaMalloc(&d[4], M * N * 4);
  CUtensorMap tm[4];
  for (int i = 0; i < 4; ++i)
    if (!make_tmap_2d_f32_sw128(&tm[i], d[i], 128, K, K, 128)) { printf("tmap fail\n"); return 1; }
  const size_t smem = 4 * 128 * 32 * 4 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int mode : {1, 3}) {
    cudaMemset(d[4], 0, M * N * 4);
    probe<<<1, 128, smem>>>(tm[0], tm[1], tm[2], tm[3], ns, mode, d[4]);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("kernel error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> D(M * N);
    cudaMemcpy(D.data(), d[4], M * N * 4, cudaMemcpyDeviceToHost);
    double emax = 0, smax = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)A[m * K + k] * B[n * K + k];
        emax = fmax(emax, fabs(ref - D[m * N + n]));
        smax = fmax(smax, fabs(ref));
      }
    printf("mode %dxTF32: max|err| %.3e  max|D| %.3e  rel %.3e  D[0]=%g D[5*128+7]=%g\n", mode,
           emax, smax, emax / smax, D[0], D[5 * 128 + 7]);
  }
  return 0;
}
