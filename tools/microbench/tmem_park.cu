// TMEM as a per-thread parking area: each thread stores 64 32-bit words to
// its own TMEM lane (tcgen05.st 32x32b), reads them back (tcgen05.ld) and
// checks; then times N park/unpark rounds.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void tm_st16(uint32_t taddr, const uint32_t *r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};\n" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]));
}
__device__ __forceinline__ void tm_ld16(uint32_t taddr, uint32_t *r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

__global__ void __launch_bounds__(128, 8) park_kernel(int rounds, int *bad, unsigned long long *cyc) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;\n" ::"r"(
        (unsigned)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t taddr = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
  uint32_t v[16];
  int errs = 0;
  long long t0 = clock64();
  for (int it = 0; it < rounds; ++it) {
    for (int blk = 0; blk < 4; ++blk) {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = (threadIdx.x * 1315423911u) ^ (it * 64 + blk * 16 + i);
      tm_st16(taddr + blk * 16, v);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    for (int blk = 0; blk < 4; ++blk) {
      tm_ld16(taddr + blk * 16, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int i = 0; i < 16; ++i)
        errs += v[i] != ((threadIdx.x * 1315423911u) ^ (it * 64 + blk * 16 + i));
    }
  }
  long long t1 = clock64();
  if (errs) atomicAdd(bad, errs);
  if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;\n" ::"r"(tbase));
}

int main() {
  int *bad;
  unsigned long long *cyc;
  cudaMalloc(&bad, 4);
  cudaMalloc(&cyc, 8);
  cudaMemset(bad, 0, 4);
  cudaMemset(cyc, 0, 8);
  const int rounds = 1000, grid = 148 * 8;
  park_kernel<<<grid, 128>>>(rounds, bad, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  int hb = 0;
  unsigned long long hc = 0;
  cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
  printf("err=%s bad=%d  cycles/round/CTA=%.1f (64 words st + ld per thread, 8 CTAs/SM)\n",
         cudaGetErrorString(e), hb, (double)hc / grid / rounds);
  return 0;
}
